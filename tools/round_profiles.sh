#!/bin/bash
# Turn a tools/measure_round.sh capture (gpurun_out/DIR) into the tracked
# profiles/ files of round TAG:  bash tools/round_profiles.sh gpurun_out/r02b r02
set -e
IN=$1; TAG=$2
for c in C2 C3 C4; do
  tail -1 $IN/bench_$c.json > profiles/${TAG}_bench_$c.json
  tail -1 $IN/bench_reference_$c.json > profiles/${TAG}_bench_reference_$c.json
done
cp $IN/smoke.txt profiles/${TAG}_smoke.txt
python tools/launch_summary.py $IN/prof/launches_C2.csv \
  "python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-probe (C2: 2000 atoms, 2J=8)" \
  > profiles/${TAG}_launches_C2.md
cp $IN/prof/launches_C2.csv profiles/${TAG}_launches_C2.csv
declare -A NA=([C2]=2000 [C3]=262144 [C4]=32768)
declare -A TJ=([C2]=8 [C3]=8 [C4]=14)
for c in C2 C3 C4; do
  { echo "# ${TAG} ncu --set full digest, config $c (tools/profile_configs.sh; cold-cache, serialised)"
    echo; echo '```'; python tools/ncu_brief.py $IN/prof/$c.ncu-rep | grep -v "ncu-rep$"; echo '```'; } \
    > profiles/${TAG}_ncu_$c.md
  python tools/fp64_report.py $IN/prof/$c.ncu-rep ${NA[$c]} $((26 * ${NA[$c]})) ${TJ[$c]} \
    > profiles/${TAG}_fp64_$c.json
done
python - "$IN" <<'PY'
import csv, io, json, subprocess, sys
out = {}
for c in ("C2", "C3", "C4"):
    raw = subprocess.run(["ncu", "-i", f"{sys.argv[1]}/prof/{c}.ncu-rep", "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u = r[0], r[1]
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    d = {}
    for row in r[2:]:
        k = row[h.index("Kernel Name")]
        key = ("U" if "compute_U" in k else "Y" if "compute_Y" in k else "dE" if "dE" in k
               else "gather")
        b = sum(float(row[h.index(m)].replace(",", "")) * sc.get(u[h.index(m)], 1)
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        d[f"{key}_bytes_per_launch"] = b
    out[c] = d
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
PY
