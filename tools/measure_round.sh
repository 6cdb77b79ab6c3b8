#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): bench lines of both arms
# at C2/C3/C4, ncu digests + FP64 counters + the launch list, smoke.
#   bash tools/measure_round.sh OUTDIR
OUT=${1:-gpurun_out/round}
mkdir -p $OUT
python bench.py > $OUT/bench_C2.json 2> $OUT/bench_C2.err
python bench.py --config C3 --steps 20 --warmup 3 > $OUT/bench_C3.json 2> $OUT/bench_C3.err
python bench.py --config C4 --steps 10 --warmup 3 > $OUT/bench_C4.json 2> $OUT/bench_C4.err
python bench.py --impl reference > $OUT/bench_reference_C2.json 2> $OUT/bench_reference_C2.err
python bench.py --impl reference --config C3 --steps 5 --warmup 3 > $OUT/bench_reference_C3.json 2> $OUT/bench_reference_C3.err
python bench.py --impl reference --config C4 --steps 5 --warmup 3 > $OUT/bench_reference_C4.json 2> $OUT/bench_reference_C4.err
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
bash tools/profile_configs.sh $OUT/prof
