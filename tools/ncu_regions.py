"""Stall attribution by SASS region from `ncu --page source --csv --print-source sass`.

    ncu -i rep --page source --csv --print-source sass > src.csv
    python tools/ncu_regions.py src.csv [top]

Groups instructions into basic blocks (split at branch targets / branches),
prints blocks by sampled stall share with their instruction mix and the
dominant stall reasons (development helper).
"""
import csv, re, sys
from collections import Counter, defaultdict

allrows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
want = sys.argv[3] if len(sys.argv) > 3 else None  # kernel-name substring
starts = [i for i, r in enumerate(allrows) if r and r[0] == 'Kernel Name']
sec = [(i, j) for i, j in zip(starts, starts[1:] + [len(allrows)])
       if want is None or want in allrows[i][1]][0]
rows = allrows[sec[0]:sec[1]]
print(rows[0][1])
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
stall_cols = [k for k in h if k.startswith('stall_') and '(Not Issued)' not in k]
ins = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    a = int(r[ix['Address']], 16)
    ins.append((a, r[ix['Source']].strip(), int(r[ix['Warp Stall Sampling (All Samples)']] or 0),
                int(r[ix['Instructions Executed']] or 0), {k: int(r[ix[k]] or 0) for k in stall_cols}))
base = ins[0][0]
targets = set()
for a, s, *_ in ins:
    m = re.search(r'BRA[^0-9x]*(0x[0-9a-f]+)', s)
    if m:
        targets.add(base + int(m.group(1), 16) if int(m.group(1), 16) < base else int(m.group(1), 16))
blocks, cur = [], []
for a, s, smp, ex, st in ins:
    if (a - base) in targets or a in targets:
        if cur: blocks.append(cur)
        cur = []
    cur.append((a, s, smp, ex, st))
    if 'BRA' in s or 'EXIT' in s or 'BRX' in s:
        blocks.append(cur); cur = []
if cur: blocks.append(cur)
tot = sum(x[2] for x in ins)
res = []
for b in blocks:
    smp = sum(x[2] for x in b)
    st = Counter()
    for x in b: st.update(x[4])
    mix = Counter(x[1].split()[0] if not x[1].startswith('@') else x[1].split()[1] for x in b)
    mix = Counter({k.split('.')[0]: 0 for k in mix}) + Counter(k.split('.')[0] for k in mix.elements())
    res.append((smp, b[0][0] - base, b[-1][0] - base, len(b), b[0][3], st, mix))
res.sort(key=lambda r: -r[0])
print(f"total samples {tot}")
for smp, a0, a1, n, ex, st, mix in res[:top]:
    s = ', '.join(f"{k[6:]} {100*v/max(1,smp):.0f}%" for k, v in st.most_common(5))
    print(f"{100*smp/tot:5.1f}% [{a0:#x}-{a1:#x}] n={n} exec={ex}  {s}\n        mix {dict(mix.most_common(8))}")

# share of samples in FP64-dense blocks vs the rest
dense = sum(r[0] for r in res if (r[6].get('DFMA', 0) + r[6].get('DMUL', 0)) >= 0.4 * r[3])
print(f"FP64-dense blocks: {100*dense/tot:.1f}% of samples; other: {100*(tot-dense)/tot:.1f}%")
other = Counter()
for r in res:
    if (r[6].get('DFMA', 0) + r[6].get('DMUL', 0)) < 0.4 * r[3]:
        other.update(r[5])
print("other-block stalls:", ', '.join(f"{k[6:]} {100*v/max(1,tot):.1f}%" for k, v in other.most_common(8)))
print("--- top non-dense blocks")
nd = [r for r in res if (r[6].get('DFMA', 0) + r[6].get('DMUL', 0)) < 0.4 * r[3]]
for smp, a0, a1, n, ex, st, mix in nd[:top]:
    s = ', '.join(f"{k[6:]} {100*v/max(1,smp):.0f}%" for k, v in st.most_common(4))
    print(f"{100*smp/tot:5.1f}% [{a0:#x}-{a1:#x}] n={n} exec={ex} {s} | {dict(mix.most_common(6))}")
