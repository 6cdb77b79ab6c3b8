"""Top SASS instructions by warp-stall samples from an ncu source page CSV
(ncu -i R --page source --csv --print-source sass -k regex:K > F):
    python tools/ncu_hot.py F [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
si = h.index('Warp Stall Sampling (All Samples)')
st = [i for i, x in enumerate(h) if x.startswith('stall_') and 'Not Issued' not in x]
body = [r for r in rows[2:] if r and r[0].startswith("0x")]
tot = sum(int(r[si] or 0) for r in body)
agg = {}
for r in body:
    for i in st:
        agg[h[i]] = agg.get(h[i], 0) + int(r[i] or 0)
print('total samples', tot, {k[6:]: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]})
order = sorted(range(len(body)), key=lambda k: -int(body[k][si] or 0))
for k in order[:N]:
    r = body[k]
    s = sorted(((int(r[i] or 0), h[i][6:]) for i in st), reverse=True)[:3]
    print(f"{k:6d} {r[0][-5:]} {int(r[si]):6d} {r[1].strip()[:60]:60s} {s}")
