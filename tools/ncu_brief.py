"""Brief ncu report digest: key metrics, stall shares, instruction mix."""
import csv, re, subprocess, sys, io
from collections import Counter

KEYS = ['gpu__time_duration.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__warps_eligible.avg.per_cycle_active', 'smsp__warps_active.avg.per_cycle_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'l1tex__t_sector_hit_rate.pct', 'launch__registers_per_thread',
        'dram__bytes_read.sum', 'dram__bytes_write.sum']

def run(path):
    raw = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    scale = {'byte': 1.0, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}
    out = []
    for r in rows[2:]:
        d = {'kernel': r[h.index('Kernel Name')][:40]}
        for k in KEYS:
            if k not in h:
                continue
            i = h.index(k)
            v = r[i]
            if units[i] in scale:  # normalise byte counts
                v = float(v.replace(',', '')) * scale[units[i]]
            elif units[i]:
                v = f"{v} {units[i]}"
            d[k] = v
        st = {}
        for k in h:
            if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued'):
                v = r[h.index(k)].replace(',', '')
                if v.isdigit():
                    st[k[len('smsp__pcsamp_warps_issue_stalled_'):]] = int(v)
        tot = sum(st.values()) or 1
        d['stalls'] = [(k, round(v / tot * 100, 1)) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]]
        out.append(d)
    src = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    # one section per kernel: a "Kernel Name" line, a header, then rows
    cur, hdr, c = None, None, None
    mixes = []
    for r in rows:
        if r and r[0] == 'Kernel Name':
            if c is not None:
                mixes.append((cur, c))
            cur, c, hdr = r[1], Counter(), None
            continue
        if hdr is None:
            hdr = r
            iS, iE = hdr.index('Source'), hdr.index('Instructions Executed')
            continue
        if len(r) <= max(iS, iE):
            continue
        op = re.sub(r'^@!?U?P\w+\s+', '', r[iS].strip()).split(' ')[0].split('.')[0]
        c[op] += int(r[iE]) if r[iE].isdigit() else 0
    if c is not None:
        mixes.append((cur, c))
    merged = {}
    for name, m in mixes:  # the page lists each kernel more than once: keep the richest
        if sum(m.values()) > sum(merged.get(name, Counter()).values()):
            merged[name] = m
    order = list(dict.fromkeys(n for n, _ in mixes))
    for d, name in zip(out, order):
        m = merged[name]
        T = sum(m.values()) or 1
        d['mix'] = [(k, round(v / T * 100, 1)) for k, v in m.most_common(12)]
    return out

if __name__ == '__main__':
    for p in sys.argv[1:]:
        for d in run(p):
            print(p)
            for k, v in d.items():
                print(f'  {k}: {v}')
