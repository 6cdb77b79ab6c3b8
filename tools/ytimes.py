import ctypes as C, sys
import numpy as np
sys.path.insert(0, '.')
import paper_2011_12875_b200 as snap
if len(sys.argv) > 1 and sys.argv[1].startswith("--lib="):  # the SNAP_Y_PROFILE build
    snap.LIB_PATH = sys.argv.pop(1)[6:]
p = snap.bcc_problem(10, 10, 10, twojmax=8)
eng = snap.SnapEngine.for_problem(p); eng.set_problem(p); eng.enable_stage_timing(True)
eng.run(); eng.synchronize()
L = snap.library(); buf = (C.c_longlong * 2112)()
L.snapgpu_debug_yprof(buf, 2112)
eng.run(); eng.synchronize()
L.snapgpu_debug_yprof(buf, 2112)
nb = int(buf[61])  # CTAs of the launch
a = np.array(buf[64:64 + 2 * nb], dtype=np.int64).reshape(-1, 2)
smid = a[:, 1] & 255
a[:, 1] = a[:, 0] + (a[:, 1] >> 8)
t0 = a[:, 0].min()
s = (a[:, 0] - t0) / 1e3; e = (a[:, 1] - t0) / 1e3
print("start us: min %.1f med %.1f max %.1f" % (s.min(), np.median(s), s.max()))
print("end   us: min %.1f med %.1f max %.1f" % (e.min(), np.median(e), e.max()))
print("dur   us: min %.1f med %.1f max %.1f" % ((e - s).min(), np.median(e - s), (e - s).max()))
print("stage times", eng.stage_times())
d = e - s
order = np.argsort(-d)
print("slowest CTAs (block, sm, start us, dur us):", [(int(i), int(smid[i]), round(float(s[i]), 1), round(float(d[i]), 1)) for i in order[:12]])
print("fastest:", [(int(i), int(smid[i]), round(float(s[i]), 1), round(float(d[i]), 1)) for i in order[-6:]])
# TPC pairing: SMs 2k and 2k+1 share a TPC; is a CTA slower when its TPC partner is busy?
busy = set(int(x) for x in smid)
pd_ = [d[i] for i in range(len(d)) if (int(smid[i]) ^ 1) in busy]
pa_ = [d[i] for i in range(len(d)) if (int(smid[i]) ^ 1) not in busy]
print("TPC partner busy: n=%d median %.1f us; partner idle: n=%d median %.1f us" %
      (len(pd_), np.median(pd_) if pd_ else 0, len(pa_), np.median(pa_) if pa_ else 0))
