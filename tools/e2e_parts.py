"""Decomposition of the one-call (host lists) step at C2 on the GPU
(development helper): device time of the uploads, the reverse-index
rebuild, the step graph and the read-back, against the wall time per call."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2011_12875_b200 as snap

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 10
p = snap.bcc_problem(nx, nx, nx, 8)
eng = snap.SnapEngine.for_problem(p)
s = torch.cuda.Stream()
eng.set_stream(s.cuda_stream)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
nn, nb, dp = pin(p.numneigh), pin(p.nbr), pin(p.disp)
f = pin(np.zeros((p.natoms, 3))).numpy(); e = pin(np.zeros(p.natoms)).numpy(); t = pin(np.zeros(1)).numpy()
args = (nn.numpy(), nb.numpy(), dp.numpy())
R = 100
def ev_time(fn, reps=R):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps): fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
def wall(fn, reps=R):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6
d = [torch.empty_like(x, device='cuda') for x in (nn, nb, dp)]
def up():
    with torch.cuda.stream(s):
        for x, y in zip(d, (nn, nb, dp)): x.copy_(y, non_blocking=True)
out = torch.empty(4 * p.natoms + 1, dtype=torch.float64, device='cuda')
hout = pin(np.zeros(4 * p.natoms + 1))
def down():
    with torch.cuda.stream(s):
        hout.copy_(out, non_blocking=True)
eng.set_neighbors(*args)
eng.run(); eng.synchronize()
print(f"N={p.natoms}")
print(f"uploads (3 H2D, {sum(x.nbytes for x in (nn, nb, dp))} B): {ev_time(up):.1f} us GPU")
print(f"read-back (D2H {hout.numel()*8} B): {ev_time(down):.1f} us GPU")
print(f"step graph: {ev_time(lambda: eng.run()):.1f} us GPU")
def dirty_run():
    eng.set_neighbors(*args)   # uploads + host validation + reverse index marked dirty
    eng.run()
print(f"set_neighbors + run (uploads, CSR rebuild, graph): {ev_time(dirty_run, 30):.1f} us GPU, {wall(dirty_run, 30):.1f} us wall")
step = lambda: eng.step(*args, forces=f, eatom=e, etotal=t)
print(f"one-call step: {ev_time(step):.1f} us GPU (events around the call), {wall(step):.1f} us wall")
pos = pin(p.positions).numpy()
sp = lambda: eng.step_positions(pos, p.box, forces=f, eatom=e, etotal=t)
print(f"positions step: {ev_time(sp):.1f} us GPU, {wall(sp):.1f} us wall")
print(f"graph only wall (sync each): {wall(lambda: (eng.run(), eng.synchronize())):.1f} us")
# host-side overhead: the Python wrapper's argument handling vs the bare C call
L, h = eng._L, eng._h
ptrs = [x.ctypes.data for x in (args[0], args[1], args[2], f, e, t)]
raw = lambda: L.snapgpu_run_host(h, p.natoms, 0, p.natoms, p.nbr.shape[1], ptrs[0], ptrs[1], ptrs[2],
                                 None, ptrs[3], ptrs[4], ptrs[5])
print(f"bare C one-call (precomputed pointers): {wall(raw):.1f} us wall")
def prep():
    nn_ = np.ascontiguousarray(args[0], np.int32); nb_ = np.ascontiguousarray(args[1], np.int32)
    dp_ = np.ascontiguousarray(args[2], np.float64)
    return (nn_.ctypes.data, nb_.ctypes.data, dp_.ctypes.data, f.ctypes.data, e.ctypes.data, t.ctypes.data)
print(f"wrapper argument handling only: {wall(prep):.1f} us wall")
print(f"bare C no-op call (last_error): {wall(lambda: L.snapgpu_last_error(h)):.2f} us wall")
