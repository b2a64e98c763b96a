"""Phase timing of the window stencil blocks (diagnostic; needs `make -B EXTRA=-DESDP_WIN_TRACE`):
marks 0 start, 1 W staged, 2 level-0 keys, 3 levels built, 4 queries + singles, 5 near-tie pass done."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_15629_b200 as E
import workloads

inst = workloads.cfg2()
s = E.Solver(inst, keep_values=True)
for _ in range(3):
    s.backward()
torch.cuda.synchronize()
buf = np.zeros((4096, 8), np.uint64)
E.lib.esdp_win_trace.argtypes = [ctypes.c_void_p]
assert E.lib.esdp_win_trace(buf.ctypes.data) == 0
b = buf[:400, :6].astype(np.float64)
t0 = b[:, 0].min()
print("block start spread (us): %.2f .. %.2f" % ((b[:, 0].min() - t0) / 1e3, (b[:, 0].max() - t0) / 1e3))
print("block end   spread (us): %.2f .. %.2f" % ((b[:, 5].min() - t0) / 1e3, (b[:, 5].max() - t0) / 1e3))
d = np.diff(b, axis=1) / 1e3
names = ["stage W", "level0+M", "levels", "queries+singles", "near-tie pass"]
for j, nm in enumerate(names):
    print("%-16s mean %.3f  p50 %.3f  max %.3f us" % (nm, d[:, j].mean(), np.median(d[:, j]), d[:, j].max()))
print("total per block mean %.3f us" % ((b[:, 5] - b[:, 0]).mean() / 1e3))
