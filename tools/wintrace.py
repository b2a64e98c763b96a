"""Phase timing of the last stage's expectation and window-stencil blocks (diagnostic; needs
`make -B EXTRA=-DESDP_WIN_TRACE`).  Marks are thread 0's %globaltimer (256 ns granularity on B200).
window:      0 start, 1 payoffs + dependency wait, 2 W staged, 3 keys + unimodality reductions,
             4 packed levels (non-unimodal only), 5 queries + singles, 6 stored
expectation (dmma3): 0 start, 1 P chunks issued, 2 after the dependency wait, 3 first chunk landed,
             4 DMMA chain done, 5 stored"""
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
buf = np.zeros((2, 4096, 8), np.uint64)
E.lib.esdp_win_trace.argtypes = [ctypes.c_void_p]
assert E.lib.esdp_win_trace(buf.ctypes.data) == 0


def report(name, bb, nb, names):
    nm = len(names) + 1
    b = bb[:nb, :nm].astype(np.float64)
    sm = bb[:nb, 7].astype(np.int64)
    t0 = b[:, 0].min()
    print("== %s (%d blocks)" % (name, nb))
    print("block start spread (us): %.2f .. %.2f" % (0.0, (b[:, 0].max() - t0) / 1e3))
    print("block end   spread (us): %.2f .. %.2f" % ((b[:, -1].min() - t0) / 1e3, (b[:, -1].max() - t0) / 1e3))
    d = np.diff(b, axis=1) / 1e3
    for j, n in enumerate(names):
        print("  %-16s mean %.3f  p50 %.3f  max %.3f us" % (n, d[:, j].mean(), np.median(d[:, j]), d[:, j].max()))
    cnt = np.bincount(sm, minlength=148)
    print("  blocks per SM histogram:", np.bincount(cnt))
    return t0, b


tw, bw = report("window", buf[0], 400, ["pay+wait", "stage W", "keys+reduce", "levels", "queries+singles",
                                         "near-tie+store"])
tc, bc = report("expectation", buf[1], 416, ["P issue", "wait", "chunk 0 landed", "DMMA chain", "store"])
print("expectation first start -> window first start: %.2f us; expectation last end -> window last wait done: %.2f us"
      % ((tw - tc) / 1e3, (bw[:, 1].max() - bc[:, 5].max()) / 1e3))
