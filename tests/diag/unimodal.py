"""How often are the window stencil's packed keys unimodal per (stage, k, tile, side)?  (diagnostic, CPU)
Emulates window.cuh's key(j) = W[j] - fl(beta j) and pack_key on the oracle's W_t."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import oracle, workloads
from helpers import to_oracle

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
gc1 = gd1 = 0.0
if name == "cfg3":
    b = workloads.cfg2(T=48)
    a0 = oracle.actions(to_oracle(b))
    inst = workloads.cfg3_gpu(a0, T=48)
    gc1, gd1 = 2.0 * inst.delta / inst.eta_c, 2.0 * inst.delta * inst.eta_d
elif name == "cfg5":
    inst = workloads.cfg5_instances([int(sys.argv[2]) if len(sys.argv) > 2 else 0], T=48)[0]
else:
    inst = {"cfg2": lambda: workloads.cfg2(T=48), "cfg4": lambda: workloads.cfg4(T=12)}[name]()
pr = to_oracle(inst)
ref = oracle.backward(pr, nthreads=os.cpu_count())
act = oracle.actions(pr)
S = ref.W.shape[2]
off = np.round(-np.where(act >= 0, act / inst.eta_d, act * inst.eta_c) / inst.delta)
a_z = int(np.where(act == 0)[0][0])
Lc = a_z - 1 if True else 0   # interior charge offsets +1..+Lc (endpoint is a single)
Ld = len(act) - a_z - 2
dc, dd = inst.delta / inst.eta_c, inst.delta * inst.eta_d
TILE = 256


def pack(v, pos):
    b = v.view(np.uint64)
    o = np.where(b >> np.uint64(63), ~b, b | np.uint64(1 << 63))
    o = np.where(np.isneginf(v), np.uint64(0), o)          # -inf: 0 for the check
    return np.where(np.isneginf(v), np.uint64(0), (o & ~np.uint64(1023)) | pos.astype(np.uint64))


def unimodal(pk):
    up = pk[1:] > pk[:-1]
    dn = pk[1:] < pk[:-1]
    ui = np.nonzero(up)[0]; di = np.nonzero(dn)[0]
    return not (len(ui) and len(di) and ui.max() > di.min())


tot = uni_c = uni_d = both = 0
for t in range(1, inst.T):
    W = ref.W[t - 1]
    for k in range(inst.K):
        lam = inst.lam[t - 1, k]
        bc, bd = lam * dc + gc1, lam * dd - gd1
        for i0 in range(0, S, TILE):
            jc = i0 + 1 + np.arange(TILE + Lc)
            jd = i0 - Ld + np.arange(TILE + Ld)
            def keys(j, beta):
                w = np.where((j >= 0) & (j < S), W[k][np.clip(j, 0, S - 1)], -np.inf)
                return pack(w - beta * j.astype(np.float64), np.arange(len(j)))
            c = unimodal(keys(jc, bc)); d = unimodal(keys(jd, bd))
            tot += 1; uni_c += c; uni_d += d; both += c and d
print(f"{name}: tiles {tot}: charge unimodal {uni_c/tot:.3f}, discharge {uni_d/tot:.3f}, both {both/tot:.3f}")
