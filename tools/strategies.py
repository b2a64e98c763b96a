"""NEXT-2: the paper's Fig. 3 strategy study on the GPU, for a sweep of storage durations:
  perfect foresight  -- deterministic DP on every realised price path (one context, K = paths, P = I);
  DP bid curves      -- ESDP_SIM_PHYSICAL: the stage's curve cleared at the realised price, real SoC;
  DP self-scheduled  -- ESDP_SIM_SELF: decided at the realised one-stage-lagged price;
  myopic             -- ESDP_SIM_FIXED: the plan of a deterministic DP on the expected ("day-ahead")
                        prices, settled at the realised prices.
python tools/strategies.py [--config cfg2-rank1|cfg2] [--paths 256] -> one JSON line per duration."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_15629_b200 as E
import workloads


def expected_prices(inst):
    """E[lambda_t] under the price model: pi_t (rank-1) or pi_1 P_1 ... P_{t-1} (Markov)."""
    T = inst.T
    if inst.P is None:
        return np.sum(inst.pi * inst.lam, axis=1)
    m = np.asarray(inst.pi, float)
    out = np.empty(T)
    for t in range(T):
        out[t] = m @ inst.lam[t]
        if t < T - 1:
            m = m @ inst.P[t]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2-rank1", choices=["cfg2-rank1", "cfg2"])
    ap.add_argument("--paths", type=int, default=256)
    ap.add_argument("--durations", type=int, default=4)
    args = ap.parse_args()
    dev = torch.device("cuda")
    n = args.paths
    rows = []
    for pbar in np.geomspace(10.42, 99.0, args.durations):
        base = workloads.cfg2(rank1=args.config == "cfg2-rank1")
        base.pbar = float(np.round(pbar, 6))
        res = {"config": args.config, "pbar_over_delta": base.pbar, "hours": 1000.0 / base.pbar / 12.0, "paths": n}
        t0 = time.perf_counter()
        with E.Solver(base, keep_values=True) as s:
            s.backward()
            out = torch.empty(n, dtype=torch.float64, device=dev)
            for name, mode in (("bids", E.ESDP_SIM_PHYSICAL), ("self", E.ESDP_SIM_SELF)):
                E.esdp_simulate_strategy_dev(s.ctx, n, 7, mode, out.data_ptr())
                torch.cuda.synchronize()
                res[name] = float(out.mean())
            lamp = torch.empty(base.T * n, dtype=torch.float64, device=dev)
            E.esdp_price_paths_dev(s.ctx, n, 7, lambda_ptr=lamp.data_ptr())
            # myopic: deterministic DP on the expected prices, its plan settled at the realised prices
            da = workloads.Instance("da", base.T, 1, base.pbar, base.sbar, base.s0, base.eta_c, base.eta_d, base.delta,
                                    expected_prices(base).reshape(-1, 1), np.ones((base.T - 1, 1, 1)), np.array([1.0]))
            with E.Solver(da, keep_values=True) as sd:
                sd.backward()
                plan = torch.empty(base.T, dtype=torch.int16, device=dev)
                one = torch.empty(1, dtype=torch.float64, device=dev)
                E.esdp_simulate_strategy_dev(sd.ctx, 1, 7, E.ESDP_SIM_PHYSICAL, one.data_ptr(), actions_ptr=plan.data_ptr())
                torch.cuda.synchronize()
            E.esdp_simulate_strategy_dev(s.ctx, n, 7, E.ESDP_SIM_FIXED, out.data_ptr(), schedule_ptr=plan.data_ptr())
            torch.cuda.synchronize()
            res["myopic"] = float(out.mean())
            lam = lamp.cpu().numpy().reshape(base.T, n)
        # perfect foresight on the same realised paths: K = n deterministic rows, identity transitions
        pf = workloads.Instance("pf", base.T, n, base.pbar, base.sbar, base.s0, base.eta_c, base.eta_d, base.delta,
                                lam.copy(), np.broadcast_to(np.eye(n), (base.T - 1, n, n)).copy(), np.full(n, 1.0 / n))
        with E.Solver(pf, keep_values=False) as sp:
            res["perfect"] = float(sp.backward())                 # = mean over paths of V_1(s0, path)
        res["gpu_wall_s"] = time.perf_counter() - t0
        for k in ("bids", "self", "myopic"):
            res[k + "_capture"] = res[k] / res["perfect"]
        rows.append(res)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
