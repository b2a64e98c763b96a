"""Multi-GPU schedule on CPU (gloo, world size 2 and 3): the K-partitioned backward induction of
SURVEY.md §8(e).1 -- every rank computes its price-state rows of each stage and all-gathers V_t in
blocks of kmax rows -- is bit-identical to the single-process backward.

The row ownership comes from the product's own host function (esdp_partition, the one esdp_create_dist
uses; no GPU involved) and the per-rank stage arithmetic from the oracle (ref_stage), so this pins the
partition and the gather layout that libesdp's NCCL path relies on."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads
from helpers import to_oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_15629_b200 as E   # host-only use: esdp_partition
        inst = workloads.cfg1("b", rank1=name.endswith("rank1")) if name.startswith("cfg1") else \
            workloads.random_instance(77, T=5, K=7, S_max=40, rank1=False)
        pr = to_oracle(inst)
        S, A = oracle.dims(pr)
        K, T = inst.K, inst.T
        k_lo, k_cnt, kmax = E.esdp_partition(K, world, rank)
        Vfull = None
        pols = []
        Vs = []
        for t in range(T, 0, -1):
            W, V, pol = oracle.stage(pr, t, k_lo, k_lo + k_cnt, Vfull)
            block = torch.zeros((kmax, S), dtype=torch.float64)
            block[:k_cnt] = torch.from_numpy(V)
            pblock = torch.zeros((kmax, S), dtype=torch.int32)   # gloo has no int16 collectives
            pblock[:k_cnt] = torch.from_numpy(pol.astype(np.int32))
            gathered = torch.zeros((world * kmax, S), dtype=torch.float64)
            pg = torch.zeros((world * kmax, S), dtype=torch.int32)
            dist.all_gather_into_tensor(gathered, block)
            dist.all_gather_into_tensor(pg, pblock)
            Vfull = gathered[:K].numpy().copy()       # rows 0..K-1 in order; padding rows at the end
            Vs.append(Vfull)
            pols.append(pg[:K].numpy().astype(np.int16))
        J = oracle.objective(pr, Vfull)
        if rank == 0:
            ref = oracle.backward(pr)
            ok = (J == ref.J and all(np.array_equal(Vs[T - t], ref.V[t - 1]) for t in range(1, T + 1))
                  and all(np.array_equal(pols[T - t], ref.pol[t - 1]) for t in range(1, T + 1)))
            q.put((ok, J, ref.J))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["cfg1b", "cfg1b-rank1", "random"])
def test_k_partitioned_backward_matches_single(world, name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    ok, J, Jref = q.get(timeout=10)
    assert ok, (J, Jref)


def test_partition_covers_rows_once():
    import paper_2511_15629_b200 as E
    for K in (1, 5, 7, 100, 200):
        for world in (1, 2, 3, 4, 8):
            rows = []
            for r in range(world):
                lo, cnt, m = E.esdp_partition(K, world, r)
                assert 0 <= cnt <= m and lo == min(K, r * m)
                rows += list(range(lo, lo + cnt))
            assert rows == list(range(K))
