"""The N>1 sample-shard protocol on CPU, world_size 2 over gloo.

The device path (handle.cuh set_comm / enqueue_exchange, epilogue.cuh) shards
the K samples into fixed 32-sample chunks, gives rank r a contiguous chunk
range, reduces each chunk to softmin partials (rho_c, eta_c, num_c[T][2])
relative to the chunk minimum, all-gathers the partials (one NCCL call per
iteration) and merges them on every rank in global chunk order.  This test
runs that protocol with torch.distributed/gloo between two processes, the
oracle as the per-sample arithmetic, and checks that (1) both ranks hold the
identical merged update, bit for bit, (2) it equals the world_size-1 merge bit
for bit, and (3) it equals the reference update_plan (controller.cpp:118-131)
to rounding.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

CHUNK = 32


def chunk_range(n_chunks, rank, world):
    """Mirror of Handle::set_comm: contiguous ceil(n/world) chunks per rank."""
    per = (n_chunks + world - 1) // world
    return min(n_chunks, rank * per), min(n_chunks, (rank + 1) * per)


def chunk_partials(costs, stored, lam, c):
    """rollout_ws_kernel tail: per-chunk (rho, eta, num) relative to the chunk min."""
    s = costs[c * CHUNK:(c + 1) * CHUNK]
    rho = s.min()
    w = np.exp(-(s - rho) / lam)
    num = np.einsum("k,kct->tc", w, stored[c * CHUNK:(c + 1) * CHUNK])
    return rho, w.sum(), num


def merge(parts, lam):
    """epilogue_kernel merge: global chunk order, log-sum-exp rescale."""
    rho = min(p[0] for p in parts)
    scale = [np.exp(-(p[0] - rho) / lam) for p in parts]
    eta = sum(s * p[1] for s, p in zip(scale, parts))
    num = sum(s * p[2] for s, p in zip(scale, parts))
    return num / eta


def problem():
    import oracle
    from paper_1707_02342_b200.api import ControlBounds, SamplingParams
    K, T = 256, 20
    p = SamplingParams(samples=K, horizon_steps=T, dt=0.05, sigma_diag=(0.04, 0.09), lambda_=1.0, gamma=0.1,
                       explore_fraction=0.05, seed=11)
    cs = oracle.OracleController(p, ControlBounds((-10.0, -10.0), (10.0, 10.0)), None, None, system="quadratic",
                                 precision="fp64", noise="ref_splitmix", quad_cost_scale=1.0)
    cs.plan = np.random.default_rng(0).uniform(-0.5, 0.5, (T, 2))
    costs, stored = cs.rollout_batch(np.array([1.0, -0.5]), threads=2, return_batch=True)
    return cs, p, costs, stored


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, p, costs, stored = problem()
        n_chunks = (p.samples + CHUNK - 1) // CHUNK
        lo, hi = chunk_range(n_chunks, rank, world)
        mine = [chunk_partials(costs, stored, p.lambda_, c) for c in range(lo, hi)]
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)  # the one exchange per iteration
        parts = [x for r in gathered for x in r]
        assert len(parts) == n_chunks
        q.put((rank, merge(parts, p.lambda_)))
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_chunk_ranges_cover_every_sample_once():
    for n, world in ((512, 1), (512, 2), (60, 8), (513, 8), (8192, 8)):
        seen = []
        for r in range(world):
            lo, hi = chunk_range(n, r, world)
            seen += list(range(lo, hi))
        assert seen == list(range(n))


def test_two_rank_exchange_matches_single_rank_and_reference(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert np.array_equal(res[0], res[1])  # every rank holds the same update

    cs, p, costs, stored = problem()
    n_chunks = p.samples // CHUNK
    single = merge([chunk_partials(costs, stored, p.lambda_, c) for c in range(n_chunks)], p.lambda_)
    assert np.array_equal(single, res[0])  # bit-identical to one GPU

    U = cs.plan.copy()
    ref = cs.update_plan(cs.compute_weights(costs))  # no SG filter: U' = U + agg
    assert np.allclose(U + res[0], ref, rtol=1e-12, atol=1e-14)
