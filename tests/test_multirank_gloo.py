"""The N>1 sample-shard protocol on CPU, world_size 2 over gloo.

The device path shards one controller's K samples as follows (group.cuh,
handle.cuh set_comm / enqueue_exchange, tail.cuh):

* K1 reduces every chunk of samples (16 on the tensor-core path, 128 on the
  generic path) to softmin partials (rho_c, eta_c, num_c[T][2]) relative to
  the chunk minimum;
* the chunks form G fixed groups (G = 8 * 2^j, a function of the chunk count
  alone); each group is merged into one row in a fixed order;
* rank r of N owns groups [r G/N, (r+1) G/N) — the partition comes from the
  library itself here (mppi_gpu_shard_plan, a host-only C-ABI function, no
  device needed) — and the exchange is ONE all-gather of the G/N group rows
  per rank (a real tensor all_gather over gloo in this test);
* every rank merges the G rows in group order.

With the oracle as the per-sample arithmetic this checks that (1) the ranks'
chunk ranges cover every sample once, (2) both ranks hold the identical merged
update, bit for bit, (3) it equals the world_size-1 run bit for bit, (4) it
equals the reference update_plan (controller.cpp:118-131) to rounding, and
(5) the exchange is G x (4 + 2T) doubles for the whole job.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1707_02342_b200 import api

HEADER = 4


def chunk_row(costs, stored, lam, lo, hi):
    """K1's chunk reduction: (rho, eta, bad, 0, num[T][2] flattened t-major)."""
    s = costs[lo:hi]
    rho = s.min()
    w = np.exp(-(s - rho) / lam)
    num = np.einsum("k,kct->tc", w, stored[lo:hi]).reshape(-1)
    return np.concatenate([[rho, w.sum(), 0.0, 0.0], num])


def group_row(rows, lam):
    """group_merge_kernel: rho_g = min, eight stripes (rows q, q+8, ...) summed
    sequentially, then a balanced tree over the stripes."""
    if len(rows) == 0:
        r = np.zeros(rows.shape[1])
        r[0] = np.inf
        return r
    rho = rows[:, 0].min()
    sc = np.exp(-(rows[:, 0] - rho) / lam)
    stripes = []
    for q in range(8):
        acc = np.zeros(rows.shape[1])
        for r in range(q, len(rows), 8):
            acc = sc[r] * rows[r] + acc
        stripes.append(acc)
    v = ((stripes[0] + stripes[1]) + (stripes[2] + stripes[3])) + ((stripes[4] + stripes[5]) + (stripes[6] + stripes[7]))
    v[0], v[2], v[3] = rho, 0.0, 0.0
    return v


def final_merge(groups, lam):
    """The tail: rho = min over group rows, rows scaled and summed in group order; agg = num / eta."""
    rho = groups[:, 0].min()
    sc = np.exp(-(groups[:, 0] - rho) / lam)
    acc = np.zeros(groups.shape[1])
    for g in range(len(groups)):
        acc = sc[g] * groups[g] + acc
    return acc[HEADER:] / acc[1]


def problem():
    import oracle
    from paper_1707_02342_b200.api import ControlBounds, SamplingParams
    K, T = 1000, 20  # 63 chunks of 16: ragged last chunk, uneven groups
    p = SamplingParams(samples=K, horizon_steps=T, dt=0.05, sigma_diag=(0.04, 0.09), lambda_=1.0, gamma=0.1,
                       explore_fraction=0.05, seed=11)
    cs = oracle.OracleController(p, ControlBounds((-10.0, -10.0), (10.0, 10.0)), None, None, system="quadratic",
                                 precision="fp64", noise="ref_splitmix", quad_cost_scale=1.0)
    cs.plan = np.random.default_rng(0).uniform(-0.5, 0.5, (T, 2))
    costs, stored = cs.rollout_batch(np.array([1.0, -0.5]), threads=2, return_batch=True)
    return cs, p, costs, stored


CHUNK = 16


def rank_update(p, costs, stored, rank, world, exchange):
    plan = api.shard_plan(p.samples, CHUNK, rank, world)
    n_chunks, G = plan["chunks"], plan["groups"]
    stride = HEADER + 2 * p.horizon_steps
    groups = np.zeros((G, stride))
    for g in range(plan["group_lo"], plan["group_hi"]):
        c0 = (g * n_chunks) // G
        c1 = ((g + 1) * n_chunks) // G
        rows = np.array([chunk_row(costs, stored, p.lambda_, c * CHUNK, min(p.samples, (c + 1) * CHUNK))
                         for c in range(c0, c1)]).reshape(-1, stride)
        groups[g] = group_row(rows, p.lambda_)
    groups = exchange(groups, plan)
    return final_merge(groups, p.lambda_), plan


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, p, costs, stored = problem()

        def allgather(groups, plan):
            per = plan["groups"] // world
            mine = torch.from_numpy(np.ascontiguousarray(groups[plan["group_lo"]:plan["group_hi"]]))
            out = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(out, mine)  # the one exchange per iteration
            full = torch.cat(out).numpy()
            assert full.shape[0] == per * world
            return full

        upd, plan = rank_update(p, costs, stored, rank, world, allgather)
        q.put((rank, upd, plan))
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("K,chunk", [(1920, 16), (16384, 16), (1048576, 32), (5000, 16), (64, 16), (1, 16),
                                     (65536, 16), (1920, 128)])
def test_shard_plan_covers_every_chunk_once(K, chunk):
    for world in (1, 2, 4, 8):
        seen, groups = [], []
        for r in range(world):
            pl = api.shard_plan(K, chunk, r, world)
            assert pl["groups"] % 8 == 0 and pl["groups"] * 128 >= pl["chunks"]
            seen += list(range(pl["chunk_lo"], pl["chunk_hi"]))
            groups += list(range(pl["group_lo"], pl["group_hi"]))
        n = (K + chunk - 1) // chunk
        assert seen == list(range(n))
        assert groups == list(range(pl["groups"]))
        # the group count (hence the merge order) does not depend on the rank count
        assert pl["groups"] == api.shard_plan(K, chunk, 0, 1)["groups"]


def test_shard_plan_rejects_non_dividing_world():
    with pytest.raises(api.Unsupported):
        api.shard_plan(16384, 16, 0, 3)
    with pytest.raises(api.InvalidArgument):
        api.shard_plan(16384, 16, 2, 2)


def test_two_rank_exchange_matches_single_rank_and_reference(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in procs:
        r, upd, plan = q.get(timeout=240)
        res[r] = (upd, plan)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert np.array_equal(res[0][0], res[1][0])  # every rank holds the same update
    assert res[0][1]["chunk_hi"] == res[1][1]["chunk_lo"]  # contiguous halves

    cs, p, costs, stored = problem()
    single, plan1 = rank_update(p, costs, stored, 0, 1, lambda g, pl: g)
    assert np.array_equal(single, res[0][0])  # bit-identical to one GPU
    # the exchange: G x (4 + 2T) doubles for the whole job
    assert plan1["groups"] * (HEADER + 2 * p.horizon_steps) * 8 == 8 * 44 * 8

    U = cs.plan.copy()
    ref = cs.update_plan(cs.compute_weights(costs))  # no SG filter: U' = U + agg
    assert np.allclose(U + res[0][0].reshape(-1, 2), ref, rtol=1e-12, atol=1e-14)
