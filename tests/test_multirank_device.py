"""The library's own sample-shard path on ONE B200 (GPU only).

Each rank is a handle of the library: `set_comm_local` makes handles[r] rank
r of N, with the partition, the fixed-group merge, the exchange of group rows
and the tail of the product path (handle.cuh, group.cuh, tail.cuh).  The only
difference from the NCCL path is the transport: peer copies of the group rows
instead of ncclAllGather, and `step_local` runs every rank's rollout + group
merge, synchronises, then every rank's exchange + tail, so no kernel of one
rank ever waits for another's.

The reference guarantee this must match is that results do not depend on how
the samples are partitioned (parallel_for_chunks, parallel.hpp:11-29;
test_controller.cpp:199-217): u0 and the plan must be bit-identical on every
rank and to the single-GPU handle, for N = 2, 4, 8, ragged K and K smaller
than the group count (ranks with no samples).
"""
import os

import numpy as np
import pytest

from paper_1707_02342_b200 import workload
from paper_1707_02342_b200.api import Controller, InvalidArgument, Unsupported

pytestmark = pytest.mark.gpu


def make(w, prec="fp32", noise="philox", **kw):
    c = Controller(w.params, w.bounds, w.sg, w.cost, hidden=w.hidden, precision=prec, noise=noise, **kw)
    c.set_mlp(w.mlp)
    c.set_costmap(w.costmap)
    return c


def run_pair(w, N, prec="fp32", noise="philox", steps=3):
    single = make(w, prec, noise)
    ranks = [make(w, prec, noise) for _ in range(N)]
    Controller.set_comm_local(ranks)
    x = w.x0[0].copy()
    for it in range(steps):
        us = single.mpc_step(x)
        ul = Controller.step_local(ranks, x)
        for r in range(N):
            assert np.array_equal(ul[r], us), (N, it, r, ul[r], us)
        ps = single.plan
        for r in range(N):
            assert np.array_equal(ranks[r].plan, ps), (N, it, r)
            assert ranks[r].iteration == it + 1
        x = x + 0.01  # a moving state
    return single, ranks


@pytest.mark.parametrize("K", [16384, 5000, 1920, 100])
@pytest.mark.parametrize("N", [2, 4, 8])
def test_local_shards_bit_identical_to_one_gpu_fp32(K, N):
    """Tensor-core path: c1 size (the single GPU with branch-form stage stores, the ranks with
    predicated ones), ragged K, c0 size, and
    K = 100 (7 chunks for 8 groups: empty groups and ranks without samples)."""
    w = workload.make("c1", samples=K)
    single, ranks = run_pair(w, N)
    info = [r.shard_info for r in ranks]
    assert [i["rank"] for i in info] == list(range(N)) and all(i["world_size"] == N for i in info)
    assert info[0]["chunk_lo"] == 0 and info[-1]["chunk_hi"] == info[0]["chunks"]
    for a, b in zip(info, info[1:]):
        assert a["chunk_hi"] == b["chunk_lo"]


@pytest.mark.parametrize("N", [2, 4])
def test_local_shards_bit_identical_fp64_generic(N):
    w = workload.make("c0", samples=3000)
    run_pair(w, N, prec="fp64", noise="ref_splitmix", steps=2)


def test_local_shards_ffma2_and_h64():
    os.environ["MPPI_KERNEL"] = "ws"  # read at handle creation: the FFMA2 warp-specialised K1
    try:
        run_pair(workload.make("c1", samples=4096), 4, steps=2)
    finally:
        del os.environ["MPPI_KERNEL"]
    run_pair(workload.make("c2", samples=8192, horizon_steps=30), 2, steps=2)  # H = 64 tensor-core K1


def test_set_comm_rejections_leave_handle_unchanged():
    w = workload.make("c1", samples=4096)
    a, b = make(w), make(w)
    with pytest.raises(Unsupported):
        a.set_comm(0, 3, None)  # 3 does not divide the 8 groups
    with pytest.raises(InvalidArgument):
        a.set_comm(2, 2, None)
    with pytest.raises(Unsupported):
        Controller.set_comm_local([a, b, make(w)])
    assert a.shard_info["world_size"] == 1 and a.shard_info["chunk_hi"] == a.shard_info["chunks"]
    assert np.array_equal(a.mpc_step(w.x0[0]), b.mpc_step(w.x0[0]))
    assert np.array_equal(a.plan, b.plan)
    other = make(workload.make("c1", samples=2048))
    with pytest.raises(InvalidArgument):
        Controller.set_comm_local([a, other])  # configurations differ
    fleet = make(workload.make("c3", samples=256, controllers=2), n_controllers=2)
    with pytest.raises(Unsupported):
        fleet.set_comm(0, 2, None)


def test_fleet_controller_offset_is_the_global_index():
    """A fleet split over ranks: controllers [2, 4) of a 4-controller fleet on
    a handle with controller_offset = 2 draw the same noise and the same
    perturbed maps as in the whole fleet, so every rank count is one workload."""
    w = workload.make("c3", samples=512, controllers=4)
    whole = make(w, n_controllers=4)
    whole.perturb_fleet_costmaps(0.02, workload.SEED)
    part = make(w, n_controllers=2, controller_offset=2)
    part.perturb_fleet_costmaps(0.02, workload.SEED)
    for _ in range(2):
        uw = whole.mpc_step(w.x0)
        up = part.mpc_step(w.x0[2:4])
        assert np.array_equal(uw[2:4], up)
    for c in range(2):
        assert np.array_equal(whole.get_plan(2 + c), part.get_plan(c))


@pytest.mark.parametrize("N", [2, 8])
def test_local_shards_bit_identical_tcgen05_kernel(N):
    """From 32 768 samples the H = 32 K1 is the tcgen05 / TMEM kernel (128
    samples per CTA): the sharded iteration is still bit-identical to one GPU."""
    w = workload.make("c1", samples=70000)
    single, ranks = run_pair(w, N, steps=2)
    assert "rollout_umma_kernel" in single.kernel_variant
