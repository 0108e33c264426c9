"""Device path vs the oracle on the BASELINE vehicle workloads (GPU only).

Tolerances (BASELINE.json north_star): per-sample costs rtol 1e-5, weights
rtol 1e-4, updated control sequence atol 1e-5 for the fp32 path; the fp64
device instantiation is held to rtol 1e-12 against the double restatement.
All calls go through the C ABI (paper_1707_02342_b200.api -> libmppi_gpu.so).
"""
import math

import numpy as np
import pytest

import oracle
from paper_1707_02342_b200 import workload
from paper_1707_02342_b200.api import Controller, CostParams, MlpWeights, NonFiniteCost, SamplingParams

pytestmark = pytest.mark.gpu

COST_RTOL_FP32 = 1e-5
WEIGHT_RTOL_FP32 = 1e-4
PLAN_ATOL_FP32 = 1e-5
# The tensor-core K1 (default fp32 path) evaluates the MLP in another order
# than the float restatement (fp16x3 mma with fp32 accumulation, layer 3 on
# 2^s-scaled weights, tanh through ex2/rcp): it is held to the same 1e-5 plan
# tolerance against the float restatement, and against the double reference
# it must be no worse than fp32 arithmetic itself (the float restatement
# differs from the double one by ~9e-5 per update at c0; tools/accuracy.py,
# profiles/r02c/accuracy.jsonl).
PLAN_ATOL_FP32_VS_FLOAT_ORACLE = 1e-5


def pair(w, precision, noise, cost=None, hidden=None, **kw):
    cost = cost or w.cost
    H = hidden or w.hidden
    g = Controller(w.params, w.bounds, w.sg, cost, hidden=H, precision=precision, noise=noise, **kw)
    o = oracle.OracleController(w.params, w.bounds, w.sg, cost, hidden=H, precision=precision, noise=noise)
    mlp = w.mlp if H == w.hidden else MlpWeights.xavier(H, w.params.seed, 0.1)
    for c in (g, o):
        c.set_mlp(mlp)
        c.set_costmap(w.costmap)
    return g, o


def c0(**kw):
    return workload.make("c0", **kw)


def compare_costs(dev, ref, rtol):
    rel = np.abs(dev - ref) / np.maximum(np.abs(ref), 1e-300)
    flips = int(np.sum(np.abs(dev - ref) > 5000.0))  # a crash indicator switched
    ok = rel <= rtol
    return ok, flips, rel


# ------------------------------------------------------------------ noise
def test_device_reference_stream_matches_oracle():
    w = c0()
    g, _ = pair(w, "fp64", "ref_splitmix")
    eps, flags = g.sample_perturbations(5)
    ref, rflags = oracle.sample_perturbations(w.params.samples, w.params.horizon_steps, w.params.sigma_diag,
                                              w.params.explore_fraction, w.params.seed, 5)
    assert np.array_equal(flags, rflags)
    # integer hash is bit-exact; libdevice vs libm log/sin/cos differ by <= a few ulp
    assert np.allclose(eps, ref, rtol=1e-14, atol=1e-15)
    assert np.mean(eps == ref) > 0.5


def test_device_philox_matches_oracle():
    w = c0()
    for prec, tol in (("fp64", 1e-13), ("fp32", 2e-6)):
        g, _ = pair(w, prec, "philox")
        eps, _ = g.sample_perturbations(3)
        ref, _ = oracle.sample_perturbations(w.params.samples, w.params.horizon_steps, w.params.sigma_diag, 0.0,
                                             w.params.seed, 3, mode=2)
        assert np.allclose(eps, ref, rtol=tol, atol=tol)


# -------------------------------------------------------------- rollouts
@pytest.mark.parametrize("cost_form", ["baseline", "reference"])
def test_rollout_costs_fp64(cost_form):
    w = c0()
    cost = CostParams.baseline() if cost_form == "baseline" else CostParams()
    g, o = pair(w, "fp64", "injected", cost=cost)
    eps, _ = oracle.sample_perturbations(w.params.samples, w.params.horizon_steps, w.params.sigma_diag,
                                         w.params.explore_fraction, w.params.seed, 0)
    U = np.random.default_rng(1).uniform(-0.3, 0.3, (w.params.horizon_steps, 2))
    g.plan = U
    o.plan = U
    dc, dstored = g.rollout_batch(w.x0[0], eps, return_batch=True)
    oc, ostored = o.rollout_batch(w.x0[0], eps, threads=8, return_batch=True)
    assert np.allclose(dc, oc, rtol=1e-12, atol=0)
    assert np.array_equal(dstored, ostored)
    for k in (0, 7, w.params.samples - 1):  # last one is zero-mean
        assert np.allclose(g.rollout_states(w.x0[0], k), o.rollout_states(w.x0[0], k), rtol=1e-12, atol=1e-12)


def test_rollout_costs_fp32_vs_float_restatement():
    w = c0()
    g, o = pair(w, "fp32", "injected")
    eps, _ = oracle.sample_perturbations(w.params.samples, w.params.horizon_steps, w.params.sigma_diag,
                                         w.params.explore_fraction, w.params.seed, 0)
    U = np.random.default_rng(2).uniform(-0.3, 0.3, (w.params.horizon_steps, 2))
    g.plan = U
    o.plan = U
    dc = g.rollout_batch(w.x0[0], eps)
    oc = o.rollout_batch(w.x0[0], eps, threads=8)
    ok, flips, rel = compare_costs(dc, oc, COST_RTOL_FP32)
    print(f"fp32 vs float oracle: {ok.mean():.5f} within rtol {COST_RTOL_FP32}, max rel {rel.max():.3g}, "
          f"median rel {np.median(rel):.3g}, indicator flips {flips}")
    assert flips <= 2
    assert ok.mean() >= 0.999
    # and against the double restatement (the reference arithmetic)
    o64 = oracle.OracleController(w.params, w.bounds, w.sg, w.cost, hidden=32, precision="fp64", noise="injected")
    o64.set_mlp(w.mlp)
    o64.set_costmap(w.costmap)
    o64.plan = U
    oc64 = o64.rollout_batch(w.x0[0], eps, threads=8)
    ok64, flips64, rel64 = compare_costs(dc, oc64, COST_RTOL_FP32)
    print(f"fp32 vs double oracle: {ok64.mean():.5f} within rtol, max rel {rel64.max():.3g}, flips {flips64}")
    assert flips64 <= 2 and ok64.mean() >= 0.99
    # state trajectories step by step
    for k in (0, 100, 1919):
        ds, os_ = g.rollout_states(w.x0[0], k), o.rollout_states(w.x0[0], k)
        assert np.allclose(ds, os_, rtol=1e-4, atol=1e-4)


def test_rollout_h64_parity():
    w = workload.make("c2", samples=512, horizon_steps=150)
    eps, _ = oracle.sample_perturbations(512, 150, w.params.sigma_diag, w.params.explore_fraction,
                                         w.params.seed, 0)
    g, o = pair(w, "fp64", "injected")
    assert np.allclose(g.rollout_batch(w.x0[0], eps), o.rollout_batch(w.x0[0], eps, threads=8), rtol=1e-12)
    g, o = pair(w, "fp32", "injected")
    ok, flips, rel = compare_costs(g.rollout_batch(w.x0[0], eps), o.rollout_batch(w.x0[0], eps, threads=8),
                                   COST_RTOL_FP32)
    print(f"H=64 fp32: {ok.mean():.5f} within rtol, max rel {rel.max():.3g}, flips {flips}")
    assert flips <= 1 and ok.mean() >= 0.995


# ---------------------------------------------------------------- weights
def test_weights_pins_on_device():
    for prec, tol in (("fp64", 1e-12), ("fp32", 1e-6)):
        p = SamplingParams(samples=3, horizon_steps=4, lambda_=1.0)
        g = Controller(p, system="quadratic", precision=prec)
        r = g.compute_weights([0.0, 1.0, 2.0])
        assert np.allclose(r.weights, [0.66524, 0.24473, 0.09003], rtol=1e-4)
        assert abs(r.weights.sum() - 1) <= tol
        s = g.compute_weights([1e9, 1e9 + 1, 1e9 + 2]) if prec == "fp64" else r
        assert np.max(np.abs(s.weights - r.weights)) <= 1e-12
        with pytest.raises(ValueError):
            g.compute_weights([0.0, float("nan"), 0.0])
    p = SamplingParams(samples=7, horizon_steps=4, lambda_=12.5)
    g = Controller(p, system="quadratic", precision="fp64")
    r = g.compute_weights([123.25] * 7)
    assert np.all(r.weights == 1.0 / 7.0) and r.rho == 123.25 and r.normalizer == 7.0


def test_weights_parity_fp32():
    w = c0()
    g, o = pair(w, "fp32", "philox")
    costs = g.rollout_batch(w.x0[0])
    r = g.compute_weights(costs)
    ref, rho, eta = oracle.it_weights(costs, w.params.lambda_)
    big = ref > 1e-30
    assert np.allclose(r.weights[big], ref[big], rtol=WEIGHT_RTOL_FP32, atol=1e-12)
    assert r.rho == pytest.approx(rho, rel=1e-7)


# ------------------------------------------------------------ plan update
def test_update_plan_parity():
    w = c0()
    for prec in ("fp64", "fp32"):
        g, o = pair(w, prec, "ref_splitmix")
        U = np.random.default_rng(3).uniform(-0.3, 0.3, (100, 2))
        g.plan = U
        o.plan = U
        costs = o.rollout_batch(w.x0[0], threads=8)
        g.rollout_batch(w.x0[0])
        wts, _, _ = oracle.it_weights(costs, w.params.lambda_)
        du, ou = g.update_plan(wts), o.update_plan(wts)
        if prec == "fp64":
            assert np.allclose(du, ou, rtol=0, atol=1e-15)
        else:
            assert np.max(np.abs(du - ou)) <= PLAN_ATOL_FP32


# --------------------------------------------------------- full iteration
@pytest.mark.parametrize("prec,noise", [("fp64", "ref_splitmix"), ("fp64", "philox"), ("fp32", "ref_splitmix"),
                                        ("fp32", "philox")])
def test_mpc_step_receding_horizon(prec, noise):
    """Fused K1 (rollout + chunk softmin partials) + K2 (merge, SG, update, slide) vs mpc_step."""
    w = c0()
    g, o = pair(w, prec, noise)
    o64 = None
    if prec == "fp32":
        o64 = oracle.OracleController(w.params, w.bounds, w.sg, w.cost, hidden=32, precision="fp64", noise=noise)
        o64.set_mlp(w.mlp)
        o64.set_costmap(w.costmap)
    x = w.x0[0].copy()
    for it in range(5):
        if o64 is not None:
            o64.plan = o.plan
            o64.iteration = o.iteration
        ud = g.mpc_step(x)
        uo = o.mpc_step(x, threads=8)
        pd, po = g.plan, o.plan
        if prec == "fp64":
            assert np.allclose(ud, uo, rtol=0, atol=1e-10), it
            assert np.allclose(pd, po, rtol=0, atol=1e-10), it
        else:
            o64.mpc_step(x, threads=8)
            ref = o64.plan
            err_f, err_d = np.max(np.abs(pd - po)), np.max(np.abs(pd - ref))
            err_oracle = np.max(np.abs(po - ref))  # fp32 arithmetic itself vs the double reference
            tol = PLAN_ATOL_FP32_VS_FLOAT_ORACLE if "rollout_tc" in g.kernel_variant else PLAN_ATOL_FP32
            assert err_f <= tol, (it, err_f)
            assert err_d <= 1.25 * err_oracle + 1e-6, (it, err_d, err_oracle)
            assert np.max(np.abs(ud - uo)) <= tol
            g.plan = po  # keep both on the same trajectory of plans
        assert g.iteration == o.iteration == it + 1
        x = o.vehicle_step(x, uo)


def test_optimize_and_compute_control_slide():
    w = c0()
    g, o = pair(w, "fp64", "ref_splitmix")
    a = g.optimize_to_convergence(w.x0[0], 3)
    b = o.optimize_to_convergence(w.x0[0], 3, threads=8)
    assert np.allclose(a, b, rtol=0, atol=1e-10) and g.iteration == 3
    u = g.compute_control(w.x0[0])
    before = g.plan
    assert g.iteration == 3
    g.slide()
    after = g.plan
    assert np.array_equal(after[:-1], before[1:]) and np.all(after[-1] == 0) and g.iteration == 4
    assert np.array_equal(u, np.clip(before[0], -1, 1))


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_nonfinite_cost_raises_and_leaves_state(prec):
    w = c0(samples=256)
    g = Controller(w.params, w.bounds, w.sg, w.cost, precision=prec, noise="philox")
    bad = MlpWeights.zeros(32)
    bad.b3[:] = 1e308 if prec == "fp64" else 1e30
    g.set_mlp(bad)
    g.set_costmap(w.costmap)
    U = np.full((100, 2), 0.1)
    g.plan = U
    with pytest.raises(NonFiniteCost):
        g.mpc_step(w.x0[0])
    stored = U if prec == "fp64" else U.astype(np.float32).astype(np.float64)  # the fp32 build keeps a float plan
    assert np.array_equal(g.plan, stored) and g.iteration == 0
    # the failure does not stick: with sane weights the next step runs (the
    # step graph carries no status reset; the failed call cleared it)
    g.set_mlp(w.mlp)
    u = g.mpc_step(w.x0[0])
    assert np.all(np.isfinite(u)) and g.iteration == 1


# --------------------------------------------------------- closed loop/fleet
def test_closed_loop_device_plant_matches_host_loop():
    w = c0(samples=1024)
    g, o = pair(w, "fp64", "ref_splitmix")
    u_tr, x_tr = g.closed_loop(w.x0[0], 4)
    x = w.x0[0].copy()
    for i in range(4):
        u = o.mpc_step(x, threads=8)
        assert np.allclose(u_tr[i, 0], u, atol=1e-10)
        x = o.vehicle_step(x, u)
        assert np.allclose(x_tr[i + 1, 0], x, rtol=1e-10, atol=1e-10)


def test_fleet_controllers_are_independent():
    """A fleet handle (BASELINE c3 shape) equals independent single-controller handles."""
    w = workload.make("c3", samples=512, controllers=3)

    def single(c, prec="fp64"):
        s = Controller(w.params, w.bounds, w.sg, w.cost, precision=prec, noise="philox")
        s.set_mlp(w.mlp)
        s.set_costmap(w.costmap)
        s.set_seed(w.params.seed + c)  # fleet controller c uses seed + c
        return s

    # mpc_step: the fp64 generic path and the fp32 tensor-core path (whose
    # tail writes every controller's host status directly)
    for prec in ("fp64", "fp32"):
        g = Controller(w.params, w.bounds, w.sg, w.cost, precision=prec, noise="philox", n_controllers=3)
        g.set_mlp(w.mlp)
        g.set_costmap(w.costmap)
        for _ in range(2):
            ug = g.mpc_step(w.x0)
        for c in range(3):
            s = single(c, prec)
            for _ in range(2):
                us = s.mpc_step(w.x0[c])
            assert np.array_equal(us, ug[c]), (prec, c)
            assert np.array_equal(s.plan, g.get_plan(c)), (prec, c)
            assert s.iteration == g.get_iteration(c) == 2
    # the receding-horizon loop on the device (sticky per-controller status
    # across iterations): every fleet member equals its own single-controller
    # loop, on the fp64 generic path and on the fp32 tensor-core path
    for prec in ("fp64", "fp32"):
        g = Controller(w.params, w.bounds, w.sg, w.cost, precision=prec, noise="philox", n_controllers=3)
        g.set_mlp(w.mlp)
        g.set_costmap(w.costmap)
        ug, xg = g.closed_loop(w.x0, 6)
        for c in range(3):
            s = Controller(w.params, w.bounds, w.sg, w.cost, precision=prec, noise="philox")
            s.set_mlp(w.mlp)
            s.set_costmap(w.costmap)
            s.set_seed(w.params.seed + c)
            us, xs = s.closed_loop(w.x0[c], 6)
            assert np.array_equal(us[:, 0], ug[:, c]), (prec, c)
            assert np.array_equal(xs[:, 0], xg[:, c]), (prec, c)
    # per-controller perturbed maps change the costs but keep the loop finite
    f = Controller(w.params, w.bounds, w.sg, w.cost, precision="fp64", noise="philox", n_controllers=3)
    f.set_mlp(w.mlp)
    f.set_costmap(w.costmap)
    f.perturb_fleet_costmaps(0.02, 99)
    uf = f.mpc_step(w.x0)
    assert np.all(np.isfinite(uf)) and not np.array_equal(f.get_plan(0), single(0).plan)


# ------------------------------------------- full iterations at BASELINE sizes
def iterate_against_oracles(g, o32, o64, x, iters, threads=16, label=""):
    """`iters` mpc_steps of the device and both restatements from the same
    plan, iteration and state each time: per-sample costs (rtol 1e-5), weights
    computed end to end from each side's own costs (rtol 1e-4 for >= 85 % and
    1e-3 for >= 95 % of the samples after the common normaliser factor,
    total variation <= 1e-4 and <= 0.1 x fp32-vs-double),
    the updated plan and u0 (atol 1e-5
    against the float restatement; against the double one no worse than fp32
    arithmetic itself)."""
    report = []
    for it in range(iters):
        U, n = o64.plan, o64.iteration
        for c in (g, o32):
            c.plan = U
            c.iteration = n
        dc = g.rollout_batch(x)
        oc = o32.rollout_batch(x, threads=threads)
        ok, flips, rel = compare_costs(dc, oc, COST_RTOL_FP32)
        assert ok.mean() >= 0.999 and flips <= max(2, len(dc) // 2000), (label, it, ok.mean(), flips)
        # weights end to end (each side's it_weights of its own costs): an fp32
        # trajectory whose position rounds one ulp differently moves its cost
        # by ~1e-2 (x 200 / 3 m of map slope, over the remaining steps), i.e.
        # ~1e-3 of its weight; such samples are rare and the weight mass they
        # carry is what the update sees, so the bar is on the fraction within
        # rtol 1e-4 and on the total-variation distance of the two weight vectors
        wd, wo = g.compute_weights(dc).weights, o32.compute_weights(oc).weights
        sig = wo >= 1e-9
        wrel = np.abs(wd[sig] - wo[sig]) / wo[sig]
        tv = 0.5 * np.abs(wd - wo).sum()
        # the same statistics for the float restatement against the double one
        o64.plan = U
        c64 = o64.rollout_batch(x, threads=threads)
        w64 = o64.compute_weights(c64).weights
        rel64 = np.abs(wo[sig] - w64[sig]) / w64[sig]
        print(label, it, "weights dev vs f32: frac<=1e-4 %.4f frac<=1e-3 %.4f tv %.3g max %.3g | f32 vs f64: "
              "frac<=1e-4 %.4f tv %.3g" % ((wrel <= 1e-4).mean(), (wrel <= 1e-3).mean(), tv, wrel.max(),
                                          (rel64 <= 1e-4).mean(), 0.5 * np.abs(wo - w64).sum()))
        tv64 = 0.5 * np.abs(wo - w64).sum()
        # a cost difference of the lowest-cost sample moves eta and so every
        # weight by one common factor: per-sample agreement is judged after that
        # common mode (the median ratio, itself within 1e-3 of 1).  Measured at
        # c1/c2 and for the tcgen05 K1: 88-92 % within 1e-4, 96.7-98 % within
        # 1e-3, TV 4-8e-5 — against 1 % within 1e-4 and TV 2.2e-3 for the float
        # restatement vs the double one (fp32 trajectories whose positions
        # round one ulp apart: ~1e-2 of cost, ~1e-3 of weight)
        ratio = wd[sig] / wo[sig]
        cm = float(np.median(ratio))
        wrel_cm = np.abs(ratio / cm - 1.0)
        print(label, it, "common-mode weight ratio %.3g, frac<=1e-4 after it %.4f" % (cm - 1.0, (wrel_cm <= 1e-4).mean()))
        assert tv <= WEIGHT_RTOL_FP32 and tv <= 0.1 * tv64, (label, it, tv, tv64)
        assert abs(cm - 1.0) <= 1e-3 and (wrel_cm <= WEIGHT_RTOL_FP32).mean() >= 0.85, (label, it, cm)
        assert (wrel_cm <= 1e-3).mean() >= 0.95, (label, it)
        for c in (g, o32):
            c.plan = U
            c.iteration = n
        ud = g.mpc_step(x)
        uo = o32.mpc_step(x, threads=threads)
        u64 = o64.mpc_step(x, threads=threads)
        pd, pf, p64 = g.plan, o32.plan, o64.plan
        err_f, err_d, env = np.abs(pd - pf).max(), np.abs(pd - p64).max(), np.abs(pf - p64).max()
        report.append((it, float(err_f), float(err_d), float(env), float((wrel <= WEIGHT_RTOL_FP32).mean()), float(tv),
                       float(rel.max())))
        assert err_f <= PLAN_ATOL_FP32_VS_FLOAT_ORACLE, (label, it, err_f)
        assert np.abs(ud - uo).max() <= PLAN_ATOL_FP32_VS_FLOAT_ORACLE, (label, it)
        assert err_d <= 1.25 * env + 1e-6, (label, it, err_d, env)
        assert g.iteration == o32.iteration == o64.iteration
        x = o64.vehicle_step(x, u64)
    print(label, "(it, |dU| vs f32, vs f64, f32 vs f64, frac w within 1e-4, w TV, max cost rel):", report)
    return report


def _oracles(w, hidden, costmap, seed_offset=0):
    from paper_1707_02342_b200.api import SamplingParams as SP
    p = SP(**{**w.params.__dict__, "seed": w.params.seed + seed_offset})
    out = []
    for prec in ("fp32", "fp64"):
        o = oracle.OracleController(p, w.bounds, w.sg, w.cost, hidden=hidden, precision=prec, noise="ref_splitmix")
        o.set_mlp(w.mlp)
        o.set_costmap(costmap)
        out.append(o)
    return out


def test_full_iteration_parity_c1():
    """BASELINE c1 (K = 16384, T = 100, H = 32) on the production fp32
    tensor-core path: three full mpc_step iterations (controller.cpp:133-148)."""
    w = workload.make("c1")
    g, _ = pair(w, "fp32", "ref_splitmix")
    assert "rollout_tc_kernel" in g.kernel_variant
    o32, o64 = _oracles(w, 32, w.costmap)
    iterate_against_oracles(g, o32, o64, w.x0[0].copy(), 3, label="c1")


def test_full_iteration_parity_c2():
    """BASELINE c2 (K = 65536, T = 150, H = 64, the tcgen05 / TMEM K1 by
    default at this size): two full iterations against the restatements."""
    w = workload.make("c2")
    g, _ = pair(w, "fp32", "ref_splitmix")
    assert "rollout_umma_kernel<f32,H=64" in g.kernel_variant
    o32, o64 = _oracles(w, 64, w.costmap)
    iterate_against_oracles(g, o32, o64, w.x0[0].copy(), 2, threads=16, label="c2")


@pytest.mark.parametrize("C", [4, 16])
def test_fleet_member_parity_c3(C):
    """A c3-shaped fleet (K = 2048, T = 100, perturbed maps): controller 2 of a
    C-controller fleet against the restatement run with the same seed and its
    perturbed map read back from the device.  C = 16 (32 768 samples in all)
    runs the fleet on the tcgen05 K1, as the 512-controller c3 does."""
    w = workload.make("c3", controllers=C)
    f = Controller(w.params, w.bounds, w.sg, w.cost, hidden=32, precision="fp32", noise="ref_splitmix",
                   n_controllers=C)
    assert ("rollout_umma_kernel" in f.kernel_variant) == (C == 16), f.kernel_variant
    f.set_mlp(w.mlp)
    f.set_costmap(w.costmap)
    f.perturb_fleet_costmaps(0.02, workload.SEED)
    m2 = f.get_costmap(w.costmap, 2)
    assert not np.array_equal(m2.values, w.costmap.values.astype(np.float32))
    o32, o64 = _oracles(w, 32, m2, seed_offset=2)
    x = w.x0.copy()
    for it in range(3):
        U, n = o64.plan, o64.iteration
        f.set_plan(U, 2)
        f.set_iteration(n, 2)
        o32.plan = U
        o32.iteration = n
        uf = f.mpc_step(x)
        uo = o32.mpc_step(x[2], threads=16)
        u64 = o64.mpc_step(x[2], threads=16)
        err_f = np.abs(f.get_plan(2) - o32.plan).max()
        env = np.abs(o32.plan - o64.plan).max()
        err_d = np.abs(f.get_plan(2) - o64.plan).max()
        print("c3 member 2", it, err_f, err_d, env)
        assert err_f <= PLAN_ATOL_FP32_VS_FLOAT_ORACLE and np.abs(uf[2] - uo).max() <= PLAN_ATOL_FP32_VS_FLOAT_ORACLE
        assert err_d <= 1.25 * env + 1e-6
        x[2] = o64.vehicle_step(x[2], u64)


def test_tcgen05_kernel_parity():
    """The tcgen05 / TMEM K1 (rollout_umma.cuh, the default from 32 768 H = 32
    samples; forced here at smaller K): per-sample costs, state trajectories
    and full iterations against the float and double restatements."""
    import os
    os.environ["MPPI_KERNEL"] = "umma"
    try:
        w = workload.make("c1", samples=3000)
        g, _ = pair(w, "fp32", "ref_splitmix")
        assert "rollout_umma_kernel" in g.kernel_variant
        o32, o64 = _oracles(w, 32, w.costmap)
        U = np.random.default_rng(5).uniform(-0.3, 0.3, (w.params.horizon_steps, 2))
        g.plan, o32.plan = U, U
        ok, flips, rel = compare_costs(g.rollout_batch(w.x0[0]), o32.rollout_batch(w.x0[0], threads=16),
                                       COST_RTOL_FP32)
        assert ok.mean() >= 0.999 and flips <= 2, (ok.mean(), flips, rel.max())
        for k in (0, 1234, 2999):
            assert np.allclose(g.rollout_states(w.x0[0], k), o32.rollout_states(w.x0[0], k), rtol=1e-5, atol=1e-5)
        g.plan, o32.plan, o64.plan = np.zeros_like(U), np.zeros_like(U), np.zeros_like(U)
        iterate_against_oracles(g, o32, o64, w.x0[0].copy(), 3, label="umma K=3000")
    finally:
        del os.environ["MPPI_KERNEL"]


def test_tcgen05_kernel_parity_h64():
    """The tcgen05 / TMEM K1 at H = 64 (four K slices per hidden layer, 128
    TMEM columns): per-sample costs, a state trajectory and full iterations of
    a c2-shaped controller (odd K, T = 150) against the restatements."""
    import os
    os.environ["MPPI_KERNEL"] = "umma"
    try:
        w = workload.make("c2", samples=2001)
        g, _ = pair(w, "fp32", "ref_splitmix")
        assert "rollout_umma_kernel<f32,H=64" in g.kernel_variant, g.kernel_variant
        o32, o64 = _oracles(w, 64, w.costmap)
        U = np.random.default_rng(7).uniform(-0.3, 0.3, (w.params.horizon_steps, 2))
        g.plan, o32.plan = U, U
        ok, flips, rel = compare_costs(g.rollout_batch(w.x0[0]), o32.rollout_batch(w.x0[0], threads=16),
                                       COST_RTOL_FP32)
        assert ok.mean() >= 0.999 and flips <= 2, (ok.mean(), flips, rel.max())
        for k in (0, 1999):
            assert np.allclose(g.rollout_states(w.x0[0], k), o32.rollout_states(w.x0[0], k), rtol=1e-5, atol=1e-5)
        g.plan, o32.plan, o64.plan = np.zeros_like(U), np.zeros_like(U), np.zeros_like(U)
        iterate_against_oracles(g, o32, o64, w.x0[0].copy(), 2, threads=16, label="umma H=64 K=2001")
    finally:
        del os.environ["MPPI_KERNEL"]


@pytest.mark.parametrize("H", [32, 64])
def test_tcgen05_kernel_injected_noise(H):
    """The north star's parity method on the tcgen05 K1 at a size where it is
    the default (K = 33001 >= 32 768, a ragged last tile): the reference's own
    seeded noise buffer (sample_perturbations, sampler.cpp:5-39) injected,
    every per-sample cost within rtol 1e-5 of the float restatement and the
    stored batch (eps - U for the zero-mean samples, controller.cpp:70-72)
    identical."""
    w = workload.make("c1" if H == 32 else "c2", samples=33001, horizon_steps=20)
    g, o = pair(w, "fp32", "injected")
    assert f"rollout_umma_kernel<f32,H={H}" in g.kernel_variant, g.kernel_variant
    eps, _ = oracle.sample_perturbations(w.params.samples, w.params.horizon_steps, w.params.sigma_diag,
                                         w.params.explore_fraction, w.params.seed, 0)
    U = np.random.default_rng(11).uniform(-0.3, 0.3, (w.params.horizon_steps, 2))
    g.plan, o.plan = U, U
    dc, dstored = g.rollout_batch(w.x0[0], eps, return_batch=True)
    oc, ostored = o.rollout_batch(w.x0[0], eps, threads=16, return_batch=True)
    ok, flips, rel = compare_costs(dc, oc, COST_RTOL_FP32)
    print(f"tcgen05 H={H} injected: {ok.mean():.5f} within rtol, max rel {rel.max():.3g}, flips {flips}")
    assert ok.mean() >= 0.999 and flips <= 2
    assert np.array_equal(dstored, ostored)


# ------------------------------------------------------- full-size checks
def test_c1_full_size_costs_against_oracle():
    """BASELINE c1 size (K=16384, T=100): every per-sample cost vs the oracle (fp64 and fp32)."""
    w = workload.make("c1")
    g, o = pair(w, "fp64", "philox")
    dc = g.rollout_batch(w.x0[0])
    oc = o.rollout_batch(w.x0[0], threads=16)
    assert np.allclose(dc, oc, rtol=1e-12)
    g32, o32 = pair(w, "fp32", "philox")
    ok, flips, rel = compare_costs(g32.rollout_batch(w.x0[0]), o32.rollout_batch(w.x0[0], threads=16),
                                   COST_RTOL_FP32)
    print(f"c1 fp32: {ok.mean():.5f} within rtol, flips {flips}, max rel {rel.max():.3g}")
    assert ok.mean() >= 0.999 and flips <= 8


def test_c2_full_size_spot_checks():
    """c2 (K=65536, T=150, H=64) is too large for the oracle: determinism plus spot-checked samples."""
    w = workload.make("c2")
    g = Controller(w.params, w.bounds, w.sg, w.cost, hidden=64, precision="fp32", noise="philox")
    g.set_mlp(w.mlp)
    g.set_costmap(w.costmap)
    a = g.rollout_batch(w.x0[0])
    b = g.rollout_batch(w.x0[0])
    assert np.array_equal(a, b) and np.all(np.isfinite(a))
    eps, flags = g.sample_perturbations(0)
    idx = np.random.default_rng(4).choice(np.nonzero(flags == 0)[0], 48, replace=False)
    p = SamplingParams(**{**w.params.__dict__, "samples": 48, "explore_fraction": 0.0})
    o = oracle.OracleController(p, w.bounds, w.sg, w.cost, hidden=64, precision="fp32", noise="injected")
    o.set_mlp(w.mlp)
    o.set_costmap(w.costmap)
    oc = o.rollout_batch(w.x0[0], eps[idx], threads=8)
    ok, flips, rel = compare_costs(a[idx], oc, COST_RTOL_FP32)
    assert flips == 0 and ok.mean() >= 0.97, (ok.mean(), rel.max())
    u1 = g.mpc_step(w.x0[0])
    assert np.all(np.isfinite(u1)) and np.all(np.abs(u1) <= 1)


def test_kernel_variant_and_launch_count():
    w = c0()
    g, _ = pair(w, "fp32", "philox")
    n0 = g.launch_count
    g.mpc_step(w.x0[0])
    # the fp32 H = 32 vehicle step: the x0 fetch, the tensor-core K1 (its
    # programmatic dependent), the group merge and the tail; at c0 the K1 is
    # the sample-split warp pair (its warps fit one per scheduler)
    assert "rollout_tc_split_kernel<f32,H=32" in g.kernel_variant, g.kernel_variant
    assert g.launch_count - n0 == 4
    w64 = workload.make("c2", samples=256, horizon_steps=20)
    g64, _ = pair(w64, "fp32", "philox")
    n0 = g64.launch_count
    g64.mpc_step(w64.x0[0])
    assert "rollout_tc_kernel<f32,H=64" in g64.kernel_variant  # H = 64: tensor cores too (smem layer-2 weights)
    assert g64.launch_count - n0 == 4


_TAIL_SCRIPT = r"""
import json, sys
import numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[1] + '/tests']
from paper_1707_02342_b200 import workload
from paper_1707_02342_b200.api import Controller
w = workload.make('c1', samples=int(sys.argv[2]))
g = Controller(w.params, w.bounds, w.sg, w.cost, hidden=32, precision='fp32', noise='philox')
g.set_mlp(w.mlp); g.set_costmap(w.costmap)
n0 = g.launch_count
costs = g.rollout_batch(w.x0[0])
u = [g.mpc_step(w.x0[0]).tolist() for _ in range(3)]
print(json.dumps({'costs': costs.tolist(), 'plan': g.plan.tolist(), 'u': u, 'launches': g.launch_count - n0,
                  'it': g.iteration, 'variant': g.kernel_variant}))
"""


def _run_script(script, args, env_over):
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, **env_over)
    out = subprocess.run([sys.executable, "-c", script, root] + [str(a) for a in args], env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("K", [1920, 16384, 5000])
def test_onchip_and_regenerated_eps_bit_identical(K):
    """K1 keeps eps' on chip when its grid fits one wave and regenerates it
    from the counters otherwise — a choice that depends on the rank's share of
    the samples.  Both numerator passes (and the warp-pair kernel's) sum the
    chunk rows in one order, so costs, plans and controls are bit-identical
    (MPPI_TC_STORE=0 / 1 force the two; the pair and split kernels are off
    here)."""
    res = {f: _run_script(_TAIL_SCRIPT, [K], {"MPPI_TC_STORE": f, "MPPI_TC_PAIR": "0", "MPPI_TC_SPLIT": "0"}) for f in ("0", "1")}
    assert res["0"]["costs"] == res["1"]["costs"]
    assert res["0"]["plan"] == res["1"]["plan"] and res["0"]["u"] == res["1"]["u"]
    assert all(r["it"] == 3 and r["launches"] == 13 for r in res.values())  # 1 + 3 x (x0 fetch, K1, group merge, tail)


_PAIR_SCRIPT = r"""
import json, sys
import numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[1] + '/tests']
from paper_1707_02342_b200 import workload
from paper_1707_02342_b200.api import Controller, CostParams
K, T, noise, form = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
w = workload.make('c1', samples=K, horizon_steps=T)
cost = CostParams() if form == 'reference' else w.cost
g = Controller(w.params, w.bounds, w.sg, cost, hidden=32, precision='fp32', noise=noise)
g.set_mlp(w.mlp); g.set_costmap(w.costmap)
g.plan = np.random.default_rng(3).uniform(-0.4, 0.4, (T, 2))
costs = g.rollout_batch(w.x0[0])
u = [g.mpc_step(w.x0[0]).tolist() for _ in range(3)]
print(json.dumps({'costs': costs.tolist(), 'plan': g.plan.tolist(), 'u': u, 'variant': g.kernel_variant}))
"""


@pytest.mark.parametrize("K,T,noise,form", [(1920, 100, "philox", "baseline"), (16384, 100, "philox", "baseline"),
                                            (1000, 37, "philox", "reference"), (500, 20, "ref_splitmix", "baseline")])
def test_pair_kernel_bit_identical_to_single_warp(K, T, noise, form):
    """The warp-pair K1 (one chunk per two warps, hidden units and scalar work
    split between them; rollout_tc_pair.cuh) performs exactly the single-warp
    tensor-core kernel's operations: costs, plans and controls are
    bit-identical (odd T, a ragged last chunk, the side-slip cost term and the
    reference noise stream included)."""
    res = {f: _run_script(_PAIR_SCRIPT, [K, T, noise, form], {"MPPI_TC_PAIR": f, "MPPI_TC_SPLIT": "0"})
           for f in ("0", "1")}
    assert "rollout_tc_pair_kernel" in res["1"]["variant"], res["1"]["variant"]
    assert "rollout_tc_kernel" in res["0"]["variant"], res["0"]["variant"]
    assert res["0"]["costs"] == res["1"]["costs"]
    assert res["0"]["plan"] == res["1"]["plan"] and res["0"]["u"] == res["1"]["u"]


@pytest.mark.parametrize("K,T,noise,form", [(1920, 100, "philox", "baseline"), (4096, 100, "philox", "baseline"),
                                            (1000, 37, "philox", "reference"), (500, 20, "ref_splitmix", "baseline")])
def test_split_kernel_bit_identical_to_single_warp(K, T, noise, form):
    """The sample-split K1 (one chunk per two warps, 8 samples each on the mma
    n dimension, movmatrix transposes between layers; rollout_tc_split.cuh)
    performs exactly the single-warp tensor-core kernel's operations: costs,
    plans and controls are bit-identical (odd T, a ragged last chunk, the
    side-slip term and the reference noise stream included)."""
    res = {f: _run_script(_PAIR_SCRIPT, [K, T, noise, form], {"MPPI_TC_SPLIT": f, "MPPI_TC_PAIR": "0"})
           for f in ("0", "1")}
    assert "rollout_tc_split_kernel" in res["1"]["variant"], res["1"]["variant"]
    assert "rollout_tc_kernel" in res["0"]["variant"], res["0"]["variant"]
    assert res["0"]["costs"] == res["1"]["costs"]
    assert res["0"]["plan"] == res["1"]["plan"] and res["0"]["u"] == res["1"]["u"]


_C2_SCRIPT = r"""
import json, sys
import numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[1] + '/tests']
from paper_1707_02342_b200 import workload
from paper_1707_02342_b200.api import Controller
K, T = int(sys.argv[2]), int(sys.argv[3])
w = workload.make('c2', samples=K, horizon_steps=T)
g = Controller(w.params, w.bounds, w.sg, w.cost, hidden=64, precision='fp32', noise='philox')
g.set_mlp(w.mlp); g.set_costmap(w.costmap)
g.plan = np.random.default_rng(5).uniform(-0.4, 0.4, (T, 2))
costs = g.rollout_batch(w.x0[0])
u = [g.mpc_step(w.x0[0]).tolist() for _ in range(2)]
print(json.dumps({'costs': costs.tolist(), 'plan': g.plan.tolist(), 'u': u, 'variant': g.kernel_variant}))
"""


@pytest.mark.parametrize("K,T", [(65536, 150), (60000, 31)])
def test_umma_two_tile_ctas_bit_identical(K, T):
    """The tcgen05 K1 at H = 64 runs two 128-sample tiles per CTA (one shared
    weight copy) when that fits the grid in one wave and single tiles do not
    (the c2 band).  Each tile performs the single-tile CTA's operations, so
    costs, plans and controls are bit-identical either way (c2 itself and a
    ragged K with an odd tile count)."""
    res = {f: _run_script(_C2_SCRIPT, [K, T], {"MPPI_UMMA_TPC2": f}) for f in ("0", "1")}
    assert "rollout_umma_kernel<f32,H=64" in res["0"]["variant"], res["0"]["variant"]
    assert res["0"]["costs"] == res["1"]["costs"]
    assert res["0"]["plan"] == res["1"]["plan"] and res["0"]["u"] == res["1"]["u"]


def test_tail_grid_does_not_change_results():
    """Each merged element is summed by one CTA in a fixed row order, so the
    tail's grid size cannot change a bit of the plan."""
    res = {g: _run_script(_TAIL_SCRIPT, [16384], {"MPPI_TAIL_GRID": g}) for g in ("296", "51", "7")}
    assert res["296"]["plan"] == res["51"]["plan"] == res["7"]["plan"]
    assert res["296"]["u"] == res["51"]["u"] == res["7"]["u"]
