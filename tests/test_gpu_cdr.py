"""Config c4 on the GPU (CdrNeumann, real fp64, packed DCT-II/III engine, upwind V) against
the reference's DCT pair (tests/golden/ref_dct.npz) and the plain-C oracle (per iterate)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
import paper_2603_18527_b200 as bs
from oracle import OracleProblem

pytestmark = pytest.mark.gpu
FIELD_TOL = 1e-10
OP_TOL = 1e-13


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def media(n, count, seed=11):
    return bs.make_cdr_instances(bs.CdrSpec(n=n, seed=seed), 0, count)


def oracle(bx, by, sigma, s0, lx=1.0):
    return OracleProblem.cdr(bx, by, sigma, float(s0), lx=lx)


@pytest.mark.parametrize("n", [16, 32, 64])
def test_cdr_transforms_match_reference(gpu, n):
    g = np.load(os.path.join(GOLDEN, "ref_dct.npz"))
    x = g[f"x_{n}x{n}"]
    z = np.zeros((2, n, n))
    with bs.CdrNeumann(z, z, z + 1.0, 1.0) as p:
        xx = np.stack([x.real, x.imag])
        fwd = p.forward_transform(xx)
        inv = p.inverse_transform(xx)
    ref_f, ref_i = g[f"fwd_{n}x{n}"], g[f"inv_{n}x{n}"]
    assert rel(fwd[0], ref_f.real) < OP_TOL and rel(fwd[1], ref_f.imag) < OP_TOL
    assert rel(inv[0], ref_i.real) < OP_TOL and rel(inv[1], ref_i.imag) < OP_TOL


@pytest.mark.parametrize("n", [8, 16, 64, 256])
def test_cdr_operators_match_oracle(gpu, n):
    bx, by, sigma, s0, f = media(n, 3)
    rng = np.random.default_rng(n)
    u = rng.standard_normal(bx.shape)
    with bs.CdrNeumann(bx, by, sigma, s0) as p:
        out = {"A": p.apply_A(u), "V": p.apply_V(u), "Lref": p.apply_Lref(u), "G": p.apply_G(u),
               "born": p.born_residual(u, f), "res": p.residual(u, f), "Vadj": p.apply_V_adjoint(u)}
    for b in range(3):
        o = oracle(bx[b], by[b], sigma[b], s0[b])
        ub, fb = u[b] + 0j, f[b] + 0j
        exp = {"A": o.apply_A(ub), "V": o.apply_V(ub), "Lref": o.apply_Lref(ub), "Vadj": o.apply_V_adjoint(ub),
               "G": o.apply_G(ub), "born": o.born_residual(ub, fb), "res": o.residual(ub, fb)}
        for k, e in exp.items():
            assert np.abs(e.imag).max() < 1e-12 * np.abs(e.real).max()
            # G: the tridiagonal column pass's forward error scales with the column system's
            # conditioning (test_gpu_tri.cdr_tol); the DCT route (BP_COL_DST=1) holds OP_TOL
            tol = max(OP_TOL, 1e-15 * (4.0 * n * n + s0[b]) / s0[b]) if k in ("G", "born") else OP_TOL
            assert rel(out[k][b], e.real) < tol, (k, b)


@pytest.mark.parametrize("n", [16, 64])
def test_cdr_run_per_iterate_matches_oracle(gpu, n):
    bx, by, sigma, s0, f = media(n, 2, seed=5)
    n_snap = 60
    with bs.CdrNeumann(bx, by, sigma, s0) as p:
        r = bs.run(p, bs.ScalarMap(1.0), f, bs.IterationConfig("cbs", 1e-8, 500), n_snap=n_snap)
    for b in range(2):
        o = oracle(bx[b], by[b], sigma[b], s0[b])
        ro = o.run(f[b] + 0j, rtol=1e-8, max_iters=500, n_snap=n_snap)
        t = r.traces[b]
        assert t.terminated == ro.terminated == "converged"
        assert abs(t.iters - ro.iters) <= 1
        k = min(t.iters, ro.iters) + 1
        np.testing.assert_allclose(t.res_l2_rel[:k], ro.res_l2[:k], rtol=1e-9, atol=1e-14)
        np.testing.assert_allclose(t.res_reta_rel[:k], ro.res_reta[:k], rtol=1e-9, atol=1e-14)
        for m in range(1, min(k, n_snap)):
            assert rel(r.snapshots[m, b], ro.snapshots[m].real) < FIELD_TOL, m
        assert rel(r.u[b], ro.u.real) < FIELD_TOL
        assert abs(t.fnorm_l2 - ro.fnorm_l2) < 1e-12 * ro.fnorm_l2
        assert abs(t.fnorm_reta - ro.fnorm_reta) < 1e-12 * ro.fnorm_reta


@pytest.mark.parametrize("metric", ["euclidean", "reta"])
@pytest.mark.parametrize("fmt", ["npbs", "cbs"])
def test_cdr_optimal_scalar_matches_oracle(gpu, metric, fmt):
    """OptimalScalarMap (correction.cpp:22-48) on the CDR family: per-iterate parity over the
    first sweeps, then the full solve's count and field."""
    from oracle import FMT_CBS, FMT_NPBS, MAP_OPTIMAL_SCALAR
    n, n_snap = 64, 20
    bx, by, sigma, s0, f = media(n, 2, seed=6)
    cmap = bs.OptimalScalarMap(metric)
    with bs.CdrNeumann(bx, by, sigma, s0) as p:
        r = bs.run(p, cmap, f, bs.IterationConfig(fmt, 1e-8, 500), n_snap=n_snap)
    for b in range(2):
        ro = oracle(bx[b], by[b], sigma[b], s0[b]).run(
            f[b] + 0j, map_kind=MAP_OPTIMAL_SCALAR, metric=0 if metric == "euclidean" else 1,
            fmt=FMT_CBS if fmt == "cbs" else FMT_NPBS, rtol=1e-8, max_iters=500, n_snap=n_snap)
        t = r.traces[b]
        assert t.terminated == ro.terminated == "converged"
        assert abs(t.iters - ro.iters) <= 1
        k = min(t.iters, ro.iters, n_snap - 1) + 1
        np.testing.assert_allclose(t.res_l2_rel[:k], ro.res_l2[:k], rtol=1e-8, atol=1e-14)
        np.testing.assert_allclose(t.res_reta_rel[:k], ro.res_reta[:k], rtol=1e-8, atol=1e-14)
        for m in range(1, k):
            assert np.abs(ro.snapshots[m].imag).max() < 1e-12 * np.abs(ro.snapshots[m].real).max()
            assert rel(r.snapshots[m, b], ro.snapshots[m].real) < FIELD_TOL, m
        assert rel(r.u[b], ro.u.real) < (FIELD_TOL if t.iters == ro.iters else 1e-7)


def test_cdr_relaxed_gamma_and_u0(gpu):
    n = 32
    bx, by, sigma, s0, f = media(n, 2, seed=8)
    u0 = 0.01 * np.random.default_rng(1).standard_normal(bx.shape)
    with bs.CdrNeumann(bx, by, sigma, s0) as p:
        r = bs.run(p, bs.ScalarMap(0.8), f, bs.IterationConfig("cbs", 1e-9, 400), u0=u0)
    for b in range(2):
        ro = oracle(bx[b], by[b], sigma[b], s0[b]).run(f[b] + 0j, gamma=0.8, rtol=1e-9,
                                                        max_iters=400, u0=u0[b] + 0j)
        assert abs(r.traces[b].iters - ro.iters) <= 1
        assert rel(r.u[b], ro.u.real) < FIELD_TOL


def test_cdr_config_c4_member_full_solve(gpu):
    """One c4 member at the full 1024^2 size: iteration count and final field vs the oracle."""
    bx, by, sigma, s0, f = bs.config_instances("c4", 0, 1)
    cfg = bs.CONFIGS["c4"]
    with bs.CdrNeumann(bx, by, sigma, s0) as p:
        r = bs.run(p, bs.ScalarMap(1.0), f, bs.IterationConfig("cbs", cfg["rtol"], 200))
    ro = oracle(bx[0], by[0], sigma[0], s0[0]).run(f[0] + 0j, rtol=cfg["rtol"], max_iters=200)
    assert r.trace.terminated == ro.terminated == "converged"
    assert abs(r.trace.iters - ro.iters) <= 1
    assert rel(r.u[0], ro.u.real) < FIELD_TOL


def test_cdr_batch_size_independent_properties(gpu):
    """c4 batch at 1024^2 (4 members): each member converges, and a member's result does not
    depend on the batch it is solved in (members are independent units)."""
    bx, by, sigma, s0, f = bs.config_instances("c4", 0, 4)
    cfg = bs.IterationConfig("cbs", 1e-8, 200)
    with bs.CdrNeumann(bx, by, sigma, s0) as p:
        r = bs.run(p, bs.ScalarMap(1.0), f, cfg)
        res = p.residual(r.u, f)
    with bs.CdrNeumann(bx[2:3], by[2:3], sigma[2:3], s0[2:3]) as p1:
        r1 = bs.run(p1, bs.ScalarMap(1.0), f[2:3], cfg)
    for b in range(4):
        assert r.traces[b].terminated == "converged"
        assert 10 <= r.traces[b].iters <= 40
        assert np.linalg.norm(res[b]) / np.linalg.norm(f[b]) < 1e-6
    assert r1.trace.iters == r.traces[2].iters
    assert np.array_equal(r1.u[0], r.u[2])


def test_cdr_errors(gpu):
    z = np.zeros((1, 32, 32))
    with pytest.raises(NotImplementedError):
        bs.CdrNeumann(np.zeros((1, 24, 24)), np.zeros((1, 24, 24)), np.zeros((1, 24, 24)), 1.0)
    with pytest.raises(RuntimeError):  # sigma0 = 0: the (0,0) DCT mode of -Lap_N is zero
        bs.CdrNeumann(z, z, z, 0.0)
    with bs.CdrNeumann(z, z, z + 1.0, 1.0) as p:
        f = np.ones((1, 32, 32))
        with pytest.raises(NotImplementedError):  # real fields: no complex relaxation, no mode-space map
            bs.run(p, bs.FourierDiagMap(np.ones((32, 32), complex)), f)
        with pytest.raises(NotImplementedError):
            bs.run(p, bs.ScalarMap(1.0 + 0.5j), f)
        with pytest.raises(ValueError):
            bs.run(p, bs.ScalarMap(1.0), np.zeros((1, 32, 32)))
        before = bs.run(p, bs.ScalarMap(1.0), f)
        with pytest.raises(ValueError):
            p.set_medium(z, z, z + np.nan, 1.0)
        after = bs.run(p, bs.ScalarMap(1.0), f)  # the rejected medium replaced nothing
        assert np.array_equal(before.u, after.u)


def test_cdr_set_medium_equals_fresh_handle(gpu):
    bx, by, sigma, s0, f = media(64, 2, seed=21)
    bx2, by2, sigma2, s02, _ = media(64, 2, seed=22)
    cfg = bs.IterationConfig("cbs", 1e-8, 300)
    with bs.CdrNeumann(bx, by, sigma, s0) as p:
        bs.run(p, bs.ScalarMap(1.0), f, cfg)
        p.set_medium(bx2, by2, sigma2, s02)
        swapped = bs.run(p, bs.ScalarMap(1.0), f, cfg)
    with bs.CdrNeumann(bx2, by2, sigma2, s02) as q:
        fresh = bs.run(q, bs.ScalarMap(1.0), f, cfg)
    assert np.array_equal(swapped.u, fresh.u)


def test_cdr_repeated_runs_and_operators_after_run(gpu):
    """A second run on the same handle reproduces the first bit for bit (incl. ||G f|| and the
    R_eta trace), and apply_G after a run still acts on every member (regression: the column
    kernel skipped members the previous run had terminated)."""
    bx, by, sigma, s0, f = media(64, 2, seed=5)
    cfg = bs.IterationConfig("cbs", 1e-8, 200)
    with bs.CdrNeumann(bx, by, sigma, s0) as p:
        g0 = p.apply_G(f)
        r1 = bs.run(p, bs.ScalarMap(1.0), f, cfg)
        r2 = bs.run(p, bs.ScalarMap(1.0), f, cfg)
        g1 = p.apply_G(f)
    assert np.array_equal(g0, g1)
    assert np.array_equal(r1.u, r2.u)
    for t1, t2 in zip(r1.traces, r2.traces):
        assert t1.fnorm_reta == t2.fnorm_reta and abs(t1.res_reta_rel[0] - 1.0) < 1e-14
        assert np.array_equal(t1.res_reta_rel, t2.res_reta_rel)
