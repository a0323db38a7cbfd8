"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle and the reference.

Tolerances (BASELINE.json north_star): fp64 complex fields within 1e-10 relative L2 per
iterate, identical iteration counts to the stated tolerance within +-1.  Transforms and
operators are held to 1e-13 (they are single fp64 passes).
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN
import paper_2603_18527_b200 as bs
from oracle import (MAP_FOURIER_DIAG, MAP_OPTIMAL_SCALAR, MAP_POINTWISE, MAP_SCALAR, Oracle,
                    OracleProblem)

pytestmark = pytest.mark.gpu

FIELD_TOL = 1e-10   # per-iterate relative L2 (north_star)
OP_TOL = 1e-13      # single transform / operator pass


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def rand_field(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def instance(n, batch=1, ppw=8.0, contrast=0.5, sigma=3.0, seed=0, **kw):
    spec = bs.InstanceSpec(n=n, ppw=ppw, contrast=contrast, sigma_cells=sigma, seed=seed, **kw)
    return bs.make_instances(spec, 0, batch)


SIZES = [8, 16, 32, 64, 128, 256, 512]


# ------------------------------------------------------------------ transforms
@pytest.mark.parametrize("n", SIZES)
def test_transforms_match_oracle(gpu, n):
    k2, f, k0, eta = instance(n, batch=2)
    rng = np.random.default_rng(n)
    x = rand_field(rng, k2.shape)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        fw = p.forward_transform(x)
        iv = p.inverse_transform(x)
        back = p.inverse_transform(fw)
    for b in range(2):
        assert rel(fw[b], Oracle.forward_dst(x[b])) < OP_TOL
        assert rel(iv[b], Oracle.inverse_dst(x[b])) < OP_TOL
        assert rel(back[b], x[b]) < 1e-12


def test_transforms_match_scipy_goldens(gpu):
    g = np.load(os.path.join(GOLDEN, "dst_scipy.npz"))
    for shape in ["15x15", "7x7", "31x31"]:
        x, y = g["x_" + shape], g["y_" + shape]
        n = x.shape[0]
        with bs.HelmholtzDirichlet(np.ones_like(x), 1.0, 1.0) as p:
            assert rel(p.forward_transform(x), y) < OP_TOL, shape


def test_unsupported_shapes_raise(gpu):
    # any 2-D shape up to 4095 per side runs (power-of-two kernels or the any-shape path,
    # test_gpu_generic.py); longer sides are not implemented
    for shape in [(4096, 4096), (8191, 8191), (5000, 12)]:
        with pytest.raises(NotImplementedError):
            bs.HelmholtzDirichlet(np.ones(shape, np.complex128), 1.0, 1.0)


# ------------------------------------------------------------------ operators
@pytest.mark.parametrize("n", SIZES)
def test_operators_match_oracle(gpu, n):
    k2, f, k0, eta = instance(n, batch=2, seed=n)
    rng = np.random.default_rng(100 + n)
    u = rand_field(rng, k2.shape)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        got = dict(A=p.apply_A(u), V=p.apply_V(u), VH=p.apply_V_adjoint(u), L=p.apply_Lref(u),
                   G=p.apply_G(u), born=p.born_residual(u, f), res=p.residual(u, f))
    for b in range(2):
        o = OracleProblem(k2[b], k0[b], eta[b])
        assert rel(got["A"][b], o.apply_A(u[b])) < 1e-15
        assert rel(got["V"][b], o.apply_V(u[b])) < 1e-15
        assert rel(got["VH"][b], o.apply_V_adjoint(u[b])) < 1e-15
        assert rel(got["res"][b], o.residual(u[b], f[b])) < 1e-15
        assert rel(got["L"][b], o.apply_Lref(u[b])) < OP_TOL
        assert rel(got["G"][b], o.apply_G(u[b])) < OP_TOL
        assert rel(got["born"][b], o.born_residual(u[b], f[b])) < OP_TOL


@pytest.mark.parametrize("n", [16, 32])
def test_operators_match_reference_fixtures(gpu, n):
    g = np.load(os.path.join(GOLDEN, f"ref_ops_n{n}.npz"))
    x, f = g["x"], g["f"]
    with bs.HelmholtzDirichlet(g["k2"], float(g["k0"]), float(g["eta"])) as p:
        assert rel(p.apply_A(x), g["A"]) < 1e-15
        assert rel(p.apply_V(x), g["V"]) < 1e-15
        assert rel(p.apply_V_adjoint(x), g["VH"]) < 1e-15
        assert rel(p.apply_Lref(x), g["Lref"]) < OP_TOL
        assert rel(p.apply_G(x), g["G"]) < OP_TOL
        assert rel(p.born_residual(x, f), g["born"]) < OP_TOL
        assert rel(p.residual(x, f), g["res"]) < 1e-15
        assert rel(p.forward_transform(x), g["fwd"]) < OP_TOL
        assert rel(p.inverse_transform(x), g["inv"]) < OP_TOL


def test_identities_at_full_size(gpu):
    """Size-independent properties at config-1 size (511^2, batch 4): key identity,
    splitting, two-sided Green inverse, round trip, linearity (proj/src/verify.cpp:168-216)."""
    k2, f, k0, eta = instance(512, batch=4, seed=5)
    rng = np.random.default_rng(9)
    r = rand_field(rng, k2.shape)
    s = rand_field(rng, k2.shape)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        lhs = r - p.apply_G(p.apply_V(r))
        rhs = p.apply_G(p.apply_A(r))
        lin = p.apply_G(2.0 * r - 3j * s) - (2.0 * p.apply_G(r) - 3j * p.apply_G(s))
        for b in range(4):
            assert np.linalg.norm(lhs[b] - rhs[b]) / np.linalg.norm(r[b]) < 1e-12
            assert np.linalg.norm(lin[b]) / np.linalg.norm(r[b]) < 1e-13
        assert rel(p.apply_Lref(r) - p.apply_V(r), p.apply_A(r)) < 1e-12
        assert rel(p.apply_Lref(p.apply_G(r)), r) < 1e-12
        assert rel(p.apply_G(p.apply_Lref(r)), r) < 1e-12
        assert rel(p.inverse_transform(p.forward_transform(r)), r) < 1e-12


# ------------------------------------------------------------------ the driver
def _oracle_run(k2, f, k0, eta, cmap, rtol, max_iters, u0=None, n_snap=0):
    o = OracleProblem(k2, k0, eta)
    if isinstance(cmap, bs.PointwiseMap):
        return o.run(f, map_kind=MAP_POINTWISE, rtol=rtol, max_iters=max_iters, u0=u0, n_snap=n_snap)
    if isinstance(cmap, bs.OptimalScalarMap):
        return o.run(f, map_kind=MAP_OPTIMAL_SCALAR, metric=0 if cmap.metric == "euclidean" else 1,
                     rtol=rtol, max_iters=max_iters, u0=u0, n_snap=n_snap)
    if isinstance(cmap, bs.FourierDiagMap):
        return o.run(f, map_kind=MAP_FOURIER_DIAG, m=cmap.m, rtol=rtol, max_iters=max_iters, u0=u0,
                     n_snap=n_snap)
    return o.run(f, map_kind=MAP_SCALAR, gamma=cmap.gamma, rtol=rtol, max_iters=max_iters, u0=u0,
                 n_snap=n_snap)


def assert_run_parity(gpu_trace, u_gpu, ref, field_tol=FIELD_TOL):
    assert gpu_trace.terminated == ref.terminated
    assert abs(gpu_trace.iters - ref.iters) <= 1
    k = min(gpu_trace.iters, ref.iters) + 1
    np.testing.assert_allclose(gpu_trace.res_l2_rel[:k], ref.res_l2[:k], rtol=1e-8, atol=1e-13)
    np.testing.assert_allclose(gpu_trace.res_reta_rel[:k], ref.res_reta[:k], rtol=1e-8, atol=1e-13)
    assert abs(gpu_trace.fnorm_l2 - ref.fnorm_l2) <= 1e-13 * ref.fnorm_l2
    assert abs(gpu_trace.fnorm_reta - ref.fnorm_reta) <= 1e-12 * ref.fnorm_reta
    if gpu_trace.iters == ref.iters:
        assert rel(u_gpu, ref.u) < field_tol


RUN_FIXTURES = {
    "c0like_n32_scalar": lambda g: bs.ScalarMap(complex(g["gamma"])),
    "n32_pointwise": lambda g: bs.PointwiseMap(),
    "n32_scalar_maxiters": lambda g: bs.ScalarMap(complex(g["gamma"])),
    "n16_optl2": lambda g: bs.OptimalScalarMap("euclidean"),
    "n16_optreta": lambda g: bs.OptimalScalarMap("reta"),
}


@pytest.mark.parametrize("name", sorted(RUN_FIXTURES))
def test_run_matches_reference_fixture(gpu, name):
    g = np.load(os.path.join(GOLDEN, f"ref_run_{name}.npz"))
    cfg = bs.IterationConfig(rtol=float(g["rtol"]), max_iters=int(g["max_iters"]))
    with bs.HelmholtzDirichlet(g["k2"], float(g["k0"]), float(g["eta"])) as p:
        res = bs.run(p, RUN_FIXTURES[name](g), g["f"], cfg)
    tr = res.trace
    assert tr.terminated == str(g["terminated"])
    assert abs(tr.iters - int(g["iters"])) <= 1
    k = min(tr.iters, int(g["iters"])) + 1
    np.testing.assert_allclose(tr.res_l2_rel[:k], g["res_l2"][:k], rtol=1e-8, atol=1e-13)
    np.testing.assert_allclose(tr.res_reta_rel[:k], g["res_reta"][:k], rtol=1e-8, atol=1e-13)
    if tr.iters == int(g["iters"]):
        assert rel(res.u, g["u"]) < FIELD_TOL


def _fd_map(n, seed=5):
    """random-init FourierDiag multiplier near the identity (the NPBS M_theta stand-in)"""
    rng = np.random.default_rng(seed)
    nd = n - 1
    return bs.FourierDiagMap(1.0 + 0.3 * (rng.standard_normal((nd, nd)) + 1j * rng.standard_normal((nd, nd))))


@pytest.mark.parametrize("n,cmap", [(32, bs.ScalarMap(1.0)), (64, bs.PointwiseMap()),
                                    (128, bs.ScalarMap(1.0)), (256, bs.PointwiseMap()),
                                    (64, bs.OptimalScalarMap("euclidean")),
                                    (128, bs.OptimalScalarMap("reta")),
                                    (64, "fd"), (512, bs.OptimalScalarMap("euclidean"))])
def test_per_iterate_parity(gpu, n, cmap):
    """u^m for m = 0..K within 1e-10 relative L2 of the oracle's iterates."""
    if cmap == "fd":
        cmap = _fd_map(n)
    k2, f, k0, eta = instance(n, ppw=10.0, contrast=0.3, seed=2)
    K = 40 if n < 512 else 12
    cfg = bs.IterationConfig(rtol=1e-12, max_iters=K)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        res = bs.run(p, cmap, f, cfg, n_snap=K + 1)
    ref = _oracle_run(k2[0], f[0], k0[0], eta[0], cmap, 1e-12, K, n_snap=K + 1)
    assert res.trace.iters == ref.iters == K
    for m in range(1, K + 1):
        assert rel(res.snapshots[m], ref.snapshots[m]) < FIELD_TOL, m
    assert_run_parity(res.trace, res.u, ref)


def test_config0_full_solve(gpu):
    """BASELINE config 0: 127^2, contrast 0.3, 10 ppw, gamma = 1, rtol 1e-6, to convergence."""
    cfg0 = bs.CONFIGS["c0"]
    k2, f, k0, eta = bs.make_instances(cfg0["spec"], 0, 1)
    cfg = bs.IterationConfig(rtol=cfg0["rtol"], max_iters=20000)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        res = bs.run(p, bs.ScalarMap(1.0), f, cfg)
    ref = _oracle_run(k2[0], f[0], k0[0], eta[0], bs.ScalarMap(1.0), cfg0["rtol"], 20000)
    assert ref.terminated == "converged"
    assert_run_parity(res.trace, res.u[0] if res.u.ndim == 3 else res.u, ref)


def test_config1_members_truncated(gpu):
    """BASELINE config 1 at full size (511^2, contrast 0.5, 8 ppw, pointwise map): the first
    members of the seeded batch over a fixed window of sweeps vs the oracle."""
    Oracle.set_threads(os.cpu_count() or 8)
    k2, f, k0, eta = bs.config_instances("c1", 0, 2)
    K = 60
    cfg = bs.IterationConfig(rtol=1e-6, max_iters=K)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        res = bs.run(p, bs.PointwiseMap(), f, cfg)
    for b in range(2):
        ref = _oracle_run(k2[b], f[b], k0[b], eta[b], bs.PointwiseMap(), 1e-6, K)
        assert res.traces[b].iters == ref.iters == K
        assert_run_parity(res.traces[b], res.u[b], ref)


@pytest.mark.slow
def test_config1_member_full_length(gpu):
    """BASELINE config 1, member 1 (511^2, pointwise map) solved to rtol 1e-6: the GPU and the
    oracle take the same number of sweeps (4708 with this seed) and end on the same iterate."""
    Oracle.set_threads(os.cpu_count() or 8)
    k2, f, k0, eta = bs.config_instances("c1", 1, 1)
    cfg = bs.IterationConfig(rtol=1e-6, max_iters=20000)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        res = bs.run(p, bs.PointwiseMap(), f, cfg)
    ref = _oracle_run(k2[0], f[0], k0[0], eta[0], bs.PointwiseMap(), 1e-6, 20000)
    t = res.traces[0]
    assert t.terminated == ref.terminated == "converged"
    assert t.iters == ref.iters
    assert np.linalg.norm(res.u[0] - ref.u) / np.linalg.norm(ref.u) < 1e-10


def test_batch_members_independent(gpu):
    """Each member of a batch iterates and terminates on its own: a batch run equals the
    members run one at a time (bit-for-bit: same kernels, same reduction order)."""
    k2, f, k0, eta = instance(64, batch=3, ppw=10.0, contrast=0.3, seed=4)
    f[1] *= 1e3  # different scale; relative criteria unchanged
    cfg = bs.IterationConfig(rtol=1e-8, max_iters=3000)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        batch = bs.run(p, bs.ScalarMap(1.0), f, cfg)
    for b in range(3):
        with bs.HelmholtzDirichlet(k2[b:b + 1], k0[b:b + 1], eta[b:b + 1]) as p1:
            one = bs.run(p1, bs.ScalarMap(1.0), f[b:b + 1], cfg)
        assert one.traces[0].iters == batch.traces[b].iters
        assert np.array_equal(one.u[0], batch.u[b])
        assert np.array_equal(one.traces[0].res_l2_rel, batch.traces[b].res_l2_rel)


def test_terminations(gpu):
    k2, f, k0, eta = instance(32, ppw=10.0, contrast=0.3, seed=6)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        # diverged: over-relaxed scalar map
        cfgd = bs.IterationConfig(rtol=1e-6, max_iters=5000)
        d = bs.run(p, bs.ScalarMap(3.0), f, cfgd)
        rd = _oracle_run(k2[0], f[0], k0[0], eta[0], bs.ScalarMap(3.0), 1e-6, 5000)
        assert d.trace.terminated == rd.terminated == "diverged"
        assert abs(d.trace.iters - rd.iters) <= 1
        # stagnated: a tolerance below the fp64 floor
        s = bs.run(p, bs.ScalarMap(1.0), f, bs.IterationConfig(rtol=1e-17, max_iters=5000))
        rs = _oracle_run(k2[0], f[0], k0[0], eta[0], bs.ScalarMap(1.0), 1e-17, 5000)
        assert s.trace.terminated == rs.terminated == "stagnated"
        assert abs(s.trace.iters - rs.iters) <= 25
        # converged at entry 0: start from the (converged) solution
        c = bs.run(p, bs.ScalarMap(1.0), f, bs.IterationConfig(rtol=1e-6, max_iters=100), u0=s.u)
        assert c.trace.terminated == "converged" and c.trace.iters == 0
        assert np.array_equal(c.u, s.u)
        # max_iters = 1
        one = bs.run(p, bs.ScalarMap(1.0), f, bs.IterationConfig(rtol=1e-6, max_iters=1))
        r1 = _oracle_run(k2[0], f[0], k0[0], eta[0], bs.ScalarMap(1.0), 1e-6, 1)
        assert one.trace.terminated == "max_iters" and one.trace.iters == 1
        assert_run_parity(one.trace, one.u, r1)


def test_warm_start_matches_oracle(gpu):
    k2, f, k0, eta = instance(64, ppw=10.0, contrast=0.3, seed=8)
    rng = np.random.default_rng(3)
    u0 = 1e-3 * rand_field(rng, k2.shape)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        res = bs.run(p, bs.PointwiseMap(), f, bs.IterationConfig(rtol=1e-7, max_iters=4000), u0=u0)
    ref = _oracle_run(k2[0], f[0], k0[0], eta[0], bs.PointwiseMap(), 1e-7, 4000, u0=u0[0])
    assert_run_parity(res.trace, res.u, ref)


def test_errors_follow_reference(gpu):
    k2, f, k0, eta = instance(16)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        with pytest.raises(ValueError, match="zero source"):
            bs.run(p, bs.ScalarMap(), np.zeros_like(f))
        with pytest.raises(ValueError, match="rtol"):
            bs.run(p, bs.ScalarMap(), f, bs.IterationConfig(rtol=0.0))
        with pytest.raises(ValueError, match="max_iters"):
            bs.run(p, bs.ScalarMap(), f, bs.IterationConfig(max_iters=0))
        with pytest.raises(ValueError, match="metric"):
            bs.run(p, bs.OptimalScalarMap("bogus"), f)
        with pytest.raises(ValueError, match="shape"):
            p.apply_G(np.zeros((3, 3), np.complex128))
    with pytest.raises(ValueError, match="eta"):
        bs.HelmholtzDirichlet(k2, k0, -1.0)
    with pytest.raises(ValueError, match="finite"):
        bad = k2.copy()
        bad[0, 3, 3] = np.nan
        bs.HelmholtzDirichlet(bad, k0, eta)


def test_rejected_medium_leaves_handle_intact(gpu):
    """set_medium validates the new k2 on the device before replacing anything: a rejected
    medium leaves the previous one (and its run result) in place."""
    k2, f, k0, eta = instance(32, batch=2, seed=12)
    cfg = bs.IterationConfig(rtol=1e-6, max_iters=300)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        before = bs.run(p, bs.ScalarMap(1.0), f, cfg)
        bad = k2.copy()
        bad[1, 5, 7] = np.inf
        with pytest.raises(ValueError, match="finite"):
            p.set_medium(bad, k0 * 1.1, eta * 2.0)
        after = bs.run(p, bs.ScalarMap(1.0), f, cfg)
        assert np.array_equal(before.u, after.u)
        # an accepted medium takes effect (same as a fresh handle)
        k2b, _, k0b, etab = instance(32, batch=2, seed=13)
        p.set_medium(k2b, k0b, etab)
        swapped = bs.run(p, bs.ScalarMap(1.0), f, cfg)
    with bs.HelmholtzDirichlet(k2b, k0b, etab) as q:
        fresh = bs.run(q, bs.ScalarMap(1.0), f, cfg)
    assert np.array_equal(swapped.u, fresh.u)


def test_cbs_equals_npbs_on_gpu(gpu):
    k2, f, k0, eta = instance(64, ppw=10.0, contrast=0.3, seed=1)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        a = bs.run(p, bs.ScalarMap(1.0), f, bs.IterationConfig(format="cbs", rtol=1e-12, max_iters=50))
        b = bs.run(p, bs.ScalarMap(1.0), f, bs.IterationConfig(format="npbs", rtol=1e-12, max_iters=50))
    assert rel(a.u, b.u) < 1e-12


def test_config0_full_solve_optimal_scalar(gpu):
    """Config 0 with the reference's default CBS map, OptimalScalar-L2 (bench.cpp:140-141)."""
    cfg0 = bs.CONFIGS["c0"]
    k2, f, k0, eta = bs.make_instances(cfg0["spec"], 0, 1)
    cmap = bs.OptimalScalarMap("euclidean")
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        res = bs.run(p, cmap, f, bs.IterationConfig(rtol=cfg0["rtol"], max_iters=20000))
    ref = _oracle_run(k2[0], f[0], k0[0], eta[0], cmap, cfg0["rtol"], 20000)
    assert ref.terminated == "converged"
    assert_run_parity(res.trace, res.u, ref)


@pytest.mark.parametrize("kind", ["reta", "fd"])
def test_other_maps_full_solve(gpu, kind):
    k2, f, k0, eta = instance(64, ppw=10.0, contrast=0.3, seed=7)
    cmap = bs.OptimalScalarMap("reta") if kind == "reta" else _fd_map(64, seed=1)
    if kind == "fd":  # a contracting multiplier: identity scaled into the CBS-stable range
        cmap = bs.FourierDiagMap(np.full((63, 63), 0.9 + 0.0j))
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        res = bs.run(p, cmap, f, bs.IterationConfig(rtol=1e-8, max_iters=5000))
    ref = _oracle_run(k2[0], f[0], k0[0], eta[0], cmap, 1e-8, 5000)
    assert_run_parity(res.trace, res.u, ref)


# ------------------------------------------------------------------ long lines (n = 1024 .. 4096)
@pytest.mark.parametrize("n", [1024, 2048, 4096])
def test_long_line_operators_match_oracle(gpu, n):
    Oracle.set_threads(os.cpu_count() or 8)
    k2, f, k0, eta = instance(n, batch=1, ppw=6.0, seed=n)
    rng = np.random.default_rng(n + 1)
    u = rand_field(rng, k2.shape)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        G, born, fw = p.apply_G(u), p.born_residual(u, f), p.forward_transform(u)
        back = p.inverse_transform(fw)
    o = OracleProblem(k2[0], k0[0], eta[0])
    assert rel(G[0], o.apply_G(u[0])) < OP_TOL
    assert rel(born[0], o.born_residual(u[0], f[0])) < OP_TOL
    assert rel(fw[0], Oracle.forward_dst(u[0])) < OP_TOL
    assert rel(back[0], u[0]) < 1e-12


@pytest.mark.parametrize("n,cmap,K", [(1024, bs.PointwiseMap(), 12), (2048, bs.ScalarMap(1.0), 6)])
def test_long_line_per_iterate(gpu, n, cmap, K):
    Oracle.set_threads(os.cpu_count() or 8)
    k2, f, k0, eta = instance(n, ppw=8.0, contrast=0.3, seed=3)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        res = bs.run(p, cmap, f, bs.IterationConfig(rtol=1e-12, max_iters=K), n_snap=K + 1)
    ref = _oracle_run(k2[0], f[0], k0[0], eta[0], cmap, 1e-12, K, n_snap=K + 1)
    for m in range(1, K + 1):
        assert rel(res.snapshots[m], ref.snapshots[m]) < FIELD_TOL, m
    assert_run_parity(res.trace, res.u, ref)


def test_config2_grid_first_sweeps(gpu):
    """BASELINE config 2 on one GPU: 4095^2, 6 ppw, contrast 0.5, 16 point sources, pointwise
    map -- the first sweeps against the oracle (a full solve is O(1e4) sweeps)."""
    Oracle.set_threads(os.cpu_count() or 8)
    k2, f, k0, eta = bs.config_instances("c2")
    K = 3
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        res = bs.run(p, bs.PointwiseMap(), f, bs.IterationConfig(rtol=1e-6, max_iters=K))
    ref = _oracle_run(k2[0], f[0], k0[0], eta[0], bs.PointwiseMap(), 1e-6, K)
    assert res.trace.iters == ref.iters == K
    assert_run_parity(res.trace, res.u, ref)


def test_column_routes_match(gpu, monkeypatch):
    """The Green column pass as a tridiagonal x-solve (default) and as the transform pair
    (BP_COL_DST=1) give the same iterates for every correction map, both against the oracle."""
    k2, f, k0, eta = instance(128, batch=2, ppw=10.0, contrast=0.3, seed=9)
    cfg = bs.IterationConfig(rtol=1e-9, max_iters=400)
    for cmap in (bs.PointwiseMap(), bs.OptimalScalarMap("euclidean"), bs.OptimalScalarMap("reta"),
                 _fd_map(128)):
        runs = []
        for route in ("0", "1"):
            monkeypatch.setenv("BP_COL_DST", route)
            with bs.HelmholtzDirichlet(k2, k0, eta) as p:
                runs.append(bs.run(p, cmap, f, cfg))
        ref = _oracle_run(k2[0], f[0], k0[0], eta[0], cmap, 1e-9, 400)
        for r in runs:
            assert_run_parity(r.traces[0], r.u[0], ref)
        assert runs[0].traces[1].iters == runs[1].traces[1].iters
        assert rel(runs[0].u, runs[1].u) < FIELD_TOL  # (the random FourierDiag map diverges)
