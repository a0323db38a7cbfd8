"""Any-shape grids on the GPU (csrc/generic_kernels.cuh): rectangular grids and sides that are
not 2^k - 1, as the reference plans them through FFTW (proj/src/transforms.cpp:39-65).

Pinned against the reference's own code (tests/golden/ref_generic.npz, make_golden.py generic:
oracle/_ref operators and bp::run trajectories), scipy's dstn (the verify suite's 16 x 12
round trip, verify.cpp:90-100) and the plain-C oracle.  Tolerances as test_gpu_parity.py:
operators 1e-13, iterates 1e-10 relative L2, iteration counts +-1."""
import os

import numpy as np
import pytest

import paper_2603_18527_b200 as bs
from conftest import GOLDEN
from oracle import MAP_POINTWISE, OracleProblem

pytestmark = pytest.mark.gpu

OP_TOL = 1e-13
FIELD_TOL = 1e-10
TAGS = ["a", "b", "c", "d"]


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLDEN, "ref_generic.npz"))


def handle(g, t, batch=1):
    lx, ly = g[f"{t}_l"]
    k2 = np.repeat(g[f"{t}_k2"][None], batch, axis=0)
    return bs.HelmholtzDirichlet(k2, float(g[f"{t}_k0"]), float(g[f"{t}_eta"]), lx=float(lx), ly=float(ly))


def test_scipy_goldens_any_shape(gpu):
    d = np.load(os.path.join(GOLDEN, "dst_scipy.npz"))
    for shape in ["16x12", "3x5", "15x15", "7x7", "31x31"]:
        x, y = d["x_" + shape], d["y_" + shape]
        with bs.HelmholtzDirichlet(np.ones_like(x), 1.0, 1.0) as p:
            assert rel(p.forward_transform(x), y) < OP_TOL, shape
            back = p.inverse_transform(p.forward_transform(x))
            assert rel(back, x) < 1e-12, shape  # verify.cpp:96-99 round trip


@pytest.mark.parametrize("t", TAGS)
def test_operators_match_reference(gpu, g, t):
    x, f = g[f"{t}_x"], g[f"{t}_f"]
    with handle(g, t) as p:
        got = dict(G=p.apply_G(x), A=p.apply_A(x), L=p.apply_Lref(x), V=p.apply_V(x),
                   born=p.born_residual(x, f), res=p.residual(x, f), fwd=p.forward_transform(x),
                   inv=p.inverse_transform(x))
    for k, v in got.items():
        assert rel(v, g[f"{t}_{k}"]) < OP_TOL, (t, k, rel(v, g[f"{t}_{k}"]))


@pytest.mark.parametrize("t", TAGS)
@pytest.mark.parametrize("name", ["pw", "sc", "dir"])
def test_runs_match_reference(gpu, g, t, name):
    cmap = bs.ScalarMap(1.0) if name == "sc" else bs.PointwiseMap()
    cfg = bs.IterationConfig("direct" if name == "dir" else "npbs", 1e-8, 3000)
    with handle(g, t, batch=2) as p:
        r = bs.run(p, cmap, np.repeat(g[f"{t}_f"][None], 2, axis=0), cfg)
    it, term = int(g[f"{t}_{name}_iters"]), str(g[f"{t}_{name}_term"])
    for b in range(2):  # batch members bit-identical to each other
        tr = r.traces[b]
        assert tr.terminated == term and abs(tr.iters - it) <= 1, (t, name, tr.iters, it, tr.terminated)
        k = min(tr.iters, it) + 1
        # (atol: the traces' last digits near rtol are roundoff of ||f - A u|| / ||f||)
        np.testing.assert_allclose(tr.res_l2_rel[:k], g[f"{t}_{name}_l2"][:k], rtol=1e-8, atol=1e-13)
        np.testing.assert_allclose(tr.res_reta_rel[:k], g[f"{t}_{name}_reta"][:k], rtol=1e-8, atol=1e-13)
        if term != "diverged":
            assert rel(r.u[b], g[f"{t}_{name}_u"]) < FIELD_TOL
    assert np.array_equal(r.u[0], r.u[1])


@pytest.mark.parametrize("shape", [(200, 150), (511, 300), (1000, 1000), (4095, 33)])
def test_larger_shapes_match_oracle(gpu, shape):
    """Bluestein lengths up to the 4096-point limit, per-iterate parity on a short run."""
    nx, ny = shape
    rng = np.random.default_rng(nx + ny)
    k2 = (400.0 * (1.0 + 0.1 * rng.standard_normal((nx, ny))) * (1.0 + 0.05j))
    k0, eta = 20.0, 1.01 * float(np.abs(k2 - 400.0).max())
    x = rng.standard_normal((nx, ny)) + 1j * rng.standard_normal((nx, ny))
    o = OracleProblem(k2, k0, eta)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        assert rel(p.apply_G(x), o.apply_G(x)) < OP_TOL
        assert rel(p.forward_transform(x), Oracle_fwd(x)) < OP_TOL
        if nx * ny <= 300_000:
            cfg = bs.IterationConfig(rtol=1e-30, max_iters=6)
            res = bs.run(p, bs.PointwiseMap(), x, cfg, n_snap=7)
            ref = o.run(x, map_kind=MAP_POINTWISE, rtol=1e-30, max_iters=6, n_snap=7)
            for m in range(1, 7):
                assert rel(res.snapshots[m], ref.snapshots[m]) < FIELD_TOL, m


def Oracle_fwd(x):
    from oracle import Oracle
    return Oracle.forward_dst(x)


def test_any_shape_limits(gpu):
    for shape in [(4096, 8), (8191, 8191)]:
        with pytest.raises(NotImplementedError):
            bs.HelmholtzDirichlet(np.ones(shape, np.complex128), 1.0, 1.0)
    with bs.HelmholtzPeriodic(np.full((16, 12), 4.0 + 0j), 2.0, 1.0) as p:
        with pytest.raises(NotImplementedError):  # the (i/eta) V map is a Dirichlet-family map
            bs.run(p, bs.PointwiseMap(), np.ones((16, 12), np.complex128))


# ------------------------------------------------------------------ periodic family, any shape
PTAGS = ["pa", "pb", "pc"]


def phandle(g, t, batch=1):
    lx, ly = g[f"{t}_l"]
    k2 = np.repeat(g[f"{t}_k2"][None], batch, axis=0)
    return bs.HelmholtzPeriodic(k2, float(g[f"{t}_k0"]), float(g[f"{t}_eta"]), lx=float(lx), ly=float(ly))


@pytest.mark.parametrize("t", PTAGS)
def test_periodic_operators_match_reference(gpu, g, t):
    x, f = g[f"{t}_x"], g[f"{t}_f"]
    with phandle(g, t) as p:
        got = dict(G=p.apply_G(x), A=p.apply_A(x), L=p.apply_Lref(x), V=p.apply_V(x),
                   born=p.born_residual(x, f), res=p.residual(x, f), fwd=p.forward_transform(x),
                   inv=p.inverse_transform(x))
    for k, v in got.items():
        assert rel(v, g[f"{t}_{k}"]) < OP_TOL, (t, k, rel(v, g[f"{t}_{k}"]))


@pytest.mark.parametrize("t", PTAGS)
@pytest.mark.parametrize("name", ["sc", "rx", "dir"])
def test_periodic_runs_match_reference(gpu, g, t, name):
    gamma = {"sc": 1.0, "rx": 0.9 + 0.05j, "dir": 2e-5}[name]
    cfg = bs.IterationConfig("direct" if name == "dir" else "npbs", 1e-8, 3000)
    with phandle(g, t, batch=2) as p:
        r = bs.run(p, bs.ScalarMap(gamma), np.repeat(g[f"{t}_f"][None], 2, axis=0), cfg)
    it, term = int(g[f"{t}_{name}_iters"]), str(g[f"{t}_{name}_term"])
    for b in range(2):
        tr = r.traces[b]
        assert tr.terminated == term and abs(tr.iters - it) <= 1, (t, name, tr.iters, it, tr.terminated)
        k = min(tr.iters, it) + 1
        np.testing.assert_allclose(tr.res_l2_rel[:k], g[f"{t}_{name}_l2"][:k], rtol=1e-8, atol=1e-13)
        np.testing.assert_allclose(tr.res_reta_rel[:k], g[f"{t}_{name}_reta"][:k], rtol=1e-8, atol=1e-13)
        if term != "diverged":
            assert rel(r.u[b], g[f"{t}_{name}_u"]) < FIELD_TOL
    assert np.array_equal(r.u[0], r.u[1])


def test_periodic_fft_round_trip_16x12(gpu):
    """verify.cpp:90-100 'roundtrip_fft' on the 16 x 12 periodic grid."""
    rng = np.random.default_rng(12)
    x = rng.standard_normal((16, 12)) + 1j * rng.standard_normal((16, 12))
    with bs.HelmholtzPeriodic(np.full((16, 12), 4.0 + 0j), 2.0, 1.0) as p:
        fw = p.forward_transform(x)
        assert rel(fw, np.fft.fft2(x)) < OP_TOL
        assert rel(p.inverse_transform(fw), x) < 1e-12


# ------------------------------------------------- OptimalScalar / FourierDiag maps, any shape
@pytest.fixture(scope="module")
def gm():
    return np.load(os.path.join(GOLDEN, "ref_generic_maps.npz"))


def _map_cfg(gm, t, name, rtol, max_iters):
    cmap = {"opt": bs.OptimalScalarMap("euclidean"), "reta": bs.OptimalScalarMap("reta"),
            "optcbs": bs.OptimalScalarMap("euclidean"), "optdir": bs.OptimalScalarMap("euclidean"),
            "fd": bs.FourierDiagMap(gm[f"{t}_m"])}[name]
    fmt = {"optcbs": "cbs", "optdir": "direct"}.get(name, "npbs")
    return cmap, bs.IterationConfig(fmt, rtol, max_iters)


@pytest.mark.parametrize("t", TAGS + PTAGS)
@pytest.mark.parametrize("name", ["opt", "reta", "optcbs", "optdir", "fd"])
def test_any_shape_maps_match_reference(gpu, g, gm, t, name):
    """OptimalScalarMap (both metrics; NPBS, CBS, Direct) and FourierDiagMap on any-shape Dirichlet
    and periodic grids against the reference's own bp::run / apply_correction (oracle/_ref,
    ref_generic_maps.npz): the iterate and both traces after 30 sweeps within 1e-10 / 1e-8, and
    the full solve's termination, iteration count (+-1) and field."""
    make = phandle if t.startswith("p") else handle
    f2 = np.repeat(g[f"{t}_f"][None], 2, axis=0)
    cmap, cfg30 = _map_cfg(gm, t, name, 1e-12, 30)
    with make(g, t, batch=2) as p:
        r = bs.run(p, cmap, f2, cfg30)
        assert np.array_equal(r.u[0], r.u[1])  # members bit-identical
        tr = r.traces[0]
        assert tr.iters == int(gm[f"{t}_{name}_iters30"]) == 30
        assert rel(r.u[0], gm[f"{t}_{name}_u30"]) < FIELD_TOL
        np.testing.assert_allclose(tr.res_l2_rel, gm[f"{t}_{name}_l2_30"], rtol=1e-8, atol=1e-13)
        np.testing.assert_allclose(tr.res_reta_rel, gm[f"{t}_{name}_reta_30"], rtol=1e-8, atol=1e-13)
        term = str(gm[f"{t}_{name}_term"])
        if term != "converged":
            return  # Direct never converges in 3000 sweeps; stagnation windows sit on roundoff
        cmap, cfg = _map_cfg(gm, t, name, 1e-8, 3000)
        full = bs.run(p, cmap, f2, cfg)
    it = int(gm[f"{t}_{name}_iters"])
    assert full.traces[0].terminated == term and abs(full.traces[0].iters - it) <= 1
    # one sweep apart at the rtol crossing differs by that sweep's update, O(rtol)
    assert rel(full.u[0], gm[f"{t}_{name}_u"]) < (FIELD_TOL if full.traces[0].iters == it else 1e-7)
