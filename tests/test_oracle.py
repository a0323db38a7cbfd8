"""Pin the CPU oracle (test infrastructure) before trusting it as the GPU checker.

Sources of truth:
  * scipy.fft DST-I golden vectors (tests/golden/dst_scipy.npz)  -- FFTW RODFT00 definition
  * SPEC.md known-answer values
  * the reference's verify-suite properties (proj/src/verify.cpp:82-216)
  * outputs of the reference's OWN code (oracle/_ref, fixtures tests/golden/ref_*.npz)
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import (FMT_CBS, FMT_NPBS, MAP_FOURIER_DIAG, MAP_OPTIMAL_SCALAR, MAP_POINTWISE,
                    MAP_SCALAR, Oracle, OracleProblem, Reference, ReferenceProblem)


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def rand_field(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


# ------------------------------------------------------------------ transforms
def test_dst_matches_scipy_goldens():
    g = np.load(os.path.join(GOLDEN, "dst_scipy.npz"))
    for key in g.files:
        if not key.startswith("x_"):
            continue
        x, y = g[key], g["y_" + key[2:]]
        assert rel(Oracle.forward_dst(x), y) < 1e-13, key


def test_dst_roundtrip_and_self_inverse():
    # proj/src/verify.cpp:94-100 (16x12 round trip <= 1e-12)
    rng = np.random.default_rng(0)
    for nx, ny in [(16, 12), (15, 15), (127, 127), (7, 31)]:
        x = rand_field(rng, (nx, ny))
        back = Oracle.inverse_dst(Oracle.forward_dst(x))
        assert rel(back, x) < 1e-12


def test_dst_eigenfunction_single_mode():
    # proj/src/verify.cpp:113-124: sin(pi x) sin(pi y) -> the (1,1) mode only
    n = 15
    h = 1.0 / (n + 1)
    xs = (np.arange(n) + 1) * h
    f = np.outer(np.sin(np.pi * xs), np.sin(np.pi * xs)).astype(np.complex128)
    m = Oracle.forward_dst(f)
    off = np.abs(m).ravel()[1:].max()
    assert off / abs(m[0, 0]) < 1e-12


@pytest.mark.parametrize("n", [3, 5, 7])
def test_dst_symbol_vs_dense_five_point(n):
    # proj/src/verify.cpp:126-152 and SPEC.md:61 (N=3, (1,1) -> 128 sin^2(pi/8))
    k2 = np.zeros((n, n), np.complex128)
    p = OracleProblem(k2, 0.0, 1e-300 + 1.0)  # lambda = L_D - i
    sym = (p.symbol() + 1j).real
    h = 1.0 / (n + 1)
    L = np.zeros((n * n, n * n))
    for i in range(n):
        for j in range(n):
            k = i * n + j
            L[k, k] = 4 / h**2
            if i > 0: L[k, k - n] = -1 / h**2
            if i < n - 1: L[k, k + n] = -1 / h**2
            if j > 0: L[k, k - 1] = -1 / h**2
            if j < n - 1: L[k, k + 1] = -1 / h**2
    ev = np.sort(np.linalg.eigvalsh(L))
    assert np.abs(np.sort(sym.ravel()) - ev).max() < 1e-10 * ev.max()
    if n == 3:
        assert abs(sym[0, 0] - 128 * np.sin(np.pi / 8) ** 2) < 1e-12
        assert abs(sym[0, 0] - 18.7450) < 5e-4  # SPEC.md:61 quotes 4 decimals


def test_green_symbol_kat_and_homogeneous_V():
    # SPEC.md:53-ish KAT restated for the Dirichlet symbol: lambda = a_p + a_q - (k0^2 + i eta);
    # homogeneous medium (k2 = k0^2) -> V u = -i eta u
    n, k0, eta = 7, 1.0, 0.5
    k2 = np.full((n, n), k0 * k0, np.complex128)
    p = OracleProblem(k2, k0, eta)
    u = rand_field(np.random.default_rng(1), (n, n))
    assert np.abs(p.apply_V(u) - (-1j * eta) * u).max() < 1e-15
    h = 1.0 / (n + 1)
    a = 4 / h**2 * np.sin(np.arange(1, n + 1) * np.pi / (2 * (n + 1))) ** 2
    assert np.abs(p.symbol() - (a[:, None] + a[None, :] - (k0**2 + 1j * eta))).max() < 1e-12


# ------------------------------------------------------------------ identities (verify.cpp:168-216)
def _problem(n=32, seed=3):
    import paper_2603_18527_b200 as bs
    spec = bs.InstanceSpec(n=n, ppw=8.0, contrast=0.5, sigma_cells=3.0, seed=seed)
    k2, f, k0, eta = bs.make_instances(spec, 0, 1)
    return OracleProblem(k2[0], k0[0], eta[0]), f[0]


def test_key_identity_splitting_green_inverse_adjoint():
    p, _ = _problem()
    rng = np.random.default_rng(2)
    for _ in range(20):
        r = rand_field(rng, (p.nx, p.ny))
        lhs = r - p.apply_G(p.apply_V(r))            # (I - GV) r
        rhs = p.apply_G(p.apply_A(r))                # G (A r)
        assert rel(lhs, rhs) * np.linalg.norm(rhs) / np.linalg.norm(r) < 1e-12
        au = p.apply_A(r)
        assert rel(p.apply_Lref(r) - p.apply_V(r), au) < 1e-12   # A = L_ref - V
        assert rel(p.apply_Lref(p.apply_G(r)), r) < 1e-12        # L_ref G = I
        assert rel(p.apply_G(p.apply_Lref(r)), r) < 1e-12        # G L_ref = I
        y = rand_field(rng, (p.nx, p.ny))
        lhs_ip = np.vdot(y, p.apply_V(r))
        rhs_ip = np.vdot(p.apply_V_adjoint(y), r)
        assert abs(lhs_ip - rhs_ip) / (np.linalg.norm(p.apply_V(r)) * np.linalg.norm(y)) < 1e-12


def test_green_matches_dense_inverse():
    # SPEC.md:584 (apply_G vs dense inverse at <= 16^2)
    p, _ = _problem(n=8)
    n = p.nx * p.ny
    E = np.eye(n, dtype=np.complex128)
    Lref = np.stack([p.apply_Lref(E[k].reshape(p.nx, p.ny)).ravel() for k in range(n)], axis=1)
    q = rand_field(np.random.default_rng(4), (p.nx, p.ny))
    dense = np.linalg.solve(Lref, q.ravel()).reshape(p.nx, p.ny)
    assert rel(p.apply_G(q), dense) < 1e-10


def test_cbs_equals_npbs_with_scalar():
    # CBS == NPBS(scalar) trajectories to 1e-12 over 50 steps
    p, f = _problem()
    a = p.run(f, map_kind=MAP_SCALAR, gamma=1.0, fmt=FMT_CBS, max_iters=50, rtol=1e-12)
    b = p.run(f, map_kind=MAP_SCALAR, gamma=1.0, fmt=FMT_NPBS, max_iters=50, rtol=1e-12)
    assert rel(a.u, b.u) < 1e-12
    assert np.abs(a.res_l2 - b.res_l2).max() < 1e-12


# ------------------------------------------------------------------ vs the reference's own code
def _load(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.mark.parametrize("n", [16, 32])
def test_oracle_operators_match_reference_fixtures(n):
    g = _load(f"ref_ops_n{n}.npz")
    p = OracleProblem(g["k2"], float(g["k0"]), float(g["eta"]))
    x, f = g["x"], g["f"]
    assert rel(p.symbol(), g["symbol"]) < 1e-15
    assert rel(p.apply_A(x), g["A"]) < 1e-15
    assert rel(p.apply_V(x), g["V"]) < 1e-15
    assert rel(p.apply_V_adjoint(x), g["VH"]) < 1e-15
    assert rel(p.apply_Lref(x), g["Lref"]) < 1e-13
    assert rel(p.apply_G(x), g["G"]) < 1e-13
    assert rel(p.born_residual(x, f), g["born"]) < 1e-13
    assert rel(p.residual(x, f), g["res"]) < 1e-15
    assert rel(Oracle.forward_dst(x), g["fwd"]) < 1e-13
    assert rel(Oracle.inverse_dst(x), g["inv"]) < 1e-13


RUNS = ["c0like_n32_scalar", "n32_pointwise", "n16_optl2", "n16_optreta", "n32_scalar_maxiters"]


@pytest.mark.parametrize("name", RUNS)
def test_oracle_run_matches_reference_fixture(name):
    g = _load(f"ref_run_{name}.npz")
    p = OracleProblem(g["k2"], float(g["k0"]), float(g["eta"]))
    r = p.run(g["f"], map_kind=int(g["map_kind"]), gamma=complex(g["gamma"]),
              metric=int(g["metric"]), rtol=float(g["rtol"]), max_iters=int(g["max_iters"]))
    assert abs(r.iters - int(g["iters"])) <= 1
    assert r.terminated == str(g["terminated"])
    k = min(len(r.res_l2), len(g["res_l2"]))
    assert np.abs(r.res_l2[:k] - g["res_l2"][:k]).max() < 1e-10
    assert np.abs(r.res_reta[:k] - g["res_reta"][:k]).max() < 1e-10
    assert rel(r.u, g["u"]) < 1e-9
    assert abs(r.fnorm_l2 - float(g["fnorm_l2"])) < 1e-13 * float(g["fnorm_l2"])
    assert abs(r.fnorm_reta - float(g["fnorm_reta"])) < 1e-12 * float(g["fnorm_reta"])


def test_run_errors_follow_reference():
    p, f = _problem(n=8)
    with pytest.raises(ValueError, match="zero source"):
        p.run(np.zeros_like(f))
    with pytest.raises(ValueError, match="rtol"):
        p.run(f, rtol=1.5)
    with pytest.raises(ValueError, match="max_iters"):
        p.run(f, max_iters=0)
    with pytest.raises(ValueError, match="eta"):
        OracleProblem(np.ones((7, 7), np.complex128), 1.0, 0.0)


@pytest.mark.skipif(not Reference.available(), reason="reference build absent")
def test_live_reference_agrees_with_oracle():
    """When oracle/_ref is present, run both on a fresh instance (not a fixture)."""
    p, f = _problem(n=16, seed=99)
    r = ReferenceProblem(p.k2, p.k0, p.eta)
    a = p.run(f, map_kind=MAP_POINTWISE, max_iters=500)
    b = r.run(f, map_kind=MAP_POINTWISE, max_iters=500)
    assert abs(a.iters - b.iters) <= 1 and a.terminated == b.terminated
    assert rel(a.u, b.u) < 1e-10
    m = np.exp(1j * np.random.default_rng(5).uniform(size=(p.nx, p.ny)))
    a = p.run(f, map_kind=MAP_FOURIER_DIAG, m=m, max_iters=5, rtol=1e-12)
    b = r.run(f, map_kind=MAP_FOURIER_DIAG, m=m, max_iters=5, rtol=1e-12)
    assert rel(a.u, b.u) < 1e-12
    a = p.run(f, map_kind=MAP_OPTIMAL_SCALAR, metric=1, max_iters=30, rtol=1e-12)
    b = r.run(f, map_kind=MAP_OPTIMAL_SCALAR, metric=1, max_iters=30, rtol=1e-12)
    assert rel(a.u, b.u) < 1e-11


def test_3d_oracle_dst_and_identities():
    """3-D extension of the oracle (config c3): DST-I vs scipy dstn golden (made by
    tests/golden/make_golden.py), round trip, splitting, Green two-sided inverse, key identity."""
    g = np.load(os.path.join(GOLDEN, "dst3_scipy.npz"))
    assert rel(Oracle.forward_dst(g["x"]), g["y"]) < 1e-13
    rng = np.random.default_rng(11)
    x = rand_field(rng, (15, 15, 15))
    assert rel(Oracle.inverse_dst(Oracle.forward_dst(x)), x) < 1e-12
    import paper_2603_18527_b200 as bs
    spec = bs.InstanceSpec(n=16, ppw=8.0, contrast=0.4, sigma_cells=2.0, dim=3)
    k2, f, k0, eta = bs.make_instances(spec, 0, 1)
    p = OracleProblem(k2[0], k0[0], eta[0])
    r = rand_field(rng, p.shape)
    assert rel(p.apply_Lref(r) - p.apply_V(r), p.apply_A(r)) < 1e-12
    assert rel(p.apply_Lref(p.apply_G(r)), r) < 1e-12
    lhs = r - p.apply_G(p.apply_V(r))
    assert np.linalg.norm(lhs - p.apply_G(p.apply_A(r))) / np.linalg.norm(r) < 1e-12
    # seven-point symbol vs the dense operator at n = 3
    k2s = np.zeros((3, 3, 3), np.complex128)
    ps = OracleProblem(k2s, 0.0, 1.0)
    e = np.eye(27, dtype=np.complex128)
    A = np.stack([ps.apply_A(e[k].reshape(3, 3, 3)).ravel() for k in range(27)], axis=1)
    ev = np.sort(np.linalg.eigvalsh(A.real))
    assert np.abs(np.sort((ps.symbol() + 1j).real.ravel()) - ev).max() < 1e-10 * ev.max()


@pytest.mark.parametrize("n", [32, 64])
def test_oracle_periodic_matches_reference_helmholtz(n):
    """The oracle's periodic family vs the reference's OWN bp::HelmholtzProblem (fixtures from
    oracle/_ref on the reference's own bench instance generator)."""
    g = _load(f"ref_periodic_n{n}.npz")
    p = OracleProblem(g["k2"], float(g["k0"]), float(g["eta"]), periodic=True)
    x, f = g["x"], g["f"]
    assert rel(p.symbol(), g["symbol"]) < 1e-15
    for name, ref in [("apply_A", "A"), ("apply_V", "V"), ("apply_V_adjoint", "VH"),
                      ("apply_Lref", "Lref"), ("apply_G", "G")]:
        assert rel(getattr(p, name)(x), g[ref]) < 1e-13, name
    assert rel(p.born_residual(x, f), g["born"]) < 1e-13
    assert rel(p.residual(x, f), g["res"]) < 1e-13
    runs = {"scalar": dict(map_kind=MAP_SCALAR, gamma=1.0),
            "scalar_relaxed": dict(map_kind=MAP_SCALAR, gamma=0.9 + 0.05j),
            "optl2": dict(map_kind=MAP_OPTIMAL_SCALAR, metric=0),
            "fd": dict(map_kind=MAP_FOURIER_DIAG, m=g["fd_m"])}
    for name, kw in runs.items():
        r = p.run(f, rtol=1e-8, max_iters=4000, **kw)
        assert abs(r.iters - int(g[f"run_{name}_iters"])) <= 1, name
        assert r.terminated == str(g[f"run_{name}_term"])
        k = min(len(r.res_l2), len(g[f"run_{name}_l2"]))
        assert np.abs(r.res_l2[:k] - g[f"run_{name}_l2"][:k]).max() < 1e-10
        if r.iters == int(g[f"run_{name}_iters"]):
            assert rel(r.u, g[f"run_{name}_u"]) < 1e-9
