"""Config c4 (convection-diffusion-reaction, Neumann, DCT-II) -- the oracle's restatement pinned
to the reference's own DCT transform pair and Neumann symbol (tests/golden/ref_dct.npz, made by
the reference's code in oracle/_ref: transforms.cpp:105-148, symbol.cpp:81-92), plus the
splitting identities of the upwind CDR operator (no reference counterpart: SURVEY.md 8(a) a16)
and the seeded c4 media generator."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
import paper_2603_18527_b200 as bs
from oracle import Oracle, OracleProblem

SHAPES = [(16, 12), (16, 16), (32, 32), (64, 64)]


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLDEN, "ref_dct.npz"))


@pytest.mark.parametrize("shape", SHAPES)
def test_oracle_dct_matches_reference(g, shape):
    key = f"{shape[0]}x{shape[1]}"
    x = g[f"x_{key}"]
    # forward: REDFT10 both axes, unnormalised (transforms.cpp:120-121)
    assert rel(Oracle.dct2(x), g[f"fwd_{key}"]) < 1e-14
    # inverse: REDFT01 both axes x 1/(4 nx ny) (transforms.cpp:100,142-143)
    inv = Oracle.dct2(x, inverse=True) / (4.0 * shape[0] * shape[1])
    assert rel(inv, g[f"inv_{key}"]) < 1e-14
    # the reference agrees with scipy's type-2 / type-3 DCT of the real part
    assert rel(g[f"fwd_{key}"].real, g[f"scipy2_{key}"]) < 1e-14
    assert rel(g[f"inv_{key}"].real * 4.0 * shape[0] * shape[1], g[f"scipy3_{key}"]) < 1e-14


@pytest.mark.parametrize("n,lx", [(32, 1.0), (64, 2.0)])
def test_oracle_cdr_symbol_matches_reference(g, n, lx):
    rng = np.random.default_rng(n)
    z = np.zeros((n, n))
    s0 = 7.5
    p = OracleProblem.cdr(z, z, z + s0, s0, lx=lx)
    lam = p.symbol()
    assert rel(lam, g[f"symbol_n{n}"] + s0) < 1e-15
    # round trip through the reference normalisation
    x = rng.standard_normal((n, n)) + 0j
    back = Oracle.dct2(Oracle.dct2(x), inverse=True) / (4.0 * n * n)
    assert rel(back, x) < 1e-14


def _cdr_problem(n=32, seed=3):
    bx, by, sigma, s0, f = bs.make_cdr_instances(bs.CdrSpec(n=n, seed=seed), 0, 1)
    return bx[0], by[0], sigma[0], float(s0[0]), f[0]


def test_oracle_cdr_splitting_identities():
    bx, by, sigma, s0, f = _cdr_problem()
    p = OracleProblem.cdr(bx, by, sigma, s0)
    rng = np.random.default_rng(0)
    u = rng.standard_normal(bx.shape) + 0j
    # A = L_ref - V
    assert rel(p.apply_A(u), p.apply_Lref(u) - p.apply_V(u)) < 1e-13
    # G L_ref = I
    assert rel(p.apply_G(p.apply_Lref(u)), u) < 1e-12
    # born residual G(V u + f) - u = G(f - A u)
    assert rel(p.born_residual(u, f), p.apply_G(p.residual(u, f))) < 1e-12
    # constants: -Lap_N 1 = 0 and the upwind gradient of a constant vanishes
    one = np.ones(bx.shape) + 0j
    assert np.abs(p.apply_A(one) - sigma).max() < 1e-10


@pytest.mark.parametrize("seed", [3, 8])
def test_oracle_cdr_adjoint_identity(seed):
    """<V u, y> = <u, V^H y> (the reference's verify-suite adjoint check, verify.cpp:196-210, on
    the upwind family: V is real, so V^H is the transposed stencil), and A^H = L_ref^H - V^H
    against a dense assembly of A on a small grid."""
    bx, by, sigma, s0, f = _cdr_problem(16, seed)
    p = OracleProblem.cdr(bx, by, sigma, s0)
    rng = np.random.default_rng(seed)
    u = rng.standard_normal(bx.shape) + 1j * rng.standard_normal(bx.shape)
    y = rng.standard_normal(bx.shape) + 1j * rng.standard_normal(bx.shape)
    lhs = np.vdot(y, p.apply_V(u))
    rhs = np.vdot(p.apply_V_adjoint(y), u)
    assert abs(lhs - rhs) < 1e-12 * abs(lhs)
    # dense V (column by column) and its transpose
    n = bx.size
    V = np.empty((n, n))
    for k in range(n):
        e = np.zeros(n, complex)
        e[k] = 1.0
        V[:, k] = p.apply_V(e.reshape(bx.shape)).real.ravel()
    assert rel(p.apply_V_adjoint(y).ravel(), V.T @ y.ravel()) < 1e-13


def test_oracle_cdr_upwind_direction():
    """A linear ramp u = x: the upwind x-difference is exact (h) inside, the reflective ghost
    zeroes the difference at the boundary cell it looks through."""
    n = 16
    h = 1.0 / n
    xs = (np.arange(n) + 0.5) * h
    u = np.repeat(xs[:, None], n, axis=1) + 0j
    z = np.zeros((n, n))
    for v in (1.0, -1.0):
        p = OracleProblem.cdr(z + v, z, z, 1.0)
        conv = -(p.apply_V(u) - (1.0 - 0.0) * u)  # V u = (s0 - sigma) u - conv
        conv = conv.real
        inner = conv[1:-1]
        assert np.allclose(inner, v * 1.0)
        if v > 0:
            assert np.isclose(conv[0, 0], 0.0) and np.isclose(conv[-1, 0], v)
        else:
            assert np.isclose(conv[-1, 0], 0.0) and np.isclose(conv[0, 0], v)


def test_oracle_cdr_run_converges():
    bx, by, sigma, s0, f = _cdr_problem(32)
    p = OracleProblem.cdr(bx, by, sigma, s0)
    r = p.run(f + 0j, rtol=1e-8, max_iters=200)
    assert r.terminated == "converged"
    assert r.iters < 40
    assert np.linalg.norm(p.residual(r.u, f + 0j)) / np.linalg.norm(f) < 1e-7


def test_cdr_instances_deterministic_and_ranged():
    spec = bs.CdrSpec(n=64, seed=9)
    a = bs.make_cdr_instances(spec, 0, 3)
    b = bs.make_cdr_instances(spec, 1, 2)
    for x, y in zip(a, b):
        assert np.array_equal(x[1:], y)  # member k is independent of the slice it is made in
    bx, by, sigma, s0, f = a
    assert np.sqrt(bx ** 2 + by ** 2).max() <= spec.b_max + 1e-12
    assert sigma.min() >= -1e-12 and sigma.max() <= spec.sigma_max + 1e-12
    assert np.allclose(s0, sigma.reshape(3, -1).mean(axis=1))
    assert np.abs(f).max() == pytest.approx(1.0)
    assert not np.array_equal(bx[0], bx[1])
