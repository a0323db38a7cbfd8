"""Full-length parity against committed CPU fixtures (tests/golden/make_long.py): the long solves
the per-iterate tests cannot reach ("next round" item 1).

  c1  members 2..9 of the 64-member batch to rtol 1e-6 (2581..6563 sweeps) vs oracle/_ref, the
      reference's own code;
  c2  the 4095^2 grid, u^20 and u^40 and their residual traces vs oracle/_ref;
  c3  the 255^3 grid solved to rtol 1e-5 (1192 sweeps) vs the plain-C oracle.
Bar (north_star): iteration counts within +-1 and the same termination; fields within 1e-10
relative L2 -- checked on the fixtures' sub-lattice samples, the full-field norms and a fixed
full-field projection <w, u>; residual traces within 1e-8 relative on the common prefix."""
import os

import numpy as np
import pytest

import paper_2603_18527_b200 as bs
from conftest import GOLDEN

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

FIELD_TOL = 1e-10


def load(name):
    path = os.path.join(GOLDEN, f"long_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    return np.load(path)


def projection(u):
    n = u.shape[-1] + 1
    grids = np.meshgrid(*[np.arange(s) for s in u.shape], indexing="ij")
    phase = sum(k * g for k, g in zip((3, 5, 7), grids))
    return complex(np.vdot(np.exp(2j * np.pi * phase / n), u))


def check_field(u, norm, proj, sample, stride):
    sl = tuple(slice(0, None, stride) for _ in range(u.ndim))
    s = u[sl]
    assert np.linalg.norm(s - sample) / np.linalg.norm(sample) < FIELD_TOL
    assert abs(np.linalg.norm(u) - norm) / norm < FIELD_TOL
    assert abs(projection(u) - proj) / abs(proj) < 1e-9


def check_trace(got, ref):
    k = min(len(got), len(ref))
    np.testing.assert_allclose(got[:k], ref[:k], rtol=1e-8, atol=0)


def check_inputs(g, k2, f):
    np.testing.assert_allclose(g["checksum"], [k2.sum(), f.sum()], rtol=1e-13)


def test_c1_members_full_length(gpu):
    g = load("c1")
    first, count = int(g["first"]), int(g["count"])
    k2, f, k0, eta = bs.config_instances("c1", first, count)
    check_inputs(g, k2, f)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        r = bs.run(p, bs.PointwiseMap(), f, bs.IterationConfig(rtol=1e-6, max_iters=20000))
    for b in range(count):
        t = r.traces[b]
        assert abs(t.iters - int(g["iters"][b])) <= 1, (b, t.iters, g["iters"][b])
        assert t.terminated == str(g["term"][b])
        check_trace(t.res_l2_rel, g[f"l2_{b}"])
        check_trace(t.res_reta_rel, g[f"reta_{b}"])
        check_field(r.u[b], float(g[f"norm_{b}"]), complex(g[f"proj_{b}"]), g[f"sample_{b}"], 8)


@pytest.mark.parametrize("m", [20, 40])
def test_c2_iterates(gpu, m):
    g = load("c2")
    k2, f, k0, eta = bs.config_instances("c2")
    check_inputs(g, k2, f)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        r = bs.run(p, bs.PointwiseMap(), f, bs.IterationConfig(rtol=1e-30, max_iters=m))
    t = r.traces[0]
    assert t.iters == m
    check_trace(t.res_l2_rel, g[f"l2_{m}"])
    check_trace(t.res_reta_rel, g[f"reta_{m}"])
    check_field(r.u[0], float(g[f"norm_{m}"]), complex(g[f"proj_{m}"]), g[f"sample_{m}"], 16)


def test_c3_full_solve(gpu):
    g = load("c3")
    k2, f, k0, eta = bs.config_instances("c3")
    check_inputs(g, k2, f)
    cmap = bs.PointwiseMap() if bs.CONFIGS["c3"]["map"] == "pointwise" else bs.ScalarMap(1.0)
    with bs.HelmholtzDirichlet(k2, k0, eta, dim=3) as p:
        r = bs.run(p, cmap, f, bs.IterationConfig(rtol=bs.CONFIGS["c3"]["rtol"], max_iters=20000))
    t = r.traces[0]
    assert abs(t.iters - int(g["iters"])) <= 1, (t.iters, int(g["iters"]))
    assert t.terminated == str(g["term"])
    check_trace(t.res_l2_rel, g["l2"])
    check_trace(t.res_reta_rel, g["reta"])
    check_field(r.u[0], float(g["norm"]), complex(g["proj"]), g["sample"], 8)
