"""IterFormat::Direct (direction = r^m, proj/src/iterate.cpp:118-123) on the Dirichlet
five-point family, every correction map, vs run() of the reference's own code (fixtures from
oracle/_ref, tests/golden/make_golden.py round2) and per iterate vs the plain-C oracle."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
import paper_2603_18527_b200 as bs
from oracle import FMT_DIRECT, MAP_OPTIMAL_SCALAR, OracleProblem

pytestmark = pytest.mark.gpu
FIELD_TOL = 1e-10


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _map(name, g, n):
    return {"optl2": bs.OptimalScalarMap("euclidean"), "optreta": bs.OptimalScalarMap("reta"),
            "scalar": bs.ScalarMap(1.0 / (8.0 * n * n)), "pointwise": bs.PointwiseMap(),
            "fd": bs.FourierDiagMap(g[f"n{n}_fd_m"] * (1.0 / (8.0 * n * n)))}[name]


@pytest.mark.parametrize("n", [16, 32])
@pytest.mark.parametrize("name", ["optl2", "optreta", "scalar", "pointwise", "fd"])
def test_direct_format_matches_reference(gpu, n, name):
    g = np.load(os.path.join(GOLDEN, "ref_direct.npz"))
    k = f"n{n}"
    with bs.HelmholtzDirichlet(g[k + "_k2"][None], np.array([g[k + "_k0"]]), np.array([g[k + "_eta"]])) as p:
        res = bs.run(p, _map(name, g, n), g[k + "_f"][None],
                     bs.IterationConfig(format="direct", rtol=1e-4, max_iters=150))
    tr, iters = res.traces[0], int(g[f"{k}_{name}_iters"])
    assert tr.terminated == str(g[f"{k}_{name}_term"])
    assert abs(tr.iters - iters) <= 1
    m = min(tr.iters, iters) + 1
    if str(g[f"{k}_{name}_term"]) == "diverged":
        m -= 1  # the diverging entry is > 1e8 (rounding grows with it); the earlier ones are pinned
    np.testing.assert_allclose(tr.res_l2_rel[:m], g[f"{k}_{name}_l2"][:m], rtol=1e-8, atol=1e-13)
    np.testing.assert_allclose(tr.res_reta_rel[:m], g[f"{k}_{name}_reta"][:m], rtol=1e-8, atol=1e-13)
    if tr.iters == iters and tr.terminated != "diverged":
        assert rel(res.u[0], g[f"{k}_{name}_u"]) < FIELD_TOL


def test_direct_optimal_scalar_per_iterate_vs_oracle(gpu):
    """u^m per iterate (Direct + OptimalScalar Euclidean: the R_FD_A / C_LREF / R_RETA_C plan)
    at n = 64 against the plain-C oracle."""
    spec = bs.InstanceSpec(n=64, ppw=8.0, contrast=0.4, sigma_cells=2.0, seed=3)
    k2, f, k0, eta = bs.make_instances(spec, 0, 2)
    K = 20
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        res = bs.run(p, bs.OptimalScalarMap("euclidean"), f,
                     bs.IterationConfig(format="direct", rtol=1e-12, max_iters=K), n_snap=K + 1)
    for b in range(2):
        ref = OracleProblem(k2[b], k0[b], eta[b]).run(f[b], map_kind=MAP_OPTIMAL_SCALAR, fmt=FMT_DIRECT,
                                                      rtol=1e-12, max_iters=K, n_snap=K + 1)
        assert res.traces[b].iters == ref.iters == K
        assert not np.any(res.snapshots[0][b])  # u^0 = 0
        for m in range(1, K + 1):
            assert rel(res.snapshots[m][b], ref.snapshots[m]) < FIELD_TOL, (b, m)
