"""Slab decomposition host logic (paper_2603_18527_b200/slab.py) on CPUs: the driver with the
numpy stand-in part (tests/slab_standin.py) -- in one process (LocalComm, 1/2/4 parts) and as
two gloo ranks (DistComm) -- against the single-grid oracle run (iterate.cpp:88-153)."""
import os
import socket
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2603_18527_b200 as bs  # noqa: E402
from oracle import MAP_POINTWISE, MAP_SCALAR, OracleProblem  # noqa: E402
from paper_2603_18527_b200.slab import DistComm, LocalComm, run_slab  # noqa: E402
from slab_standin import NumpySlabPart, NumpySlabPart3  # noqa: E402

FIELD_TOL = 1e-10


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def instance(n, seed=3):
    spec = bs.InstanceSpec(n=n, ppw=10.0, contrast=0.3, sigma_cells=3.0, seed=seed)
    k2, f, k0, eta = bs.make_instances(spec, 0, 1)
    return k2[0], f[0], float(k0[0]), float(eta[0])


def oracle_run(k2, f, k0, eta, cmap, rtol, max_iters, u0=None):
    p = OracleProblem(k2, k0, eta)
    if isinstance(cmap, bs.PointwiseMap):
        return p.run(f, map_kind=MAP_POINTWISE, rtol=rtol, max_iters=max_iters, u0=u0)
    return p.run(f, map_kind=MAP_SCALAR, gamma=cmap.gamma, rtol=rtol, max_iters=max_iters, u0=u0)


@pytest.mark.parametrize("nranks", [1, 2, 4])
@pytest.mark.parametrize("cmap", [bs.ScalarMap(1.0), bs.PointwiseMap()], ids=["scalar", "pointwise"])
def test_local_slab_driver_matches_oracle(nranks, cmap):
    k2, f, k0, eta = instance(32)
    cfg = bs.IterationConfig(rtol=1e-8, max_iters=3000)
    parts = [NumpySlabPart(k2, k0, eta, r, nranks) for r in range(nranks)]
    res = run_slab(parts, LocalComm(), cmap, f, cfg)
    ref = oracle_run(k2, f, k0, eta, cmap, 1e-8, 3000)
    assert res.trace.terminated == ref.terminated == "converged"
    assert abs(res.trace.iters - ref.iters) <= 1
    assert rel(res.u, ref.u) < FIELD_TOL
    k = min(res.trace.iters, ref.iters) + 1
    np.testing.assert_allclose(res.trace.res_l2_rel[:k], ref.res_l2[:k], rtol=1e-9, atol=1e-13)
    np.testing.assert_allclose(res.trace.res_reta_rel[:k], ref.res_reta[:k], rtol=1e-9, atol=1e-13)


def fd_multiplier(shape, seed=11):
    """a non-trivial FourierDiag multiplier close enough to 1 that the iteration still converges"""
    rng = np.random.default_rng(seed)
    return 0.9 + 0.05 * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def oracle_map_run(k2, f, k0, eta, cmap, rtol, max_iters):
    from oracle import MAP_FOURIER_DIAG, MAP_OPTIMAL_SCALAR, METRIC_EUCLIDEAN, METRIC_RETA
    p = OracleProblem(k2, k0, eta)
    if isinstance(cmap, bs.FourierDiagMap):
        return p.run(f, map_kind=MAP_FOURIER_DIAG, m=cmap.m, rtol=rtol, max_iters=max_iters)
    metric = METRIC_EUCLIDEAN if cmap.metric == "euclidean" else METRIC_RETA
    return p.run(f, map_kind=MAP_OPTIMAL_SCALAR, metric=metric, rtol=rtol, max_iters=max_iters)


def staged_maps(shape):
    return [bs.OptimalScalarMap("euclidean"), bs.OptimalScalarMap("reta"), bs.FourierDiagMap(fd_multiplier(shape))]


@pytest.mark.parametrize("nranks", [1, 2, 4])
@pytest.mark.parametrize("which", [0, 1, 2], ids=["optimal_l2", "optimal_reta", "fourier_diag"])
def test_local_slab_driver_staged_maps_match_oracle(nranks, which):
    """OptimalScalarMap (both metrics) and FourierDiagMap (correction.cpp:22-76) on slabs: the
    extra global reductions and the distributed-layout multiplier."""
    k2, f, k0, eta = instance(32)
    cmap = staged_maps(k2.shape)[which]
    cfg = bs.IterationConfig(rtol=1e-8, max_iters=3000)
    parts = [NumpySlabPart(k2, k0, eta, r, nranks) for r in range(nranks)]
    res = run_slab(parts, LocalComm(), cmap, f, cfg)
    ref = oracle_map_run(k2, f, k0, eta, cmap, 1e-8, 3000)
    assert res.trace.terminated == ref.terminated == "converged"
    assert abs(res.trace.iters - ref.iters) <= 1
    assert rel(res.u, ref.u) < FIELD_TOL
    k = min(res.trace.iters, ref.iters) + 1
    np.testing.assert_allclose(res.trace.res_l2_rel[:k], ref.res_l2[:k], rtol=1e-8, atol=1e-13)
    np.testing.assert_allclose(res.trace.res_reta_rel[:k], ref.res_reta[:k], rtol=1e-8, atol=1e-13)


@pytest.mark.parametrize("which", [0, 1, 2], ids=["optimal_l2", "optimal_reta", "fourier_diag"])
def test_local_slab3d_driver_staged_maps_match_oracle(which):
    k2, f, k0, eta = instance3(16)
    cmap = staged_maps(k2.shape)[which]
    parts = [NumpySlabPart3(k2, k0, eta, r, 2) for r in range(2)]
    res = run_slab(parts, LocalComm(), cmap, f, bs.IterationConfig(rtol=1e-8, max_iters=3000))
    ref = oracle_map_run(k2, f, k0, eta, cmap, 1e-8, 3000)
    assert res.trace.terminated == ref.terminated == "converged"
    assert abs(res.trace.iters - ref.iters) <= 1
    assert rel(res.u, ref.u) < FIELD_TOL


@pytest.mark.parametrize("name", ["scalar", "pointwise", "optimal_l2", "optimal_reta", "fourier_diag"])
def test_local_slab_driver_direct_format_matches_oracle(name):
    """IterFormat::Direct (direction = r, iterate.cpp:118-123) on slabs with every map; the
    Euclidean optimal scalar then needs w = A r through a distributed L_ref application."""
    from oracle import (FMT_DIRECT, MAP_FOURIER_DIAG, MAP_OPTIMAL_SCALAR, METRIC_EUCLIDEAN, METRIC_RETA)
    k2, f, k0, eta = instance(32)
    h2 = (1.0 / 32) ** 2
    m = 0.1 * h2 * fd_multiplier(k2.shape)  # Richardson on A needs a step of the order of h^2
    cmap, kw = {
        "scalar": (bs.ScalarMap(0.1 * h2), dict(map_kind=MAP_SCALAR, gamma=0.1 * h2)),
        "pointwise": (bs.PointwiseMap(), dict(map_kind=MAP_POINTWISE)),
        "optimal_l2": (bs.OptimalScalarMap("euclidean"), dict(map_kind=MAP_OPTIMAL_SCALAR, metric=METRIC_EUCLIDEAN)),
        "optimal_reta": (bs.OptimalScalarMap("reta"), dict(map_kind=MAP_OPTIMAL_SCALAR, metric=METRIC_RETA)),
        "fourier_diag": (bs.FourierDiagMap(m), dict(map_kind=MAP_FOURIER_DIAG, m=m)),
    }[name]
    cfg = bs.IterationConfig("direct", 1e-8, 25)
    parts = [NumpySlabPart(k2, k0, eta, r, 2) for r in range(2)]
    res = run_slab(parts, LocalComm(), cmap, f, cfg)
    ref = OracleProblem(k2, k0, eta).run(f, fmt=FMT_DIRECT, rtol=1e-8, max_iters=25, **kw)
    assert res.trace.terminated == ref.terminated and res.trace.iters == ref.iters
    assert rel(res.u, ref.u) < FIELD_TOL
    np.testing.assert_allclose(res.trace.res_l2_rel, ref.res_l2, rtol=1e-8, atol=1e-13)
    np.testing.assert_allclose(res.trace.res_reta_rel, ref.res_reta, rtol=1e-8, atol=1e-13)


def test_local_slab_driver_warm_start_and_max_iters():
    k2, f, k0, eta = instance(32, seed=5)
    u0 = 1e-3 * (np.random.default_rng(2).standard_normal(k2.shape) + 0j)
    parts = [NumpySlabPart(k2, k0, eta, r, 2) for r in range(2)]
    res = run_slab(parts, LocalComm(), bs.ScalarMap(1.0), f, bs.IterationConfig(rtol=1e-8, max_iters=7), u0=u0)
    ref = oracle_run(k2, f, k0, eta, bs.ScalarMap(1.0), 1e-8, 7, u0=u0)
    assert res.trace.terminated == ref.terminated == "max_iters"
    assert res.trace.iters == ref.iters == 7
    assert rel(res.u, ref.u) < FIELD_TOL


def test_local_slab_zero_source_raises():
    k2, f, k0, eta = instance(16)
    parts = [NumpySlabPart(k2, k0, eta, r, 2) for r in range(2)]
    with pytest.raises(ValueError, match="zero source"):
        run_slab(parts, LocalComm(), bs.ScalarMap(1.0), np.zeros_like(f))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def instance3(n, seed=2):
    spec = bs.InstanceSpec(n=n, ppw=10.0, contrast=0.3, sigma_cells=3.0, seed=seed, dim=3)
    k2, f, k0, eta = bs.make_instances(spec, 0, 1)
    return k2[0], f[0], float(k0[0]), float(eta[0])


@pytest.mark.parametrize("nranks", [1, 2, 4])
def test_local_slab3d_driver_matches_oracle(nranks):
    """3-D x-plane slabs (bp_slab_create3d protocol: y-block all-to-all, halo planes)."""
    k2, f, k0, eta = instance3(16)
    parts = [NumpySlabPart3(k2, k0, eta, r, nranks) for r in range(nranks)]
    res = run_slab(parts, LocalComm(), bs.PointwiseMap(), f, bs.IterationConfig(rtol=1e-8, max_iters=3000))
    ref = oracle_run(k2, f, k0, eta, bs.PointwiseMap(), 1e-8, 3000)
    assert res.trace.terminated == ref.terminated == "converged"
    assert abs(res.trace.iters - ref.iters) <= 1
    assert rel(res.u, ref.u) < FIELD_TOL


def _worker(rank, world, port, q, dim=2, which=-1):
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from slab_standin import NumpySlabPart, NumpySlabPart3
    Part = NumpySlabPart3 if dim == 3 else NumpySlabPart
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        k2, f, k0, eta = instance3(16) if dim == 3 else instance(32)
        part = Part(k2, k0, eta, rank, world)
        cmap = bs.PointwiseMap() if which < 0 else staged_maps(k2.shape)[which]
        res = run_slab([part], DistComm(), cmap, f, bs.IterationConfig(rtol=1e-8, max_iters=3000))
        q.put((rank, part.row0, part.rows, res.u, res.trace.iters, res.trace.terminated,
               res.trace.res_l2_rel, res.sweeps_launched))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dim,which", [(2, -1), (3, -1), (2, 0), (2, 1), (2, 2)],
                         ids=["2d", "3d", "2d_optimal_l2", "2d_optimal_reta", "2d_fourier_diag"])
def test_two_rank_gloo_slab_matches_oracle(dim, which):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, dim, which)) for r in range(2)]
    for p in procs:
        p.start()
    results = sorted([q.get(timeout=300) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    k2, f, k0, eta = instance3(16) if dim == 3 else instance(32)
    if which < 0:
        ref = oracle_run(k2, f, k0, eta, bs.PointwiseMap(), 1e-8, 3000)
    else:
        ref = oracle_map_run(k2, f, k0, eta, staged_maps(k2.shape)[which], 1e-8, 3000)
    u = np.zeros_like(ref.u)
    for rank, row0, rows, ur, iters, term, l2, launched in results:
        lo, hi = max(row0 - 1, 0), min(row0 + rows - 1, k2.shape[0])
        u[lo:hi] = ur[lo:hi]  # each rank filled only its own rows
        assert term == ref.terminated == "converged"
        assert abs(iters - ref.iters) <= 1
    # both ranks saw the same trace and stopped at the same sweep
    assert results[0][4] == results[1][4] and results[0][7] == results[1][7]
    assert np.array_equal(results[0][6], results[1][6])
    assert rel(u, ref.u) < FIELD_TOL
