"""Repeat-run determinism of every kernel family (compute-sanitizer is closed on the GPU pool:
the runner refuses it).  Shared-memory races, reads of uninitialised shared or global memory
and barrier mistakes show up as run-to-run differences; every reduction here has a fixed order,
so three runs of the same solve must agree BIT FOR BIT -- including on the tridiagonal column
pass's cp.async double buffer, the named-barrier engines and the slab exchanges.  Small grids
(many CTAs per SM, different co-scheduling each run) and the production sizes' kernels
(n = 512 / 1024 / 4096 instances) are both exercised."""
import numpy as np
import pytest

import paper_2603_18527_b200 as bs
from paper_2603_18527_b200.slab import LocalComm, SlabPart, run_slab

pytestmark = pytest.mark.gpu


def same3(fn):
    outs = [fn() for _ in range(3)]
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)


def inst(n, batch=2, dim=2, seed=0):
    return bs.make_instances(bs.InstanceSpec(n=n, ppw=8.0, contrast=0.5, sigma_cells=2.0, dim=dim,
                                             seed=seed), 0, batch)


@pytest.mark.parametrize("n", [64, 512, 4096])
@pytest.mark.parametrize("route", ["tri", "dst"])
def test_dirichlet_deterministic(gpu, monkeypatch, n, route):
    monkeypatch.setenv("BP_COL_DST", "1" if route == "dst" else "0")
    k2, f, k0, eta = inst(n, batch=2 if n < 4096 else 1)
    cfg = bs.IterationConfig(rtol=1e-30, max_iters=12)

    def go():
        with bs.HelmholtzDirichlet(k2, k0, eta) as p:
            outs = []
            for cmap in (bs.PointwiseMap(), bs.OptimalScalarMap("reta")):
                r = bs.run(p, cmap, f, cfg)
                outs += [r.u, r.traces[0].res_l2_rel]
            return outs
    same3(go)


def test_3d_periodic_cdr_deterministic(gpu):
    k3, f3, k03, eta3 = inst(64, batch=1, dim=3)
    bx, by, sg, s0, fc = bs.make_cdr_instances(bs.CdrSpec(n=1024), 0, 2)
    rng = np.random.default_rng(1)
    k2p = 400.0 * (1.0 + 0.2 * rng.standard_normal((2, 256, 256))) * (1.0 + 0.1j)
    etap = 1.01 * np.abs(k2p - 400.0).reshape(2, -1).max(axis=1)
    fp = rng.standard_normal((2, 256, 256)) + 0j
    cfg = bs.IterationConfig(rtol=1e-30, max_iters=10)

    def go():
        with bs.HelmholtzDirichlet(k3, k03, eta3, dim=3) as p:
            a = bs.run(p, bs.PointwiseMap(), f3, cfg).u
        with bs.CdrNeumann(bx, by, sg, s0) as p:
            b = bs.run(p, bs.ScalarMap(1.0), fc, cfg).u
        with bs.HelmholtzPeriodic(k2p, np.full(2, 20.0), etap) as p:
            c = bs.run(p, bs.OptimalScalarMap("euclidean"), fp, cfg).u
        return [a, b, c]
    same3(go)


@pytest.mark.parametrize("fused", [False, True])
def test_slab_deterministic(gpu, fused):
    k2, f, k0, eta = inst(512, batch=1)
    cfg = bs.IterationConfig(rtol=1e-30, max_iters=20)

    def go():
        parts = [SlabPart(k2[0], float(k0[0]), float(eta[0]), r, 4) for r in range(4)]
        try:
            return [run_slab(parts, LocalComm(fused=fused), bs.PointwiseMap(), f[0], cfg).u]
        finally:
            for p in parts:
                p.close()
    same3(go)


@pytest.mark.parametrize("n,batch", [(256, 2), (512, 3), (512, 8), (1024, 5)])
def test_split_batch_bit_identical(gpu, monkeypatch, n, batch):
    """Small batches run as two concurrently replayed half-batch graphs (BP_SPLIT, default on
    below 8 row waves): members are independent, so every member's u and traces are bit-identical
    to the single-graph run, terminations included (members converge at different sweeps)."""
    k2, f, k0, eta = inst(n, batch=batch, seed=batch)
    f[0] *= 10.0
    cfg = bs.IterationConfig(rtol=1e-5, max_iters=400)
    res = []
    for split in ("0", "1"):
        monkeypatch.setenv("BP_SPLIT", split)
        with bs.HelmholtzDirichlet(k2, k0, eta) as p:
            res.append(bs.run(p, bs.PointwiseMap(), f, cfg))
    for b in range(batch):
        assert res[0].traces[b].iters == res[1].traces[b].iters
        assert res[0].traces[b].terminated == res[1].traces[b].terminated
        assert np.array_equal(res[0].traces[b].res_l2_rel, res[1].traces[b].res_l2_rel)
        assert np.array_equal(res[0].u[b], res[1].u[b])


def test_waves_bit_identical(gpu, monkeypatch):
    """n = 512 batches are swept in waves of 8 members, each member its own concurrently replayed
    graph (BP_GROUP / BP_SPLIT; here 19 members: waves of 8, 8 and 3): every member's u and
    traces are bit-identical to the single-graph run and to the member solved alone."""
    batch = 19
    k2, f, k0, eta = inst(512, batch=batch, seed=7)
    f[3] *= 10.0
    cfg = bs.IterationConfig(rtol=0.5, max_iters=200)  # members stop at different sweeps
    monkeypatch.delenv("BP_GROUP", raising=False)
    monkeypatch.delenv("BP_SPLIT", raising=False)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        waves = bs.run(p, bs.PointwiseMap(), f, cfg)
    assert len({t.iters for t in waves.traces}) > 1
    # Multi-member launches, several times each: members that terminate flip their status while
    # the persistent column CTAs of the same launch read it (the race fixed in tri_kernel, r02j:
    # before, neighbours of an early-terminating member converged sweeps late in ~half the runs)
    for env in ({"BP_SPLIT": "0"}, {"BP_GROUP": "0", "BP_SPLIT": "2"}) * 3:
        for k in ("BP_GROUP", "BP_SPLIT"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        with bs.HelmholtzDirichlet(k2, k0, eta) as p:
            one = bs.run(p, bs.PointwiseMap(), f, cfg)
        for b in range(batch):
            assert waves.traces[b].iters == one.traces[b].iters, (env, b)
            assert waves.traces[b].terminated == one.traces[b].terminated
            assert np.array_equal(waves.traces[b].res_l2_rel, one.traces[b].res_l2_rel)
            assert np.array_equal(waves.u[b], one.u[b])
    with bs.HelmholtzDirichlet(k2[11:12], k0[11:12], eta[11:12]) as p:
        alone = bs.run(p, bs.PointwiseMap(), f[11:12], cfg)
    assert np.array_equal(waves.u[11], alone.u[0])
    assert np.array_equal(waves.traces[11].res_reta_rel, alone.traces[0].res_reta_rel)


@pytest.mark.parametrize("batch", [2, 5])
def test_cdr_split_batch_bit_identical(gpu, monkeypatch, batch):
    """The CDR family's split-batch graphs (run_core_cdr): members bit-identical to one graph."""
    bx, by, sg, s0, f = bs.make_cdr_instances(bs.CdrSpec(n=256, seed=batch), 0, batch)
    f[0] *= 3.0
    cfg = bs.IterationConfig(rtol=1e-9, max_iters=200)
    res = []
    for split in ("0", "1"):
        monkeypatch.setenv("BP_SPLIT", split)
        with bs.CdrNeumann(bx, by, sg, s0) as p:
            res.append(bs.run(p, bs.ScalarMap(1.0), f, cfg))
    for b in range(batch):
        assert res[0].traces[b].iters == res[1].traces[b].iters
        assert res[0].traces[b].terminated == res[1].traces[b].terminated
        assert np.array_equal(res[0].traces[b].res_l2_rel, res[1].traces[b].res_l2_rel)
        assert np.array_equal(res[0].u[b], res[1].u[b])
