"""bs.Pipeline (bp_pipeline_*): overlapped set_medium + run jobs over several handles give
results bit-identical to the direct calls, for every family the pipeline takes, and report the
first job error like bp_run does.  Every job is also checked against the CPU oracle."""
import numpy as np
import pytest

import paper_2603_18527_b200 as bs
from oracle import MAP_POINTWISE, OracleProblem

pytestmark = pytest.mark.gpu


def _same(ra, rb):
    for t in ra.traces:  # r^0 = f: entry 0 of the R_eta trace is 1 (iterate.cpp:93-102)
        assert abs(t.res_reta_rel[0] - 1.0) < 1e-12
    assert np.array_equal(ra.u, rb.u)
    for ta, tb in zip(ra.traces, rb.traces):
        assert ta.iters == tb.iters and ta.terminated == tb.terminated
        assert np.array_equal(ta.res_l2_rel, tb.res_l2_rel)
        assert np.array_equal(ta.res_reta_rel, tb.res_reta_rel)


def test_pipeline_helmholtz_bit_identical(gpu):
    spec = bs.InstanceSpec(n=64, ppw=8.0, contrast=0.5)
    jobs = [bs.make_instances(spec, 3 * j, 3) for j in range(5)]  # 5 batches of 3 media
    cfg = bs.IterationConfig(rtol=1e-6, max_iters=400)
    cmap = bs.PointwiseMap()
    k2, f, k0, eta = jobs[0]
    slots = [bs.HelmholtzDirichlet(k2, k0, eta) for _ in range(2)]
    with bs.Pipeline(slots) as pipe:
        for k2, f, k0, eta in jobs:
            pipe.submit(cmap, f, cfg, medium=(k2, k0, eta))
        got = pipe.wait()
        # medium=None keeps the slot's medium: round robin puts the next job on slot 1 (last
        # held jobs[3]'s medium) and the one after on slot 0 (jobs[4]'s)
        pipe.submit(cmap, jobs[4][1], cfg)
        pipe.submit(cmap, jobs[3][1], cfg)
        kept = pipe.wait()
    with bs.HelmholtzDirichlet(*[jobs[0][i] for i in (0, 2, 3)]) as direct:
        for (k2, f, k0, eta), r in zip(jobs, got):
            direct.set_medium(k2, k0, eta)
            _same(r, bs.run(direct, cmap, f, cfg))
        direct.set_medium(jobs[3][0], jobs[3][2], jobs[3][3])
        _same(kept[0], bs.run(direct, cmap, jobs[4][1], cfg))
        direct.set_medium(jobs[4][0], jobs[4][2], jobs[4][3])
        _same(kept[1], bs.run(direct, cmap, jobs[3][1], cfg))
    for p in slots:
        p.close()
    # and the oracle agrees on one member of every job (SURVEY.md 8(c) parity bar)
    for (k2, f, k0, eta), r in zip(jobs, got):
        ref = OracleProblem(k2[1], k0[1], eta[1]).run(f[1], map_kind=MAP_POINTWISE, rtol=1e-6,
                                                      max_iters=400)
        assert abs(r.traces[1].iters - ref.iters) <= 1
        assert np.linalg.norm(r.u[1] - ref.u) / np.linalg.norm(ref.u) < 1e-10


def test_pipeline_cdr_bit_identical(gpu):
    media = [bs.make_cdr_instances(bs.CdrSpec(n=64, seed=5 + j), 0, 2) for j in range(3)]
    cfg = bs.IterationConfig("cbs", 1e-8, 200)
    cmap = bs.ScalarMap(1.0)
    bx, by, sg, s0, f = media[0]
    slots = [bs.CdrNeumann(bx, by, sg, s0) for _ in range(3)]
    with bs.Pipeline(slots) as pipe:
        for bx, by, sg, s0, f in media:
            pipe.submit(cmap, f, cfg, medium=(bx, by, sg, s0))
        got = pipe.wait()
    with bs.CdrNeumann(*media[0][:4]) as direct:
        for (bx, by, sg, s0, f), r in zip(media, got):
            direct.set_medium(bx, by, sg, s0)
            _same(r, bs.run(direct, cmap, f, cfg))
    for p in slots:
        p.close()


def test_pipeline_reports_job_errors(gpu):
    k2, f, k0, eta = bs.make_instances(bs.InstanceSpec(n=32, ppw=8.0, contrast=0.3), 0, 2)
    cfg = bs.IterationConfig(rtol=1e-6, max_iters=50)
    slots = [bs.HelmholtzDirichlet(k2, k0, eta) for _ in range(2)]
    with bs.Pipeline(slots) as pipe:
        pipe.submit(bs.ScalarMap(1.0), f, cfg)
        pipe.submit(bs.ScalarMap(1.0), np.zeros_like(f), cfg)  # zero source (iterate.cpp:94)
        with pytest.raises(ValueError, match="zero source"):
            pipe.wait()
        # the pipeline stays usable after a failed job
        pipe.submit(bs.ScalarMap(1.0), f, cfg)
        (r,) = pipe.wait()
        assert r.traces[0].iters > 0
    for p in slots:
        p.close()


def test_direct_run_on_a_slot_handle_and_second_pipeline(gpu):
    """A direct bs.run on a slot handle between jobs (another thread than the slot's worker)
    does not take a compute turn (it used to wait forever for a ticket); a handle cannot be a
    slot of two pipelines at once."""
    import threading
    k2, f, k0, eta = bs.make_instances(bs.InstanceSpec(n=32, ppw=8.0, contrast=0.3), 0, 2)
    cfg = bs.IterationConfig(rtol=1e-6, max_iters=60)
    slots = [bs.HelmholtzDirichlet(k2, k0, eta) for _ in range(2)]
    with bs.Pipeline(slots) as pipe:
        pipe.submit(bs.ScalarMap(1.0), f, cfg)
        (first,) = pipe.wait()
        out = {}
        th = threading.Thread(target=lambda: out.setdefault("r", bs.run(slots[0], bs.ScalarMap(1.0), f, cfg)))
        th.start()
        th.join(timeout=60)
        assert not th.is_alive(), "direct bp_run on a pipeline slot hung"
        _same(out["r"], first)
        with pytest.raises(ValueError, match="already a slot"):
            bs.Pipeline(slots)
        pipe.submit(bs.ScalarMap(1.0), f, cfg)  # the pipeline still works afterwards
        (again,) = pipe.wait()
        _same(again, first)
    for p in slots:
        p.close()
