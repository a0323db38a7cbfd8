"""Problem manifests on the GPU path: the reference-written helmholtz manifest
(tests/golden/ref_io) loads into the periodic family and runs like the arrays it holds;
save_problem -> load_problem round trips for the Dirichlet and CDR families."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
import paper_2603_18527_b200 as bs
from paper_2603_18527_b200 import bpfd

pytestmark = pytest.mark.gpu


def test_reference_manifest_loads_and_runs(gpu):
    g = np.load(os.path.join(GOLDEN, "io_inputs.npz"))
    p = bpfd.load_problem(os.path.join(GOLDEN, "ref_io", "helm.problem"))
    assert isinstance(p, bs.HelmholtzPeriodic)
    cfg = bs.IterationConfig(rtol=1e-8, max_iters=3000)
    a = bs.run(p, bs.ScalarMap(1.0), g["f"], cfg)
    with bs.HelmholtzPeriodic(g["k2"], float(g["k0"]), float(g["eta"])) as q:
        b = bs.run(q, bs.ScalarMap(1.0), g["f"], cfg)
    assert a.trace.iters == b.trace.iters and np.array_equal(a.u, b.u)
    p.close()


def test_save_load_round_trips(gpu, tmp_path):
    k2, f, k0, eta = bs.make_instances(bs.InstanceSpec(n=64, ppw=10.0, contrast=0.3), 0, 2)
    cfg = bs.IterationConfig(rtol=1e-7, max_iters=2000)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        path = bpfd.save_problem(str(tmp_path), "m1", p, member=1)
        ref = bs.run(p, bs.ScalarMap(1.0), f, cfg)
    q = bpfd.load_problem(path)
    assert isinstance(q, bs.HelmholtzDirichlet) and not isinstance(q, bs.HelmholtzPeriodic)
    r = bs.run(q, bs.ScalarMap(1.0), f[1], cfg)
    assert r.trace.iters == ref.traces[1].iters and np.array_equal(r.u, ref.u[1])
    q.close()
    bx, by, sg, s0, fc = bs.make_cdr_instances(bs.CdrSpec(n=64, seed=4), 0, 1)
    with bs.CdrNeumann(bx, by, sg, s0) as c:
        path = bpfd.save_problem(str(tmp_path), "cdr", c)
        rc = bs.run(c, bs.ScalarMap(1.0), fc, bs.IterationConfig("cbs", 1e-8, 300))
    d = bpfd.load_problem(path)
    rd = bs.run(d, bs.ScalarMap(1.0), fc[0], bs.IterationConfig("cbs", 1e-8, 300))
    assert rd.trace.iters == rc.trace.iters and np.array_equal(rd.u, rc.u[0])
    bpfd.write_trace_csv(str(tmp_path / "t.csv"), rd.trace)
    rows = (tmp_path / "t.csv").read_text().splitlines()
    assert rows[0] == "step,res_l2_rel,res_Reta_rel" and len(rows) == rd.trace.iters + 2
    d.close()
