"""The header-only C++ mirror (include/bornsweep.hpp) gives the same runs as the Python API and
maps errors to the reference's exception types (tools/cpp_api_check.cpp)."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT
import paper_2603_18527_b200 as bs

pytestmark = pytest.mark.gpu


def test_cpp_mirror_matches_python_api(gpu):
    exe = os.path.join(ROOT, "paper_2603_18527_b200", "bornsweep_cpp_check")
    out = subprocess.run([exe, "32", "2"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = out.stdout.strip().splitlines()
    assert lines[-1].startswith("invalid_argument: run: zero source")
    spec = bs.InstanceSpec(n=32, ppw=10.0, contrast=0.3, sigma_cells=3.0)
    k2, f, k0, eta = bs.make_instances(spec, 0, 2)
    with bs.HelmholtzDirichlet(k2, k0, eta) as p:
        res = bs.run(p, bs.ScalarMap(1.0), f, bs.IterationConfig(rtol=1e-6, max_iters=5000))
    assert [l for l in lines if l.startswith("pipe")] == [f"pipe {j} same" for j in range(3)]
    for b, line in enumerate(lines[:2]):
        mb, iters, term, last, csum = line.split()
        assert int(mb) == b
        assert int(iters) == res.traces[b].iters
        assert int(term) == 0 and res.traces[b].terminated == "converged"
        assert float(last) == res.traces[b].res_l2_rel[-1]
        assert np.isclose(float(csum), np.abs(res.u[b]).sum(), rtol=1e-12)
