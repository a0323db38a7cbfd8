"""The bench's reference arm synthesises its inputs from the reference's own RngState and
samplers (oracle/instances.py) so that it never loads the product package; pin those arrays
against the product's host synthesis (libbornsweep_host.so) to rounding."""
import numpy as np
import pytest

import paper_2603_18527_b200 as bs
from oracle import Reference
from oracle.instances import cdr_c4, helmholtz_c1

pytestmark = pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("n", [64, 128])
def test_helmholtz_c1_synthesis_matches_product(n):
    k2, f, k0, eta = helmholtz_c1(3, 2, n=n)
    pk2, pf, pk0, peta = bs.make_instances(bs.InstanceSpec(n=n, ppw=8.0, contrast=0.5), 3, 2)
    assert np.max(np.abs(k2 - pk2)) <= 1e-12 * np.max(np.abs(pk2))
    assert np.array_equal(f, pf)
    np.testing.assert_allclose(k0, pk0, rtol=1e-13)
    np.testing.assert_allclose(eta, peta, rtol=1e-12)


def test_cdr_c4_synthesis_matches_product():
    bx, by, sg, s0, f = cdr_c4(1, 2, n=64)
    pbx, pby, psg, ps0, pf = bs.make_cdr_instances(bs.CdrSpec(n=64), 1, 2)
    for a, b in ((bx, pbx), (by, pby), (sg, psg), (f, pf)):
        assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))
    np.testing.assert_allclose(s0, ps0, rtol=1e-13)
