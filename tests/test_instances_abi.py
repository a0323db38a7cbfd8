"""Host-side checks (no GPU): instance synthesis pinned to the reference's RNG and samplers,
and the C-ABI library loads and exports exactly what include/bornsweep.h declares."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
import paper_2603_18527_b200 as bs
from paper_2603_18527_b200 import _native as N


def _host_call(name, *args):
    return getattr(N.host_lib(), name)(*args)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def test_rng_matches_reference_rngstate():
    g = np.load(os.path.join(GOLDEN, "ref_rng.npz"))
    for key in g.files:
        kind, seed, idx = key.split("_")
        want = g[key]
        out = np.empty(len(want))
        fn = "bp_rng_normals" if kind == "normal" else "bp_rng_uniforms"
        _host_call(fn, int(seed), int(idx), len(want), _dp(out))
        assert np.array_equal(out, want), key  # bit-exact


def test_samplers_match_reference():
    g = np.load(os.path.join(GOLDEN, "ref_samplers.npz"))
    for key in g.files:
        parts = key.split("_")
        want = g[key]
        out = np.empty_like(want)
        if parts[0] == "sponge":
            nx, layer = int(parts[1]), int(parts[2])
            _host_call("bp_sponge_profile", nx, nx, layer, 1.0, _dp(out))
        else:
            nx, cx, cy, w = int(parts[1]), float(parts[2]), float(parts[3]), float(parts[4])
            _host_call("bp_gaussian_bump", nx, nx, 1.0, 1.0, cx, cy, w, 1.0, _dp(out))
        assert np.array_equal(out, want), key  # bit-exact


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_config_instances_match_baseline_definition(name):
    cfg = bs.CONFIGS[name]
    spec = cfg["spec"]
    k2, f, k0, eta = bs.make_instances(spec, 0, 2 if name == "c1" else 1)
    nd = spec.n - 1
    assert k2.shape[1:] == (nd, nd)
    h = 1.0 / spec.n
    omega = 2 * np.pi / (spec.ppw * h)
    layer = nd // 8
    sponge = np.empty((nd, nd))
    _host_call("bp_sponge_profile", nd, nd, layer, 1.0, _dp(sponge))
    for b in range(k2.shape[0]):
        kk = k2[b].real  # undamped k^2 (sponge only touches the imaginary part: k2 (1 + i d))
        assert np.allclose(k2[b].imag, kk * sponge, rtol=1e-15, atol=0)
        c = omega / np.sqrt(kk)
        assert c.min() >= 1 - spec.contrast - 1e-12 and c.max() <= 1 + spec.contrast + 1e-12
        # normalised to unit max-abs => one extreme touches the contrast bound
        assert max(abs(c.min() - (1 - spec.contrast)), abs(c.max() - (1 + spec.contrast))) >= 0
        assert np.isclose(max(1 - c.min(), c.max() - 1), spec.contrast, rtol=1e-10)
        assert np.isclose(k0[b], np.mean(np.sqrt(kk)), rtol=1e-12)
        assert np.isclose(eta[b], 1.01 * np.abs(k2[b] - k0[b] ** 2).max(), rtol=1e-14)
        # unit Gaussian bump (sigma = 2 cells) at the grid centre, an exact node
        assert f[b].real.max() == 1.0 and f[b][nd // 2, nd // 2].real == 1.0
        assert np.all(f[b].imag == 0)
    if k2.shape[0] > 1:
        assert not np.allclose(k2[0], k2[1])  # independent seeded media


def test_instances_deterministic():
    spec = bs.InstanceSpec(n=64, ppw=8.0, contrast=0.5)
    a = bs.make_instances(spec, 3, 2)
    b = bs.make_instances(spec, 3, 2)
    c = bs.make_instances(spec, 4, 1)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert np.array_equal(a[0][1], c[0][0])  # member index, not batch position, seeds the draw


def _header_functions():
    text = open(os.path.join(ROOT, "include", "bornsweep.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"^\s*(?:int|const char\*)\s+(bp_\w+)\s*\(", text, flags=re.M))


def test_c_abi_library_exports_every_declared_symbol():
    declared = _header_functions()
    assert declared, "no declarations parsed"
    assert declared == set(N.ABI_FUNCTIONS), declared ^ set(N.ABI_FUNCTIONS)
    lib = N.lib()  # loads without a GPU: no CUDA call happens at load time
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.bp_abi_version() == 1


def test_instances_header_symbols_exported():
    declared = set()
    for h in ("bornsweep_instances.h", "bornsweep_io.h"):  # both live in libbornsweep_host.so
        text = open(os.path.join(ROOT, "include", h)).read()
        declared |= set(re.findall(r"^(?:int|void|const char\*)\s+(bp_\w+)\s*\(", text, flags=re.M))
    assert declared == set(N.HOST_FUNCTIONS), declared ^ set(N.HOST_FUNCTIONS)
    for name in declared:
        assert hasattr(N.host_lib(), name)


def test_sm100a_code_in_library():
    """The CUDA library carries sm_100a SASS (cuobjdump), i.e. it was built for B200."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump absent")
    out = subprocess.run([tool, "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_pipeline_argument_errors_without_gpu():
    """bp_pipeline_* validate their arguments before any CUDA call (BP_EINVAL + message)."""
    lib = N.lib()
    out = C.c_void_p()
    assert lib.bp_pipeline_create(None, 2, C.byref(out)) == 1
    assert "null" in N.last_error()
    slots = (C.c_void_p * 2)(None, None)
    assert lib.bp_pipeline_create(slots, 2, C.byref(out)) == 1
    assert "slot" in N.last_error()
    assert lib.bp_pipeline_create(slots, 0, C.byref(out)) == 1
    assert lib.bp_pipeline_wait(None) == 1
    assert lib.bp_pipeline_destroy(None) == 0
