"""ctypes bindings of the two native libraries (built in-tree by ``__graft_entry__.build()``).

* ``libbornsweep.so``      -- the sm_100a CUDA path behind ``include/bornsweep.h``
* ``libbornsweep_host.so`` -- seeded instance synthesis behind ``include/bornsweep_instances.h``

There is no fallback: if the CUDA library is missing, loading raises ``NativeLibraryMissing``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# BP_LIB_PATH: load an alternative build of the same ABI (A/B kernel experiments only)
LIB_PATH = os.environ.get("BP_LIB_PATH") or os.path.join(HERE, "libbornsweep.so")
HOST_LIB_PATH = os.path.join(HERE, "libbornsweep_host.so")

_dp = C.POINTER(C.c_double)


class NativeLibraryMissing(ImportError):
    pass


class Grid(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("lx", C.c_double), ("ly", C.c_double),
                ("bc", C.c_int32)]


class Grid3(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("lx", C.c_double),
                ("ly", C.c_double), ("lz", C.c_double), ("bc", C.c_int32)]


class Map(C.Structure):
    _fields_ = [("kind", C.c_int32), ("gamma_re", C.c_double), ("gamma_im", C.c_double),
                ("metric", C.c_int32), ("m", _dp)]


class IterConfig(C.Structure):
    _fields_ = [("format", C.c_int32), ("rtol", C.c_double), ("max_iters", C.c_int32)]


class Trace(C.Structure):
    _fields_ = [("iters", C.c_int32), ("terminated", C.c_int32), ("fnorm_l2", C.c_double),
                ("fnorm_reta", C.c_double)]


class SlabView(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("rows", C.c_int32), ("row0", C.c_int32),
                ("n", C.c_int32), ("block_elems", C.c_int64), ("t_rows", C.c_void_p),
                ("t_cols", C.c_void_p), ("sums", C.c_void_p), ("u_first", C.c_void_p * 2),
                ("u_last", C.c_void_p * 2), ("u_halo_lo", C.c_void_p * 2),
                ("u_halo_hi", C.c_void_p * 2), ("stream", C.c_void_p), ("dim", C.c_int32),
                ("halo_elems", C.c_int64)]


class Medium(C.Structure):
    _fields_ = [("k2", _dp), ("k0", _dp), ("eta", _dp), ("bx", _dp), ("by", _dp), ("sigma", _dp),
                ("sigma0", _dp)]


class InstanceSpec(C.Structure):
    _fields_ = [("n", C.c_int32), ("ppw", C.c_double), ("contrast", C.c_double),
                ("sigma_cells", C.c_double), ("src_sigma_cells", C.c_double),
                ("n_sources", C.c_int32), ("seed", C.c_uint64), ("sponge_points", C.c_int32),
                ("sponge_strength", C.c_double), ("eta_factor", C.c_double), ("dim", C.c_int32)]


class CdrSpec(C.Structure):
    _fields_ = [("n", C.c_int32), ("b_max", C.c_double), ("sigma_max", C.c_double),
                ("smooth_cells", C.c_double), ("src_smooth_cells", C.c_double), ("seed", C.c_uint64)]


# Every symbol include/bornsweep.h declares (tests/test_abi.py checks the header agrees).
ABI_FUNCTIONS = {
    "bp_last_error": (C.c_char_p, []),
    "bp_abi_version": (C.c_int, []),
    "bp_problem_create": (C.c_int, [C.POINTER(Grid), C.c_int32, _dp, _dp, _dp, C.c_int32,
                                    C.POINTER(C.c_void_p)]),
    "bp_problem_create3d": (C.c_int, [C.POINTER(Grid3), C.c_int32, _dp, _dp, _dp, C.c_int32,
                                      C.POINTER(C.c_void_p)]),
    "bp_problem_create_cdr": (C.c_int, [C.POINTER(Grid), C.c_int32, _dp, _dp, _dp, _dp, C.c_int32,
                                        C.POINTER(C.c_void_p)]),
    "bp_problem_set_cdr_medium": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp]),
    "bp_problem_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "bp_slab_create": (C.c_int, [C.POINTER(Grid), C.c_int32, C.c_int32, _dp, C.c_double, C.c_double,
                                 C.c_int32, C.POINTER(C.c_void_p)]),
    "bp_slab_create3d": (C.c_int, [C.POINTER(Grid3), C.c_int32, C.c_int32, _dp, C.c_double, C.c_double,
                                   C.c_int32, C.POINTER(C.c_void_p)]),
    "bp_slab_view": (C.c_int, [C.c_void_p, C.POINTER(SlabView)]),
    "bp_slab_set_exchange": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                       C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "bp_slab_set_fields": (C.c_int, [C.c_void_p, _dp, _dp]),
    "bp_slab_set_multiplier": (C.c_int, [C.c_void_p, _dp]),
    "bp_slab_stage": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(Map), C.POINTER(IterConfig),
                                C.c_double, C.c_double]),
    "bp_slab_active": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "bp_slab_result": (C.c_int, [C.c_void_p, _dp, _dp, _dp, C.POINTER(Trace)]),
    "bp_problem_destroy": (C.c_int, [C.c_void_p]),
    "bp_problem_batch": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(Grid)]),
    "bp_problem_set_medium": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "bp_problem_stream": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "bp_apply_A": (C.c_int, [C.c_void_p, _dp, _dp]),
    "bp_apply_V": (C.c_int, [C.c_void_p, _dp, _dp]),
    "bp_apply_V_adjoint": (C.c_int, [C.c_void_p, _dp, _dp]),
    "bp_apply_Lref": (C.c_int, [C.c_void_p, _dp, _dp]),
    "bp_apply_G": (C.c_int, [C.c_void_p, _dp, _dp]),
    "bp_born_residual": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "bp_residual": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "bp_forward_transform": (C.c_int, [C.c_void_p, _dp, _dp]),
    "bp_inverse_transform": (C.c_int, [C.c_void_p, _dp, _dp]),
    "bp_run": (C.c_int, [C.c_void_p, C.POINTER(Map), _dp, C.POINTER(IterConfig), _dp, _dp, _dp,
                         _dp, C.POINTER(Trace)]),
    "bp_run_device": (C.c_int, [C.c_void_p, C.POINTER(Map), C.c_void_p, C.POINTER(IterConfig),
                                C.c_void_p, C.c_void_p, _dp, _dp, C.POINTER(Trace)]),
    "bp_run_snapshots": (C.c_int, [C.c_void_p, C.POINTER(Map), _dp, C.POINTER(IterConfig), _dp,
                                   _dp, _dp, _dp, C.POINTER(Trace), _dp, C.c_int32]),
    "bp_set_kernel_timing": (C.c_int, [C.c_void_p, C.c_int32]),
    "bp_pipeline_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(C.c_void_p)]),
    "bp_pipeline_submit": (C.c_int, [C.c_void_p, C.POINTER(Medium), C.POINTER(Map), _dp,
                                     C.POINTER(IterConfig), _dp, _dp, _dp, _dp, C.POINTER(Trace),
                                     C.POINTER(C.c_int32)]),
    "bp_pipeline_wait": (C.c_int, [C.c_void_p]),
    "bp_pipeline_destroy": (C.c_int, [C.c_void_p]),
    "bp_last_run_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                    _dp, _dp, C.POINTER(C.c_int64)]),
}

HOST_FUNCTIONS = {
    "bp_make_instances": (C.c_int, [C.POINTER(InstanceSpec), C.c_int64, C.c_int32, _dp, _dp, _dp,
                                    _dp, C.c_int32]),
    "bp_make_cdr_instances": (C.c_int, [C.POINTER(CdrSpec), C.c_int64, C.c_int32, _dp, _dp, _dp,
                                        _dp, _dp, C.c_int32]),
    "bp_rng_normals": (None, [C.c_uint64, C.c_int64, C.c_int32, _dp]),
    "bp_rng_uniforms": (None, [C.c_uint64, C.c_int64, C.c_int32, _dp]),
    "bp_sponge_profile": (None, [C.c_int32, C.c_int32, C.c_int32, C.c_double, _dp]),
    "bp_gaussian_bump": (None, [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                                C.c_double, C.c_double, C.c_double, _dp]),
    "bp_gaussian_smooth": (None, [C.c_int32, C.c_int32, C.c_double, _dp, _dp]),
    # include/bornsweep_io.h
    "bp_io_last_error": (C.c_char_p, []),
    "bp_bpfd_save": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, _dp]),
    "bp_bpfd_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                               C.POINTER(C.c_int32)]),
    "bp_bpfd_load": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, _dp]),
    "bp_csv_export": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, _dp]),
    "bp_trace_csv_write": (C.c_int, [C.c_char_p, C.c_int32, _dp, _dp]),
}

_lib = None
_host = None


def _bind(lib, table):
    for name, (res, args) in table.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """The CUDA library.  Raises if it was not built -- there is no CPU fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        _lib = _bind(C.CDLL(LIB_PATH), ABI_FUNCTIONS)
    return _lib


def host_lib():
    global _host
    if _host is None:
        if not os.path.exists(HOST_LIB_PATH):
            raise NativeLibraryMissing(f"{HOST_LIB_PATH} is missing: build the package first")
        _host = _bind(C.CDLL(HOST_LIB_PATH), HOST_FUNCTIONS)
    return _host


def last_error() -> str:
    return lib().bp_last_error().decode()
