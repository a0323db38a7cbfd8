"""CPU ORACLE for the Born-series hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference`` arm) may import this package, and only as the checker / CPU baseline.
The product package ``paper_2603_18527_b200`` never imports it.

Two backends, both driven through ctypes over numpy ``complex128`` arrays:

* ``Oracle``    -- ``liboracle.so``: plain-C restatement (``bp_oracle.c``) of the reference's
  transforms, Green operator, Dirichlet five-point Helmholtz operators and ``bp::run``.
* ``Reference`` -- ``_ref/libbpref.so``: the reference's OWN sources
  (``/root/reference/proj/src/{parallel,kernels,field,transforms,symbol,problem,helmholtz,
  newton_problem,samplers}.cpp``) compiled in place against a project-owned FFTW-API shim,
  plus an Eigen-free restatement of ``run``/``apply_correction`` (``ref/ref_driver.cpp``).
  FFTW itself is absent from the image, so this is "the reference with a non-FFTW FFT".
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbpref.so")

MAP_SCALAR, MAP_OPTIMAL_SCALAR, MAP_FOURIER_DIAG, MAP_POINTWISE = 0, 1, 2, 3
METRIC_EUCLIDEAN, METRIC_RETA = 0, 1
FMT_DIRECT, FMT_CBS, FMT_NPBS = 0, 1, 2
TERM_NAMES = {0: "converged", 1: "max_iters", 2: "diverged", 3: "stagnated"}

_dp = C.POINTER(C.c_double)


def _ptr(a):
    if a is None:
        return None
    assert a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _c(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    if shape is not None:
        a = a.reshape(shape)
    return a


class _Trace(C.Structure):
    _fields_ = [("iters", C.c_int), ("terminated", C.c_int), ("fnorm_l2", C.c_double),
                ("fnorm_reta", C.c_double)]


@dataclass
class RunResult:
    u: np.ndarray
    res_l2: np.ndarray
    res_reta: np.ndarray
    iters: int
    terminated: str
    fnorm_l2: float
    fnorm_reta: float
    snapshots: np.ndarray | None = None


class OracleError(RuntimeError):
    pass


def build(ref: bool = True) -> None:
    """Compile liboracle.so (and _ref/libbpref.so when /root/reference is present)."""
    import subprocess
    targets = ["oracle"]
    if ref and os.path.isdir(os.environ.get("BP_REFERENCE", "/root/reference")):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


# --------------------------------------------------------------------------- plain-C oracle
class Oracle:
    """ctypes front-end of the plain-C restatement (bp_oracle.c)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                build(ref=False)
            lib = C.CDLL(ORACLE_SO)
            lib.bpo_last_error.restype = C.c_char_p
            lib.bpo_problem_create.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _dp,
                                               C.c_double, C.c_double, C.POINTER(C.c_void_p)]
            lib.bpo_problem_create3.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _dp,
                                                C.c_double, C.c_double, C.POINTER(C.c_void_p)]
            lib.bpo_forward_dst3.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp]
            lib.bpo_problem_create_periodic.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double,
                                                        _dp, C.c_double, C.c_double,
                                                        C.POINTER(C.c_void_p)]
            lib.bpo_fft2.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp]
            lib.bpo_problem_create_cdr.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _dp,
                                                   _dp, _dp, C.c_double, C.POINTER(C.c_void_p)]
            lib.bpo_dct2.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp]
            lib.bpo_inverse_dst3.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp]
            for name in ("bpo_apply_A", "bpo_apply_V", "bpo_apply_V_adjoint", "bpo_apply_Lref"):
                getattr(lib, name).argtypes = [C.c_void_p, _dp, _dp]
                getattr(lib, name).restype = None
            lib.bpo_apply_G.argtypes = [C.c_void_p, _dp, _dp]
            lib.bpo_born_residual.argtypes = [C.c_void_p, _dp, _dp, _dp]
            lib.bpo_residual.argtypes = [C.c_void_p, _dp, _dp, _dp]
            lib.bpo_residual.restype = None
            lib.bpo_problem_destroy.argtypes = [C.c_void_p]
            lib.bpo_problem_destroy.restype = None
            lib.bpo_problem_symbol.argtypes = [C.c_void_p, _dp]
            lib.bpo_problem_symbol.restype = None
            lib.bpo_forward_dst.argtypes = [C.c_int, C.c_int, _dp, _dp]
            lib.bpo_inverse_dst.argtypes = [C.c_int, C.c_int, _dp, _dp]
            lib.bpo_dst1_1d.argtypes = [C.c_int, _dp, _dp]
            lib.bpo_set_threads.argtypes = [C.c_int]

            class Map(C.Structure):
                _fields_ = [("kind", C.c_int), ("gamma_re", C.c_double), ("gamma_im", C.c_double),
                            ("metric", C.c_int), ("m", _dp)]
            cls.Map = Map
            lib.bpo_run.argtypes = [C.c_void_p, C.POINTER(Map), _dp, C.c_int, C.c_double, C.c_int,
                                    _dp, _dp, _dp, _dp, C.POINTER(_Trace), _dp, C.c_int]
            cls._lib = lib
        return cls._lib

    @classmethod
    def set_threads(cls, n: int) -> None:
        cls.lib().bpo_set_threads(int(n))

    # transforms (reference normalisation: forward = plain sine sum, inverse carries 4/((nx+1)(ny+1)))
    @classmethod
    def forward_dst(cls, x):
        x = _c(x)
        out = np.empty_like(x)
        if x.ndim == 3:
            cls.lib().bpo_forward_dst3(*x.shape, _ptr(x), _ptr(out))
        else:
            cls.lib().bpo_forward_dst(x.shape[0], x.shape[1], _ptr(x), _ptr(out))
        return out

    @classmethod
    def inverse_dst(cls, x):
        x = _c(x)
        out = np.empty_like(x)
        if x.ndim == 3:
            cls.lib().bpo_inverse_dst3(*x.shape, _ptr(x), _ptr(out))
        else:
            cls.lib().bpo_inverse_dst(x.shape[0], x.shape[1], _ptr(x), _ptr(out))
        return out

    @classmethod
    def dct2(cls, x, inverse=False):
        """REDFT10 both axes (inverse: REDFT01 both axes, unnormalised) of a complex array"""
        x = _c(x)
        out = np.empty_like(x)
        cls.lib().bpo_dct2(x.shape[0], x.shape[1], int(inverse), _ptr(x), _ptr(out))
        return out

    @classmethod
    def dst1_1d(cls, x):
        x = _c(x)
        out = np.empty_like(x)
        cls.lib().bpo_dst1_1d(x.shape[0], _ptr(x), _ptr(out))
        return out


class OracleProblem:
    """Dirichlet five-point Helmholtz problem held by the plain-C oracle."""

    backend = "oracle"

    def __init__(self, k2, k0: float, eta: float, lx: float = 1.0, ly: float = 1.0,
                 periodic: bool = False):
        """k2 of shape (nx, ny) -> the 2-D Dirichlet problem; (nx, ny, nz) -> 3-D extension;
        periodic=True -> the reference's own periodic pseudospectral HelmholtzProblem."""
        k2 = _c(k2)
        self.shape = k2.shape
        self.nx, self.ny = k2.shape[:2]
        self.k2, self.k0, self.eta, self.lx, self.ly = k2, float(k0), float(eta), lx, ly
        self._lib = Oracle.lib()
        h = C.c_void_p()
        if periodic:
            rc = self._lib.bpo_problem_create_periodic(self.nx, self.ny, lx, ly, _ptr(k2), k0, eta,
                                                       C.byref(h))
        elif k2.ndim == 3:
            rc = self._lib.bpo_problem_create3(*k2.shape, lx, _ptr(k2), k0, eta, C.byref(h))
        else:
            rc = self._lib.bpo_problem_create(self.nx, self.ny, lx, ly, _ptr(k2), k0, eta, C.byref(h))
        if rc:
            raise (ValueError if rc == 1 else OracleError)(self._lib.bpo_last_error().decode())
        self._h = h

    @classmethod
    def cdr(cls, bx, by, sigma, sigma0: float, lx: float = 1.0):
        """Config-c4 convection-diffusion-reaction problem (Neumann, DCT-II, upwind)."""
        self = cls.__new__(cls)
        bx, by, sigma = (np.ascontiguousarray(a, np.float64) for a in (bx, by, sigma))
        self.shape = bx.shape
        self.nx, self.ny = bx.shape
        self.k0, self.eta, self.lx, self.ly = 0.0, 1.0, lx, lx
        self._lib = Oracle.lib()
        h = C.c_void_p()
        rc = self._lib.bpo_problem_create_cdr(self.nx, self.ny, lx, lx, _ptr(bx), _ptr(by),
                                              _ptr(sigma), float(sigma0), C.byref(h))
        if rc:
            raise (ValueError if rc == 1 else OracleError)(self._lib.bpo_last_error().decode())
        self._h = h
        return self

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.bpo_problem_destroy(self._h)
            self._h = None

    def _un(self, name, u):
        u = _c(u, self.shape)
        out = np.empty_like(u)
        rc = getattr(self._lib, name)(self._h, _ptr(u), _ptr(out))
        if rc:
            raise OracleError(self._lib.bpo_last_error().decode())
        return out

    def symbol(self):
        out = np.empty(self.shape, np.complex128)
        self._lib.bpo_problem_symbol(self._h, _ptr(out))
        return out

    def apply_A(self, u): return self._un("bpo_apply_A", u)
    def apply_V(self, u): return self._un("bpo_apply_V", u)
    def apply_V_adjoint(self, u): return self._un("bpo_apply_V_adjoint", u)
    def apply_Lref(self, u): return self._un("bpo_apply_Lref", u)
    def apply_G(self, q): return self._un("bpo_apply_G", q)

    def born_residual(self, u, f):
        u, f = _c(u, self.shape), _c(f, self.shape)
        out = np.empty_like(u)
        if self._lib.bpo_born_residual(self._h, _ptr(u), _ptr(f), _ptr(out)):
            raise OracleError(self._lib.bpo_last_error().decode())
        return out

    def residual(self, u, f):
        u, f = _c(u, self.shape), _c(f, self.shape)
        out = np.empty_like(u)
        self._lib.bpo_residual(self._h, _ptr(u), _ptr(f), _ptr(out))
        return out

    def run(self, f, *, map_kind=MAP_SCALAR, gamma=1.0 + 0j, metric=METRIC_EUCLIDEAN, m=None,
            fmt=FMT_NPBS, rtol=1e-6, max_iters=1000, u0=None, n_snap=0) -> RunResult:
        f = _c(f, self.shape)
        u0 = None if u0 is None else _c(u0, self.shape)
        mm = None if m is None else _c(m, self.shape)
        u = np.empty_like(f)
        l2 = np.full(max_iters + 1, np.nan)
        rt = np.full(max_iters + 1, np.nan)
        tr = _Trace()
        snaps = np.zeros((n_snap,) + self.shape, np.complex128) if n_snap else None
        mp = Oracle.Map(map_kind, complex(gamma).real, complex(gamma).imag, metric, _ptr(mm))
        rc = self._lib.bpo_run(self._h, C.byref(mp), _ptr(f), fmt, rtol, max_iters, _ptr(u0),
                               _ptr(u), _ptr(l2), _ptr(rt), C.byref(tr), _ptr(snaps), n_snap)
        if rc:
            raise (ValueError if rc == 1 else OracleError)(self._lib.bpo_last_error().decode())
        k = tr.iters + 1
        return RunResult(u, l2[:k].copy(), rt[:k].copy(), tr.iters, TERM_NAMES[tr.terminated],
                         tr.fnorm_l2, tr.fnorm_reta, None if snaps is None else snaps[:k])


# --------------------------------------------------------------------------- reference build
class Reference:
    """ctypes front-end of oracle/_ref/libbpref.so (the reference's own code)."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(REF_SO):
                raise OracleError("oracle/_ref/libbpref.so not built (needs /root/reference at build time)")
            lib = C.CDLL(REF_SO)
            lib.bpref_last_error.restype = C.c_char_p
            lib.bpref_problem_create.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _dp,
                                                 C.c_double, C.c_double, C.POINTER(C.c_void_p)]
            lib.bpref_periodic_create.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _dp,
                                                  C.c_double, C.c_double, C.POINTER(C.c_void_p)]
            lib.bpref_periodic_bench_instance.argtypes = [C.c_int, C.c_double, C.c_double,
                                                          C.c_uint64, _dp, _dp, _dp, _dp]
            lib.bpref_problem_destroy.argtypes = [C.c_void_p]
            lib.bpref_problem_destroy.restype = None
            lib.bpref_symbol.argtypes = [C.c_void_p, _dp]
            lib.bpref_apply.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
            lib.bpref_born_residual.argtypes = [C.c_void_p, _dp, _dp, _dp]
            lib.bpref_residual.argtypes = [C.c_void_p, _dp, _dp, _dp]
            lib.bpref_run.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int, _dp,
                                      _dp, C.c_int, C.c_double, C.c_int, _dp, _dp, _dp, _dp,
                                      C.POINTER(_Trace)]
            lib.bpref_run_batch.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                            _dp, _dp, _dp, C.c_int, C.c_double, C.c_double,
                                            C.c_int, _dp, C.c_int, C.c_double, C.c_int, _dp, _dp,
                                            _dp, C.POINTER(_Trace), C.c_int]
            lib.bpref_run_handles.argtypes = [C.c_int, C.POINTER(C.c_void_p), C.c_int, C.c_double,
                                              C.c_double, C.c_int, _dp, C.c_long, C.c_int,
                                              C.c_double, C.c_int, _dp, _dp, _dp,
                                              C.POINTER(_Trace), C.c_int]
            lib.bpref_set_mode.argtypes = [C.c_int]
            lib.bpref_set_mode.restype = None
            lib.bpref_sponge_profile.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _dp]
            lib.bpref_gaussian_bump.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                                C.c_double, C.c_double, C.c_double, C.c_double, _dp]
            lib.bpref_rng_normals.argtypes = [C.c_uint64, C.c_int64, C.c_int, _dp]
            lib.bpref_rng_normals.restype = None
            lib.bpref_rng_uniforms.argtypes = [C.c_uint64, C.c_int64, C.c_int, _dp]
            lib.bpref_rng_uniforms.restype = None
            lib.bpref_laplacian_symbol.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _dp]
            lib.bpref_five_point.argtypes = [_dp, C.c_int, C.c_int, C.c_double, _dp]
            lib.bpref_dct.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp]
            lib.bpref_save_field.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, _dp]
            lib.bpref_load_field.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, _dp]
            lib.bpref_export_csv.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, _dp]
            lib.bpref_save_problem_helmholtz.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int,
                                                         C.c_double, C.c_double, _dp, C.c_double,
                                                         C.c_double]
            lib.bpref_load_problem_helmholtz.argtypes = [C.c_char_p] + [C.POINTER(C.c_int)] * 2 + \
                [C.POINTER(C.c_double)] * 4 + [_dp, C.c_int]
            lib.bpref_five_point.restype = None
            lib.bpref_thread_count.restype = C.c_int
            cls._lib = lib
        return cls._lib

    @classmethod
    def set_mode(cls, mode: str) -> None:
        cls.lib().bpref_set_mode({"serial": 0, "parallel": 1, "auto": 2}[mode])

    @classmethod
    def thread_count(cls) -> int:
        return cls.lib().bpref_thread_count()

    @classmethod
    def periodic_bench_instance(cls, n, ppw, contrast, seed):
        """The reference's Helmholtz bench instance (make_layered_helmholtz + bump source)."""
        k2 = np.empty((n, n), np.complex128)
        f = np.empty((n, n), np.complex128)
        k0, eta = C.c_double(), C.c_double()
        if cls.lib().bpref_periodic_bench_instance(n, ppw, contrast, seed, _ptr(k2), _ptr(f),
                                                   C.byref(k0), C.byref(eta)):
            raise OracleError(cls.lib().bpref_last_error().decode())
        return k2, f, k0.value, eta.value

    # ---- the reference's file formats (field.cpp, problem_io.cpp)
    @classmethod
    def _chk(cls, rc):
        if rc:
            raise OracleError(cls.lib().bpref_last_error().decode())

    @classmethod
    def save_field(cls, path, a):
        a = np.asarray(a)
        cx = int(np.iscomplexobj(a))
        a = np.ascontiguousarray(a, np.complex128 if cx else np.float64)
        cls._chk(cls.lib().bpref_save_field(os.fsencode(path), a.shape[0], a.shape[1], cx, _ptr(a)))

    @classmethod
    def load_field(cls, path, nx, ny, complex_=True):
        out = np.empty((nx, ny), np.complex128 if complex_ else np.float64)
        cls._chk(cls.lib().bpref_load_field(os.fsencode(path), nx, ny, int(complex_), _ptr(out)))
        return out

    @classmethod
    def export_csv(cls, path, a):
        a = np.asarray(a)
        cx = int(np.iscomplexobj(a))
        a = np.ascontiguousarray(a, np.complex128 if cx else np.float64)
        cls._chk(cls.lib().bpref_export_csv(os.fsencode(path), a.shape[0], a.shape[1], cx, _ptr(a)))

    @classmethod
    def save_problem_helmholtz(cls, directory, stem, k2, k0, eta, lx=1.0, ly=1.0):
        k2 = _c(k2)
        cls._chk(cls.lib().bpref_save_problem_helmholtz(os.fsencode(directory), stem.encode(),
                                                         k2.shape[0], k2.shape[1], lx, ly, _ptr(k2),
                                                         k0, eta))

    @classmethod
    def load_problem_helmholtz(cls, path, cap=1 << 22):
        nx, ny = C.c_int(), C.c_int()
        lx, ly, k0, eta = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        buf = np.empty(cap, np.complex128)
        cls._chk(cls.lib().bpref_load_problem_helmholtz(os.fsencode(path), C.byref(nx), C.byref(ny),
                                                         C.byref(lx), C.byref(ly), C.byref(k0),
                                                         C.byref(eta), _ptr(buf), cap))
        return dict(nx=nx.value, ny=ny.value, lx=lx.value, ly=ly.value, k0=k0.value, eta=eta.value,
                    k2=buf[:nx.value * ny.value].reshape(nx.value, ny.value).copy())

    @classmethod
    def dct(cls, x, inverse=False):
        """the reference's forward/inverse DCT transform pair on a Neumann grid"""
        x = _c(x)
        out = np.empty_like(x)
        if cls.lib().bpref_dct(x.shape[0], x.shape[1], int(inverse), _ptr(x), _ptr(out)):
            raise OracleError(cls.lib().bpref_last_error().decode())
        return out

    @classmethod
    def sponge_profile(cls, nx, ny, layer, strength=1.0, bc=1):
        out = np.empty((nx, ny))
        if cls.lib().bpref_sponge_profile(nx, ny, bc, layer, strength, _ptr(out)):
            raise ValueError(cls.lib().bpref_last_error().decode())
        return out

    @classmethod
    def gaussian_bump(cls, nx, ny, cx, cy, width, amp=1.0, lx=1.0, ly=1.0, bc=1):
        out = np.empty((nx, ny))
        if cls.lib().bpref_gaussian_bump(nx, ny, lx, ly, bc, cx, cy, width, amp, _ptr(out)):
            raise ValueError(cls.lib().bpref_last_error().decode())
        return out

    @classmethod
    def rng_normals(cls, seed, index, count):
        out = np.empty(count)
        cls.lib().bpref_rng_normals(seed, index, count, _ptr(out))
        return out

    @classmethod
    def rng_uniforms(cls, seed, index, count):
        out = np.empty(count)
        cls.lib().bpref_rng_uniforms(seed, index, count, _ptr(out))
        return out

    @classmethod
    def laplacian_symbol(cls, nx, ny, lx=1.0, ly=1.0, bc=1):
        out = np.empty((nx, ny), np.complex128)
        if cls.lib().bpref_laplacian_symbol(nx, ny, lx, ly, bc, _ptr(out)):
            raise ValueError(cls.lib().bpref_last_error().decode())
        return out

    @classmethod
    def run_batch(cls, k2, k0, eta, f, *, map_kind=MAP_SCALAR, gamma=1.0 + 0j, metric=0,
                  fmt=FMT_NPBS, rtol=1e-6, max_iters=1000, nthreads=None, lx=1.0, ly=1.0):
        k2, f = _c(k2), _c(f)
        batch, nx, ny = k2.shape
        k0 = np.ascontiguousarray(k0, np.float64)
        eta = np.ascontiguousarray(eta, np.float64)
        u = np.empty_like(f)
        l2 = np.full((batch, max_iters + 1), np.nan)
        rt = np.full((batch, max_iters + 1), np.nan)
        tr = (_Trace * batch)()
        nthreads = nthreads or os.cpu_count()
        g = complex(gamma)
        rc = cls.lib().bpref_run_batch(nx, ny, lx, ly, batch, _ptr(k2), _ptr(k0), _ptr(eta),
                                       map_kind, g.real, g.imag, metric, _ptr(f), fmt, rtol,
                                       max_iters, _ptr(u), _ptr(l2), _ptr(rt), tr, nthreads)
        if rc:
            raise OracleError(cls.lib().bpref_last_error().decode())
        return u, l2, rt, [(t.iters, TERM_NAMES[t.terminated]) for t in tr]


class ReferenceBatch:
    """Reference problems of a batch created ONCE (the reference's Problem constructors), then
    run repeatedly with OpenMP over members (bpref_run_handles, the sample-parallel loop of
    proj/src/bench.cpp:143-151): the bench's reference arm times only the runs."""

    def __init__(self, k2, k0, eta, lx: float = 1.0, ly: float = 1.0):
        k2 = _c(k2)
        self.batch, self.nx, self.ny = k2.shape
        lib = Reference.lib()
        self.handles = (C.c_void_p * self.batch)()
        for b in range(self.batch):
            h = C.c_void_p()
            if lib.bpref_problem_create(self.nx, self.ny, lx, ly, _ptr(k2[b]), float(k0[b]),
                                        float(eta[b]), C.byref(h)):
                raise OracleError(lib.bpref_last_error().decode())
            self.handles[b] = h

    def close(self):
        lib = Reference.lib()
        for b in range(self.batch):
            if self.handles[b]:
                lib.bpref_problem_destroy(self.handles[b])
                self.handles[b] = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, f, *, map_kind=MAP_SCALAR, gamma=1.0 + 0j, metric=0, fmt=FMT_NPBS, rtol=1e-6,
            max_iters=1000, nthreads=None):
        f = _c(f)
        u = np.empty_like(f)
        l2 = np.full((self.batch, max_iters + 1), np.nan)
        rt = np.full((self.batch, max_iters + 1), np.nan)
        tr = (_Trace * self.batch)()
        g = complex(gamma)
        rc = Reference.lib().bpref_run_handles(self.batch, self.handles, map_kind, g.real, g.imag,
                                               metric, _ptr(f), self.nx * self.ny, fmt, rtol,
                                               max_iters, _ptr(u), _ptr(l2), _ptr(rt), tr,
                                               nthreads or os.cpu_count())
        if rc:
            raise OracleError(Reference.lib().bpref_last_error().decode())
        return u, l2, rt, [(t.iters, TERM_NAMES[t.terminated]) for t in tr]


class ReferenceProblem(OracleProblem):
    """Same interface as OracleProblem, backed by the reference's own code (oracle/_ref)."""

    backend = "reference"

    def __init__(self, k2, k0: float, eta: float, lx: float = 1.0, ly: float = 1.0,
                 periodic: bool = False):
        k2 = _c(k2)
        self.shape = k2.shape
        self.nx, self.ny = k2.shape
        self.k2, self.k0, self.eta, self.lx, self.ly = k2, float(k0), float(eta), lx, ly
        self._rl = Reference.lib()
        h = C.c_void_p()
        create = self._rl.bpref_periodic_create if periodic else self._rl.bpref_problem_create
        rc = create(self.nx, self.ny, lx, ly, _ptr(k2), k0, eta, C.byref(h))
        if rc:
            raise (ValueError if rc == 1 else OracleError)(self._rl.bpref_last_error().decode())
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            self._rl.bpref_problem_destroy(self._h)
            self._h = None

    def _op(self, op, u):
        u = _c(u, self.shape)
        out = np.empty_like(u)
        rc = self._rl.bpref_apply(self._h, op, _ptr(u), _ptr(out))
        if rc:
            raise (ValueError if rc == 1 else OracleError)(self._rl.bpref_last_error().decode())
        return out

    def symbol(self):
        out = np.empty((self.nx, self.ny), np.complex128)
        self._rl.bpref_symbol(self._h, _ptr(out))
        return out

    def apply_A(self, u): return self._op(0, u)
    def apply_V(self, u): return self._op(1, u)
    def apply_V_adjoint(self, u): return self._op(2, u)
    def apply_Lref(self, u): return self._op(3, u)
    def apply_G(self, q): return self._op(4, q)
    def forward_dst(self, x): return self._op(5, x)
    def inverse_dst(self, x): return self._op(6, x)

    def born_residual(self, u, f):
        u, f = _c(u, self.shape), _c(f, self.shape)
        out = np.empty_like(u)
        if self._rl.bpref_born_residual(self._h, _ptr(u), _ptr(f), _ptr(out)):
            raise OracleError(self._rl.bpref_last_error().decode())
        return out

    def residual(self, u, f):
        u, f = _c(u, self.shape), _c(f, self.shape)
        out = np.empty_like(u)
        if self._rl.bpref_residual(self._h, _ptr(u), _ptr(f), _ptr(out)):
            raise OracleError(self._rl.bpref_last_error().decode())
        return out

    def run(self, f, *, map_kind=MAP_SCALAR, gamma=1.0 + 0j, metric=METRIC_EUCLIDEAN, m=None,
            fmt=FMT_NPBS, rtol=1e-6, max_iters=1000, u0=None, n_snap=0) -> RunResult:
        f = _c(f, self.shape)
        u0 = None if u0 is None else _c(u0, self.shape)
        mm = None if m is None else _c(m, self.shape)
        u = np.empty_like(f)
        l2 = np.full(max_iters + 1, np.nan)
        rt = np.full(max_iters + 1, np.nan)
        tr = _Trace()
        g = complex(gamma)
        rc = self._rl.bpref_run(self._h, map_kind, g.real, g.imag, metric, _ptr(mm), _ptr(f), fmt,
                                rtol, max_iters, _ptr(u0), _ptr(u), _ptr(l2), _ptr(rt), C.byref(tr))
        if rc:
            raise (ValueError if rc == 1 else OracleError)(self._rl.bpref_last_error().decode())
        k = tr.iters + 1
        return RunResult(u, l2[:k].copy(), rt[:k].copy(), tr.iters, TERM_NAMES[tr.terminated],
                         tr.fnorm_l2, tr.fnorm_reta)
