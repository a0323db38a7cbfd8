"""Python mirror of the reference's operator / preconditioner / driver API over the C ABI.

Reference interface (all under /root/reference/proj):
  bp::Problem          include/bp/problem.hpp:16-49   -> HelmholtzDirichlet
  bp::CorrectionMap    include/bp/correction.hpp:16-40 -> ScalarMap, PointwiseMap, ...
  bp::IterationConfig  include/bp/iterate.hpp:14-18   -> IterationConfig
  bp::run / RunResult  include/bp/iterate.hpp:57-67   -> run() / RunResult
Error behaviour follows the reference's exceptions: std::invalid_argument -> ValueError,
std::runtime_error -> RuntimeError.  Fields are numpy complex128 arrays shaped
(batch, nx, ny) (or (nx, ny) for a single member), row-major x slow like bp::ComplexField.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

BC_PERIODIC, BC_DIRICHLET, BC_NEUMANN = 0, 1, 2
FORMATS = {"direct": 0, "cbs": 1, "npbs": 2}
TERMINATION = {0: "converged", 1: "max_iters", 2: "diverged", 3: "stagnated"}


class BornSweepError(RuntimeError):
    pass


class CudaError(BornSweepError):
    pass


def _raise(rc: int) -> None:
    msg = N.last_error()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise RuntimeError(msg)
    if rc == 5:
        raise NotImplementedError(msg)
    if rc == 3:
        raise CudaError(msg)
    raise BornSweepError(f"status {rc}: {msg}")


def _check(rc: int) -> None:
    if rc != 0:
        _raise(rc)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


# ---------------------------------------------------------------------------- maps
@dataclass
class ScalarMap:
    """bp::ScalarMap (classical CBS coefficient), correction.hpp:16-18."""
    gamma: complex = 1.0 + 0.0j

    def _c(self):
        g = complex(self.gamma)
        return N.Map(0, g.real, g.imag, 0, None)


@dataclass
class PointwiseMap:
    """Diagonal relaxation gamma(x) = (i/eta) V(x) (Osnabrugge CBS)."""

    def _c(self):
        return N.Map(3, 0.0, 0.0, 0, None)


@dataclass
class OptimalScalarMap:
    """bp::OptimalScalarMap (correction.hpp:20-23): per-step least-squares gamma in the
    Euclidean ("euclidean", the reference's default CBS map, bench.cpp:140-141) or the
    R_eta ("reta") metric."""
    metric: str = "euclidean"

    def _c(self):
        if self.metric not in ("euclidean", "reta"):
            raise ValueError(f"unknown optimal-scalar metric {self.metric!r}")
        return N.Map(1, 0.0, 0.0, 0 if self.metric == "euclidean" else 1, None)


class FourierDiagMap:
    """bp::FourierDiagMap (correction.hpp:25-32): du = T^{-1}(m * T(x)) in the DST-I basis,
    one multiplier m (nx x ny complex, mode layout) shared by the batch -- the learned M_theta
    of the paper's NPBS in its desk-scale form.  The identity m == 1 is plain
    preconditioned Richardson (make_identity_fourier_diag, correction.cpp:78-84)."""

    def __init__(self, m):
        self.m = np.ascontiguousarray(np.asarray(m, dtype=np.complex128))

    def _c(self):
        return N.Map(2, 0.0, 0.0, 0, _ptr(self.m))


@dataclass
class IterationConfig:
    """bp::IterationConfig (iterate.hpp:14-18)."""
    format: str = "npbs"
    rtol: float = 1e-6
    max_iters: int = 1000

    def _c(self):
        return N.IterConfig(FORMATS[self.format], float(self.rtol), int(self.max_iters))


@dataclass
class IterationTrace:
    """bp::IterationTrace (iterate.hpp:25-32); entry 0 is the initial residual."""
    res_l2_rel: np.ndarray
    res_reta_rel: np.ndarray
    iters: int
    terminated: str
    fnorm_l2: float
    fnorm_reta: float


@dataclass
class RunResult:
    u: np.ndarray
    traces: list = field(default_factory=list)
    snapshots: np.ndarray | None = None

    @property
    def trace(self) -> IterationTrace:
        return self.traces[0]


# ---------------------------------------------------------------------------- problem
class HelmholtzDirichlet:
    """Batch of Dirichlet five-point Helmholtz problems on the GPU.

    A = L_D - k2, L_ref = L_D - (k0^2 + i eta), V = k2 - (k0^2 + i eta): the reference's
    HelmholtzProblem splitting (helmholtz.cpp:11-25) on the DirichletInterior / DST-I /
    five-point pattern of NewtonJacobianProblem (newton_problem.cpp:17-44).
    """

    BC = BC_DIRICHLET
    DTYPE = np.complex128

    def __init__(self, k2, k0, eta, lx: float = 1.0, device: int = 0, dim: int = 2,
                 ly: float | None = None):
        """k2: (batch, nx, ny) -- or (nx, ny) for one member; dim=3: (batch, n, n, n) or
        (n, n, n), the seven-point 3-D extension (config c3).  Grids with nx + 1 = ny + 1 = 2^k
        and lx == ly run the fused power-of-two kernels; any other 2-D Dirichlet shape runs the
        any-shape path (generic_kernels.cuh: radix-2 / Bluestein line transforms)."""
        k2 = np.asarray(k2, dtype=np.complex128)
        self.dim = dim
        self.single = k2.ndim == dim
        k2 = np.ascontiguousarray(k2.reshape((1,) + k2.shape) if self.single else k2)
        self.batch = k2.shape[0]
        self.grid_shape = k2.shape[1:]
        self.nx, self.ny = self.grid_shape[:2]
        k0 = np.ascontiguousarray(np.broadcast_to(np.asarray(k0, np.float64), (self.batch,)))
        eta = np.ascontiguousarray(np.broadcast_to(np.asarray(eta, np.float64), (self.batch,)))
        self.k0, self.eta, self.lx, self.device = k0, eta, lx, device
        self.ly = lx if ly is None else ly
        self.k2 = k2  # host copy of the media (save_problem)
        h = C.c_void_p()
        self._lib = N.lib()
        if dim == 3:
            g3 = N.Grid3(*self.grid_shape, lx, lx, lx, BC_DIRICHLET)
            rc = self._lib.bp_problem_create3d(C.byref(g3), self.batch, _ptr(k2), _ptr(k0),
                                               _ptr(eta), device, C.byref(h))
        else:
            g = N.Grid(self.nx, self.ny, lx, self.ly, self.BC)
            rc = self._lib.bp_problem_create(C.byref(g), self.batch, _ptr(k2), _ptr(k0), _ptr(eta),
                                             device, C.byref(h))
        _check(rc)
        self._h = h

    # context management / lifetime
    def close(self):
        if getattr(self, "_h", None):
            self._lib.bp_problem_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    @property
    def shape(self):
        return (self.batch,) + tuple(self.grid_shape)

    def _field(self, x):
        x = np.asarray(x, dtype=self.DTYPE)
        if x.shape == tuple(self.grid_shape) and self.batch == 1:
            x = x.reshape(self.shape)
        if x.shape != self.shape:
            raise ValueError(f"field shape {x.shape} does not match problem {self.shape}")
        return np.ascontiguousarray(x)

    def _out(self, out):
        return out.reshape(self.grid_shape) if self.single else out

    def _unary(self, fn, x):
        x = self._field(x)
        out = np.empty_like(x)
        _check(getattr(self._lib, fn)(self._h, _ptr(x), _ptr(out)))
        return self._out(out)

    def apply_A(self, u): return self._unary("bp_apply_A", u)
    def apply_V(self, u): return self._unary("bp_apply_V", u)
    def apply_V_adjoint(self, u): return self._unary("bp_apply_V_adjoint", u)
    def apply_Lref(self, u): return self._unary("bp_apply_Lref", u)
    def apply_G(self, q): return self._unary("bp_apply_G", q)
    def forward_transform(self, x): return self._unary("bp_forward_transform", x)
    def inverse_transform(self, x): return self._unary("bp_inverse_transform", x)

    def born_residual(self, u, f):
        u, f = self._field(u), self._field(f)
        out = np.empty_like(u)
        _check(self._lib.bp_born_residual(self._h, _ptr(u), _ptr(f), _ptr(out)))
        return self._out(out)

    def residual(self, u, f):
        u, f = self._field(u), self._field(f)
        out = np.empty_like(u)
        _check(self._lib.bp_residual(self._h, _ptr(u), _ptr(f), _ptr(out)))
        return self._out(out)

    def set_medium(self, k2, k0, eta) -> None:
        """Swap in new media (same grid/batch) without re-allocating device workspace."""
        k2 = self._field(k2)
        k0 = np.ascontiguousarray(np.broadcast_to(np.asarray(k0, np.float64), (self.batch,)))
        eta = np.ascontiguousarray(np.broadcast_to(np.asarray(eta, np.float64), (self.batch,)))
        _check(self._lib.bp_problem_set_medium(self._h, _ptr(k2), _ptr(k0), _ptr(eta)))
        self.k0, self.eta, self.k2 = k0, eta, k2

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(self._lib.bp_problem_stream(self._h, C.byref(s)))
        return s.value or 0

    def set_kernel_timing(self, enable: bool) -> None:
        _check(self._lib.bp_set_kernel_timing(self._h, int(bool(enable))))

    def last_run_stats(self) -> dict:
        la, sw, tm = C.c_int64(), C.c_int64(), C.c_int64()
        r, c = C.c_double(), C.c_double()
        _check(self._lib.bp_last_run_stats(self._h, C.byref(la), C.byref(sw), C.byref(r),
                                           C.byref(c), C.byref(tm)))
        return {"kernel_launches": la.value, "active_sweeps": sw.value, "row_ms": r.value,
                "col_ms": c.value, "timed_sweeps": tm.value}


class HelmholtzPeriodic(HelmholtzDirichlet):
    """The reference's own family: bp::HelmholtzProblem (helmholtz.cpp:11-53), periodic
    pseudospectral, A = F^-1(|xi|^2 F u) - k2 u, FFT basis, h = lx/nx.  nx = ny = 2^k with
    lx == ly: fused FFT kernels, iterate carried in Fourier space (maps: ScalarMap,
    OptimalScalarMap, FourierDiagMap); any other nx x ny <= 4096: the any-shape path
    (radix-2 / Bluestein DFT lines, ScalarMap)."""

    BC = BC_PERIODIC


class CdrNeumann(HelmholtzDirichlet):
    """Config c4: convection-diffusion-reaction batch on the Neumann cell-centred grid
    (h = lx/nx), A = -Lap_N + b . grad_upwind + sigma, L_ref = -Lap_N + sigma0 (DCT-II basis,
    transforms.cpp:120-121,142-143; symbol.cpp:81-92), V = L_ref - A.  REAL float64 fields
    (batch, n, n); maps: real ScalarMap.  No reference problem family exists for it (SURVEY.md
    8(a) a16): the oracle (oracle/bp_oracle.c, bpo_problem_create_cdr) is the parity anchor."""

    BC = BC_NEUMANN
    DTYPE = np.float64

    def __init__(self, bx, by, sigma, sigma0=None, lx: float = 1.0, device: int = 0):
        bx = np.asarray(bx, np.float64)
        self.dim = 2
        self.single = bx.ndim == 2
        shape = ((1,) + bx.shape) if self.single else bx.shape
        bx = np.ascontiguousarray(bx.reshape(shape))
        by = np.ascontiguousarray(np.asarray(by, np.float64).reshape(shape))
        sigma = np.ascontiguousarray(np.asarray(sigma, np.float64).reshape(shape))
        self.batch = shape[0]
        self.grid_shape = shape[1:]
        self.nx, self.ny = self.grid_shape
        if sigma0 is None:  # the reference CDR default sigma0 = mean sigma (cdr.cpp:215)
            sigma0 = sigma.reshape(self.batch, -1).mean(axis=1)
        sigma0 = np.ascontiguousarray(np.broadcast_to(np.asarray(sigma0, np.float64), (self.batch,)))
        self.sigma0, self.lx, self.device = sigma0, lx, device
        self.bx, self.by, self.sigma = bx, by, sigma  # host copies (save_problem)
        h = C.c_void_p()
        self._lib = N.lib()
        g = N.Grid(self.nx, self.ny, lx, lx, BC_NEUMANN)
        _check(self._lib.bp_problem_create_cdr(C.byref(g), self.batch, _ptr(bx), _ptr(by),
                                               _ptr(sigma), _ptr(sigma0), device, C.byref(h)))
        self._h = h

    def set_medium(self, bx, by, sigma, sigma0=None) -> None:
        bx, by, sigma = self._field(bx), self._field(by), self._field(sigma)
        if sigma0 is None:
            sigma0 = sigma.reshape(self.batch, -1).mean(axis=1)
        sigma0 = np.ascontiguousarray(np.broadcast_to(np.asarray(sigma0, np.float64), (self.batch,)))
        _check(self._lib.bp_problem_set_cdr_medium(self._h, _ptr(bx), _ptr(by), _ptr(sigma),
                                                   _ptr(sigma0)))
        self.sigma0, self.bx, self.by, self.sigma = sigma0, bx, by, sigma


def run(problem: HelmholtzDirichlet, cmap, f, config: IterationConfig | None = None, u0=None,
        n_snap: int = 0) -> RunResult:
    """bp::run (iterate.cpp:88-153) over every member of the batch."""
    config = config or IterationConfig()
    f = problem._field(f)
    u0 = None if u0 is None else problem._field(u0)
    u = np.empty_like(f)
    stride = config.max_iters + 1
    l2 = np.empty((problem.batch, stride))
    rt = np.empty((problem.batch, stride))
    info = (N.Trace * problem.batch)()
    mp, cfg = cmap._c(), config._c()
    lib = problem._lib
    snaps = None
    if n_snap:
        snaps = np.zeros((n_snap,) + problem.shape, problem.DTYPE)
        rc = lib.bp_run_snapshots(problem.handle, C.byref(mp), _ptr(f), C.byref(cfg), _ptr(u0),
                                  _ptr(u), _ptr(l2), _ptr(rt), info, _ptr(snaps), n_snap)
    else:
        rc = lib.bp_run(problem.handle, C.byref(mp), _ptr(f), C.byref(cfg), _ptr(u0), _ptr(u),
                        _ptr(l2), _ptr(rt), info)
    _check(rc)
    traces = []
    for b in range(problem.batch):
        k = info[b].iters + 1
        traces.append(IterationTrace(l2[b, :k].copy(), rt[b, :k].copy(), info[b].iters,
                                     TERMINATION[info[b].terminated], info[b].fnorm_l2,
                                     info[b].fnorm_reta))
    if snaps is not None and problem.single:
        snaps = snaps[:, 0]
    return RunResult(problem._out(u), traces, snaps)


class Pipeline:
    """Overlapped solves over ``depth`` problem handles of one shape (bp_pipeline_*): each
    ``submit`` is ``set_medium`` (when a medium is given) + ``run`` on the next slot, executed by
    that slot's native worker thread on the slot's own stream, so the PCIe copies of one job run
    under the sweeps of the others.  The reference solves one batch at a time
    (proj/src/bench.cpp:143-151); every job's result is bit-identical to calling
    ``problem.set_medium(...)`` + ``run(problem, ...)`` directly.

    ``submit`` returns a handle; ``wait()`` blocks for every submitted job and returns their
    RunResults in submission order.  Host buffers are held until then (pass pinned arrays for
    overlapped copies)."""

    def __init__(self, problems):
        self.problems = list(problems)
        if not self.problems:
            raise ValueError("Pipeline needs at least one problem handle")
        p0 = self.problems[0]
        for p in self.problems[1:]:
            if type(p) is not type(p0) or p.shape != p0.shape:
                raise ValueError("Pipeline slots must be problems of one family and shape")
        self._lib = N.lib()
        self._h = None
        self._jobs = []
        hs = (C.c_void_p * len(self.problems))(*[p.handle for p in self.problems])
        h = C.c_void_p()
        _check(self._lib.bp_pipeline_create(hs, len(self.problems), C.byref(h)))
        self._h = h

    def submit(self, cmap, f, config: IterationConfig | None = None, medium=None, u0=None,
               u_out=None) -> int:
        """medium: None (keep the slot's medium), (k2, k0, eta) for Helmholtz problems or
        (bx, by, sigma[, sigma0]) for CdrNeumann.  u_out: optional preallocated (pinned) output
        of the problem's shape.  Returns the job index into wait()'s list."""
        config = config or IterationConfig()
        p = self.problems[0]
        f = p._field(f)
        u0 = None if u0 is None else p._field(u0)
        u = np.empty_like(f) if u_out is None else u_out
        if u.shape != f.shape or u.dtype != f.dtype or not u.flags["C_CONTIGUOUS"]:
            raise ValueError("u_out must be a C-contiguous array of the problem's shape and dtype")
        keep = []
        md = N.Medium()
        if medium is not None:
            if isinstance(p, CdrNeumann):
                bx, by, sg = (p._field(a) for a in medium[:3])
                s0 = medium[3] if len(medium) > 3 and medium[3] is not None else \
                    sg.reshape(p.batch, -1).mean(axis=1)
                s0 = np.ascontiguousarray(np.broadcast_to(np.asarray(s0, np.float64), (p.batch,)))
                md.bx, md.by, md.sigma, md.sigma0 = _ptr(bx), _ptr(by), _ptr(sg), _ptr(s0)
                keep += [bx, by, sg, s0]
            else:
                k2 = p._field(medium[0])
                k0 = np.ascontiguousarray(np.broadcast_to(np.asarray(medium[1], np.float64), (p.batch,)))
                eta = np.ascontiguousarray(np.broadcast_to(np.asarray(medium[2], np.float64), (p.batch,)))
                md.k2, md.k0, md.eta = _ptr(k2), _ptr(k0), _ptr(eta)
                keep += [k2, k0, eta]
        stride = config.max_iters + 1
        l2 = np.empty((p.batch, stride))
        rt = np.empty((p.batch, stride))
        info = (N.Trace * p.batch)()
        mp, cfg = cmap._c(), config._c()
        slot = C.c_int32()
        _check(self._lib.bp_pipeline_submit(self._h, C.byref(md), C.byref(mp), _ptr(f), C.byref(cfg),
                                            _ptr(u0), _ptr(u), _ptr(l2), _ptr(rt), info,
                                            C.byref(slot)))
        self._jobs.append((slot.value, u, l2, rt, info, keep + [f, u0, md, mp, cfg, cmap]))
        return len(self._jobs) - 1

    def wait(self) -> list:
        """Block until every submitted job finished; RunResults in submission order."""
        rc = self._lib.bp_pipeline_wait(self._h)
        jobs, self._jobs = self._jobs, []
        _check(rc)
        out = []
        for slot, u, l2, rt, info, _ in jobs:
            p = self.problems[slot]
            traces = []
            for b in range(p.batch):
                k = info[b].iters + 1
                traces.append(IterationTrace(l2[b, :k].copy(), rt[b, :k].copy(), info[b].iters,
                                             TERMINATION[info[b].terminated], info[b].fnorm_l2,
                                             info[b].fnorm_reta))
            out.append(RunResult(p._out(u), traces, None))
        return out

    def close(self):
        if getattr(self, "_h", None):
            self._lib.bp_pipeline_wait(self._h)
            self._lib.bp_pipeline_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        self.close()
