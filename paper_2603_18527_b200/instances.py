"""Seeded synthetic instances of BASELINE.json's configs (host-side input synthesis).

Wraps ``libbornsweep_host.so`` (include/bornsweep_instances.h).  Every arm -- the CUDA path,
the plain-C oracle and the reference build -- consumes the arrays returned here.

Decisions: an "n x n grid, h = 1/n" config is the reference's
DirichletInterior grid with N = n-1 interior points per side (proj/include/bp/grid.hpp:12-24),
so the DST-I length n-1 maps onto a power-of-two transform of length n.  The reference's
default sponge (N/8 points, strength 1; proj/src/helmholtz.cpp:67-72) is folded into k2,
because the lossless cavity the configs literally describe does not converge.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from . import _native as N


@dataclass(frozen=True)
class InstanceSpec:
    n: int
    ppw: float
    contrast: float
    sigma_cells: float = 4.0
    src_sigma_cells: float = 2.0
    n_sources: int = 0
    seed: int = 0
    sponge_points: int = -1
    sponge_strength: float = 1.0
    eta_factor: float = 1.01
    dim: int = 2

    def _c(self):
        return N.InstanceSpec(self.n, self.ppw, self.contrast, self.sigma_cells,
                              self.src_sigma_cells, self.n_sources, self.seed, self.sponge_points,
                              self.sponge_strength, self.eta_factor, self.dim)


# BASELINE.json configs (synthetic stand-ins)
CONFIGS = {
    # c0: 2D CBS, 128x128 (h = 1/128), contrast 0.3, 10 ppw, single RHS, gamma = 1
    "c0": dict(spec=InstanceSpec(n=128, ppw=10.0, contrast=0.3), batch=1, map="scalar",
               rtol=1e-6),
    # c1: 64 independent media on 512x512, contrast 0.5, 8 ppw, pointwise gamma(x) = iV/eta
    "c1": dict(spec=InstanceSpec(n=512, ppw=8.0, contrast=0.5), batch=64, map="pointwise",
               rtol=1e-6),
    # c2: one high-frequency 4096x4096 grid, 6 ppw, contrast 0.5, 16 seeded point sources
    "c2": dict(spec=InstanceSpec(n=4096, ppw=6.0, contrast=0.5, n_sources=16), batch=1,
               map="pointwise", rtol=1e-6),
    # c3: 3-D 256^3 cube (255^3 interior), seven-point, sigma 3 cells, contrast 0.4, 8 ppw
    "c3": dict(spec=InstanceSpec(n=256, ppw=8.0, contrast=0.4, sigma_cells=3.0, dim=3), batch=1,
               map="pointwise", rtol=1e-5),
}


def make_instances(spec: InstanceSpec, first: int = 0, count: int = 1, nthreads: int = 0):
    """(k2, f, k0, eta) for members first..first+count-1: complex (count, N[, N], N) arrays."""
    nd = spec.n - 1
    shape = (count,) + (nd,) * spec.dim
    k2 = np.empty(shape, np.complex128)
    f = np.empty(shape, np.complex128)
    k0 = np.empty(count)
    eta = np.empty(count)
    dp = C.POINTER(C.c_double)
    s = spec._c()
    rc = N.host_lib().bp_make_instances(C.byref(s), first, count, k2.ctypes.data_as(dp),
                                        f.ctypes.data_as(dp), k0.ctypes.data_as(dp),
                                        eta.ctypes.data_as(dp), nthreads)
    if rc:
        raise ValueError(f"invalid instance spec {spec}")
    return k2, f, k0, eta


def config_instances(name: str, first: int = 0, count: int | None = None, **overrides):
    if name == "c4":
        spec = replace(CONFIGS["c4"]["spec"], **overrides) if overrides else CONFIGS["c4"]["spec"]
        return make_cdr_instances(spec, first, CONFIGS["c4"]["batch"] if count is None else count)
    cfg = CONFIGS[name]
    spec = replace(cfg["spec"], **overrides) if overrides else cfg["spec"]
    return make_instances(spec, first, cfg["batch"] if count is None else count)


@dataclass(frozen=True)
class CdrSpec:
    """Config c4 media (include/bornsweep_instances.h bp_cdr_spec)."""
    n: int = 1024
    b_max: float = 20.0
    sigma_max: float = 50.0
    smooth_cells: float = 0.0
    src_smooth_cells: float = 0.0
    seed: int = 0

    def _c(self):
        return N.CdrSpec(self.n, self.b_max, self.sigma_max, self.smooth_cells,
                         self.src_smooth_cells, self.seed)


CONFIGS["c4"] = dict(spec=CdrSpec(n=1024), batch=32, map="scalar", rtol=1e-8)


def make_cdr_instances(spec: CdrSpec, first: int = 0, count: int = 1, nthreads: int = 0):
    """(bx, by, sigma, sigma0, f): real (count, n, n) arrays and sigma0 (count)."""
    n = spec.n
    arrs = [np.empty((count, n, n)) for _ in range(4)]
    s0 = np.empty(count)
    dp = C.POINTER(C.c_double)
    s = spec._c()
    rc = N.host_lib().bp_make_cdr_instances(C.byref(s), first, count, arrs[0].ctypes.data_as(dp),
                                            arrs[1].ctypes.data_as(dp), arrs[2].ctypes.data_as(dp),
                                            s0.ctypes.data_as(dp), arrs[3].ctypes.data_as(dp), nthreads)
    if rc:
        raise ValueError(f"invalid CDR spec {spec}")
    bx, by, sigma, f = arrs
    return bx, by, sigma, s0, f
