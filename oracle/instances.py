"""Instance synthesis for the bench's REFERENCE arm (ORACLE infrastructure, test/bench only).

The reference arm must not load anything from the product package, so it builds the c1 / c4
inputs here from the reference's OWN generators in oracle/_ref/libbpref.so:
  * white noise  -- RngState(seed).split(member) Box-Muller normals (proj/include/bp/rng.hpp:10-62)
  * sponge       -- sponge_profile (proj/src/samplers.cpp:130-150), DirichletInterior grid
  * source       -- gaussian_bump (proj/src/samplers.cpp:86-105)
and restates, in numpy, the BASELINE construction the product's host synthesis uses
(decision 5): separable Gaussian smoothing truncated at 4 sigma, zero
padded (c4: reflective, truncated at 3 sigma), normalised to unit max-abs, c = 1 + contrast g
clipped, k = omega / c, k0 = mean k, k^2 -> k^2 (1 + i d), eta = 1.01 max|k^2 - k0^2|
(proj/src/helmholtz.cpp:62-87 rules).  The summation order of the smoothing differs from the
product's C++ loops, so the arrays agree to rounding (tests/test_ref_instances.py pins them
at <= 1e-12), not bit for bit; the reference arm only needs the same workload.
"""
from __future__ import annotations

import math

import numpy as np
from scipy.ndimage import convolve1d

from . import Reference


def _weights(sigma: float, trunc: float) -> np.ndarray:
    r = int(math.ceil(trunc * sigma))
    d = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-0.5 * d * d / (sigma * sigma))
    return w / w.sum()


def _smooth(a: np.ndarray, sigma: float, trunc: float, mode: str) -> np.ndarray:
    w = _weights(sigma, trunc)
    out = convolve1d(a, w, axis=1, mode=mode, cval=0.0)
    return convolve1d(out, w, axis=0, mode=mode, cval=0.0)


def helmholtz_c1(first: int, count: int, *, n: int = 512, ppw: float = 8.0,
                 contrast: float = 0.5, sigma_cells: float = 4.0, src_sigma_cells: float = 2.0,
                 seed: int = 0, eta_factor: float = 1.01):
    """(k2, f, k0, eta) of BASELINE c1 members first..first+count-1 (N = n-1 interior)."""
    N = n - 1
    h = 1.0 / n
    omega = 2.0 * math.pi / (ppw * h)
    layer = N // 8
    d = Reference.sponge_profile(N, N, layer, 1.0)
    src = Reference.gaussian_bump(N, N, 0.5, 0.5, src_sigma_cells * h)
    k2 = np.empty((count, N, N), np.complex128)
    f = np.empty((count, N, N), np.complex128)
    k0 = np.empty(count)
    eta = np.empty(count)
    for i in range(count):
        noise = Reference.rng_normals(seed, first + i, N * N).reshape(N, N)
        g = _smooth(noise, sigma_cells, 4.0, "constant")
        gmax = float(np.abs(g).max()) or 1.0
        c = np.clip(1.0 + contrast * (g / gmax), 1.0 - contrast, 1.0 + contrast)
        kk = omega / c
        k0[i] = kk.mean()
        k2[i] = (kk * kk) * (1.0 + 1j * d)
        eta[i] = max(eta_factor * float(np.abs(k2[i] - k0[i] * k0[i]).max()), 1e-3)
        f[i] = src
    return k2, f, k0, eta


def cdr_c4(first: int, count: int, *, n: int = 1024, b_max: float = 20.0,
           sigma_max: float = 50.0, seed: int = 0):
    """(bx, by, sigma, sigma0, f) of BASELINE c4 members (Neumann cell-centred n x n)."""
    sm, sf = n / 16.0, n / 32.0
    outs = [np.empty((count, n, n)) for _ in range(4)]  # sigma, bx, by, f
    s0 = np.empty(count)
    for i in range(count):
        noise = Reference.rng_normals(seed, first + i, 4 * n * n).reshape(4, n, n)
        for k in range(4):
            g = _smooth(noise[k], sf if k == 3 else sm, 3.0, "reflect")
            g /= float(np.abs(g).max()) or 1.0
            outs[k][i] = g
        outs[0][i] = 0.5 * sigma_max * (1.0 + outs[0][i])
        s0[i] = outs[0][i].mean()
        outs[1][i] *= b_max / math.sqrt(2.0)
        outs[2][i] *= b_max / math.sqrt(2.0)
    sigma, bx, by, f = outs
    return bx, by, sigma, s0, f
