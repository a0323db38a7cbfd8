"""CPU stand-in for one rank's slab part (the interface of paper_2603_18527_b200.slab.SlabPart)
so the slab driver's host logic -- partition, blocked all-to-all layout, halo exchange,
all-reduced sums, identical termination on every rank -- runs under gloo on CPUs.

Same stage semantics as the CUDA slab stages (include/bornsweep.h BP_SLAB_*), computed with
scipy's DST-I (== FFTW RODFT00): forward = plain sine sum (transforms.cpp:117), Green weights
4/(n^2 lambda) (symbol.cpp:69-80, transforms.cpp:99), termination restating iterate.cpp:134-150.
Test infrastructure only."""
import math

import numpy as np
import scipy.fft as sf
import torch

from paper_2603_18527_b200.api import TERMINATION, IterationTrace
from paper_2603_18527_b200.slab import (COL, COL_FD, COL_LREF, FD_A, FD_B, FINALIZE, FWD_BORN, FWD_F, GAMMA, INIT,
                                        INV_NORM, OPT_A, OPT_B, RETA_A, RETA_C, SWEEP, ZERO_U)


def _sine(a):
    """plain sine sum over the interior (index 1..n-1) along the last axis of padded rows"""
    out = np.zeros_like(a)
    out[..., 1:] = 0.5 * sf.dst(a[..., 1:], type=1, axis=-1)
    return out


class NumpySlabPart:
    def __init__(self, k2, k0, eta, rank, nranks, lx=1.0):
        k2 = np.asarray(k2, np.complex128)
        self.nx, self.ny = k2.shape
        self.shape = k2.shape
        n = self.nx + 1
        R = n // nranks
        self.n, self.rows, self.rank, self.nranks, self.row0 = n, R, rank, nranks, rank * R
        self.h = lx / n
        self.k0sq, self.eta = k0 * k0, eta
        self.k2 = self._pack(k2)
        self.V = self.k2 - (self.k0sq + 1j * eta)
        j = np.arange(n)
        self.lap = 4.0 / self.h ** 2 * np.sin(j * np.pi / (2 * n)) ** 2
        self._T = np.zeros((nranks, R, R), np.complex128)
        self._Tc = np.zeros((nranks, R, R), np.complex128)
        self._sums = np.zeros(8)
        self._u = [np.zeros((R + 2, n), np.complex128) for _ in range(2)]
        self.t_rows, self.t_cols = torch.from_numpy(self._T), torch.from_numpy(self._Tc)
        self.sums = torch.from_numpy(self._sums)
        self.u_first = [torch.from_numpy(u[1]) for u in self._u]
        self.u_last = [torch.from_numpy(u[R]) for u in self._u]
        self.u_halo_lo = [torch.from_numpy(u[0]) for u in self._u]
        self.u_halo_hi = [torch.from_numpy(u[R + 1]) for u in self._u]
        self.f = np.zeros((R, n), np.complex128)
        self.y = np.zeros((R, n), np.complex128)
        self.valid = (self.row0 + np.arange(R)) % n != 0

    def _pack(self, dense):
        out = np.zeros((self.rows, self.n), np.complex128)
        for i in range(self.rows):
            x = self.row0 + i
            if 1 <= x <= self.nx:
                out[i, 1:] = dense[x - 1]
        return out

    # blocked [dest][row][col in block] <-> rows x n
    def _block(self, rows):
        R, P = self.rows, self.nranks
        self._T[...] = rows.reshape(R, P, R).transpose(1, 0, 2)

    def _unblock(self):
        R, P = self.rows, self.nranks
        return self._T.transpose(1, 0, 2).reshape(R, P * R).copy()

    def set_fields(self, f, u0=None):
        self.f = self._pack(np.asarray(f, np.complex128))
        self._u[0][...] = 0
        if u0 is not None:
            self._u[0][1:self.rows + 1] = self._pack(np.asarray(u0, np.complex128))

    def host_sums(self):
        return self._sums.copy()

    def _finalize(self, s0, s1):
        m = self.sweep
        rel, rel_reta = math.sqrt(s0) / self.fn, math.sqrt(s1) / self.gn
        self.l2[m], self.rt[m] = rel, rel_reta
        term = -1
        if m == 0:
            if rel <= self.rtol:
                term = 0
        else:
            if not math.isfinite(rel) or rel > 1e8:
                term = 2
            elif rel <= self.rtol:
                term = 0
            elif m + 1 > 20:
                past = self.l2[m - 20]
                if abs(past - rel) < 1e-14 * max(1.0, past):
                    term = 3
        if term < 0 and m >= self.max_iters:
            term = 1
        if term >= 0:
            self.iters, self.term, self.result_buf, self.status = m, term, m & 1, 1
        self.sweep = m + 1

    # ---- primitives of the staged OptimalScalar / FourierDiag sweeps (2-D; overridden in 3-D)
    def _rows_fwd(self, field):
        self._block(_sine(field))

    def _rows_inv(self):
        return _sine(self._unblock())

    def _interior(self):
        return self.valid[:, None] & (np.arange(self.n) != 0)[None, :]

    def _stencil(self, ua):
        R = self.rows
        u = ua[1:R + 1]
        uw = np.zeros_like(u)
        uw[:, 1:] = u[:, :-1]
        ue = np.zeros_like(u)
        ue[:, :-1] = u[:, 1:]
        return 4.0 * u - ua[0:R] - ua[2:R + 2] - uw - ue

    def _mode_weights(self):
        """(x mode, local column) mask of the non-zero Dirichlet modes, t_cols layout"""
        n, R = self.n, self.rows
        q = self.rank * R + np.arange(R)
        w = np.ones((n, R))
        w[0, :] = 0
        w[:, q == 0] = 0
        return w

    def set_multiplier(self, m):
        n, R = self.n, self.rows
        full = np.zeros((n, n), np.complex128)
        full[1:, 1:] = np.asarray(m, np.complex128)
        self.fd = full[:, self.rank * R:(self.rank + 1) * R].copy()

    def _col_fd(self):
        n, R = self.n, self.rows
        M = self._Tc.reshape(n, -1)
        scale = (2.0 / n) ** (3 if M.shape[1] != R else 2)  # forward x inverse sine sums
        M[...] = _sine_ax(_sine_ax(M, 0) * (self.fd.reshape(n, -1) * scale), 0)

    def _col_lref(self):
        """x-DST, x lambda x (2/n)^dim, inverse x-DST on the received block (L_ref of the direction)"""
        n, R = self.n, self.rows
        M = self._Tc.reshape(n, -1)
        q = self.rank * R + np.arange(R)
        if M.shape[1] == R:
            lam = self.lap[:, None] + self.lap[q][None, :] - (self.k0sq + 1j * self.eta)
            scale = (2.0 / n) ** 2
        else:
            lam = (self.lap[:, None, None] + self.lap[q][None, :, None] + self.lap[None, None, :]
                   - (self.k0sq + 1j * self.eta)).reshape(n, -1)
            scale = (2.0 / n) ** 3
        M[...] = _sine_ax(_sine_ax(M, 0) * (lam * scale * self._mode_weights_flat()), 0)

    def _mode_weights_flat(self):
        n, R = self.n, self.rows
        q = self.rank * R + np.arange(R)
        if self._Tc.size == n * R:
            w = np.ones((n, R))
            w[0, :] = 0
            w[:, q == 0] = 0
            return w
        w = np.ones((n, R, n))
        w[0], w[:, :, 0] = 0, 0
        w[:, q == 0, :] = 0
        return w.reshape(n, -1)

    def _map_stage(self, code, lw=False):
        """OPT_A / OPT_B / RETA_A / RETA_C / FD_A / FD_B (csrc/sweep_kernels.cuh RowMode)."""
        if self.status != 0:
            return
        R = self.rows
        mask = self._interior()
        if code in (OPT_A, RETA_A, FD_A):  # entry modes: m = sweep
            ua = self._u[self.sweep & 1]
            u = ua[1:R + 1]
            r = (self.f - (self._stencil(ua) / self.h ** 2 - self.k2 * u)) * mask
            x = (self._rows_inv() - u) * mask
            self._sums[0] = np.sum((np.abs(r) ** 2)[mask])
            self._sums[1] = np.sum((np.abs(x) ** 2)[mask])
            d = r if self.direct else x  # the direction (iterate.cpp:118-123)
            if code == OPT_A:  # w = A x = r - V x (key identity), gamma = <w, r> / <w, w>
                w = (r - self.V * x)[mask]
                num = np.vdot(w, r[mask])
                self._sums[2:5] = num.real, num.imag, np.sum(np.abs(w) ** 2)
                self.x = x
            elif code == RETA_A:
                self.x = d
                self._rows_fwd(self.V * d)
            else:
                if lw:
                    self.x = d
                self._rows_fwd(d)
            return
        m = self.sweep - 1  # post modes: entry m was recorded
        if code == RETA_C:
            # R_eta metric: w = x - G V x; Direct + Euclidean (lw): w = L_ref x - V x = A x
            w = ((self._rows_inv() - self.V * self.x) if lw else (self.x - self._rows_inv()))[mask]
            num = np.vdot(w, self.x[mask])
            self._sums[0:3] = num.real, num.imag, np.sum(np.abs(w) ** 2)
            return
        u = self._u[m & 1][1:R + 1]
        du = self.gamma * self.x if code == OPT_B else self._rows_inv()
        unew = (u + du) * mask
        nxt = self._u[(m + 1) & 1][1:R + 1]
        nxt[self.valid] = unew[self.valid]
        self._rows_fwd(self.V * nxt + self.f)

    def _gamma(self, off):
        if self.status != 0:
            return
        num = complex(self._sums[off], self._sums[off + 1])
        den = self._sums[off + 2]
        self.gamma = num / den if den > 0 and math.isfinite(den) else 0.0

    def stage(self, code, cmap=None, config=None, a0=0.0, a1=0.0):
        R, n = self.rows, self.n
        if code in (OPT_A, OPT_B, RETA_A, RETA_C, FD_A, FD_B):
            self._map_stage(code, lw=a0 == 1.0)
        elif code == COL_LREF:
            if self.status == 0:
                self._col_lref()
        elif code == GAMMA:
            self._gamma(0)
        elif code == COL_FD:
            if self.status == 0:
                self._col_fd()
        elif code == FWD_F:
            self._block(_sine(self.f))
            self._sums[0] = np.sum(np.abs(self.f) ** 2)
        elif code == COL:
            if getattr(self, "status", 0) != 0:
                return
            M = self._Tc.reshape(n, R)
            q = self.rank * R + np.arange(R)
            X = _sine(M.T)  # x-DST of every column
            lam = self.lap[None, :] + self.lap[q][:, None] - (self.k0sq + 1j * self.eta)
            w = 4.0 / (n * n) / lam
            w[:, 0] = 0
            w[q == 0, :] = 0
            M[...] = _sine(X * w).T
        elif code == INV_NORM:
            self.y = _sine(self._unblock()) * self.valid[:, None]
            self._sums[1] = np.sum(np.abs(self.y) ** 2)
        elif code == INIT:
            if not a0 > 0:
                raise ValueError("run: zero source")
            self.fn, self.gn = a0, a1
            self.rtol, self.max_iters = config.rtol, config.max_iters
            self.direct = config.format == "direct"
            self.l2 = np.full(config.max_iters + 1, np.nan)
            self.rt = np.full(config.max_iters + 1, np.nan)
            self.status, self.sweep = 0, 0
            self._u[1][...] = 0
        elif code == FWD_BORN:
            u = self._u[0][1:R + 1]
            self._block(_sine(self.V * u + self.f))
        elif code == SWEEP:
            if self.status != 0:
                return
            m = self.sweep
            ua = self._u[m & 1]
            u = ua[1:R + 1]
            z = _sine(self._unblock())
            un, us = ua[0:R], ua[2:R + 2]
            uw = np.zeros_like(u)
            uw[:, 1:] = u[:, :-1]
            ue = np.zeros_like(u)
            ue[:, :-1] = u[:, 1:]
            s = 4.0 * u - un - us - uw - ue
            r = self.f - (s / self.h ** 2 - self.k2 * u)
            x = z - u
            mask = self.valid[:, None] & (np.arange(n) != 0)[None, :]
            self._sums[0] = np.sum((np.abs(r) ** 2)[mask])
            self._sums[1] = np.sum((np.abs(x) ** 2)[mask])
            g = 1j / self.eta * self.V if cmap.__class__.__name__ == "PointwiseMap" else complex(cmap.gamma)
            unew = u + g * (r if self.direct else x)
            unew[:, 0] = 0
            nxt = self._u[(m + 1) & 1][1:R + 1]
            nxt[self.valid] = unew[self.valid]
            self._block(_sine(self.V * nxt + self.f))
        elif code == FINALIZE:
            if self.status == 0:
                if a0 == 1.0:
                    self._gamma(2)
                self._finalize(self._sums[0], self._sums[1])
        elif code == ZERO_U:
            self._u[0][...] = 0

    def active(self):
        return 1 if self.status == 0 else 0

    def result(self, u_dense, max_iters):
        rows = self._u[self.result_buf][1:self.rows + 1]
        for i in range(self.rows):
            x = self.row0 + i
            if 1 <= x <= self.nx:
                u_dense[x - 1] = rows[i, 1:]
        k = self.iters + 1
        return IterationTrace(self.l2[:k].copy(), self.rt[:k].copy(), self.iters, TERMINATION[self.term],
                              self.fn, self.gn)


def _sine_ax(a, axis):
    """plain sine sum over the interior (index 1..n-1) along `axis` of padded data"""
    a = np.moveaxis(a, axis, -1)
    out = np.zeros_like(a)
    out[..., 1:] = 0.5 * sf.dst(a[..., 1:], type=1, axis=-1)
    return np.moveaxis(out, -1, axis)


class NumpySlabPart3(NumpySlabPart):
    """3-D x-plane slab (bp_slab_create3d): planes [R][y][z]; t_rows = [dest][x_local][y_local][z]
    (dest = y-block); the SWEEP / FWD_* stages end with the y-DST, SWEEP / INV_NORM start with
    the inverse one; COL = x-DST, x 8/(n^3 lambda), inverse x-DST on the received y-block."""

    def __init__(self, k2, k0, eta, rank, nranks, lx=1.0):
        k2 = np.asarray(k2, np.complex128)
        self.shape = k2.shape
        self.nx, self.ny = k2.shape[:2]
        n = self.nx + 1
        R = n // nranks
        self.n, self.rows, self.rank, self.nranks, self.row0 = n, R, rank, nranks, rank * R
        self.h = lx / n
        self.k0sq, self.eta = k0 * k0, eta
        self.k2 = self._pack(k2)
        self.V = self.k2 - (self.k0sq + 1j * eta)
        j = np.arange(n)
        self.lap = 4.0 / self.h ** 2 * np.sin(j * np.pi / (2 * n)) ** 2
        self._T = np.zeros((nranks, R * R * n), np.complex128)
        self._Tc = np.zeros((nranks, R * R * n), np.complex128)
        self._sums = np.zeros(8)
        self._u = [np.zeros((R + 2, n, n), np.complex128) for _ in range(2)]
        self.t_rows, self.t_cols = torch.from_numpy(self._T), torch.from_numpy(self._Tc)
        self.sums = torch.from_numpy(self._sums)
        self.u_first = [torch.from_numpy(u[1]) for u in self._u]
        self.u_last = [torch.from_numpy(u[R]) for u in self._u]
        self.u_halo_lo = [torch.from_numpy(u[0]) for u in self._u]
        self.u_halo_hi = [torch.from_numpy(u[R + 1]) for u in self._u]
        self.f = np.zeros((R, n, n), np.complex128)
        self.y = np.zeros((R, n, n), np.complex128)
        self.valid = (self.row0 + np.arange(R)) % n != 0

    def _pack(self, dense):
        out = np.zeros((self.rows, self.n, self.n), np.complex128)
        for i in range(self.rows):
            x = self.row0 + i
            if 1 <= x <= self.nx:
                out[i, 1:, 1:] = dense[x - 1]
        return out

    def _block(self, planes):  # z- then y-DST'd planes -> [dest][xl][yb][z]
        R, P, n = self.rows, self.nranks, self.n
        self._T[...] = planes.reshape(R, P, R, n).transpose(1, 0, 2, 3).reshape(P, -1)

    def _unblock(self):
        R, P, n = self.rows, self.nranks, self.n
        return self._T.reshape(P, R, R, n).transpose(1, 0, 2, 3).reshape(R, P * R, n).copy()

    @staticmethod
    def _yz(planes):
        return _sine_ax(_sine_ax(planes, 2), 1)

    def set_fields(self, f, u0=None):
        self.f = self._pack(np.asarray(f, np.complex128))
        self._u[0][...] = 0
        if u0 is not None:
            self._u[0][1:self.rows + 1] = self._pack(np.asarray(u0, np.complex128))

    def _rows_fwd(self, field):
        self._block(self._yz(field))

    def _rows_inv(self):
        return self._yz(self._unblock())

    def _interior(self):
        j = np.arange(self.n) != 0
        return self.valid[:, None, None] & j[None, :, None] & j[None, None, :]

    def _stencil(self, ua):
        R = self.rows
        u = ua[1:R + 1]
        s = 6.0 * u - ua[0:R] - ua[2:R + 2]
        for ax in (1, 2):
            lo, hi = np.zeros_like(u), np.zeros_like(u)
            a, b = [slice(None)] * 3, [slice(None)] * 3
            a[ax], b[ax] = slice(1, None), slice(None, -1)
            lo[tuple(a)] = u[tuple(b)]
            hi[tuple(b)] = u[tuple(a)]
            s = s - lo - hi
        return s

    def set_multiplier(self, m):
        n, R = self.n, self.rows
        full = np.zeros((n, n, n), np.complex128)
        full[1:, 1:, 1:] = np.asarray(m, np.complex128)
        self.fd = full[:, self.rank * R:(self.rank + 1) * R, :].copy()

    def stage(self, code, cmap=None, config=None, a0=0.0, a1=0.0):
        R, n = self.rows, self.n
        if code in (OPT_A, OPT_B, RETA_A, RETA_C, FD_A, FD_B, GAMMA, COL_FD, COL_LREF):
            NumpySlabPart.stage(self, code, cmap, config, a0, a1)
        elif code == FWD_F:
            self._block(self._yz(self.f))
            self._sums[0] = np.sum(np.abs(self.f) ** 2)
        elif code == COL:
            if getattr(self, "status", 0) != 0:
                return
            M = self._Tc.reshape(n, R, n)  # (x, y_local, z)
            yq = self.rank * R + np.arange(R)
            lam = (self.lap[:, None, None] + self.lap[yq][None, :, None] + self.lap[None, None, :]
                   - (self.k0sq + 1j * self.eta))
            w = 8.0 / n ** 3 / lam
            w[0], w[:, :, 0] = 0, 0
            w[:, yq == 0, :] = 0
            M[...] = _sine_ax(_sine_ax(M, 0) * w, 0)
        elif code == INV_NORM:
            self.y = self._yz(self._unblock()) * self.valid[:, None, None]
            self._sums[1] = np.sum(np.abs(self.y) ** 2)
        elif code in (INIT, FINALIZE, ZERO_U):
            super().stage(code, cmap, config, a0, a1)
            if code == INIT:
                self._u[1][...] = 0
        elif code == FWD_BORN:
            u = self._u[0][1:R + 1]
            self._block(self._yz(self.V * u + self.f))
        elif code == SWEEP:
            if self.status != 0:
                return
            m = self.sweep
            ua = self._u[m & 1]
            u = ua[1:R + 1]
            z = self._yz(self._unblock())
            s = 6.0 * u - ua[0:R] - ua[2:R + 2]
            for ax in (1, 2):
                lo = np.zeros_like(u)
                hi = np.zeros_like(u)
                sl = [slice(None)] * 3
                sl[ax] = slice(1, None)
                sr = [slice(None)] * 3
                sr[ax] = slice(None, -1)
                lo[tuple(sl)] = u[tuple(sr)]
                hi[tuple(sr)] = u[tuple(sl)]
                s = s - lo - hi
            r = self.f - (s / self.h ** 2 - self.k2 * u)
            x = z - u
            mask = self.valid[:, None, None] & (np.arange(n) != 0)[None, :, None] & (np.arange(n) != 0)[None, None, :]
            self._sums[0] = np.sum((np.abs(r) ** 2)[mask])
            self._sums[1] = np.sum((np.abs(x) ** 2)[mask])
            g = 1j / self.eta * self.V if cmap.__class__.__name__ == "PointwiseMap" else complex(cmap.gamma)
            unew = u + g * (r if self.direct else x)
            unew[:, 0, :], unew[:, :, 0] = 0, 0
            nxt = self._u[(m + 1) & 1][1:R + 1]
            nxt[self.valid] = unew[self.valid]
            self._block(self._yz(self.V * nxt + self.f))

    def result(self, u_dense, max_iters):
        planes = self._u[self.result_buf][1:self.rows + 1]
        for i in range(self.rows):
            x = self.row0 + i
            if 1 <= x <= self.nx:
                u_dense[x - 1] = planes[i, 1:, 1:]
        k = self.iters + 1
        return IterationTrace(self.l2[:k].copy(), self.rt[:k].copy(), self.iters, TERMINATION[self.term],
                              self.fn, self.gn)
