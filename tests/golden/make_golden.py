"""Generate the committed golden fixtures (run HERE, where /root/reference and scipy exist).

    python tests/golden/make_golden.py

* dst_scipy.npz      -- 2-D DST-I vectors from scipy.fft.dstn(type=1) (== FFTW RODFT00), scaled
                        to the reference's forward convention (x0.25, proj/src/transforms.cpp:117)
* ref_rng.npz        -- RngState normals / uniforms from the reference's own rng.hpp
* ref_samplers.npz   -- sponge_profile / gaussian_bump from the reference's samplers.cpp
* ref_dct.npz        -- the reference's DCT-II / DCT-III transform pair (Neumann grids,
                        transforms.cpp:105-148) and Neumann five-point symbol (symbol.cpp:81-92),
                        plus scipy.fft.dctn(type=2/3) of the same real inputs (config c4)
* ref_io/            -- BPFD field files, CSV exports and a helmholtz problem manifest written by
                        the reference's own field.cpp / problem_io.cpp (io_inputs.npz: the data)
* ref_ops_n{16,32}.npz, ref_run_*.npz
                     -- operator outputs and run() trajectories produced by the reference's own
                        L1-L3 code (oracle/_ref) on instances from libbornsweep_host.so
The GPU box never reads /root/reference: tests consume only these files.
"""
import os
import sys

import numpy as np
import scipy.fft as sf

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import (FMT_CBS, FMT_DIRECT, MAP_FOURIER_DIAG, MAP_OPTIMAL_SCALAR, MAP_POINTWISE,  # noqa: E402
                    MAP_SCALAR, Reference, ReferenceProblem)
import paper_2603_18527_b200 as bs  # noqa: E402


def dst_golden():
    rng = np.random.default_rng(20261020)
    out = {}
    for nx, ny in [(16, 12), (15, 15), (7, 7), (31, 31), (3, 5)]:
        x = rng.standard_normal((nx, ny)) + 1j * rng.standard_normal((nx, ny))
        y = (sf.dstn(x.real, type=1) + 1j * sf.dstn(x.imag, type=1)) * 0.25
        out[f"x_{nx}x{ny}"] = x
        out[f"y_{nx}x{ny}"] = y
    np.savez_compressed(os.path.join(HERE, "dst_scipy.npz"), **out)


def dst3_golden():
    rng = np.random.default_rng(7)
    x = rng.standard_normal((7, 15, 31)) + 1j * rng.standard_normal((7, 15, 31))
    y = (sf.dstn(x.real, type=1) + 1j * sf.dstn(x.imag, type=1)) / 8
    np.savez_compressed(os.path.join(HERE, "dst3_scipy.npz"), x=x, y=y)


def rng_golden():
    out = {}
    for seed, idx in [(0, -1), (0, 0), (0, 7), (12345, 3), (2**63 + 5, 63)]:
        out[f"normal_{seed}_{idx}"] = Reference.rng_normals(seed, idx, 257)
        out[f"uniform_{seed}_{idx}"] = Reference.rng_uniforms(seed, idx, 64)
    np.savez_compressed(os.path.join(HERE, "ref_rng.npz"), **out)


def sampler_golden():
    out = {}
    for nx, layer in [(15, 1), (31, 3), (127, 15), (12, 0)]:
        out[f"sponge_{nx}_{layer}"] = Reference.sponge_profile(nx, nx, layer, 1.0)
    for nx, cx, cy, w in [(15, 0.5, 0.5, 2 / 16), (31, 0.3, 0.7, 0.05), (127, 0.5, 0.5, 2 / 128)]:
        out[f"bump_{nx}_{cx}_{cy}_{w}"] = Reference.gaussian_bump(nx, nx, cx, cy, w)
    np.savez_compressed(os.path.join(HERE, "ref_samplers.npz"), **out)


def ops_golden():
    rng = np.random.default_rng(7)
    for n in (16, 32):
        spec = bs.InstanceSpec(n=n, ppw=8.0, contrast=0.4, sigma_cells=2.0)
        k2, f, k0, eta = bs.make_instances(spec, 0, 1)
        p = ReferenceProblem(k2[0], k0[0], eta[0])
        x = rng.standard_normal(k2[0].shape) + 1j * rng.standard_normal(k2[0].shape)
        np.savez_compressed(
            os.path.join(HERE, f"ref_ops_n{n}.npz"), k2=k2[0], f=f[0], k0=k0[0], eta=eta[0], x=x,
            A=p.apply_A(x), V=p.apply_V(x), VH=p.apply_V_adjoint(x), Lref=p.apply_Lref(x),
            G=p.apply_G(x), born=p.born_residual(x, f[0]), res=p.residual(x, f[0]),
            fwd=p.forward_dst(x), inv=p.inverse_dst(x), symbol=p.symbol())


def run_golden():
    cases = {
        # name: (n, ppw, contrast, map, gamma, metric, rtol, max_iters)
        "c0like_n32_scalar": (32, 10.0, 0.3, MAP_SCALAR, 1.0, 0, 1e-6, 2000),
        "n32_pointwise": (32, 8.0, 0.5, MAP_POINTWISE, 0.0, 0, 1e-6, 3000),
        "n16_optl2": (16, 8.0, 0.4, MAP_OPTIMAL_SCALAR, 0.0, 0, 1e-8, 2000),
        "n16_optreta": (16, 8.0, 0.4, MAP_OPTIMAL_SCALAR, 0.0, 1, 1e-8, 2000),
        "n32_scalar_maxiters": (32, 10.0, 0.3, MAP_SCALAR, 0.8 + 0.1j, 0, 1e-6, 37),
    }
    for name, (n, ppw, contrast, mk, gamma, metric, rtol, mi) in cases.items():
        spec = bs.InstanceSpec(n=n, ppw=ppw, contrast=contrast, sigma_cells=2.0, seed=11)
        k2, f, k0, eta = bs.make_instances(spec, 0, 1)
        p = ReferenceProblem(k2[0], k0[0], eta[0])
        r = p.run(f[0], map_kind=mk, gamma=gamma, metric=metric, rtol=rtol, max_iters=mi)
        np.savez_compressed(os.path.join(HERE, f"ref_run_{name}.npz"), k2=k2[0], f=f[0], k0=k0[0],
                            eta=eta[0], map_kind=mk, gamma=gamma, metric=metric, rtol=rtol,
                            max_iters=mi, u=r.u, res_l2=r.res_l2, res_reta=r.res_reta,
                            iters=r.iters, terminated=r.terminated, fnorm_l2=r.fnorm_l2,
                            fnorm_reta=r.fnorm_reta)
        print(name, r.iters, r.terminated)


def periodic_golden():
    """The reference's OWN HelmholtzProblem (periodic pseudospectral) on its own bench instance
    generator (make_layered_helmholtz + bump source, bench.cpp:25-67)."""
    rng = np.random.default_rng(3)
    for n, seed in [(32, 5), (64, 7)]:
        k2, f, k0, eta = Reference.periodic_bench_instance(n, 16.0, 2.0, seed)
        p = ReferenceProblem(k2, k0, eta, periodic=True)
        x = rng.standard_normal(k2.shape) + 1j * rng.standard_normal(k2.shape)
        out = dict(k2=k2, f=f, k0=k0, eta=eta, x=x, A=p.apply_A(x), V=p.apply_V(x),
                   VH=p.apply_V_adjoint(x), Lref=p.apply_Lref(x), G=p.apply_G(x),
                   born=p.born_residual(x, f), res=p.residual(x, f), fwd=p.forward_dst(x),
                   inv=p.inverse_dst(x), symbol=p.symbol())
        m = 0.8 + 0.1 * (rng.standard_normal(k2.shape) + 1j * rng.standard_normal(k2.shape))
        out["fd_m"] = m
        for name, kw in [("scalar", dict(map_kind=MAP_SCALAR, gamma=1.0)),
                         ("scalar_relaxed", dict(map_kind=MAP_SCALAR, gamma=0.9 + 0.05j)),
                         ("optl2", dict(map_kind=MAP_OPTIMAL_SCALAR, metric=0)),
                         ("fd", dict(map_kind=2, m=m))]:
            r = p.run(f, rtol=1e-8, max_iters=4000, **kw)
            out[f"run_{name}_u"] = r.u
            out[f"run_{name}_l2"] = r.res_l2
            out[f"run_{name}_reta"] = r.res_reta
            out[f"run_{name}_iters"] = r.iters
            out[f"run_{name}_term"] = r.terminated
            print("periodic", n, name, r.iters, r.terminated)
        np.savez_compressed(os.path.join(HERE, f"ref_periodic_n{n}.npz"), **out)


def round2_golden():
    """Round-2 fixtures (new files only; the round-1 fixtures are left as committed).
    ref_periodic_more.npz -- the reference's OWN periodic HelmholtzProblem (n = 32 instance of
        ref_periodic_n32.npz): OptimalScalar with the R_eta metric, and the Direct format
        (iterate.cpp:118-123) with OptimalScalar (Euclidean) and a small scalar gamma.
    ref_direct.npz -- the Direct format on the Dirichlet five-point family (n = 16 / 32
        instances of run_golden): scalar, pointwise, OptimalScalar (both metrics), FourierDiag."""
    g = np.load(os.path.join(HERE, "ref_periodic_n32.npz"))
    p = ReferenceProblem(g["k2"], float(g["k0"]), float(g["eta"]), periodic=True)
    out = {}
    cases = {"optreta": dict(map_kind=MAP_OPTIMAL_SCALAR, metric=1, rtol=1e-8, max_iters=4000),
             "direct_optl2": dict(map_kind=MAP_OPTIMAL_SCALAR, metric=0, fmt=FMT_DIRECT, rtol=1e-3,
                                  max_iters=300),
             "direct_scalar": dict(map_kind=MAP_SCALAR, gamma=2e-5, fmt=FMT_DIRECT, rtol=1e-3,
                                   max_iters=200)}
    for name, kw in cases.items():
        r = p.run(g["f"], **kw)
        for k, v in dict(u=r.u, l2=r.res_l2, reta=r.res_reta, iters=r.iters, term=r.terminated).items():
            out[f"run_{name}_{k}"] = v
        print("periodic", name, r.iters, r.terminated)
    np.savez_compressed(os.path.join(HERE, "ref_periodic_more.npz"), **out)

    out = {}
    rng = np.random.default_rng(5)
    for n in (16, 32):
        spec = bs.InstanceSpec(n=n, ppw=8.0, contrast=0.4, sigma_cells=2.0)
        k2, f, k0, eta = bs.make_instances(spec, 0, 1)
        out[f"n{n}_k2"], out[f"n{n}_f"], out[f"n{n}_k0"], out[f"n{n}_eta"] = k2[0], f[0], k0[0], eta[0]
        p = ReferenceProblem(k2[0], k0[0], eta[0])
        m = 0.5 + 0.05 * (rng.standard_normal(k2[0].shape) + 1j * rng.standard_normal(k2[0].shape))
        out[f"n{n}_fd_m"] = m
        cases = {"optl2": dict(map_kind=MAP_OPTIMAL_SCALAR, metric=0),
                 "optreta": dict(map_kind=MAP_OPTIMAL_SCALAR, metric=1),
                 "scalar": dict(map_kind=MAP_SCALAR, gamma=1.0 / (8.0 * n * n)),
                 "pointwise": dict(map_kind=MAP_POINTWISE),
                 "fd": dict(map_kind=2, m=m * (1.0 / (8.0 * n * n)))}
        for name, kw in cases.items():
            r = p.run(f[0], fmt=FMT_DIRECT, rtol=1e-4, max_iters=150, **kw)
            for k, v in dict(u=r.u, l2=r.res_l2, reta=r.res_reta, iters=r.iters,
                             term=r.terminated).items():
                out[f"n{n}_{name}_{k}"] = v
            print("direct", n, name, r.iters, r.terminated)
    np.savez_compressed(os.path.join(HERE, "ref_direct.npz"), **out)


def dct_golden():
    rng = np.random.default_rng(44)
    out = {}
    for nx, ny in [(16, 12), (16, 16), (32, 32), (64, 64)]:
        x = rng.standard_normal((nx, ny)) + 1j * rng.standard_normal((nx, ny))
        out[f"x_{nx}x{ny}"] = x
        out[f"fwd_{nx}x{ny}"] = Reference.dct(x)
        out[f"inv_{nx}x{ny}"] = Reference.dct(x, inverse=True)
        out[f"scipy2_{nx}x{ny}"] = sf.dctn(x.real, type=2)
        out[f"scipy3_{nx}x{ny}"] = sf.dctn(x.real, type=3)
    for n, lx in [(32, 1.0), (64, 2.0)]:
        out[f"symbol_n{n}"] = Reference.laplacian_symbol(n, n, lx, lx, bc=2)
    np.savez_compressed(os.path.join(HERE, "ref_dct.npz"), **out)


def generic_golden():
    """ref_generic.npz -- any-shape Dirichlet grids (rectangular, sides not 2^k - 1, lx != ly):
    the reference's own operators (oracle/_ref, FFTW-API shim) and bp::run trajectories with the
    scalar and pointwise maps (NPBS) and the Direct format, for the GPU any-shape path
    (tests/test_gpu_generic.py).  Media: c = 1 + 0.3 g (g smoothed seeded noise, unit max-abs),
    k = omega / c, 10 points per wavelength in x, absorption 5 %, k0 = mean k,
    eta = 1.01 max|k^2 - k0^2|, a Gaussian source at the grid centre."""
    from scipy.ndimage import gaussian_filter
    rng = np.random.default_rng(2026)
    out = {}
    # a, b, d: hx == hy (ly = lx (ny+1)/(nx+1)): A = five_point - k2 and L_ref - V agree and the
    # solves converge; c: hx != hy -- five_point takes hx^2 only (kernels.cpp:56-69) while the
    # symbol uses both spacings, so the reference's own run stagnates; the GPU must too
    for tag, (nx, ny, lx, ly) in {"a": (16, 12, 1.0, 13 / 17), "b": (13, 21, 1.0, 22 / 14),
                                  "c": (100, 37, 2.0, 1.0), "d": (96, 127, 1.0, 128 / 97)}.items():
        hx, hy = lx / (nx + 1), ly / (ny + 1)
        g = gaussian_filter(rng.standard_normal((nx, ny)), 2.0)
        g /= np.abs(g).max()
        kk = 2 * np.pi / (10.0 * hx) / (1.0 + 0.2 * g)
        k2 = (kk * kk) * (1.0 + 0.05j)
        k0 = float(kk.mean())
        eta = float(1.01 * np.abs(k2 - k0 * k0).max())
        X, Y = np.meshgrid((np.arange(nx) + 1) * hx, (np.arange(ny) + 1) * hy, indexing="ij")
        f = np.exp(-((X - lx / 2) ** 2 + (Y - ly / 2) ** 2) / (2 * (3 * hx) ** 2)) + 0j
        x = rng.standard_normal((nx, ny)) + 1j * rng.standard_normal((nx, ny))
        r = ReferenceProblem(k2, k0, eta, lx, ly)
        out.update({f"{tag}_shape": np.array([nx, ny]), f"{tag}_l": np.array([lx, ly]), f"{tag}_k2": k2,
                    f"{tag}_f": f, f"{tag}_k0": k0, f"{tag}_eta": eta, f"{tag}_x": x,
                    f"{tag}_G": r.apply_G(x), f"{tag}_A": r.apply_A(x), f"{tag}_L": r.apply_Lref(x),
                    f"{tag}_V": r.apply_V(x), f"{tag}_born": r.born_residual(x, f),
                    f"{tag}_res": r.residual(x, f),
                    f"{tag}_fwd": (sf.dstn(x.real, type=1) + 1j * sf.dstn(x.imag, type=1)) * 0.25,
                    f"{tag}_inv": (sf.dstn(x.real, type=1) + 1j * sf.dstn(x.imag, type=1)) / ((nx + 1) * (ny + 1))})
        for name, kw in {"pw": dict(map_kind=MAP_POINTWISE), "sc": dict(map_kind=MAP_SCALAR, gamma=1.0),
                         "dir": dict(map_kind=MAP_POINTWISE, fmt=FMT_DIRECT)}.items():
            u, l2, rt, info = Reference.run_batch(k2[None], np.array([k0]), np.array([eta]), f[None],
                                                  rtol=1e-8, max_iters=3000, lx=lx, ly=ly, **kw)
            it, term = info[0]
            out[f"{tag}_{name}_u"] = u[0]
            out[f"{tag}_{name}_l2"] = l2[0, :it + 1]
            out[f"{tag}_{name}_reta"] = rt[0, :it + 1]
            out[f"{tag}_{name}_iters"] = it
            out[f"{tag}_{name}_term"] = term
            print("generic", tag, name, it, term)
    # the reference's own periodic HelmholtzProblem on any shape (pa: 16 x 12, pb: 24 x 20 with
    # lx != ly, pc: 100 x 37): operators, transforms and scalar-map runs (NPBS, relaxed, Direct)
    for tag, (nx, ny, lx, ly) in {"pa": (16, 12, 1.0, 1.0), "pb": (24, 20, 1.0, 0.8),
                                  "pc": (100, 37, 2.0, 1.0)}.items():
        g = gaussian_filter(rng.standard_normal((nx, ny)), 2.0, mode="wrap")
        g /= np.abs(g).max()
        kk = 2 * np.pi / (12.0 * lx / nx) / (1.0 + 0.2 * g)
        k2 = (kk * kk) * (1.0 + 0.05j)
        k0 = float(kk.mean())
        eta = float(1.01 * np.abs(k2 - k0 * k0).max())
        X, Y = np.meshgrid(np.arange(nx) * lx / nx, np.arange(ny) * ly / ny, indexing="ij")
        f = np.exp(-((X - lx / 2) ** 2 + (Y - ly / 2) ** 2) / (2 * (3 * lx / nx) ** 2)) + 0j
        x = rng.standard_normal((nx, ny)) + 1j * rng.standard_normal((nx, ny))
        r = ReferenceProblem(k2, k0, eta, lx, ly, periodic=True)
        out.update({f"{tag}_shape": np.array([nx, ny]), f"{tag}_l": np.array([lx, ly]), f"{tag}_k2": k2,
                    f"{tag}_f": f, f"{tag}_k0": k0, f"{tag}_eta": eta, f"{tag}_x": x,
                    f"{tag}_G": r.apply_G(x), f"{tag}_A": r.apply_A(x), f"{tag}_L": r.apply_Lref(x),
                    f"{tag}_V": r.apply_V(x), f"{tag}_born": r.born_residual(x, f),
                    f"{tag}_res": r.residual(x, f), f"{tag}_fwd": r.forward_dst(x), f"{tag}_inv": r.inverse_dst(x)})
        for name, kw in {"sc": dict(map_kind=MAP_SCALAR, gamma=1.0),
                         "rx": dict(map_kind=MAP_SCALAR, gamma=0.9 + 0.05j),
                         "dir": dict(map_kind=MAP_SCALAR, gamma=2e-5, fmt=FMT_DIRECT)}.items():
            rr = r.run(f, rtol=1e-8, max_iters=3000, **kw)
            out[f"{tag}_{name}_u"] = rr.u
            out[f"{tag}_{name}_l2"] = rr.res_l2
            out[f"{tag}_{name}_reta"] = rr.res_reta
            out[f"{tag}_{name}_iters"] = rr.iters
            out[f"{tag}_{name}_term"] = rr.terminated
            print("generic periodic", tag, name, rr.iters, rr.terminated)
    np.savez_compressed(os.path.join(HERE, "ref_generic.npz"), **out)


def generic_maps_golden():
    """ref_generic_maps.npz -- OptimalScalarMap (both metrics, NPBS and Direct) and FourierDiagMap
    runs of the reference's own bp::run / apply_correction (oracle/_ref; iterate.cpp:88-153,
    correction.cpp:22-76) on the any-shape grids of ref_generic.npz (Dirichlet a-d, periodic
    pa-pc): the iterate and traces after 30 sweeps (per-iterate parity; the optimal-scalar
    trajectory amplifies roundoff over long runs) and the full solve's count / termination / u."""
    g = np.load(os.path.join(HERE, "ref_generic.npz"))
    rng = np.random.default_rng(4242)
    out = {}
    for tag in ["a", "b", "c", "d", "pa", "pb", "pc"]:
        per = tag.startswith("p")
        k2, f = g[f"{tag}_k2"], g[f"{tag}_f"]
        lx, ly = (float(v) for v in g[f"{tag}_l"])
        r = ReferenceProblem(k2, float(g[f"{tag}_k0"]), float(g[f"{tag}_eta"]), lx, ly, periodic=per)
        m = 0.9 + 0.05 * (rng.standard_normal(k2.shape) + 1j * rng.standard_normal(k2.shape))
        out[f"{tag}_m"] = m
        runs = {"opt": dict(map_kind=MAP_OPTIMAL_SCALAR, metric=0),
                "reta": dict(map_kind=MAP_OPTIMAL_SCALAR, metric=1),
                "optcbs": dict(map_kind=MAP_OPTIMAL_SCALAR, metric=0, fmt=FMT_CBS),
                "optdir": dict(map_kind=MAP_OPTIMAL_SCALAR, metric=0, fmt=FMT_DIRECT),
                "fd": dict(map_kind=MAP_FOURIER_DIAG, m=m)}
        for name, kw in runs.items():
            r30 = r.run(f, rtol=1e-12, max_iters=30, **kw)
            full = r.run(f, rtol=1e-8, max_iters=3000, **kw)
            out[f"{tag}_{name}_u30"] = r30.u
            out[f"{tag}_{name}_l2_30"] = r30.res_l2
            out[f"{tag}_{name}_reta_30"] = r30.res_reta
            out[f"{tag}_{name}_iters30"] = r30.iters
            out[f"{tag}_{name}_u"] = full.u
            out[f"{tag}_{name}_iters"] = full.iters
            out[f"{tag}_{name}_term"] = full.terminated
            out[f"{tag}_{name}_l2_last"] = full.res_l2[-1]
            print("generic maps", tag, name, r30.iters, full.iters, full.terminated)
    np.savez_compressed(os.path.join(HERE, "ref_generic_maps.npz"), **out)


def io_golden():
    d = os.path.join(HERE, "ref_io")
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng(77)
    fc = rng.standard_normal((5, 7)) + 1j * rng.standard_normal((5, 7))
    fr = rng.standard_normal((6, 4))
    fr[0, 0], fr[1, 1] = 1.0, 1e-300  # formatting edge cases in the CSV
    k2, f, k0, eta = Reference.periodic_bench_instance(16, 8.0, 1.0, 3)
    Reference.save_field(os.path.join(d, "field_c.bpfd"), fc)
    Reference.save_field(os.path.join(d, "field_r.bpfd"), fr)
    Reference.export_csv(os.path.join(d, "field_c.csv"), fc)
    Reference.export_csv(os.path.join(d, "field_r.csv"), fr)
    Reference.save_problem_helmholtz(d, "helm", k2, k0, eta)
    np.savez_compressed(os.path.join(HERE, "io_inputs.npz"), fc=fc, fr=fr, k2=k2, f=f, k0=k0, eta=eta)


if __name__ == "__main__":
    Reference.set_mode("serial")
    if sys.argv[1:] in (["dct"], ["io"], ["round2"], ["generic"], ["generic_maps"]):
        {"dct": dct_golden, "io": io_golden, "round2": round2_golden, "generic": generic_golden,
         "generic_maps": generic_maps_golden}[sys.argv[1]]()
        sys.exit(0)
    io_golden()
    dct_golden()
    dst_golden()
    dst3_golden()
    rng_golden()
    sampler_golden()
    ops_golden()
    run_golden()
    periodic_golden()
    round2_golden()
    generic_golden()
    generic_maps_golden()
    print("golden fixtures written to", HERE)
