// sweep_launch.cuh -- per-size launch entry points (one translation unit per LOG2N, see
// sweep_L*.cu, so the instantiations compile in parallel).
#pragma once

#include "cdr_kernels.cuh"
#include "periodic_kernels.cuh"
#include "sweep_kernels.cuh"
#include "tri_kernels.cuh"
#include "tri_wide_kernels.cuh"
#include "cluster_kernels.cuh"

namespace bs {

constexpr int kRowWarps = 8;   // warps per row-kernel CTA
// experiment knobs (r01: 4-warp row CTAs equal, 4-column n = 512 column CTAs 47 % slower)
#ifndef BS_ROW_NW
#define BS_ROW_NW 8            // warps per CTA of the Dirichlet row kernel for single-warp lines
#endif
#ifndef BS_COLC9
#define BS_COLC9 8             // columns per column-kernel CTA for n = 512
#endif
template <int L, int PP>
struct RowWarps {
    static constexpr int value = Geom<L, PP>::T <= 32 ? BS_ROW_NW : kRowWarps;
};
// columns per column-kernel CTA: 8 (128-B row segments) while a CTA of 8 lines fits; long
// lines (n >= 1024) hold fewer columns per CTA so the shared-memory lines still fit
template <int L>
struct ColCols {
    static constexpr int value = L == 9 ? BS_COLC9 : L <= 8 ? 8 : (L == 10 ? 4 : 2);
};

// lines per Dirichlet row-kernel CTA (RowGeom::EPB of the launched instance), for the host
inline int row_lines_per_cta(int log2n, int pp) {
    const int n = 1 << log2n, p = (n / 2) < pp ? (n / 2) : pp, t = n / p;
    const int nw = t <= 32 ? BS_ROW_NW : kRowWarps;
    return nw * 32 / t;
}

template <int L, int MODE, int PP, int DIM, bool SLAB = false>
cudaError_t launch_row_t(const RowArgs& a, cudaStream_t s, bool prepare) {
    constexpr int NWR = RowWarps<L, PP>::value;
    using RG = RowGeom<L, PP, NWR>;
    // slab launches (2-D, row-major handoff, the modes the slab driver uses) -> SLAB instance
    constexpr bool SLAB_OK = PP == 16;
    if constexpr (SLAB_OK && !SLAB) {
        if (a.slab_log2 || prepare) {
            const cudaError_t e = launch_row_t<L, MODE, PP, DIM, true>(a, s, prepare);
            if (!prepare || e != cudaSuccess) return e;
        }
    }
    if (!SLAB && a.slab_log2 && !prepare) return cudaErrorInvalidValue;
    auto k = row_kernel<L, MODE, NWR, PP, DIM, SLAB>;
    if (prepare) return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RG::SMEM);
    const long rows = (long)a.batch << (SLAB ? a.slab_log2 + (DIM - 2) * L : (DIM - 1) * L);
    const int grid = (int)((rows + RG::EPB - 1) / RG::EPB);
    k<<<grid, NWR * 32, RG::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int L, int MODE, int PP, int LAYOUT>
cudaError_t launch_col_t(const ColArgs& a, cudaStream_t s, bool prepare) {
    constexpr int C = ColCols<L>::value;
    using CG = ColGeom<L, PP, C>;
    auto k = col_kernel<L, MODE, C, PP, LAYOUT>;
    if (prepare) return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CG::SMEM);
    // CL_PLANE: one CTA per (plane, column group), planes = batch * planes_per_member;
    // CL_X3: one CTA per (member, y, column group)
    // CL_SLAB: one CTA per (member, column group of the rank's block)
    // CL_YBLK: one CTA per (local x-plane, column group); batch 1
    const long groups = LAYOUT == CL_YBLK ? (1L << a.slab_log2)
                                          : (long)a.batch * (LAYOUT == CL_X3 ? (1L << L) : a.planes_per_member);
    const int grid = LAYOUT == CL_SLAB ? (int)((long)a.batch * (a.slab_cols / C))
                                       : (int)(groups * ((1 << L) / C));
    if (LAYOUT == CL_SLAB && (a.slab_cols % C) != 0) return cudaErrorInvalidValue;
    k<<<grid, CG::THREADS, CG::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int L, int PP, int DIM = 2>
cudaError_t launch_row_p(int mode, const RowArgs& a, cudaStream_t s, bool prepare) {
    switch (mode) {
        case R_FWD: return launch_row_t<L, R_FWD, PP, DIM>(a, s, prepare);
        case R_FWD_BORN: return launch_row_t<L, R_FWD_BORN, PP, DIM>(a, s, prepare);
        case R_INV: return launch_row_t<L, R_INV, PP, DIM>(a, s, prepare);
        case R_SWEEP: return launch_row_t<L, R_SWEEP, PP, DIM>(a, s, prepare);
        case R_SWEEP_D: return launch_row_t<L, R_SWEEP_D, PP, DIM>(a, s, prepare);
        case R_OPT_A: return launch_row_t<L, R_OPT_A, PP, DIM>(a, s, prepare);
        case R_OPT_B: return launch_row_t<L, R_OPT_B, PP, DIM>(a, s, prepare);
        case R_RETA_A: return launch_row_t<L, R_RETA_A, PP, DIM>(a, s, prepare);
        case R_RETA_C: return launch_row_t<L, R_RETA_C, PP, DIM>(a, s, prepare);
        case R_FD_A: return launch_row_t<L, R_FD_A, PP, DIM>(a, s, prepare);
        default: return launch_row_t<L, R_FD_B, PP, DIM>(a, s, prepare);
    }
}

template <int L, int PP, int LAYOUT = CL_PLANE>
cudaError_t launch_col_p(int mode, const ColArgs& a, cudaStream_t s, bool prepare) {
    switch (mode) {
        case C_ONE: return launch_col_t<L, C_ONE, PP, LAYOUT>(a, s, prepare);
        case C_GREEN: return launch_col_t<L, C_GREEN, PP, LAYOUT>(a, s, prepare);
        case C_FD: return launch_col_t<L, C_FD, PP, LAYOUT>(a, s, prepare);
        default: return launch_col_t<L, C_LREF, PP, LAYOUT>(a, s, prepare);
    }
}

// columns per CTA of the tridiagonal column pass (host side of TriGeom::C)
inline int tri_cols_per_cta(int log2n) {
    const int segs = (1 << log2n) / kTriP;
    return segs >= TRI_THREADS ? 2 : TRI_THREADS / segs;
}

// ---- long lines (n >= 2048), 2-D whole members: wide tiles over 4-CTA clusters
// (tri_wide_kernels.cuh); BP_TRI_WIDE=0 keeps the two-column tiles.  Returns
// cudaErrorNotSupported when the wide kernel does not apply (caller falls back).
template <int L>
cudaError_t launch_tri_wide_t(const ColArgs& a, cudaStream_t s, bool prepare) {
    if constexpr (L >= 11 && (1 << L) / BS_TRIW_CLW / kTriP >= 32) {
        using TW = TriWide<L>;
        auto k = tri_wide_kernel<L>;
        cudaLaunchConfig_t cfg{};
        cfg.blockDim = dim3(TW::THREADS);
        cfg.gridDim = dim3(TW::CLW);
        cfg.dynamicSmemBytes = TW::SMEM;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = TW::CLW;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        static int clusters = [&] {  // co-resident clusters on this device (0: not launchable)
            int n = 0;
            if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TW::SMEM) != cudaSuccess ||
                cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) {
                cudaGetLastError();
                n = 0;
            }
            return n;
        }();
        const char* env = std::getenv("BP_TRI_WIDE");  // read per launch (tests toggle it)
        if (clusters <= 0 || (env && env[0] == '0')) return cudaErrorNotSupported;
        if (prepare) return cudaSuccess;
        const long tiles = (long)a.batch * ((1 << L) / TW::WC);
        const long ncl = tiles < clusters ? tiles : clusters;
        if (ncl == 0) return cudaSuccess;
        cfg.gridDim = dim3((unsigned)(ncl * TW::CLW));
        return cudaLaunchKernelEx(&cfg, k, a);
    }
    return cudaErrorNotSupported;
}

// ---- Green column pass as a tridiagonal x-solve (n >= 64): persistent CTAs, one per
// resident slot (occupancy queried once per instance)
template <int L, int LAYOUT>
cudaError_t launch_tri_t(const ColArgs& a, cudaStream_t s, bool prepare) {
    if constexpr (L >= 11 && LAYOUT == CL_PLANE) {
        const cudaError_t e = launch_tri_wide_t<L>(a, s, prepare);
        if (e != cudaErrorNotSupported && !prepare) return e;
    }
    if constexpr (L >= 6) {
        using TG = TriGeom<L>;
        using TT = TriTile<L, LAYOUT == CL_CDR>;
        auto k = tri_kernel<L, LAYOUT, LAYOUT == CL_CDR>;
        if (prepare) return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TT::SMEM);
        static int slots = [&] {
            int dev = 0, sms = 0, per = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, TG::THREADS, TT::SMEM);
            return sms * (per > 0 ? per : 1);
        }();
        const long tiles = LAYOUT == CL_SLAB  ? (long)(a.slab_cols / TG::C)
                           : LAYOUT == CL_CDR ? (long)a.batch * ((1 << L) / 2 / TG::C)
                                              : (long)a.batch * (LAYOUT == CL_X3 ? (1L << L) : 1L) * ((1 << L) / TG::C);
        if (LAYOUT == CL_SLAB && (a.slab_cols % TG::C) != 0) return cudaErrorInvalidValue;
        if (LAYOUT == CL_CDR && (1 << L) / 2 < TG::C) return cudaErrorInvalidValue;
        const int grid = (int)(tiles < slots ? tiles : slots);
        if (grid == 0) return cudaSuccess;
        k<<<grid, TG::THREADS, TT::SMEM, s>>>(a);
        return cudaGetLastError();
    }
    return cudaErrorInvalidValue;
}

// ---- whole-solve cluster kernel (n = 64 / 128: the grid in one cluster's shared memory)
template <int L>
cudaError_t launch_cluster_t(const ClArgs& a, int batch, cudaStream_t s, bool prepare) {
    if constexpr (L == 6 || L == 7) {
        using CG = ClGeom<L>;
        auto k = cluster_solve_kernel<L>;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)(batch * CG::CL));
        cfg.blockDim = dim3(CG::THREADS);
        cfg.dynamicSmemBytes = CG::SMEM;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CG::CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (prepare) {  // attributes + can this device co-schedule the cluster at all
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CG::SMEM);
            if (e == cudaSuccess && CG::CL > 8)
                e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            int clusters = 0;
            if (e == cudaSuccess) e = cudaOccupancyMaxActiveClusters(&clusters, k, &cfg);
            return e != cudaSuccess ? e : (clusters > 0 ? cudaSuccess : cudaErrorInvalidConfiguration);
        }
        return cudaLaunchKernelEx(&cfg, k, a);
    }
    return cudaErrorInvalidValue;
}

// ---- config c4 (CDR, DCT engine, real packed pairs)
template <int L, int MODE>
cudaError_t launch_crow_t(const CdrArgs& a, cudaStream_t s, bool prepare) {
    using RG = RowGeom<L, 16, kRowWarps>;
    auto k = crow_kernel<L, MODE, kRowWarps, 16>;
    if (prepare) return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RG::SMEM);
    const long pairs = (long)a.batch << (L - 1);
    k<<<(int)((pairs + RG::EPB - 1) / RG::EPB), kRowWarps * 32, RG::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int L, int MODE>
cudaError_t launch_ccol_t(const CdrArgs& a, cudaStream_t s, bool prepare) {
    constexpr int C = ColCols<L>::value >= 8 ? 4 : ColCols<L>::value;  // column pairs per CTA
    using CG = ColGeom<L, 16, C>;
    auto k = ccol_kernel<L, MODE, C, 16>;
    if (prepare) return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CG::SMEM);
    k<<<a.batch * ((1 << L) / (2 * C)), CG::THREADS, CG::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int L>
cudaError_t launch_cdr_p(bool row, int mode, const CdrArgs& a, cudaStream_t s, bool prep) {
    if (row) {
        switch (mode) {
            case RC_FWD: return launch_crow_t<L, RC_FWD>(a, s, prep);
            case RC_INV: return launch_crow_t<L, RC_INV>(a, s, prep);
            case RC_A: return launch_crow_t<L, RC_A>(a, s, prep);
            default: return launch_crow_t<L, RC_B>(a, s, prep);
        }
    }
    switch (mode) {
        case CC_ONE: return launch_ccol_t<L, CC_ONE>(a, s, prep);
        case CC_INV: return launch_ccol_t<L, CC_INV>(a, s, prep);
        case CC_LREF: return launch_ccol_t<L, CC_LREF>(a, s, prep);
        default: return launch_ccol_t<L, CC_GREEN>(a, s, prep);
    }
}

// ---- periodic family (FFT engine)
template <int L, int MODE, int PP>
cudaError_t launch_prow_t(const PerArgs& a, cudaStream_t s, bool prepare) {
    using RG = RowGeom<L, PP, kRowWarps>;
    auto k = prow_kernel<L, MODE, kRowWarps, PP>;
    if (prepare) return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RG::SMEM);
    const long rows = (long)a.batch << L;
    k<<<(int)((rows + RG::EPB - 1) / RG::EPB), kRowWarps * 32, RG::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int L, int MODE, int PP>
cudaError_t launch_pcol_t(const PerArgs& a, cudaStream_t s, bool prepare) {
    constexpr int C = ColCols<L>::value;
    using CG = ColGeom<L, PP, C>;
    auto k = pcol_kernel<L, MODE, C, PP>;
    if (prepare) return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CG::SMEM);
    k<<<a.batch * ((1 << L) / C), CG::THREADS, CG::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int L>
cudaError_t launch_periodic_p(bool row, int mode, const PerArgs& a, cudaStream_t s, bool prep) {
    if (row) {
        switch (mode) {
            case RP_FWD: return launch_prow_t<L, RP_FWD, 16>(a, s, prep);
            case RP_FWD_BORN: return launch_prow_t<L, RP_FWD_BORN, 16>(a, s, prep);
            case RP_INV: return launch_prow_t<L, RP_INV, 16>(a, s, prep);
            case RP_OPT_B: return launch_prow_t<L, RP_OPT_B, 16>(a, s, prep);
            case RP_RETA_B: return launch_prow_t<L, RP_RETA_B, 16>(a, s, prep);
            default: return launch_prow_t<L, RP_SWEEP, 16>(a, s, prep);
        }
    }
    switch (mode) {
        case CP_ONE: return launch_pcol_t<L, CP_ONE, 16>(a, s, prep);
        case CP_GREEN: return launch_pcol_t<L, CP_GREEN, 16>(a, s, prep);
        case CP_LREF: return launch_pcol_t<L, CP_LREF, 16>(a, s, prep);
        case CP_INV: return launch_pcol_t<L, CP_INV, 16>(a, s, prep);
        case CP_OPT_A: return launch_pcol_t<L, CP_OPT_A, 16>(a, s, prep);
        case CP_OPT_C: return launch_pcol_t<L, CP_OPT_C, 16>(a, s, prep);
        case CP_RETA_C: return launch_pcol_t<L, CP_RETA_C, 16>(a, s, prep);
        default: return launch_pcol_t<L, CP_SWEEP, 16>(a, s, prep);
    }
}

// 3-D kernels exist for n <= 512 (P = 16)
constexpr int kMaxLog2_3d = 9;


// P = 8 needs T = n/8 <= 256 threads per line; longer lines always use P = 16
template <int L>
struct Pp8 {
    static constexpr int value = ((1 << L) / 8 <= 256) ? 8 : 16;
};

#define BS_DEFINE_SIZE(L)                                                                       \
    cudaError_t launch_row_L##L(int pp, int dim, int mode, const RowArgs& a, cudaStream_t s,     \
                                bool prep) {                                                    \
        if (dim == 3) {                                                                         \
            if constexpr (L <= kMaxLog2_3d) return launch_row_p<L, 16, 3>(mode, a, s, prep);    \
            return cudaErrorInvalidValue;                                                       \
        }                                                                                       \
        if (pp == 8) return launch_row_p<L, Pp8<L>::value>(mode, a, s, prep);                   \
        return launch_row_p<L, 16>(mode, a, s, prep);                                           \
    }                                                                                           \
    cudaError_t launch_col_L##L(int pp, int layout, int mode, const ColArgs& a, cudaStream_t s,  \
                                bool prep) {                                                    \
        if (layout == CL_X3) {                                                                  \
            if constexpr (L <= kMaxLog2_3d) return launch_col_p<L, 16, CL_X3>(mode, a, s, prep); \
            return cudaErrorInvalidValue;                                                       \
        }                                                                                       \
        if (layout == CL_SLAB) {                                                                \
            if (mode == C_ONE) return launch_col_t<L, C_ONE, 16, CL_SLAB>(a, s, prep);          \
            if (mode == C_GREEN) return launch_col_t<L, C_GREEN, 16, CL_SLAB>(a, s, prep);      \
            if (mode == C_FD) return launch_col_t<L, C_FD, 16, CL_SLAB>(a, s, prep);            \
            if (mode == C_LREF) return launch_col_t<L, C_LREF, 16, CL_SLAB>(a, s, prep);        \
            return cudaErrorInvalidValue;                                                       \
        }                                                                                       \
        if (layout == CL_YBLK) {                                                                \
            if constexpr (L <= kMaxLog2_3d)                                                     \
                if (mode == C_ONE) return launch_col_t<L, C_ONE, 16, CL_YBLK>(a, s, prep);      \
            return cudaErrorInvalidValue;                                                       \
        }                                                                                       \
        if (pp == 8) return launch_col_p<L, Pp8<L>::value>(mode, a, s, prep);                   \
        return launch_col_p<L, 16>(mode, a, s, prep);                                           \
    }                                                                                           \
    cudaError_t launch_periodic_L##L(bool row, int mode, const PerArgs& a, cudaStream_t s,      \
                                     bool prep) {                                               \
        return launch_periodic_p<L>(row, mode, a, s, prep);                                     \
    }                                                                                           \
    cudaError_t launch_cdr_L##L(bool row, int mode, const CdrArgs& a, cudaStream_t s, bool prep) { \
        return launch_cdr_p<L>(row, mode, a, s, prep);                                          \
    }                                                                                           \
    cudaError_t launch_cluster_L##L(const ClArgs& a, int batch, cudaStream_t s, bool prep) {   \
        return launch_cluster_t<L>(a, batch, s, prep);                                          \
    }                                                                                           \
    cudaError_t launch_tri_L##L(int layout, const ColArgs& a, cudaStream_t s, bool prep) {     \
        if (layout == CL_PLANE) return launch_tri_t<L, CL_PLANE>(a, s, prep);                   \
        if (layout == CL_SLAB) return launch_tri_t<L, CL_SLAB>(a, s, prep);                     \
        if (layout == CL_CDR) return launch_tri_t<L, CL_CDR>(a, s, prep);                       \
        if constexpr (L <= kMaxLog2_3d)                                                         \
            if (layout == CL_X3) return launch_tri_t<L, CL_X3>(a, s, prep);                     \
        return cudaErrorInvalidValue;                                                           \
    }

#define BS_DECLARE_SIZE(L)                                                                      \
    cudaError_t launch_row_L##L(int pp, int dim, int mode, const RowArgs& a, cudaStream_t s,     \
                                bool prep);                                                     \
    cudaError_t launch_col_L##L(int pp, int layout, int mode, const ColArgs& a, cudaStream_t s,  \
                                bool prep);                                                     \
    cudaError_t launch_periodic_L##L(bool row, int mode, const PerArgs& a, cudaStream_t s,      \
                                     bool prep);                                                \
    cudaError_t launch_cdr_L##L(bool row, int mode, const CdrArgs& a, cudaStream_t s, bool prep); \
    cudaError_t launch_tri_L##L(int layout, const ColArgs& a, cudaStream_t s, bool prep);       \
    cudaError_t launch_cluster_L##L(const ClArgs& a, int batch, cudaStream_t s, bool prep);

BS_DECLARE_SIZE(3)
BS_DECLARE_SIZE(4)
BS_DECLARE_SIZE(5)
BS_DECLARE_SIZE(6)
BS_DECLARE_SIZE(7)
BS_DECLARE_SIZE(8)
BS_DECLARE_SIZE(9)
BS_DECLARE_SIZE(10)
BS_DECLARE_SIZE(11)
BS_DECLARE_SIZE(12)

}  // namespace bs
