// sweep_launch.cuh -- per-size launch entry points (one translation unit per LOG2N, see
// sweep_L*.cu, so the instantiations compile in parallel).
#pragma once

#include "sweep_kernels.cuh"

namespace bs {

constexpr int kRowWarps = 8;   // warps per row-kernel CTA
constexpr int kColCols = 8;    // columns per column-kernel CTA (128-B row segments)

template <int L, int MODE, int PP>
cudaError_t launch_row_t(const RowArgs& a, cudaStream_t s, bool prepare) {
    using RG = RowGeom<L, PP, kRowWarps>;
    auto k = row_kernel<L, MODE, kRowWarps, PP>;
    if (prepare) return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RG::SMEM);
    const long rows = (long)a.batch << L;
    const int grid = (int)((rows + RG::EPB - 1) / RG::EPB);
    k<<<grid, kRowWarps * 32, RG::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int L, int MODE, int PP>
cudaError_t launch_col_t(const ColArgs& a, cudaStream_t s, bool prepare) {
    using CG = ColGeom<L, PP, kColCols>;
    auto k = col_kernel<L, MODE, kColCols, PP>;
    if (prepare) return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CG::SMEM);
    const int grid = a.batch * ((1 << L) / kColCols);
    k<<<grid, CG::THREADS, CG::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int L, int PP>
cudaError_t launch_row_p(int mode, const RowArgs& a, cudaStream_t s, bool prepare) {
    switch (mode) {
        case R_FWD: return launch_row_t<L, R_FWD, PP>(a, s, prepare);
        case R_FWD_BORN: return launch_row_t<L, R_FWD_BORN, PP>(a, s, prepare);
        case R_INV: return launch_row_t<L, R_INV, PP>(a, s, prepare);
        case R_SWEEP: return launch_row_t<L, R_SWEEP, PP>(a, s, prepare);
        case R_OPT_A: return launch_row_t<L, R_OPT_A, PP>(a, s, prepare);
        case R_OPT_B: return launch_row_t<L, R_OPT_B, PP>(a, s, prepare);
        case R_RETA_A: return launch_row_t<L, R_RETA_A, PP>(a, s, prepare);
        case R_RETA_C: return launch_row_t<L, R_RETA_C, PP>(a, s, prepare);
        case R_FD_A: return launch_row_t<L, R_FD_A, PP>(a, s, prepare);
        default: return launch_row_t<L, R_FD_B, PP>(a, s, prepare);
    }
}

template <int L, int PP>
cudaError_t launch_col_p(int mode, const ColArgs& a, cudaStream_t s, bool prepare) {
    switch (mode) {
        case C_ONE: return launch_col_t<L, C_ONE, PP>(a, s, prepare);
        case C_GREEN: return launch_col_t<L, C_GREEN, PP>(a, s, prepare);
        case C_FD: return launch_col_t<L, C_FD, PP>(a, s, prepare);
        default: return launch_col_t<L, C_LREF, PP>(a, s, prepare);
    }
}

// entry points defined in sweep_L<L>.cu
cudaError_t launch_row_size(int log2n, int pp, int mode, const RowArgs& a, cudaStream_t s, bool prepare);
cudaError_t launch_col_size(int log2n, int pp, int mode, const ColArgs& a, cudaStream_t s, bool prepare);

#define BS_DEFINE_SIZE(L)                                                                        \
    cudaError_t launch_row_L##L(int pp, int mode, const RowArgs& a, cudaStream_t s, bool prep) {  \
        if (pp == 8) return launch_row_p<L, 8>(mode, a, s, prep);                                \
        return launch_row_p<L, 16>(mode, a, s, prep);                                            \
    }                                                                                            \
    cudaError_t launch_col_L##L(int pp, int mode, const ColArgs& a, cudaStream_t s, bool prep) {  \
        if (pp == 8) return launch_col_p<L, 8>(mode, a, s, prep);                                \
        return launch_col_p<L, 16>(mode, a, s, prep);                                            \
    }

#define BS_DECLARE_SIZE(L)                                                                       \
    cudaError_t launch_row_L##L(int pp, int mode, const RowArgs& a, cudaStream_t s, bool prep);   \
    cudaError_t launch_col_L##L(int pp, int mode, const ColArgs& a, cudaStream_t s, bool prep);

BS_DECLARE_SIZE(3)
BS_DECLARE_SIZE(4)
BS_DECLARE_SIZE(5)
BS_DECLARE_SIZE(6)
BS_DECLARE_SIZE(7)
BS_DECLARE_SIZE(8)
BS_DECLARE_SIZE(9)

}  // namespace bs
