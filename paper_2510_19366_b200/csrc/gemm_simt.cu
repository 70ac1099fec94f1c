// gemm_simt.cu -- grouped SwiGLU FFN on CUDA cores (DFMA), the fp32 parity
// mode (1e-5 relative vs the double-accumulating oracle).  Tensor cores have
// no true-fp32 MMA, so fp32 mode stays on SIMT (hard part 3).
//   gemm1: H[r][c] = silu(A[r] . W1_gate[c]) * (A[r] . W1_up[c])
//   gemm2: O[r][i] = H[r] . W2[i]
// Rows of sub-expert g are [offsets[g], offsets[g+1]) of the permuted row
// space; tiles are enumerated (g, n, m) from the device-side prefix of
// ceil(count_g / 64), so the grid is an upper bound and spare CTAs exit.
#include "mp_common.cuh"
#include "mp_kernels.h"

namespace mp {

namespace {

constexpr uint32_t BM = kSimtBM;  // 64 rows
constexpr uint32_t BN = 64;       // 64 neurons (gemm1) / outputs (gemm2)
constexpr uint32_t BK = 16;

__device__ __forceinline__ bool map_tile(uint32_t tile, const uint32_t* __restrict__ mprefix, uint32_t G,
                                         uint32_t NT, uint32_t& g, uint32_t& m, uint32_t& n) {
    const uint32_t total = mprefix[G] * NT;
    if (tile >= total) return false;
    uint32_t lo = 0, hi = G;  // first index with prefix*NT > tile, minus one
    while (lo < hi) {
        const uint32_t mid = (lo + hi) / 2;
        if (mprefix[mid] * NT <= tile)
            lo = mid + 1;
        else
            hi = mid;
    }
    g = lo - 1;
    const uint32_t local = tile - mprefix[g] * NT;
    const uint32_t mt = mprefix[g + 1] - mprefix[g];
    n = local / mt;
    m = local % mt;
    return true;
}

// fp64 accumulation, as the reference does (inc/expert.hpp:64-72): products of
// fp32 operands are exact in double, so the per-neuron activation rounds to the
// same float as the reference's in all but astronomically rare cases -- which
// is what the 1e-5 * (1 + |y|) contract needs where |y| is near zero.
__device__ __forceinline__ float swiglu_f64(double g, double u) { return static_cast<float>(g / (1.0 + exp(-g)) * u); }

template <typename T>
__global__ void __launch_bounds__(256) gemm1_simt_kernel(const T* __restrict__ A, const T* __restrict__ W1,
                                                         T* __restrict__ H, uint32_t G, uint32_t K, uint32_t w_pad,
                                                         const uint32_t* __restrict__ offsets,
                                                         const uint32_t* __restrict__ mprefix) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bg[BK][BN + 4];
    __shared__ float Bu[BK][BN + 4];
    uint32_t g, m, n;
    if (!map_tile(blockIdx.x, mprefix, G, w_pad / BN, g, m, n)) return;
    const uint32_t row0 = offsets[g] + m * BM;
    const uint32_t cnt = offsets[g + 1] - offsets[g];
    const uint32_t rows_here = min(BM, cnt - m * BM);
    const uint32_t c0 = n * BN;
    const uint32_t tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const size_t wbase = (size_t)g * 2 * w_pad;
    double accg[4][4] = {}, accu[4][4] = {};
    for (uint32_t k0 = 0; k0 < K; k0 += BK) {
        for (uint32_t q = threadIdx.x; q < BM * BK; q += 256) {
            const uint32_t r = q / BK, kk = q % BK;
            As[kk][r] = r < rows_here ? to_f32(A[(size_t)(row0 + r) * K + k0 + kk]) : 0.0f;
        }
        for (uint32_t q = threadIdx.x; q < BN * BK; q += 256) {
            const uint32_t c = q / BK, kk = q % BK;
            const uint32_t cg = c0 + c;
            const uint32_t rg = (cg / kIlv) * 2 * kIlv + (cg % kIlv);
            Bg[kk][c] = to_f32(W1[(wbase + rg) * K + k0 + kk]);
            Bu[kk][c] = to_f32(W1[(wbase + rg + kIlv) * K + k0 + kk]);
        }
        __syncthreads();
#pragma unroll
        for (uint32_t kk = 0; kk < BK; ++kk) {
            float a[4], bg[4], bu[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                bg[j] = Bg[kk][tx * 4 + j];
                bu[j] = Bu[kk][tx * 4 + j];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    accg[i][j] = fma(static_cast<double>(a[i]), static_cast<double>(bg[j]), accg[i][j]);
                    accu[i][j] = fma(static_cast<double>(a[i]), static_cast<double>(bu[j]), accu[i][j]);
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t r = ty * 4 + i;
        if (r >= rows_here) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            H[(size_t)(row0 + r) * w_pad + c0 + tx * 4 + j] = from_f32<T>(swiglu_f64(accg[i][j], accu[i][j]));
    }
}

template <typename T, typename TO>
__global__ void __launch_bounds__(256) gemm2_simt_kernel(const T* __restrict__ Hm, const T* __restrict__ W2,
                                                         TO* __restrict__ O, uint32_t G, uint32_t K, uint32_t d_pad,
                                                         const uint32_t* __restrict__ offsets,
                                                         const uint32_t* __restrict__ mprefix) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    uint32_t g, m, n;
    const uint32_t NT = (d_pad + BN - 1) / BN;
    if (!map_tile(blockIdx.x, mprefix, G, NT, g, m, n)) return;
    const uint32_t row0 = offsets[g] + m * BM;
    const uint32_t cnt = offsets[g + 1] - offsets[g];
    const uint32_t rows_here = min(BM, cnt - m * BM);
    const uint32_t i0 = n * BN;
    const uint32_t tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const size_t wbase = (size_t)g * d_pad;
    double acc[4][4] = {};
    for (uint32_t k0 = 0; k0 < K; k0 += BK) {
        for (uint32_t q = threadIdx.x; q < BM * BK; q += 256) {
            const uint32_t r = q / BK, kk = q % BK;
            As[kk][r] = r < rows_here ? to_f32(Hm[(size_t)(row0 + r) * K + k0 + kk]) : 0.0f;
        }
        for (uint32_t q = threadIdx.x; q < BN * BK; q += 256) {
            const uint32_t c = q / BK, kk = q % BK;
            Bs[kk][c] = i0 + c < d_pad ? to_f32(W2[(wbase + i0 + c) * K + k0 + kk]) : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (uint32_t kk = 0; kk < BK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(static_cast<double>(a[i]), static_cast<double>(b[j]), acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t r = ty * 4 + i;
        if (r >= rows_here) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t c = i0 + tx * 4 + j;
            if (c < d_pad) {
                if constexpr (sizeof(TO) == 8)
                    O[(size_t)(row0 + r) * d_pad + c] = acc[i][j];
                else
                    O[(size_t)(row0 + r) * d_pad + c] = from_f32<TO>(static_cast<float>(acc[i][j]));
            }
        }
    }
}

uint32_t simt_grid(const GemmShape& sh, uint32_t NT) {
    // upper bound of sum_g ceil(count_g / BM)
    return (sh.max_rows / BM + sh.G) * NT;
}

}  // namespace

void launch_gemm1_simt(int dtype, const void* A, const void* W1, void* H, const GemmShape& sh,
                       const uint32_t* offsets, const uint32_t* mprefix, cudaStream_t s) {
    const uint32_t w_pad = sh.N_group / 2;
    const uint32_t grid = simt_grid(sh, w_pad / BN);
    if (dtype == 1)
        gemm1_simt_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(
            static_cast<const __nv_bfloat16*>(A), static_cast<const __nv_bfloat16*>(W1),
            static_cast<__nv_bfloat16*>(H), sh.G, sh.K, w_pad, offsets, mprefix);
    else
        gemm1_simt_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(A), static_cast<const float*>(W1),
                                                      static_cast<float*>(H), sh.G, sh.K, w_pad, offsets, mprefix);
}

void launch_gemm2_simt(int dtype, const void* Hm, const void* W2, void* O, const GemmShape& sh,
                       const uint32_t* offsets, const uint32_t* mprefix, cudaStream_t s) {
    const uint32_t grid = simt_grid(sh, (sh.N_group + BN - 1) / BN);
    if (dtype == 1)
        gemm2_simt_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, s>>>(
            static_cast<const __nv_bfloat16*>(Hm), static_cast<const __nv_bfloat16*>(W2),
            static_cast<__nv_bfloat16*>(O), sh.G, sh.K, sh.N_group, offsets, mprefix);
    else
        gemm2_simt_kernel<float, double><<<grid, 256, 0, s>>>(static_cast<const float*>(Hm),
                                                              static_cast<const float*>(W2), static_cast<double*>(O), sh.G, sh.K, sh.N_group, offsets,
                                                      mprefix);
}

}  // namespace mp
