// calib.cu -- the calibration side of MoE-Prism on the GPU:
// the activation profile |a| that the offline refactoring engine partitions
// experts with, its per-row top-k binarisation, and the co-activation counts.
//
//   collect_activation_matrix  inc/expert.hpp:137-151   (gemm_tc.cu kEpiActAbs)
//   binarize_topk              inc/activation.hpp:213-240 (binarize_topk_kernel)
//   coactivation               inc/activation.hpp:242-266 (gemm_tc.cu kEpiCount
//                              over the transposed 0/1 matrix: C = B^T B,
//                              exact in fp32 for up to 2^24 rows)
//
// binarize_topk: CTA per row.  |v| of a float is ordered like its bit
// pattern, so the k-th largest magnitude is found by a 4-pass 8-bit radix
// select on the keys (shared-memory histograms); then every key above it is
// set and, among keys equal to it, the lowest column indices (the
// reference's tie rule: value desc, index asc) -- an ordered block scan over
// contiguous column chunks.  Exact and deterministic.
#include "mp_common.cuh"
#include "mp_kernels.h"

namespace mp {

namespace {

constexpr uint32_t kBinThreads = 1024;

__device__ __forceinline__ uint32_t mag_key(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }

__global__ void __launch_bounds__(kBinThreads) binarize_topk_kernel(const float* __restrict__ act, uint32_t cols,
                                                                    uint32_t k_a, uint8_t* __restrict__ bits) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_prefix, s_remaining;
    __shared__ uint32_t wsum[32];
    const uint32_t row = blockIdx.x, tid = threadIdx.x;
    const float* a = act + (size_t)row * cols;
    if (tid == 0) {
        s_prefix = 0;
        s_remaining = k_a;
    }
    uint32_t mask = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (uint32_t b = tid; b < 256; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        const uint32_t prefix = s_prefix;
        for (uint32_t c = tid; c < cols; c += blockDim.x) {
            const uint32_t key = mag_key(a[c]);
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t rem = s_remaining, b = 255;
            for (;; --b) {
                if (hist[b] >= rem || b == 0) break;
                rem -= hist[b];
            }
            s_prefix = prefix | (b << shift);
            s_remaining = rem;
        }
        mask |= 255u << shift;
        __syncthreads();
    }
    const uint32_t kstar = s_prefix, take_eq = s_remaining;  // take the first take_eq keys == kstar
    // ordered pass: thread tid owns columns [tid*chunk, (tid+1)*chunk)
    const uint32_t chunk = (cols + blockDim.x - 1) / blockDim.x;
    const uint32_t c0 = tid * chunk, c1 = min(c0 + chunk, cols);
    uint32_t eq = 0;
    for (uint32_t c = c0; c < c1; ++c) eq += mag_key(a[c]) == kstar;
    // block exclusive scan of eq
    const uint32_t lane = tid & 31, warp = tid >> 5;
    uint32_t inc = eq;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t n = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= (uint32_t)off) inc += n;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t v = wsum[lane];
        uint32_t si = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t n = __shfl_up_sync(0xffffffffu, si, off);
            if (lane >= (uint32_t)off) si += n;
        }
        wsum[lane] = si - v;
    }
    __syncthreads();
    uint32_t rank = wsum[warp] + inc - eq;
    uint8_t* out = bits + (size_t)row * cols;
    for (uint32_t c = c0; c < c1; ++c) {
        const uint32_t key = mag_key(a[c]);
        uint8_t bit = key > kstar;
        if (key == kstar) bit = rank++ < take_eq;
        out[c] = bit;
    }
}

// bits [rows][cols] u8 -> bf16 [cols][ld] (0 / 1), zero for rows >= `rows`
// (ld = rows rounded up to 64: the K padding of the co-activation GEMM)
__global__ void bits_to_bf16_t_kernel(const uint8_t* __restrict__ bits, uint32_t rows, uint32_t cols, uint32_t ld,
                                      __nv_bfloat16* __restrict__ out) {
    __shared__ uint8_t tile[32][33];
    const uint32_t r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    const uint32_t tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (uint32_t q = ty; q < 32; q += 8) {
        const uint32_t r = r0 + q, c = c0 + tx;
        tile[q][tx] = (r < rows && c < cols) ? bits[(size_t)r * cols + c] : 0;
    }
    __syncthreads();
    for (uint32_t q = ty; q < 32; q += 8) {
        const uint32_t c = c0 + q, r = r0 + tx;
        if (c < cols && r < ld) out[(size_t)c * ld + r] = __float2bfloat16_rn(tile[tx][q] ? 1.0f : 0.0f);
    }
}

__global__ void set_group_meta_kernel(uint32_t* meta, uint32_t rows) {
    meta[0] = 0;
    meta[1] = rows;
    meta[2] = 0;
    meta[3] = (rows + kTcBM - 1) / kTcBM;
}

}  // namespace

void launch_binarize_topk(const float* act, uint32_t rows, uint32_t cols, uint32_t k_a, uint8_t* bits,
                          cudaStream_t s) {
    binarize_topk_kernel<<<rows, kBinThreads, 0, s>>>(act, cols, k_a, bits);
}

void launch_bits_to_bf16_t(const uint8_t* bits, uint32_t rows, uint32_t cols, uint32_t ld, void* out,
                           cudaStream_t s) {
    const dim3 grid((cols + 31) / 32, (ld + 31) / 32), block(32, 8);
    bits_to_bf16_t_kernel<<<grid, block, 0, s>>>(bits, rows, cols, ld, static_cast<__nv_bfloat16*>(out));
}

void launch_set_group_meta(uint32_t* meta, uint32_t rows, cudaStream_t s) {
    set_group_meta_kernel<<<1, 1, 0, s>>>(meta, rows);
}

}  // namespace mp
