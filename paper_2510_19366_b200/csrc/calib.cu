// calib.cu -- the calibration side of MoE-Prism on the GPU:
// the activation profile |a| that the offline refactoring engine partitions
// experts with, its per-row top-k binarisation, and the co-activation counts.
//
//   collect_activation_matrix  inc/expert.hpp:137-151   (gemm_tc.cu kEpiActAbs)
//   binarize_topk              inc/activation.hpp:213-240 (binarize_topk_kernel)
//   coactivation               inc/activation.hpp:242-266 (gemm_tc.cu kEpiCount
//                              over the transposed 0/1 matrix: C = B^T B,
//                              exact in fp32 for up to 2^24 rows)
//   centrality_scores +        inc/gating.hpp:47-103 (centrality_kernel,
//   select_gate_neurons        gate_select_kernel: exact u64 sums, block argmax
//                              on (score desc, neuron asc))
//   gating_fidelity            inc/gating.hpp:149-174 + subexpert_norms
//                              inc/partition.hpp:78-95 (fidelity_kernel: the
//                              reference's double sums in its order, bit-exact)
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

// centrality of neuron i = sum of co[i][j] over the other members j of its
// sub-expert (u64, exact; order-free).  Warp per neuron.
__global__ void __launch_bounds__(256) centrality_kernel(const uint32_t* __restrict__ co, uint32_t dim,
                                                         const uint32_t* __restrict__ label,
                                                         const uint32_t* __restrict__ mem_off,
                                                         const uint32_t* __restrict__ members,
                                                         unsigned long long* __restrict__ score) {
    const uint32_t i = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x & 31;
    if (i >= dim) return;
    const uint32_t s = label[i];
    unsigned long long sum = 0;
    for (uint32_t q = mem_off[s] + lane; q < mem_off[s + 1]; q += 32) {
        const uint32_t j = members[q];
        if (j != i) sum += co[(size_t)i * dim + j];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (lane == 0) score[i] = sum;
}

// top-r members of sub-expert s by (centrality desc, neuron asc): r rounds of a
// block argmax on the packed key score << 24 | (2^24 - 1 - neuron); the picks
// are written ascending to out[out_off[s] ..).  Block per sub-expert.
__global__ void __launch_bounds__(256) gate_select_kernel(const unsigned long long* __restrict__ score,
                                                          const uint32_t* __restrict__ mem_off,
                                                          const uint32_t* __restrict__ members, uint32_t r,
                                                          const uint32_t* __restrict__ out_off,
                                                          uint32_t* __restrict__ out) {
    __shared__ unsigned long long wbest[8];
    __shared__ unsigned long long best_key;
    const uint32_t s = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t b = mem_off[s], n = mem_off[s + 1] - b;
    const uint32_t take = r < n ? r : n;
    unsigned long long last = ~0ull;  // keys strictly below the previous pick
    for (uint32_t round = 0; round < take; ++round) {
        unsigned long long bk = 0;
        for (uint32_t q = tid; q < n; q += blockDim.x) {
            const uint32_t j = members[b + q];
            const unsigned long long key = (score[j] << 24) | (0xFFFFFFull - j);
            if (key < last && key > bk) bk = key;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long o = __shfl_xor_sync(0xffffffffu, bk, off);
            bk = o > bk ? o : bk;
        }
        if (lane == 0) wbest[warp] = bk;
        __syncthreads();
        if (tid == 0) {
            unsigned long long m = 0;
            for (uint32_t w = 0; w < blockDim.x / 32; ++w) m = wbest[w] > m ? wbest[w] : m;
            best_key = m;
            out[out_off[s] + round] = 0xFFFFFFu - static_cast<uint32_t>(m & 0xFFFFFFull);
        }
        __syncthreads();
        last = best_key;
    }
    __syncthreads();
    if (tid == 0) {  // ascending neuron order (insertion sort of <= r ids)
        uint32_t* o = out + out_off[s];
        for (uint32_t a = 1; a < take; ++a) {
            const uint32_t v = o[a];
            uint32_t c = a;
            while (c > 0 && o[c - 1] > v) {
                o[c] = o[c - 1];
                --c;
            }
            o[c] = v;
        }
    }
}

// Per (row, sub-expert): the true norm sum_{c in members ascending} act[b][c]
// and the proxy mean over the gate neurons (both double, sequential in the
// reference's order), then per row the top-k recall of proxy vs truth.
__global__ void fidelity_norms_kernel(const float* __restrict__ act, uint32_t rows, uint32_t cols, uint32_t n_sub,
                                      const uint32_t* __restrict__ mem_off, const uint32_t* __restrict__ members,
                                      const uint32_t* __restrict__ gate_off, const uint32_t* __restrict__ gate_ids,
                                      double* __restrict__ norm, double* __restrict__ proxy) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= rows * n_sub) return;
    const uint32_t b = q / n_sub, s = q % n_sub;
    const float* row = act + (size_t)b * cols;
    double acc = 0.0;
    for (uint32_t m = mem_off[s]; m < mem_off[s + 1]; ++m) acc += row[members[m]];
    norm[q] = acc;
    double sum = 0.0;
    for (uint32_t g = gate_off[s]; g < gate_off[s + 1]; ++g) sum += row[gate_ids[g]];
    proxy[q] = sum / static_cast<double>(gate_off[s + 1] - gate_off[s]);
}

__device__ void row_topk(const double* v, uint32_t n, uint32_t k, uint32_t* picked) {
    // the k largest, ties to the lower index (select_topk_subexperts), as a
    // bitmask over n <= 256 candidates
    for (uint32_t w = 0; w < 8; ++w) picked[w] = 0;
    for (uint32_t r = 0; r < k; ++r) {
        uint32_t bi = 0xFFFFFFFFu;
        for (uint32_t i = 0; i < n; ++i) {
            if ((picked[i >> 5] >> (i & 31)) & 1u) continue;
            if (bi == 0xFFFFFFFFu || v[i] > v[bi]) bi = i;
        }
        picked[bi >> 5] |= 1u << (bi & 31);
    }
}

__global__ void fidelity_rows_kernel(const double* __restrict__ norm, const double* __restrict__ proxy, uint32_t rows,
                                     uint32_t n_sub, uint32_t k, double* __restrict__ recall) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= rows) return;
    uint32_t pm[8], tm[8];
    row_topk(proxy + (size_t)b * n_sub, n_sub, k, pm);
    row_topk(norm + (size_t)b * n_sub, n_sub, k, tm);
    uint32_t hits = 0;
    for (uint32_t w = 0; w < 8; ++w) hits += __popc(pm[w] & tm[w]);
    recall[b] = static_cast<double>(hits) / static_cast<double>(k);
}

}  // namespace

void launch_centrality(const uint32_t* co, uint32_t dim, const uint32_t* label, const uint32_t* mem_off,
                       const uint32_t* members, unsigned long long* score, cudaStream_t s) {
    centrality_kernel<<<(dim + 7) / 8, 256, 0, s>>>(co, dim, label, mem_off, members, score);
}
void launch_gate_select(const unsigned long long* score, const uint32_t* mem_off, const uint32_t* members,
                        uint32_t n_sub, uint32_t r, const uint32_t* out_off, uint32_t* out, cudaStream_t s) {
    gate_select_kernel<<<n_sub, 256, 0, s>>>(score, mem_off, members, r, out_off, out);
}
void launch_fidelity(const float* act, uint32_t rows, uint32_t cols, uint32_t n_sub, const uint32_t* mem_off,
                     const uint32_t* members, const uint32_t* gate_off, const uint32_t* gate_ids, uint32_t k,
                     double* norm, double* proxy, double* recall, cudaStream_t s) {
    const uint32_t nq = rows * n_sub;
    fidelity_norms_kernel<<<(nq + 255) / 256, 256, 0, s>>>(act, rows, cols, n_sub, mem_off, members, gate_off,
                                                           gate_ids, norm, proxy);
    fidelity_rows_kernel<<<(rows + 127) / 128, 128, 0, s>>>(norm, proxy, rows, n_sub, k, recall);
}

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
