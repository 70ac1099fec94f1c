// route.cu -- router (linear fp32 logits + elastic per-token top-k +
// softmax renormalisation), bucketing (warp-level histogram + prefix scan +
// stable scatter), token dispatch (permute/gather) and the weighted combine.
//
// Reference anchors: select_topk_subexperts inc/gating.hpp:129-145 (total
// order score desc / index asc, ascending output); the linear router and
// softmax renormalisation are the SURVEY 8(c) restatement;
// bucketing / combine are SURVEY 8(a) a14/a15.  All HBM-bound: coalesced
// 16-byte vector accesses, no atomics, fixed reduction orders (deterministic).
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <string>
#include <cmath>
#include <type_traits>

#include "mp_common.cuh"
#include "mp_kernels.h"
#include "mp_topk.cuh"

namespace mp {

namespace {

constexpr uint32_t TB = kRouteTokensPerBlock;  // tokens per CTA
constexpr uint32_t GB = 64;                    // router outputs per pass
constexpr uint32_t KC = 32;                    // K chunk staged in smem
constexpr uint32_t kRouterThreads = 256;
constexpr uint32_t kWarpSplits = 8;  // route_bucket: more router K splits are summed CTA-wide

// Per-token certification bound of the tensor-core router logits (RouterGuard,
// mp_kernels.h): coef * sum |x_t| + 2^-23 max_g |logit_tg| + floor, with
// xn = sum |x_t| (warp_row_abs_sum).  Warp-wide; every lane gets the value.
// Non-finite (bad input, raised elsewhere): 0, so nothing is queued for the
// exact pass.
__device__ __forceinline__ double warp_router_guard(const RouterGuard& rg, double xn, double maxabs) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) maxabs = fmax(maxabs, __shfl_xor_sync(0xffffffffu, maxabs, off));
    const double g = rg.coef * xn + 0x1.0p-23 * maxabs + rg.floor_abs;
    return isfinite(g) ? g : 0.0;
}

// ---------------------------------------------------------------- linear router
// logits[t][g] = sum_i x[t][i] * W_r[i][g] with fp64 FMAs in ascending i
// (products of fp32 / bf16 inputs are exact in fp64): the oracle's own
// arithmetic, so the selection is exact up to fp64 rounding -- no
// certification pass is needed.  Used for fp32 layers and for bf16 layers the
// tensor-core router cannot take (d % 8 != 0).  CTA: 32 tokens x all G.
template <typename Tx>
__global__ void __launch_bounds__(kRouterThreads) router_linear_kernel(
    const Tx* __restrict__ x, uint32_t T, uint32_t d, const float* __restrict__ wrT, uint32_t G, uint32_t k_max,
    const uint32_t* __restrict__ kpt, uint32_t k_scalar, int weight_mode, uint32_t* __restrict__ sel,
    float* __restrict__ wout, int* __restrict__ err, uint32_t* __restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* lg = reinterpret_cast<double*>(smem_raw);                 // [TB][G]
    float* xs = reinterpret_cast<float*>(lg + TB * G);                // [KC][TB+1]
    float* ws = xs + KC * (TB + 1);                                   // [KC][GB+4]
    const uint32_t tid = threadIdx.x;
    const uint32_t t0 = blockIdx.x * TB;
    const uint32_t tx = tid % 16, ty = tid / 16;  // 4 outputs (g) x 2 tokens per thread
    bool nonfinite = false;

    for (uint32_t g0 = 0; g0 < G; g0 += GB) {
        double acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
        for (uint32_t k0 = 0; k0 < d; k0 += KC) {
            __syncthreads();
            for (uint32_t q = tid; q < TB * KC; q += kRouterThreads) {
                const uint32_t t = q / KC, kk = q % KC;
                float v = 0.0f;
                if (t0 + t < T && k0 + kk < d) {
                    v = to_f32(x[(size_t)(t0 + t) * d + k0 + kk]);
                    if (g0 == 0 && !isfinite(v)) nonfinite = true;
                }
                xs[kk * (TB + 1) + t] = v;
            }
            for (uint32_t q = tid; q < GB * KC; q += kRouterThreads) {
                const uint32_t g = q / KC, kk = q % KC;
                float v = 0.0f;
                if (g0 + g < G && k0 + kk < d) v = wrT[(size_t)(g0 + g) * d + k0 + kk];
                ws[kk * (GB + 4) + g] = v;
            }
            __syncthreads();
#pragma unroll
            for (uint32_t kk = 0; kk < KC; ++kk) {
                const float xa = xs[kk * (TB + 1) + 2 * ty];
                const float xb = xs[kk * (TB + 1) + 2 * ty + 1];
                const float4 wv = *reinterpret_cast<const float4*>(&ws[kk * (GB + 4) + 4 * tx]);
                const double wvd[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    acc[0][b] = fma(static_cast<double>(xa), wvd[b], acc[0][b]);
                    acc[1][b] = fma(static_cast<double>(xb), wvd[b], acc[1][b]);
                }
            }
        }
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const uint32_t g = g0 + 4 * tx + b;
                if (g < G) lg[(2 * ty + a) * G + g] = acc[a][b];
            }
    }
    if (nonfinite && err) atomicOr(err, 2);
    __syncthreads();
    const uint32_t warp = tid / 32;
    for (uint32_t t = warp; t < TB; t += kRouterThreads / 32) {
        const uint32_t tg = t0 + t;
        if (tg >= T) break;
        const uint32_t kt = token_k(kpt, k_scalar, tg, k_max, G, err);
        const double gap = warp_topk_token(lg + t * G, G, kt, k_max, weight_mode, sel + (size_t)tg * k_max,
                                           wout + (size_t)tg * k_max);
        if (stats && gap < kNearTie && (tid & 31) == 0) atomicAdd(stats + 1, 1u);
    }
}

// Top-k over precomputed double scores [T][G] (proxy router).
__global__ void __launch_bounds__(256) scores_topk_kernel(const double* __restrict__ scores, uint32_t T, uint32_t G,
                                                          uint32_t k_max, const uint32_t* __restrict__ kpt,
                                                          uint32_t k_scalar, int weight_mode,
                                                          uint32_t* __restrict__ sel, float* __restrict__ wout,
                                                          int* __restrict__ err, uint32_t* __restrict__ stats) {
    const uint32_t t = blockIdx.x * 8 + threadIdx.x / 32;
    if (t >= T) return;
    const uint32_t kt = token_k(kpt, k_scalar, t, k_max, G, err);
    const double gap = warp_topk_token(scores + (size_t)t * G, G, kt, k_max, weight_mode, sel + (size_t)t * k_max,
                                       wout + (size_t)t * k_max);
    if (stats && gap < kNearTie && (threadIdx.x & 31) == 0) atomicAdd(stats + 1, 1u);
}

// Tensor-core router epilogue: logits[t][g] = sum_{s ascending} partial[s][t][g]
// (fixed order, fp64), then the per-token top-k.  Warp per token.
__global__ void __launch_bounds__(256) partials_topk_kernel(const double* __restrict__ partial, uint32_t ks,
                                                            uint32_t T, uint32_t G, uint32_t Npad, uint32_t k_max,
                                                            const uint32_t* __restrict__ kpt, uint32_t k_scalar,
                                                            int weight_mode, uint32_t* __restrict__ sel,
                                                            float* __restrict__ wout, int* __restrict__ err,
                                                            RouterGuard rg, const __nv_bfloat16* __restrict__ x,
                                                            uint32_t d, uint32_t* __restrict__ flagged) {
    __shared__ double sc[8][kMaxG];
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t t = blockIdx.x * 8 + warp;
    if (t >= T) return;
    const double xn = warp_row_abs_sum(x + (size_t)t * d, d);
    double maxabs = 0.0;
    for (uint32_t g = lane; g < G; g += 32) {
        double v = 0.0;
        for (uint32_t s = 0; s < ks; ++s) v += partial[((size_t)s * T + t) * Npad + g];
        sc[warp][g] = v;
        maxabs = fmax(maxabs, fabs(v));
    }
    const double guard = warp_router_guard(rg, xn, maxabs);
    __syncwarp();
    const uint32_t kt = token_k(kpt, k_scalar, t, k_max, G, err);
    const double gap = warp_topk_token(sc[warp], G, kt, k_max, weight_mode, sel + (size_t)t * k_max,
                                       wout + (size_t)t * k_max);
    // the selection is certified only when the k-th / (k+1)-th gap exceeds
    // twice the tensor-core error bound; otherwise recompute exactly (fp64)
    if (gap < 2.0 * guard + kNearTie && lane == 0) flagged[2 + atomicAdd(&flagged[0], 1u)] = t;
}

// Exact fp64 logits for the flagged tokens (x bf16/f32 . W_r fp32, products
// exact in double, fixed-order reduction), then the top-k again.  CTA per
// flagged token: the row of x is staged in smem as double, each warp owns
// G/8 outputs and its lanes stride over K with coalesced W_r row reads.
template <typename Tx>
__global__ void __launch_bounds__(1024) router_fixup_kernel(const Tx* __restrict__ x, uint32_t d,
                                                           const float* __restrict__ wrT, uint32_t G, uint32_t k_max,
                                                           const uint32_t* __restrict__ kpt, uint32_t k_scalar,
                                                           int weight_mode, uint32_t* __restrict__ sel,
                                                           float* __restrict__ wout, int* __restrict__ err,
                                                           uint32_t* __restrict__ flagged) {
    extern __shared__ double xs_d[];  // [d]
    __shared__ double lg[kMaxG];
    const uint32_t n = flagged[0];
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (uint32_t f = blockIdx.x; f < n; f += gridDim.x) {
        const uint32_t t = flagged[2 + f];
        const Tx* xr = x + (size_t)t * d;
        for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) xs_d[i] = static_cast<double>(to_f32(xr[i]));
        __syncthreads();
        const uint32_t nwarps = blockDim.x / 32;
        for (uint32_t g = warp; g < G; g += nwarps) {
            const float* wrow = wrT + (size_t)g * d;
            // float4 loads, 8 in flight per lane, 8 independent accumulators
            // combined in a fixed order (deterministic)
            double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            const uint32_t d4 = (d % 4 == 0) ? d / 4 : 0;
            const float4* w4 = reinterpret_cast<const float4*>(wrow);
            uint32_t i4 = lane;
            for (; i4 + 7 * 32 < d4; i4 += 8 * 32) {
                float4 wv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) wv[u] = __ldg(w4 + i4 + u * 32);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double* xd = xs_d + 4 * (i4 + u * 32);
                    acc[u] = fma(xd[0], (double)wv[u].x, acc[u]);
                    acc[u] = fma(xd[1], (double)wv[u].y, acc[u]);
                    acc[u] = fma(xd[2], (double)wv[u].z, acc[u]);
                    acc[u] = fma(xd[3], (double)wv[u].w, acc[u]);
                }
            }
            for (; i4 < d4; i4 += 32) {
                const float4 wv = __ldg(w4 + i4);
                const double* xd = xs_d + 4 * i4;
                acc[0] = fma(xd[0], (double)wv.x, acc[0]);
                acc[0] = fma(xd[1], (double)wv.y, acc[0]);
                acc[0] = fma(xd[2], (double)wv.z, acc[0]);
                acc[0] = fma(xd[3], (double)wv.w, acc[0]);
            }
            for (uint32_t i = 4 * d4 + lane; i < d; i += 32) acc[1] = fma(xs_d[i], (double)__ldg(wrow + i), acc[1]);
            double a = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
            if (lane == 0) lg[g] = a;
        }
        __syncthreads();
        if (warp == 0) {
            const uint32_t kt = token_k(kpt, k_scalar, t, k_max, G, err);
            const double gap =
                warp_topk_token(lg, G, kt, k_max, weight_mode, sel + (size_t)t * k_max, wout + (size_t)t * k_max);
            if (gap < kNearTie && lane == 0) atomicAdd(const_cast<uint32_t*>(flagged) + 1, 1u);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- bucketing
// Per CTA of 32 tokens: selection bitmasks in smem, then one thread per
// sub-expert walks the tokens in order -> rank of each (t, slot) inside its
// (CTA, bucket) and the CTA's histogram.  Stable by construction.
__global__ void __launch_bounds__(256) bucket_local_kernel(const uint32_t* __restrict__ sel, uint32_t T,
                                                           uint32_t k_max, uint32_t G, uint32_t* __restrict__ lrank,
                                                           uint32_t* __restrict__ block_counts,
                                                           int* __restrict__ err) {
    __shared__ uint32_t msk[TB][kMaxG / 32];
    __shared__ uint16_t slot_of[TB][kMaxG];  // slot index of g in token t (valid where selected)
    const uint32_t t0 = blockIdx.x * TB;
    const uint32_t words = (G + 31) / 32;
    for (uint32_t q = threadIdx.x; q < TB * words; q += blockDim.x) msk[q / words][q % words] = 0;
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < TB * k_max; q += blockDim.x) {
        const uint32_t t = q / k_max, j = q % k_max;
        if (t0 + t >= T) continue;
        const uint32_t g = sel[(size_t)(t0 + t) * k_max + j];
        if (g == kSelNone) continue;
        if (g >= G) {
            atomicOr(err, 1);
            continue;
        }
        const uint32_t old = atomicOr(&msk[t][g >> 5], 1u << (g & 31));
        if (old & (1u << (g & 31))) atomicOr(err, 1);  // duplicate (inc/expert.hpp:117)
        slot_of[t][g] = static_cast<uint16_t>(j);
    }
    __syncthreads();
    for (uint32_t g = threadIdx.x; g < G; g += blockDim.x) {
        uint32_t cnt = 0;
        for (uint32_t t = 0; t < TB && t0 + t < T; ++t) {
            if ((msk[t][g >> 5] >> (g & 31)) & 1u) lrank[(size_t)(t0 + t) * k_max + slot_of[t][g]] = cnt++;
        }
        block_counts[(size_t)blockIdx.x * G + g] = cnt;
    }
}

// Exclusive scans: over CTAs per bucket (-> block_base), over buckets
// (-> offsets), and the GEMM tile prefixes.  One CTA of 1024 threads.
#if MP_ROUTE_TRACE
__device__ unsigned long long g_scan_tr[8];
#define MP_SCAN_STAMP(i) \
    if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_scan_tr[i]))
#else
#define MP_SCAN_STAMP(i)
#endif

// V independent exclusive scans over the 1024 threads of the CTA with one
// set of barriers (the bucket offsets and the GEMM tile prefixes)
template <int V>
__device__ void block_exclusive_scan_1024_multi(uint32_t (&v)[V], uint32_t (&total)[V], uint32_t (*wsum)[32]) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc[V];
#pragma unroll
    for (int j = 0; j < V; ++j) inc[j] = v[j];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const uint32_t n = __shfl_up_sync(0xffffffffu, inc[j], off);
            if (lane >= (uint32_t)off) inc[j] += n;
        }
    }
    if (lane == 31) {
#pragma unroll
        for (int j = 0; j < V; ++j) wsum[j][warp] = inc[j];
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t sv[V], si[V];
#pragma unroll
        for (int j = 0; j < V; ++j) sv[j] = si[j] = wsum[j][lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const uint32_t n = __shfl_up_sync(0xffffffffu, si[j], off);
                if (lane >= (uint32_t)off) si[j] += n;
            }
        }
#pragma unroll
        for (int j = 0; j < V; ++j) wsum[j][lane] = si[j] - sv[j];
        if (lane == 31) {
#pragma unroll
            for (int j = 0; j < V; ++j) wsum[V][j] = si[j];  // totals row
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < V; ++j) {
        total[j] = wsum[V][j];
        v[j] = wsum[j][warp] + inc[j] - v[j];
    }
    __syncthreads();
}

__device__ void bucket_scan_body(uint32_t nblk, uint32_t G, const uint32_t* __restrict__ block_counts,
                                 uint32_t* __restrict__ block_base, uint32_t* __restrict__ offsets,
                                 uint32_t* __restrict__ mprefix_tc, uint32_t* __restrict__ mprefix_simt,
                                 uint32_t* __restrict__ mprefix_tc2, uint8_t* s_cnt) {
    // thread (g, q): bucket g, q-th contiguous range of CTA-blocks; consecutive
    // threads read consecutive buckets of one block row (coalesced).
    // s_cnt (nullable): nblk x G bytes of shared memory -- the counts (<= 32
    // tokens per block and bucket) are staged there with one coalesced pass, so
    // both sweeps over them (sums, then bases) read shared memory instead of
    // chains of L2 loads
    constexpr int V = 4;
    if (s_cnt) {
        const uint32_t n = nblk * G;
        const uint32_t n4 = (n % 4 == 0) ? n / 4 : 0;
        for (uint32_t i = threadIdx.x; i < n4; i += blockDim.x) {
            const uint4 v = __ldcg(reinterpret_cast<const uint4*>(block_counts) + i);
            reinterpret_cast<uint32_t*>(s_cnt)[i] = v.x | (v.y << 8) | (v.z << 16) | (v.w << 24);
        }
        for (uint32_t i = 4 * n4 + threadIdx.x; i < n; i += blockDim.x) s_cnt[i] = static_cast<uint8_t>(__ldcg(block_counts + i));
        __syncthreads();
    }
    auto cnt = [&](uint32_t b, uint32_t gg) -> uint32_t {
        return s_cnt ? s_cnt[(size_t)b * G + gg] : block_counts[(size_t)b * G + gg];
    };
    __shared__ uint32_t part[1024];
    __shared__ uint32_t goff[kMaxG];
    __shared__ uint32_t wsum[V + 1][32];
    const uint32_t Q = blockDim.x / G;
    const uint32_t g = threadIdx.x % G, q = threadIdx.x / G;
    const bool active = q < Q;
    const uint32_t per = (nblk + Q - 1) / Q;
    const uint32_t b0 = q * per, b1 = min(b0 + per, nblk);
    MP_SCAN_STAMP(0);
    uint32_t sum = 0;
    // independent loads in flight (Qwen prefill: 256 blocks x 240 buckets,
    // 64 blocks per thread): the last CTA's scan is on the critical path
    if (active) {
#pragma unroll 16
        for (uint32_t b = b0; b < b1; ++b) sum += cnt(b, g);
    }
    part[threadIdx.x] = sum;
    __syncthreads();
    // exclusive prefix over the Q ranges of each bucket, and bucket totals
    uint32_t qbase = 0, total = 0;
    if (active) {
        for (uint32_t r = 0; r < Q; ++r) {
            const uint32_t v = part[r * G + g];
            if (r < q) qbase += v;
            total += v;
        }
    }
    __syncthreads();
    const uint32_t gi = threadIdx.x;
    if (active && q == 0) goff[g] = total;
    __syncthreads();
    const uint32_t c = gi < G ? goff[gi] : 0;
    MP_SCAN_STAMP(1);
    // bucket offsets and the GEMM tile prefixes, scanned together:
    //   offsets (rows), 128-row tiles, 64-row SIMT tiles, 256-row pair tiles
    uint32_t sv[V] = {c, gi < G ? (c + kTcBM - 1) / kTcBM : 0u, gi < G ? (c + kSimtBM - 1) / kSimtBM : 0u,
                      gi < G ? (c + 255) / 256 : 0u};
    uint32_t tot[V];
    block_exclusive_scan_1024_multi<V>(sv, tot, wsum);
    const uint32_t off = sv[0];
    if (gi < G) {
        offsets[gi] = off;
        mprefix_tc[gi] = sv[1];
        mprefix_simt[gi] = sv[2];
        mprefix_tc2[gi] = sv[3];
    }
    if (gi == 0) {
        offsets[G] = tot[0];
        mprefix_tc[G] = tot[1];
        mprefix_simt[G] = tot[2];
        mprefix_tc2[G] = tot[3];
    }
    __syncthreads();
    if (gi < G) goff[gi] = off;
    __syncthreads();
    MP_SCAN_STAMP(2);
    if (active) {
        uint32_t running = goff[g] + qbase;
        constexpr uint32_t U = 16;
        for (uint32_t b = b0; b < b1; b += U) {
            uint32_t v[U];
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) v[u] = b + u < b1 ? cnt(b + u, g) : 0u;
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
                if (b + u < b1) block_base[(size_t)(b + u) * G + g] = running;
                running += v[u];
            }
        }
    }
}

// Grid-scan variant (every CTA b of a co-resident grid, after a grid barrier):
// block_base[b][g] = offsets[g] + sum_{b' < b} counts[b'][g] for this CTA's
// row only; offsets / tile prefixes scanned redundantly per CTA, written by
// CTA 0.  Thread (g, q) sums the q-th range of blocks.
__device__ void bucket_bases_grid(uint32_t nblk, uint32_t b, uint32_t G, const uint32_t* __restrict__ block_counts,
                                  uint32_t* __restrict__ block_base, uint32_t* __restrict__ offsets,
                                  uint32_t* __restrict__ mprefix_tc, uint32_t* __restrict__ mprefix_simt,
                                  uint32_t* __restrict__ mprefix_tc2) {
    constexpr int V = 4;
    __shared__ uint32_t part_all[1024], part_pre[1024];
    __shared__ uint32_t wsum[V + 1][32];
    const uint32_t Q = blockDim.x / G;
    const uint32_t g = threadIdx.x % G, q = threadIdx.x / G;
    const bool active = q < Q;
    const uint32_t per = (nblk + Q - 1) / Q;
    const uint32_t b0 = q * per, b1 = min(b0 + per, nblk);
    uint32_t all = 0, pre = 0;
    if (active) {
#pragma unroll 8
        for (uint32_t bb = b0; bb < b1; ++bb) {
            const uint32_t c = __ldcg(block_counts + (size_t)bb * G + g);
            all += c;
            pre += bb < b ? c : 0u;
        }
    }
    part_all[threadIdx.x] = all;
    part_pre[threadIdx.x] = pre;
    __syncthreads();
    const uint32_t gi = threadIdx.x;
    uint32_t total = 0, prefix = 0;
    if (gi < G) {
        for (uint32_t r = 0; r < Q; ++r) {
            total += part_all[r * G + gi];
            prefix += part_pre[r * G + gi];
        }
    }
    uint32_t sv[V] = {total, gi < G ? (total + kTcBM - 1) / kTcBM : 0u, gi < G ? (total + kSimtBM - 1) / kSimtBM : 0u,
                      gi < G ? (total + 255) / 256 : 0u};
    uint32_t tot[V];
    block_exclusive_scan_1024_multi<V>(sv, tot, wsum);
    if (gi < G) block_base[(size_t)b * G + gi] = sv[0] + prefix;
    if (b == 0) {
        if (gi < G) {
            offsets[gi] = sv[0];
            mprefix_tc[gi] = sv[1];
            mprefix_simt[gi] = sv[2];
            mprefix_tc2[gi] = sv[3];
        }
        if (gi == 0) {
            offsets[G] = tot[0];
            mprefix_tc[G] = tot[1];
            mprefix_simt[G] = tot[2];
            mprefix_tc2[G] = tot[3];
        }
    }
}

__global__ void __launch_bounds__(1024) bucket_scan_kernel(uint32_t nblk, uint32_t G,
                                                           const uint32_t* __restrict__ block_counts,
                                                           uint32_t* __restrict__ block_base,
                                                           uint32_t* __restrict__ offsets,
                                                           uint32_t* __restrict__ mprefix_tc,
                                                           uint32_t* __restrict__ mprefix_simt,
                                                           uint32_t* __restrict__ mprefix_tc2) {
    bucket_scan_body(nblk, G, block_counts, block_base, offsets, mprefix_tc, mprefix_simt, mprefix_tc2, nullptr);
}

// Exact fp64 logit x_t . W_r[:, g] by one warp: bf16 x and fp32 W_r are exact
// in double, 4 fixed accumulators per lane + a fixed shuffle tree
// (deterministic).  d % 4 == 0.
__device__ double warp_exact_logit(const __nv_bfloat16* __restrict__ xr, const float* __restrict__ wrow, uint32_t d) {
    const uint32_t lane = lane_id();
    double acc[4] = {0, 0, 0, 0};
    // 4 independent 16-byte loads per lane in flight: this runs for a handful
    // of (token, candidate) pairs per forward and is pure load latency
    constexpr uint32_t U = 4;
    for (uint32_t i0 = 4 * lane; i0 < d; i0 += U * 128) {
        float4 wv[U];
        uint2 xv[U];
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) {
            const uint32_t i = i0 + u * 128;
            wv[u] = i < d ? __ldg(reinterpret_cast<const float4*>(wrow + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
            xv[u] = i < d ? __ldg(reinterpret_cast<const uint2*>(xr + i)) : make_uint2(0u, 0u);
        }
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) {
            const float2 x01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xv[u].x));
            const float2 x23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xv[u].y));
            acc[0] = fma((double)x01.x, (double)wv[u].x, acc[0]);
            acc[1] = fma((double)x01.y, (double)wv[u].y, acc[1]);
            acc[2] = fma((double)x23.x, (double)wv[u].z, acc[2]);
            acc[3] = fma((double)x23.y, (double)wv[u].w, acc[3]);
        }
    }
    double a = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
    return a;
}

// Device-wide exclusive scans of the bucketing, run by one CTA of 1024
// threads (bucket_scan_kernel, or the last CTA of route_bucket_kernel).
__device__ void bucket_scan_body(uint32_t nblk, uint32_t G, const uint32_t* __restrict__ block_counts,
                                 uint32_t* __restrict__ block_base, uint32_t* __restrict__ offsets,
                                 uint32_t* __restrict__ mprefix_tc, uint32_t* __restrict__ mprefix_simt,
                                 uint32_t* __restrict__ mprefix_tc2, uint8_t* s_cnt);

// Fused routing epilogue of the tensor-core router, CTA = 32 tokens (warp per
// token), replacing partials_topk + router_fixup + bucket_local + bucket_scan:
//   1. logits = fixed-order fp64 sum of the K-split partials, top-k, weights;
//   2. near-tie certification: with a, b the k-th / (k+1)-th selection keys
//      (fp32-rounded tensor-core logits) and |key - exact| < guard, a gap
//      a - b < 2 guard leaves only the window
//      W = {g : b - 2 guard <= logit_g <= a + 2 guard} uncertain (above W:
//      certainly selected, below: certainly not); W is recomputed in exact
//      fp64 and the token re-selected on (+inf above W, exact in W, -inf
//      below) -- the same selection the exact logits give;
//   3. per-CTA bucket ranks / histogram (bucket_local_kernel's scheme);
//   4. the last CTA to finish (threadfence + atomic ticket) runs the
//      device-wide scans, then resets the ticket.
template <int NC>
__global__ void __launch_bounds__(1024) route_bucket_kernel(
    const double* __restrict__ partial, uint32_t ks, uint32_t T, uint32_t G, uint32_t Npad, uint32_t k_max,
    const uint32_t* __restrict__ kpt, uint32_t k_scalar, int weight_mode, uint32_t* __restrict__ sel,
    float* __restrict__ wout, int* __restrict__ err, RouterGuard rg, const __nv_bfloat16* __restrict__ x, uint32_t d,
    const float* __restrict__ wrT, uint32_t* __restrict__ ticket, uint32_t* __restrict__ stats, uint32_t* lrank,
    uint32_t* block_counts, uint32_t* block_base, uint32_t* offsets, uint32_t* mprefix_tc, uint32_t* mprefix_simt,
    uint32_t* mprefix_tc2, uint32_t tb, uint32_t smem_bytes, uint32_t grid_scan, uint32_t* perm_tok, float* perm_w,
    uint32_t* slot_row) {
    extern __shared__ double rsm[];  // [tb][G] logits, then [tb][G] keys; the last CTA: staged counts
    double* sc = rsm + (size_t)(threadIdx.x / 32) * G;        // used by warps < tb only
    double* key = rsm + (size_t)(tb + threadIdx.x / 32) * G;
    __shared__ double vk[TB][2];
    __shared__ uint32_t msk[TB][kMaxG / 32];
    __shared__ uint16_t slot_of[TB][kMaxG];
    __shared__ uint32_t is_last;
    constexpr uint32_t kMaxPairs = 1024, kPairBatch = 8;
    __shared__ uint32_t n_pairs;
    __shared__ uint32_t pair_tg[kMaxPairs];  // (token in CTA << 16) | candidate
    __shared__ double pair_part[kPairBatch][4];
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
#if MP_ROUTE_TRACE
    uint64_t tr_[8], tr_coop = 0, tr_row = 0, tr_topk = 0;
    uint32_t ntr_ = 0;
    auto stamp = [&]() { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_[ntr_++])); };
    stamp();
#define MP_RT_STAMP() stamp()
#else
#define MP_RT_STAMP()
#endif
    // tb tokens per block (warps >= tb only help with the CTA-wide phases):
    // small batches use tb = 8 so the token work spreads over 4x the SMs.
    // Grid-scan launches are persistent (grid <= SMs): a CTA takes token
    // blocks blockIdx.x, + gridDim.x, ... (Qwen prefill: 256 blocks on 148
    // SMs) so the grid barrier below stays deadlock-free.
    const uint32_t nblk = (T + tb - 1) / tb;
    const uint32_t words = (G + 31) / 32;
    griddep_wait();
    griddep_launch();
    for (uint32_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const bool first_blk = blk == blockIdx.x;
    const uint32_t t0 = blk * tb, t = warp < tb ? t0 + warp : T;
    for (uint32_t q = threadIdx.x; q < TB * words; q += blockDim.x) msk[q / words][q % words] = 0;
    if (threadIdx.x == 0) n_pairs = 0;
    __syncthreads();
    // many K splits (small batches: 64-deep router chunks) and few tokens per
    // CTA: the whole CTA sums the splits, one (token, sub-expert) per thread,
    // into the logit rows (replaces a separate partials_reduce launch; same
    // ascending fixed order)
    const bool coop = ks > kWarpSplits;
    if (coop) {
        for (uint32_t q = threadIdx.x; q < tb * G; q += blockDim.x) {
            const uint32_t tl = q / G, g = q - tl * G;
            if (t0 + tl >= T) continue;
            const double* pp = partial + (size_t)(t0 + tl) * Npad + g;
            double v = 0.0;
#pragma unroll 8
            for (uint32_t s = 0; s < ks; ++s) v += __ldcg(pp + (size_t)s * T * Npad);
            rsm[(size_t)tl * G + g] = v;
        }
    }
    __syncthreads();
#if MP_ROUTE_TRACE
    if (first_blk) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_coop));
#endif
    bool flagged = false;
    uint32_t kt = 0;
    double guard = 0.0;
    if (t < T) {
        const double xn = warp_row_abs_sum(x + (size_t)t * d, d);  // certification bound input
#if MP_ROUTE_TRACE
        if (first_blk) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_row));
#endif
        if (!isfinite(xn) && lane == 0 && err) atomicOr(err, 2);    // the reference's check_input
        // fixed-order sum over the K splits; all NC loads of a split in flight
        // (the partials come from L2 / HBM: a load per candidate in turn left
        // this phase latency-bound, 7 us for 240 candidates)
        double v[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) v[c] = 0.0;
        const double* prow = partial + (size_t)t * Npad + lane;
        if (coop) {
#pragma unroll
            for (int c = 0; c < NC; ++c) v[c] = lane + 32u * c < G ? sc[lane + 32u * c] : 0.0;
        } else {
#pragma unroll 4
            for (uint32_t s = 0; s < ks; ++s) {
                double u[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c) u[c] = lane + 32u * c < G ? __ldcg(prow + (size_t)s * T * Npad + 32u * c) : 0.0;
#pragma unroll
                for (int c = 0; c < NC; ++c) v[c] += u[c];
            }
        }
        double maxabs = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if (lane + 32u * c < G) {
                sc[lane + 32u * c] = v[c];
                maxabs = fmax(maxabs, fabs(v[c]));
            }
        guard = warp_router_guard(rg, xn, maxabs);
        __syncwarp();
        kt = token_k(kpt, k_scalar, t, k_max, G, err);
        const double gap = warp_topk_fast<NC>(sc, G, kt, k_max, weight_mode, sel + (size_t)t * k_max,
                                          wout + (size_t)t * k_max, vk[warp], msk[warp], slot_of[warp]);
#if MP_ROUTE_TRACE
        if (first_blk) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_topk));
#endif
        __syncwarp();
        // the exact pass also takes every token that may be an oracle near tie
        // (exact gap < 1e-6), so near ties are counted exactly
        flagged = gap < 2.0 * guard + kNearTie;
        if (flagged) {  // queue the uncertainty window for the CTA-wide exact pass
            const double a = vk[warp][0], b = vk[warp][1];
            for (uint32_t g0 = 0; g0 < G; g0 += 32) {
                const uint32_t g = g0 + lane;
                const double v = g < G ? static_cast<double>(static_cast<float>(sc[g])) : -DBL_MAX;  // the keys
                const bool in_w = g < G && v >= b - 2.0 * guard && v <= a + 2.0 * guard;
                if (g < G) key[g] = v > a + 2.0 * guard ? DBL_MAX : (in_w ? v : -DBL_MAX);
                if (in_w) {
                    const uint32_t slot = atomicAdd(&n_pairs, 1u);
                    if (slot < kMaxPairs) pair_tg[slot] = (warp << 16) | g;
                }
            }
        }
    }
    __syncthreads();
    if (first_blk) MP_RT_STAMP();  // 1: top-k done
    // exact fp64 logits of every queued (token, candidate), 4 warps per pair
    // (d split in quarters, fixed-order combination: deterministic)
    const uint32_t np = min(n_pairs, kMaxPairs);
    if (np) {
        for (uint32_t p0 = 0; p0 < np; p0 += 8) {
            const uint32_t pi = p0 + warp / 4, qq = warp % 4;
            if (pi < np) {
                const uint32_t tl = pair_tg[pi] >> 16, g = pair_tg[pi] & 0xFFFFu;
                const uint32_t dq = (d / 4 + 127) / 128 * 128;  // quarter, multiple of 128
                const uint32_t lo = qq * dq, hi = min(d, lo + dq);
                const double part = lo < hi ? warp_exact_logit(x + (size_t)(t0 + tl) * d + lo,
                                                               wrT + (size_t)g * d + lo, hi - lo)
                                            : 0.0;
                if (lane == 0) pair_part[pi % kPairBatch][qq] = part;
            }
            __syncthreads();
            for (uint32_t q2 = threadIdx.x; q2 < 8 && p0 + q2 < np; q2 += blockDim.x) {
                const uint32_t pj = p0 + q2, tl = pair_tg[pj] >> 16, g = pair_tg[pj] & 0xFFFFu;
                const double* pp = pair_part[pj % kPairBatch];
                const double e = ((pp[0] + pp[1]) + pp[2]) + pp[3];
                rsm[(size_t)(tb + tl) * G + g] = e;  // key
                rsm[(size_t)tl * G + g] = e;         // logit (weights)
            }
            __syncthreads();
        }
    }
    if (flagged) {
        if (n_pairs > kMaxPairs) {  // overflow (only with an absurd guard): serial exact pass
            for (uint32_t g = 0; g < G; ++g)
                if (key[g] != DBL_MAX && key[g] != -DBL_MAX) {
                    const double e = warp_exact_logit(x + (size_t)t * d, wrT + (size_t)g * d, d);
                    if (lane == 0) key[g] = sc[g] = e;
                    __syncwarp();
                }
        }
        __syncwarp();
        // the k-th and (k+1)-th exact keys both lie in the window: gap is exact
        const double egap = warp_topk_token<NC>(sc, G, kt, k_max, weight_mode, sel + (size_t)t * k_max,
                                                wout + (size_t)t * k_max, key, nullptr, msk[warp], slot_of[warp]);
        if (lane == 0) {
            atomicAdd(stats, 1u);
            if (egap < kNearTie) atomicAdd(stats + 1, 1u);
        }
    }
    __syncthreads();  // this CTA's selections are visible to the CTA
    if (first_blk) {
        MP_RT_STAMP();  // 2: exact pass done
        // (the selection masks / slots were written by the top-k emissions)
        MP_RT_STAMP();  // 3: selection masks built
    }
    // warp per bucket, lane per token (tb <= 32): the stable rank of token tt
    // in bucket g is the number of earlier tokens of the CTA selecting g
    for (uint32_t g = warp; g < G; g += blockDim.x / 32) {
        const bool has = lane < tb && t0 + lane < T && ((msk[lane][g >> 5] >> (g & 31)) & 1u);
        const uint32_t bal = __ballot_sync(0xffffffffu, has);
        if (has) lrank[(size_t)(t0 + lane) * k_max + slot_of[lane][g]] = __popc(bal & ((1u << lane) - 1u));
        if (lane == 0) block_counts[(size_t)blk * G + g] = __popc(bal);
    }
    // this CTA's writes (selection, weights, ranks, counts) are ordered before
    // the ticket by the barrier + one gpu-scope fence of the ticket thread
    // (fences are cumulative over what the barrier made visible to it)
    __syncthreads();
    }  // token blocks
    MP_RT_STAMP();  // 4: ranks done
    if (grid_scan) {
        // grid-wide barrier (the grid fits on the GPU at once: one 1024-thread
        // CTA per SM, gridDim <= SMs) -- then EVERY CTA forms its own bucket
        // bases from all CTAs' counts, instead of one last CTA writing all of
        // them after the others retire
        if (threadIdx.x == 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            atomicAdd(ticket + 1, 1u);
            uint32_t seen;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(ticket + 1) : "memory");
            } while (seen < gridDim.x);
        }
        __syncthreads();
        MP_RT_STAMP();  // 5: barrier passed
        for (uint32_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
            if (blk != blockIdx.x) __syncthreads();  // the previous block's scan scratch is free
            bucket_bases_grid(nblk, blk, G, block_counts, block_base, offsets, mprefix_tc, mprefix_simt,
                              mprefix_tc2);
        }
        if (perm_tok) {
            // the permutation tables of this CTA's tokens (what the dispatch
            // kernel writes when the GEMM gathers its rows from x itself:
            // decode batches), from its own bucket bases and ranks
            __syncthreads();
            for (uint32_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
                for (uint32_t tl = warp; tl < tb; tl += blockDim.x / 32) {
                    const uint32_t tt = blk * tb + tl;
                    if (tt >= T) continue;
                    for (uint32_t j = lane; j < k_max; j += 32) {
                        const uint32_t g = sel[(size_t)tt * k_max + j];
                        uint32_t pos = kSelNone;
                        if (g != kSelNone && g < G) {
                            pos = block_base[(size_t)blk * G + g] + lrank[(size_t)tt * k_max + j];
                            perm_tok[pos] = tt;
                            perm_w[pos] = wout[(size_t)tt * k_max + j];
                        }
                        slot_row[(size_t)tt * k_max + j] = pos;
                    }
                }
            }
        }
        if (threadIdx.x == 0 && atomicAdd(ticket + 2, 1u) == gridDim.x - 1) {
            ticket[1] = 0;  // every CTA is past the barrier: reset for the next forward (stream-ordered)
            ticket[2] = 0;
        }
#if MP_ROUTE_TRACE
        __syncthreads();
        MP_RT_STAMP();  // 6: bases done
        if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
            printf("route_bucket(grid) blk %u: topk %llu [partials %llu, warp0 row|x| %llu, warp0 top-k %llu] exact %llu "
                   "masks %llu ranks %llu barrier %llu bases %llu ns\n",
                   blockIdx.x, tr_[1] - tr_[0], tr_coop - tr_[0], tr_row - tr_coop, tr_topk - tr_row, tr_[2] - tr_[1],
                   tr_[3] - tr_[2], tr_[4] - tr_[3], tr_[5] - tr_[4], tr_[6] - tr_[5]);
#endif
        return;
    }
    if (threadIdx.x == 0) {
        // release (acq_rel: not the heavier sequentially consistent fence)
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        if (is_last) asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire every CTA's writes
    }
    __syncthreads();
    MP_RT_STAMP();  // 5: ticket taken
#if MP_ROUTE_TRACE
    if (threadIdx.x == 0 && blockIdx.x == 0 && !is_last)
        printf("route_bucket blk %u: topk %llu exact %llu masks %llu ranks %llu ticket %llu ns (start %llu)\n",
               blockIdx.x, tr_[1] - tr_[0], tr_[2] - tr_[1], tr_[3] - tr_[2], tr_[4] - tr_[3], tr_[5] - tr_[4],
               tr_[0]);
#endif
    if (!is_last) return;  // the barrier above extends thread 0's acquire to the CTA
    // the CTA's routing smem is free now: stage the counts there when they fit
    const bool stage = (size_t)gridDim.x * G <= smem_bytes;
    bucket_scan_body(gridDim.x, G, block_counts, block_base, offsets, mprefix_tc, mprefix_simt, mprefix_tc2,
                     stage ? reinterpret_cast<uint8_t*>(rsm) : nullptr);
#if MP_ROUTE_TRACE
    __syncthreads();
    MP_RT_STAMP();  // 6: scan done
    if (threadIdx.x == 0)
        printf("route_bucket last blk %u: topk %llu exact %llu masks %llu ranks %llu ticket %llu scan %llu ns [stage "
               "%llu counts %llu scans %llu base %llu] (start %llu)\n",
               blockIdx.x, tr_[1] - tr_[0], tr_[2] - tr_[1], tr_[3] - tr_[2], tr_[4] - tr_[3], tr_[5] - tr_[4],
               tr_[6] - tr_[5], g_scan_tr[0] - tr_[5], g_scan_tr[1] - g_scan_tr[0], g_scan_tr[2] - g_scan_tr[1],
               tr_[6] - g_scan_tr[2], tr_[0]);
#endif
    if (threadIdx.x == 0) *ticket = 0;  // ready for the next forward (stream-ordered)
}

// ---------------------------------------------------------------- dispatch
// Warp per token: position of each selected slot, permutation tables, and
// the token's row copied (zero padded to d_pad) to every selected bucket.
template <typename Tx>
__global__ void __launch_bounds__(256) dispatch_kernel(const Tx* __restrict__ x, uint32_t T, uint32_t d,
                                                       uint32_t d_pad, const uint32_t* __restrict__ sel,
                                                       const float* __restrict__ w, uint32_t k_max, uint32_t G,
                                                       const uint32_t* __restrict__ lrank,
                                                       const uint32_t* __restrict__ block_base,
                                                       uint32_t* __restrict__ perm_tok, float* __restrict__ perm_w,
                                                       uint32_t* __restrict__ slot_row, Tx* __restrict__ x_perm,
                                                       int* __restrict__ err, bool check_finite, uint32_t tb) {
    const uint32_t t = blockIdx.x * 8 + threadIdx.x / 32;
    const uint32_t lane = threadIdx.x & 31;
    griddep_wait();  // every CTA waits before exiting: completion stays transitive
    griddep_launch();
    if (t >= T) return;
    const uint32_t blk = t / tb;
    for (uint32_t j = lane; j < k_max; j += 32) {
        const uint32_t g = sel[(size_t)t * k_max + j];
        uint32_t pos = kSelNone;
        if (g != kSelNone && g < G) {
            pos = block_base[(size_t)blk * G + g] + lrank[(size_t)t * k_max + j];
            perm_tok[pos] = t;
            perm_w[pos] = w ? w[(size_t)t * k_max + j] : 1.0f;
        }
        slot_row[(size_t)t * k_max + j] = pos;
    }
    __syncwarp();
    // slot positions in registers for the first 64 slots (lane j holds slots j,
    // j + 32); slots >= 64 (k_max up to E*S) are read back from slot_row
    uint32_t pos_a = lane < k_max ? slot_row[(size_t)t * k_max + lane] : kSelNone;
    uint32_t pos_b = lane + 32 < k_max ? slot_row[(size_t)t * k_max + lane + 32] : kSelNone;
    constexpr uint32_t VE = 16 / sizeof(Tx);  // elements per 16-byte vector
    const bool vec_ok = (d % VE) == 0;
    const Tx* xr = x + (size_t)t * d;
    bool bad = false;
    if (!x_perm && !check_finite) return;  // tables only: the GEMM gathers the rows itself
    // each 16-byte chunk of the row is read once and stored to every bucket;
    // U chunks per lane in flight (memory-level parallelism of the HBM-bound copy)
    constexpr uint32_t U = 4;
    for (uint32_t c0 = 0; c0 < d_pad; c0 += U * 32 * VE) {
        uint4 v[U];
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) {
            const uint32_t c = c0 + (u * 32 + lane) * VE;
            v[u] = make_uint4(0, 0, 0, 0);
            if (vec_ok) {
                if (c < d) v[u] = __ldg(reinterpret_cast<const uint4*>(xr + c));
            } else {
                Tx tmp[VE];
#pragma unroll
                for (uint32_t q = 0; q < VE; ++q) tmp[q] = (c + q < d) ? xr[c + q] : from_f32<Tx>(0.0f);
                v[u] = *reinterpret_cast<uint4*>(tmp);
            }
        }
        if (check_finite) {
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
                const Tx* tv = reinterpret_cast<const Tx*>(&v[u]);
#pragma unroll
                for (uint32_t q = 0; q < VE; ++q) bad |= !isfinite(to_f32(tv[q]));
            }
        }
        if (!x_perm) continue;
        for (uint32_t j = 0; j < k_max; ++j) {
            const uint32_t pos =
                j < 64 ? __shfl_sync(0xffffffffu, j < 32 ? pos_a : pos_b, j & 31) : slot_row[(size_t)t * k_max + j];
            if (pos == kSelNone) continue;
            Tx* dst = x_perm + (size_t)pos * d_pad;
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
                const uint32_t c = c0 + (u * 32 + lane) * VE;
                if (c < d_pad) *reinterpret_cast<uint4*>(dst + c) = v[u];
            }
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0 && err) atomicOr(err, 2);
}

// Bulk-copy dispatch (bf16, d == d_pad, rows 16-byte multiples): warp per
// token; lane 0 pulls the token's row into shared memory with one bulk copy
// and pushes it to each of its k bucket rows with k bulk stores -- the copy
// engine streams at HBM rate with no per-16-byte instructions; the warp checks
// the row for non-finite values from shared memory meanwhile.
constexpr uint32_t kBulkRowMax = 16384;  // bytes of one staged row (d <= 8192 bf16)
__global__ void __launch_bounds__(256) dispatch_bulk_kernel(const __nv_bfloat16* __restrict__ x, uint32_t T,
                                                            uint32_t d, const uint32_t* __restrict__ sel,
                                                            const float* __restrict__ w, uint32_t k_max, uint32_t G,
                                                            const uint32_t* __restrict__ lrank,
                                                            const uint32_t* __restrict__ block_base,
                                                            uint32_t* __restrict__ perm_tok,
                                                            float* __restrict__ perm_w,
                                                            uint32_t* __restrict__ slot_row,
                                                            __nv_bfloat16* __restrict__ x_perm,
                                                            int* __restrict__ err, uint32_t tb) {
    extern __shared__ __align__(128) uint8_t drow[];  // [warps][row bytes]
    __shared__ __align__(8) uint64_t bar[8];
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const uint32_t t = blockIdx.x * (blockDim.x / 32) + warp;
    const uint32_t row_bytes = d * 2;
    uint8_t* srow = drow + (size_t)warp * row_bytes;
    if (lane == 0) {
        mbar_init(&bar[warp], 1);
        fence_mbar_init();
    }
    __syncwarp();
    griddep_wait();
    griddep_launch();
    if (t >= T) return;
    if (lane == 0) {
        mbar_expect_tx(&bar[warp], row_bytes);
        bulk_load_g2s(srow, x + (size_t)t * d, row_bytes, &bar[warp]);
    }
    const uint32_t blk = t / tb;
    uint32_t pos_a = kSelNone, pos_b = kSelNone;
    for (uint32_t j = lane; j < k_max; j += 32) {
        const uint32_t g = sel[(size_t)t * k_max + j];
        uint32_t pos = kSelNone;
        if (g != kSelNone && g < G) {
            pos = block_base[(size_t)blk * G + g] + lrank[(size_t)t * k_max + j];
            perm_tok[pos] = t;
            perm_w[pos] = w ? w[(size_t)t * k_max + j] : 1.0f;
        }
        slot_row[(size_t)t * k_max + j] = pos;
        if (j < 32) pos_a = pos;
        else pos_b = pos;
    }
    mbar_wait(&bar[warp], 0);
    // lane 0 issues one bulk store per selected slot (positions via shuffles)
    for (uint32_t j = 0; j < k_max; ++j) {
        const uint32_t pos = __shfl_sync(0xffffffffu, j < 32 ? pos_a : pos_b, j & 31);
        if (pos != kSelNone && lane == 0) bulk_store_s2g(x_perm + (size_t)pos * d, srow, row_bytes);
    }
    if (lane == 0) bulk_commit();
    // non-finite scan of the staged row (the reference's check_input)
    bool bad = false;
    for (uint32_t c = lane * 8; c < d; c += 256) {
        const uint4 v = *reinterpret_cast<const uint4*>(srow + (size_t)c * 2);
        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
        for (int q = 0; q < 8; ++q) bad |= !isfinite(__bfloat162float(h[q]));
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0 && err) atomicOr(err, 2);
    // the staged row must stay until the bulk stores have read it out; their
    // global writes are visible to the next kernel at the grid boundary
    if (lane == 0) bulk_wait_read0();
    __syncwarp();
}

// ---------------------------------------------------------------- combine
// y[t] = sum_{j ascending} w[t][j] * o[slot_row[t][j]] in a fixed order
// (ascending sub-expert id), no atomics.  CTA per token.
// bf16 mode: o is bf16, fp32 accumulate, 16-byte vector loads / stores.
template <int U>
__global__ void __launch_bounds__(256, U >= 8 ? 3 : 5) combine_bf16_kernel(const __nv_bfloat16* __restrict__ o, uint32_t d,
                                                           uint32_t d_pad, const uint32_t* __restrict__ slot_row,
                                                           const float* __restrict__ w, uint32_t k_max,
                                                           const __nv_bfloat16* __restrict__ o_sh,
                                                           const float* __restrict__ w_sh,
                                                           const float* __restrict__ o_sh32, uint32_t sh_splits,
                                                           size_t sh_stride,
                                                           const __nv_bfloat16* __restrict__ x_res,
                                                           __nv_bfloat16* __restrict__ y) {
    __shared__ uint32_t rows[kMaxG];
    __shared__ float wts[kMaxG];
    const uint32_t t = blockIdx.x;
    griddep_wait();
    griddep_launch();
    // the token's selected slots, compacted in ascending slot order (the
    // summation order); warp 0, k_max <= kMaxG
    __shared__ uint32_t n_rows;
    if (threadIdx.x < 32) {
        uint32_t base = 0;
        for (uint32_t j0 = 0; j0 < k_max; j0 += 32) {
            const uint32_t j = j0 + threadIdx.x;
            const uint32_t r = j < k_max ? slot_row[(size_t)t * k_max + j] : kSelNone;
            const bool has = r != kSelNone;
            const uint32_t bal = __ballot_sync(0xffffffffu, has);
            if (has) {
                const uint32_t at = base + __popc(bal & ((1u << threadIdx.x) - 1u));
                rows[at] = r;
                wts[at] = w ? w[(size_t)t * k_max + j] : 1.0f;
            }
            base += __popc(bal);
        }
        if (threadIdx.x == 0) n_rows = base;
    }
    __syncthreads();
    __nv_bfloat16* yr = y + (size_t)t * d;
    if ((d % 8) == 0) {
        for (uint32_t c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
            float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if (x_res) {  // fused residual: y = x + MoE(x)
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(x_res + (size_t)t * d + c));
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 f = __bfloat1622float2(h[q]);
                    acc[2 * q] = f.x;
                    acc[2 * q + 1] = f.y;
                }
            }
            // U selected rows in flight per lane, then accumulated in
            // ascending slot order (one load in turn left the kernel
            // latency-bound: 16 us for a 64-token decode batch)
            const uint32_t nr = n_rows;
            for (uint32_t j0 = 0; j0 < nr; j0 += U) {
                uint4 v[U];
#pragma unroll
                for (uint32_t u = 0; u < U; ++u)
                    v[u] = j0 + u < nr ? __ldg(reinterpret_cast<const uint4*>(o + (size_t)rows[j0 + u] * d_pad + c))
                                       : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
                for (uint32_t u = 0; u < U; ++u) {
                    if (j0 + u >= nr) break;
                    const float wj = wts[j0 + u];
                    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float2 f = __bfloat1622float2(h[q]);
                        acc[2 * q] = fmaf(wj, f.x, acc[2 * q]);
                        acc[2 * q + 1] = fmaf(wj, f.y, acc[2 * q + 1]);
                    }
                }
            }
            if (o_sh32) {  // shared expert from split-K fp32 partials, summed in split order
                float sum[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                constexpr uint32_t SU = U >= 8 ? 6 : 2;  // splits in flight
                for (uint32_t sp0 = 0; sp0 < sh_splits; sp0 += SU) {
                    float4 a[SU], b[SU];
#pragma unroll
                    for (uint32_t u = 0; u < SU; ++u) {
                        const float* pr = o_sh32 + (sp0 + u) * sh_stride + (size_t)t * d_pad + c;
                        const bool ok = sp0 + u < sh_splits;
                        a[u] = ok ? __ldg(reinterpret_cast<const float4*>(pr)) : make_float4(0.f, 0.f, 0.f, 0.f);
                        b[u] = ok ? __ldg(reinterpret_cast<const float4*>(pr + 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (uint32_t u = 0; u < SU; ++u) {
                        if (sp0 + u >= sh_splits) break;
                        sum[0] += a[u].x, sum[1] += a[u].y, sum[2] += a[u].z, sum[3] += a[u].w;
                        sum[4] += b[u].x, sum[5] += b[u].y, sum[6] += b[u].z, sum[7] += b[u].w;
                    }
                }
                const float ws = w_sh[t];
#pragma unroll
                for (int q = 0; q < 8; ++q) acc[q] = fmaf(ws, sum[q], acc[q]);
            } else if (o_sh) {  // shared expert last (its ids follow the routed ones)
                const float ws = w_sh[t];
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(o_sh + (size_t)t * d_pad + c));
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 f = __bfloat1622float2(h[q]);
                    acc[2 * q] = fmaf(ws, f.x, acc[2 * q]);
                    acc[2 * q + 1] = fmaf(ws, f.y, acc[2 * q + 1]);
                }
            }
            uint4 out;
            out.x = pack_bf16x2(acc[0], acc[1]);
            out.y = pack_bf16x2(acc[2], acc[3]);
            out.z = pack_bf16x2(acc[4], acc[5]);
            out.w = pack_bf16x2(acc[6], acc[7]);
            *reinterpret_cast<uint4*>(yr + c) = out;
        }
    } else {
        for (uint32_t c = threadIdx.x; c < d; c += blockDim.x) {
            float acc = x_res ? __bfloat162float(x_res[(size_t)t * d + c]) : 0.0f;
            for (uint32_t j = 0; j < n_rows; ++j) acc = fmaf(wts[j], __bfloat162float(o[(size_t)rows[j] * d_pad + c]), acc);
            if (o_sh32) {
                float sum = 0.0f;
                for (uint32_t sp = 0; sp < sh_splits; ++sp) sum += o_sh32[sp * sh_stride + (size_t)t * d_pad + c];
                acc = fmaf(w_sh[t], sum, acc);
            } else if (o_sh) {
                acc = fmaf(w_sh[t], __bfloat162float(o_sh[(size_t)t * d_pad + c]), acc);
            }
            yr[c] = __float2bfloat16_rn(acc);
        }
    }
}

// fp32 (reference-exact) mode: o holds each sub-expert's output in double; the
// reference rounds partitioned_forward to float per call (inc/expert.hpp:133),
// so: weighted mode rounds per sub-expert then sums w * float(o) in double;
// unit mode (group_S > 0) sums the selected sub-experts of one parent expert
// in double and rounds once per expert (one reference call per expert).
__global__ void __launch_bounds__(256) combine_f64_kernel(const double* __restrict__ o, uint32_t d, uint32_t d_pad,
                                                          const uint32_t* __restrict__ slot_row,
                                                          const uint32_t* __restrict__ sel,
                                                          const float* __restrict__ w, uint32_t k_max,
                                                          uint32_t group_S, float* __restrict__ y) {
    __shared__ uint32_t rows[kMaxG];
    __shared__ uint32_t gid[kMaxG];
    __shared__ float wts[kMaxG];
    const uint32_t t = blockIdx.x;
    griddep_wait();
    griddep_launch();
    for (uint32_t j = threadIdx.x; j < k_max; j += blockDim.x) {
        rows[j] = slot_row[(size_t)t * k_max + j];
        gid[j] = sel[(size_t)t * k_max + j];
        wts[j] = w ? w[(size_t)t * k_max + j] : 1.0f;
    }
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < d; c += blockDim.x) {
        double acc = 0.0, part = 0.0;
        uint32_t cur = kSelNone;
        for (uint32_t j = 0; j < k_max; ++j) {
            const uint32_t r = rows[j];
            if (r == kSelNone) continue;
            const double v = o[(size_t)r * d_pad + c];
            if (group_S) {
                const uint32_t e = gid[j] / group_S;
                if (e != cur && cur != kSelNone) {
                    acc += static_cast<double>(static_cast<float>(part));
                    part = 0.0;
                }
                cur = e;
                part += v;
            } else {
                acc += static_cast<double>(wts[j]) * static_cast<double>(static_cast<float>(v));
            }
        }
        if (group_S && cur != kSelNone) acc += static_cast<double>(static_cast<float>(part));
        y[(size_t)t * d + c] = static_cast<float>(acc);
    }
}

}  // namespace

// ---------------------------------------------------------------- launchers

void launch_router_linear(int dtype, const void* x, uint32_t T, uint32_t d, const float* wrT, uint32_t G,
                          uint32_t k_max, const uint32_t* kpt, uint32_t k, int weight_mode, uint32_t* sel, float* w,
                          int* err, uint32_t* stats, cudaStream_t s) {
    const size_t smem = sizeof(double) * TB * G + sizeof(float) * (KC * (TB + 1) + KC * (GB + 4));
    const dim3 grid((T + TB - 1) / TB);
    if (dtype == 1) {
        auto kern = router_linear_kernel<__nv_bfloat16>;
        func_attr_once(reinterpret_cast<const void*>(kern), (int)(sizeof(double) * TB * kMaxG + 16 * 1024));
        kern<<<grid, kRouterThreads, smem, s>>>(static_cast<const __nv_bfloat16*>(x), T, d, wrT, G, k_max, kpt, k,
                                                weight_mode, sel, w, err, stats);
    } else {
        auto kern = router_linear_kernel<float>;
        func_attr_once(reinterpret_cast<const void*>(kern), (int)(sizeof(double) * TB * kMaxG + 16 * 1024));
        kern<<<grid, kRouterThreads, smem, s>>>(static_cast<const float*>(x), T, d, wrT, G, k_max, kpt, k,
                                                weight_mode, sel, w, err, stats);
    }
}

void launch_partials_topk(const double* partial, uint32_t ks, uint32_t T, uint32_t G, uint32_t Npad, uint32_t k_max,
                          const uint32_t* kpt, uint32_t k, int weight_mode, uint32_t* sel, float* w, int* err,
                          const RouterGuard& rg, const void* x, uint32_t d, uint32_t* flagged, cudaStream_t s) {
    partials_topk_kernel<<<(T + 7) / 8, 256, 0, s>>>(partial, ks, T, G, Npad, k_max, kpt, k, weight_mode, sel, w,
                                                     err, rg, static_cast<const __nv_bfloat16*>(x), d, flagged);
}

// In-place fixed-order reduction of the K-split router partials into plane 0
// (ascending split order, the same sum route_bucket_kernel forms): for small
// batches the splits are many (64-deep chunks) and the tokens few, so the
// reduction is spread over (token, 32 sub-experts) warps instead of one warp
// per token.
__global__ void __launch_bounds__(256) partials_reduce_kernel(double* __restrict__ partial, uint32_t ks, uint32_t T,
                                                              uint32_t G, uint32_t Npad) {
    const uint32_t gw = (G + 31) / 32;
    const uint32_t wid = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
    griddep_wait();
    griddep_launch();
    if (wid >= T * gw) return;
    const uint32_t t = wid / gw, g = (wid % gw) * 32 + lane;
    if (g >= G) return;
    double v = 0.0;
    for (uint32_t s = 0; s < ks; ++s) v += partial[((size_t)s * T + t) * Npad + g];
    partial[(size_t)t * Npad + g] = v;
}

void launch_partials_reduce(double* partial, uint32_t ks, uint32_t T, uint32_t G, uint32_t Npad, cudaStream_t s) {
    const uint32_t warps = T * ((G + 31) / 32);
    launch_k(partials_reduce_kernel, dim3((warps + 7) / 8), dim3(256), 0, s, partial, ks, T, G, Npad);
}

bool launch_route_bucket(const double* partial, uint32_t ks, uint32_t T, uint32_t G, uint32_t Npad, uint32_t k_max,
                         const uint32_t* kpt, uint32_t k, int weight_mode, uint32_t* sel, float* w,
                         const RouterGuard& rg, const void* x, uint32_t d, const float* wrT, uint32_t* ticket,
                         uint32_t* stats, BucketWs& ws, cudaStream_t s, uint32_t tb, int num_sms, bool tables) {
    // the routing arrays, or the last CTA's staged counts (1 byte per block and
    // bucket) when they are larger and fit
    const size_t nblk = (T + tb - 1) / tb;
    // one 1024-thread CTA per SM: a persistent grid of <= SMs CTAs (each
    // taking every gridDim-th token block) is on the GPU at once, can
    // synchronise (grid barrier) and form its bucket bases in parallel; the
    // last-CTA scan (MOEPRISM_GRID_SCAN=0) took 23-28 us at Qwen prefill
    // (256 blocks x 240 buckets, profiles/r02e_route_trace.txt)
    static const bool grid_env = [] {  // MOEPRISM_GRID_SCAN=0: last-CTA scans only (A/B)
        const char* e = std::getenv("MOEPRISM_GRID_SCAN");
        return !(e && e[0] == '0');
    }();
    const bool grid_scan = grid_env;
    const size_t grid = grid_scan ? std::min<size_t>(nblk, static_cast<size_t>(num_sms)) : nblk;
    size_t smem = sizeof(double) * 2 * tb * G;
    if (nblk * G > smem && nblk * G <= 160 * 1024) smem = (nblk * G + 15) & ~size_t(15);
    auto launch = [&](auto kern) {
        // same shared-memory carveout as the GEMMs around it: no L1/smem
        // reconfiguration between the kernels of the chain
        func_attr_once(reinterpret_cast<const void*>(kern), (int)std::max<size_t>(sizeof(double) * 2 * TB * kMaxG,
                                                                                  160 * 1024), true);
        launch_k(kern, dim3(static_cast<uint32_t>(grid)), dim3(1024), smem, s,
            partial, ks, T, G, Npad, k_max, kpt, k, weight_mode, sel, w, ws.err, rg,
            static_cast<const __nv_bfloat16*>(x), d, wrT, ticket, stats, ws.lrank, ws.block_counts, ws.block_base,
            ws.offsets, ws.mprefix_tc, ws.mprefix_simt, ws.mprefix_tc2, tb, static_cast<uint32_t>(smem),
            grid_scan ? 1u : 0u, (tables && grid_scan) ? ws.perm_tok : nullptr, ws.perm_w, ws.slot_row);
    };
    if (G <= 64)
        launch(route_bucket_kernel<2>);
    else if (G <= 128)
        launch(route_bucket_kernel<4>);
    else
        launch(route_bucket_kernel<8>);
    return tables && grid_scan;
}

void launch_router_fixup(int dtype, const void* x, uint32_t d, const float* wrT, uint32_t G, uint32_t k_max,
                         const uint32_t* kpt, uint32_t k, int weight_mode, uint32_t* sel, float* w, int* err,
                         uint32_t* flagged, int num_sms, cudaStream_t s) {
    const size_t smem = sizeof(double) * d;
    func_attr_once(reinterpret_cast<const void*>(router_fixup_kernel<__nv_bfloat16>), 200 * 1024);
    func_attr_once(reinterpret_cast<const void*>(router_fixup_kernel<float>), 200 * 1024);
    if (dtype == 1)
        router_fixup_kernel<__nv_bfloat16><<<num_sms, 1024, smem, s>>>(static_cast<const __nv_bfloat16*>(x), d, wrT,
                                                                      G, k_max, kpt, k, weight_mode, sel, w, err,
                                                                      flagged);
    else
        router_fixup_kernel<float><<<num_sms, 1024, smem, s>>>(static_cast<const float*>(x), d, wrT, G, k_max, kpt, k,
                                                              weight_mode, sel, w, err, flagged);
}

void launch_router_scores_topk(const float* scores, uint32_t T, uint32_t G, uint32_t k_max, const uint32_t* kpt,
                               uint32_t k, int weight_mode, uint32_t* sel, float* w, int* err, uint32_t* stats,
                               cudaStream_t s) {
    scores_topk_kernel<<<(T + 7) / 8, 256, 0, s>>>(reinterpret_cast<const double*>(scores), T, G, k_max, kpt, k,
                                                   weight_mode, sel, w, err, stats);
}

void launch_bucket_local(const uint32_t* sel, uint32_t T, uint32_t k_max, uint32_t G, BucketWs& ws,
                         cudaStream_t s) {
    bucket_local_kernel<<<(T + TB - 1) / TB, 256, 0, s>>>(sel, T, k_max, G, ws.lrank, ws.block_counts, ws.err);
}

void launch_bucket_scan(uint32_t T, uint32_t G, BucketWs& ws, cudaStream_t s) {
    bucket_scan_kernel<<<1, 1024, 0, s>>>((T + TB - 1) / TB, G, ws.block_counts, ws.block_base, ws.offsets,
                                          ws.mprefix_tc, ws.mprefix_simt, ws.mprefix_tc2);
}

void launch_dispatch(int dtype, const void* x, uint32_t T, uint32_t d, uint32_t d_pad, const uint32_t* sel,
                     const float* w, uint32_t k_max, uint32_t G, BucketWs& ws, void* x_perm, cudaStream_t s,
                     bool check_finite, uint32_t tb) {
    static const bool bulk_env = [] {  // MOEPRISM_DISPATCH=vector: the 16-byte vector kernel (A/B)
        const char* e = std::getenv("MOEPRISM_DISPATCH");
        return !(e && std::string(e) == "vector");
    }();
    if (dtype == 1 && x_perm && d == d_pad && (d % 8) == 0 && d * 2 <= kBulkRowMax && bulk_env &&
        (reinterpret_cast<uintptr_t>(x) % 16) == 0) {
        // warps (staged rows) per CTA.  Measured (ncu, Mixtral T=4096, medians
        // of 5): 3 -> 50.6 / 90.8 us at k=8 / 16, 4 -> 57.7 / 94.7, 2 -> 53.4 /
        // 93.2, 1 -> 54.0 / 94.4 (9 CTAs x 3 rows of 8 KB per SM)
        static const uint32_t wpc = [] {
            const char* e = std::getenv("MOEPRISM_DISPATCH_WARPS");
            const int v = e ? std::atoi(e) : 3;
            return static_cast<uint32_t>(v < 1 ? 1 : v > 8 ? 8 : v);
        }();
        const size_t smem = wpc * (size_t)d * 2;
        func_attr_once(reinterpret_cast<const void*>(dispatch_bulk_kernel), (int)(8 * kBulkRowMax), true);
        launch_k(dispatch_bulk_kernel, dim3((T + wpc - 1) / wpc), dim3(32 * wpc), smem, s,
            static_cast<const __nv_bfloat16*>(x), T, d, sel, w, k_max, G, ws.lrank, ws.block_base, ws.perm_tok,
            ws.perm_w, ws.slot_row, static_cast<__nv_bfloat16*>(x_perm), check_finite ? ws.err : nullptr, tb);
        return;
    }
    const dim3 grid((T + 7) / 8);
    if (dtype == 1)
        launch_k(dispatch_kernel<__nv_bfloat16>, grid, dim3(256), 0, s,
            static_cast<const __nv_bfloat16*>(x), T, d, d_pad, sel, w, k_max, G, ws.lrank, ws.block_base,
            ws.perm_tok, ws.perm_w, ws.slot_row, static_cast<__nv_bfloat16*>(x_perm), ws.err, check_finite, tb);
    else
        launch_k(dispatch_kernel<float>, grid, dim3(256), 0, s, static_cast<const float*>(x), T, d, d_pad, sel, w, k_max, G,
                                                    ws.lrank, ws.block_base, ws.perm_tok, ws.perm_w, ws.slot_row,
                                                    static_cast<float*>(x_perm), ws.err, check_finite, tb);
}

// Shared expert gate (Qwen-style): w_sh[t] = sigmoid(x_t . gate)
// (1 when gate is null), warp per token, fixed-order fp32 reduction; block 0
// also writes the one-group offsets {0, T} and 128-row tile prefix of the
// shared expert's grouped GEMMs.
__global__ void __launch_bounds__(256) shared_gate_kernel(const __nv_bfloat16* __restrict__ x, uint32_t T, uint32_t d,
                                                          const float* __restrict__ gate, float* __restrict__ w_sh,
                                                          uint32_t* __restrict__ sh_off,
                                                          uint32_t* __restrict__ sh_mprefix) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        sh_off[0] = 0;
        sh_off[1] = T;
        sh_mprefix[0] = 0;
        sh_mprefix[1] = (T + kTcBM - 1) / kTcBM;
        sh_mprefix[2] = 0;  // 256-row (CTA pair) tiles
        sh_mprefix[3] = (T + 255) / 256;
    }
    const uint32_t t = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x & 31;
    if (t >= T) return;
    if (!gate) {
        if (lane == 0) w_sh[t] = 1.0f;
        return;
    }
    const __nv_bfloat16* xr = x + (size_t)t * d;
    float acc = 0.0f;
    if ((d % 8) == 0) {  // 16-byte loads of x, all of a lane's loads in flight
        for (uint32_t c = lane * 8; c < d; c += 256) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(xr + c));
            const float4 g0 = __ldg(reinterpret_cast<const float4*>(gate + c));
            const float4 g1 = __ldg(reinterpret_cast<const float4*>(gate + c + 4));
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
            const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
            const float2 e = __bfloat1622float2(h[2]), f = __bfloat1622float2(h[3]);
            acc = fmaf(a.x, g0.x, acc);
            acc = fmaf(a.y, g0.y, acc);
            acc = fmaf(b.x, g0.z, acc);
            acc = fmaf(b.y, g0.w, acc);
            acc = fmaf(e.x, g1.x, acc);
            acc = fmaf(e.y, g1.y, acc);
            acc = fmaf(f.x, g1.z, acc);
            acc = fmaf(f.y, g1.w, acc);
        }
    } else {
        for (uint32_t c = lane; c < d; c += 32) acc = fmaf(__bfloat162float(xr[c]), gate[c], acc);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) w_sh[t] = 1.0f / (1.0f + expf(-acc));
}

void launch_shared_gate(const void* x, uint32_t T, uint32_t d, const float* gate, float* w_sh, uint32_t* sh_off,
                        uint32_t* sh_mprefix, cudaStream_t s) {
    shared_gate_kernel<<<(T + 7) / 8, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x), T, d, gate, w_sh, sh_off,
                                                   sh_mprefix);
}

void launch_combine(int dtype, const void* o, uint32_t d, uint32_t d_pad, const uint32_t* slot_row,
                    const uint32_t* sel, const float* w, uint32_t k_max, uint32_t group_S, uint32_t T, void* y,
                    cudaStream_t s, const void* o_sh, const float* w_sh, const void* x_res, uint32_t sh_splits,
                    size_t sh_stride, uint32_t k_hint, int num_sms) {
    // sh_splits > 0: o_sh holds fp32 split-K partials [sh_splits][stride]
    const float* o_sh32 = sh_splits ? static_cast<const float*>(o_sh) : nullptr;
    // rows in flight per lane: many tokens (CTAs) hide the load latency by
    // occupancy, few (decode) need it per lane; measured (mixtral_quick /
    // qwen_quick): U = 8 cut a 64-token combine 16 -> 10 us but slowed
    // 4096-token k <= 4 batches (registers -> fewer resident CTAs)
    const uint32_t kh = k_hint ? k_hint : k_max;
    const int U = (T <= 4u * (uint32_t)num_sms || kh >= 12) ? 8 : kh >= 6 ? 4 : 2;
    auto go = [&](auto kern) {
        launch_k(kern, dim3(T), dim3(256), 0, s, static_cast<const __nv_bfloat16*>(o), d, d_pad, slot_row, w, k_max,
                 sh_splits ? nullptr : static_cast<const __nv_bfloat16*>(o_sh), w_sh, o_sh32, sh_splits, sh_stride,
                 static_cast<const __nv_bfloat16*>(x_res), static_cast<__nv_bfloat16*>(y));
    };
    if (dtype == 1) {
        if (U == 8)
            go(combine_bf16_kernel<8>);
        else if (U == 4)
            go(combine_bf16_kernel<4>);
        else
            go(combine_bf16_kernel<2>);
    }
    if (dtype != 1)
        combine_f64_kernel<<<T, 256, 0, s>>>(static_cast<const double*>(o), d, d_pad, slot_row, sel, w, k_max, group_S,
                                             static_cast<float*>(y));
}

}  // namespace mp
