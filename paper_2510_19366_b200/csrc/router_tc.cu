// router_tc.cu -- the linear router on the tensor cores, accurate enough for
// bit-exact routing (SURVEY 7 hard part 2: the near-tie window is 1e-6 in
// logit, so 1xTF32 / plain bf16 is far too coarse).
//
// x is bf16 (exact).  W_r (fp32) is split into three bf16 planes
// W = hi + mid + lo (8+8+8 mantissa bits: exact up to the last bit of fp32), so
// every product x * plane is exact in the MMA and
//     logits = x.hi + x.mid + x.lo
// differs from the fp64 oracle only by the accumulation rounding (the MMA adds
// into fp32).  Every 256-deep K chunk (64-deep for few token tiles) gets its
// own fresh TMEM accumulators (one for the hi plane, one for mid+lo) and the
// chunk sums are added in fp64 in the epilogue, so the error of a logit is at
// most depth * 2^-23 * sum_i |x_i| |W_ig| (every fp32 addition inside a
// chunk, however the MMA orders them, loses at most one ulp of a running sum
// bounded by the chunk's sum of |products|; 2^-23 also covers truncation).
// The consumers form that bound per token (route.cu warp_router_guard, with
// sum_i |x_i| from the bf16 row), and -- because a bound is not bit-exactness --
// every token whose k-th/(k+1)-th gap is within twice its bound is re-selected
// from exact fp64 logits (route.cu route_bucket_kernel / router_fixup_kernel):
// the selection is certified for every token, at any input scale.
// K is further split across CTAs (grid = token tiles x K splits ~ 148 CTAs);
// the per-split fp64 partials are added in a fixed order by the top-k kernel
// (deterministic, no atomics).  Warp roles and pipelines as in gemm_tc.cu.
#include "mp_common.cuh"
#include "mp_kernels.h"

namespace mp {

namespace {

constexpr uint32_t BM = 128, BK = 64, kChunkKb = 4;  // 256-deep chunks (64-deep for few token tiles)
constexpr uint32_t kThreads = 192;
constexpr uint32_t kMaxStages = 6;

struct RouterTcParams {
    uint32_t T, Npad, kb_total, kb_per_split, stages, chunk_kb;
    uint32_t ncta, nsplit;  // columns per CTA, column splits (blockIdx.y = K split * nsplit + column split)
    void* partial;          // [KS][T][Npad] fp64, or fp32 when out_f32 (rounded once per split)
    uint32_t out_f32;
};

__global__ void __launch_bounds__(kThreads, 1)
    router_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                     RouterTcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t a_bytes = BM * BK * 2;
    const uint32_t plane_bytes = p.ncta * BK * 2;
    const uint32_t ksplit = blockIdx.y / p.nsplit, n0 = (blockIdx.y % p.nsplit) * p.ncta;
    const uint32_t stage_bytes = a_bytes + 3 * plane_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(base + p.stages * stage_bytes);
    uint64_t* empty = full + kMaxStages;
    uint64_t* tfull = empty + kMaxStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t m0 = blockIdx.x * BM;
    const uint32_t kb0 = ksplit * p.kb_per_split;
    const uint32_t kb1 = min(kb0 + p.kb_per_split, p.kb_total);

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmX);
        tma_prefetch_desc(&tmW);
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    griddep_wait();
    griddep_launch();

    if (warp == 0) {
        if (lane == 0) {
            for (uint32_t kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
                const uint32_t s = it % p.stages, ph = (it / p.stages) & 1u;
                mbar_wait(&empty[s], ph ^ 1u);
                mbar_expect_tx(&full[s], stage_bytes);
                uint8_t* st = base + s * stage_bytes;
                tma_load_2d(st, &tmX, &full[s], static_cast<int32_t>(kb * BK), static_cast<int32_t>(m0));
                for (uint32_t q = 0; q < 3; ++q)
                    tma_load_2d(st + a_bytes + q * plane_bytes, &tmW, &full[s], static_cast<int32_t>(kb * BK),
                                static_cast<int32_t>(q * p.Npad + n0));
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = umma_idesc_bf16(BM, p.ncta);
            for (uint32_t kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
                const uint32_t s = it % p.stages, ph = (it / p.stages) & 1u;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t chunk = (kb - kb0) / p.chunk_kb;
                const bool first = ((kb - kb0) % p.chunk_kb) == 0;
                // hi plane and (mid + lo) planes in separate accumulators: the
                // small planes never round at the hi accumulator's ulp
                const uint32_t d_hi = tmem_base + chunk * 2 * p.ncta;
                const uint32_t d_ml = d_hi + p.ncta;
                const uint32_t a0 = smem_u32(base + s * stage_bytes);
#pragma unroll
                for (uint32_t k = 0; k < BK / 16; ++k) {
                    const uint64_t ad = umma_desc_sw128(a0 + k * 32);
                    umma_bf16(d_hi, ad, umma_desc_sw128(a0 + a_bytes + k * 32), idesc, !(first && k == 0));
                    umma_bf16(d_ml, ad, umma_desc_sw128(a0 + a_bytes + plane_bytes + k * 32), idesc,
                              !(first && k == 0));
                    umma_bf16(d_ml, ad, umma_desc_sw128(a0 + a_bytes + 2 * plane_bytes + k * 32), idesc, 1u);
                }
                umma_commit(&empty[s]);
            }
            umma_commit(tfull);
        }
        __syncwarp();
    } else {
        const uint32_t q = warp & 3u;
        mbar_wait(tfull, 0);
        tc_fence_after();
        const uint32_t t = m0 + q * 32 + lane;
        const uint32_t nchunks = (kb1 - kb0 + p.chunk_kb - 1) / p.chunk_kb;
        const size_t orow = (static_cast<size_t>(ksplit) * p.T + t) * p.Npad + n0;
        for (uint32_t grp = 0; grp < p.ncta / 32 && n0 + grp * 32 < p.Npad; ++grp) {
            double acc[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = 0.0;
            for (uint32_t c = 0; c < nchunks; ++c) {
                uint32_t rh[32], rl[32];
                const uint32_t col = tmem_base + ((q * 32u) << 16) + c * 2 * p.ncta + grp * 32;
                tmem_ld32(col, rh);
                tmem_ld32(col + p.ncta, rl);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    acc[i] += static_cast<double>(__uint_as_float(rh[i])) + static_cast<double>(__uint_as_float(rl[i]));
            }
            if (t < p.T && p.out_f32) {
                float* out = static_cast<float*>(p.partial) + orow + grp * 32;
#pragma unroll
                for (int i = 0; i < 32; i += 4)
                    *reinterpret_cast<float4*>(out + i) = make_float4(static_cast<float>(acc[i]), static_cast<float>(acc[i + 1]),
                                                                      static_cast<float>(acc[i + 2]), static_cast<float>(acc[i + 3]));
            } else if (t < p.T) {
                double* out = static_cast<double*>(p.partial) + orow + grp * 32;
#pragma unroll
                for (int i = 0; i < 32; i += 2)
                    *reinterpret_cast<double2*>(out + i) = make_double2(acc[i], acc[i + 1]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

// W_r (d x G row-major fp32) -> three bf16 planes [3][Npad][d] (K-major).
__global__ void split_router_kernel(const float* __restrict__ wr, uint32_t d, uint32_t G, uint32_t Npad,
                                    __nv_bfloat16* __restrict__ planes) {
    const size_t n = static_cast<size_t>(Npad) * d;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
        const uint32_t g = q / d, i = q % d;
        const float w = g < G ? wr[static_cast<size_t>(i) * G + g] : 0.0f;
        const __nv_bfloat16 hi = __float2bfloat16_rn(w);
        const float r1 = w - __bfloat162float(hi);  // exact
        const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
        const float r2 = r1 - __bfloat162float(mid);  // exact
        const __nv_bfloat16 lo = __float2bfloat16_rn(r2);
        planes[q] = hi;
        planes[n + q] = mid;
        planes[2 * n + q] = lo;
    }
}

// Two fp32 row blocks ([n_a][d] then [n_b][d], row-major) -> three bf16 planes
// [3][Npad][d]: the proxy router's gate and up columns of its gate neurons.
__global__ void split_rows_kernel(const float* __restrict__ ra, const float* __restrict__ rb, uint32_t n_a,
                                  uint32_t n_b, uint32_t d, uint32_t Npad, __nv_bfloat16* __restrict__ planes) {
    const size_t n = static_cast<size_t>(Npad) * d;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
        const uint32_t g = q / d, i = q % d;
        const float w = g < n_a ? ra[q] : (g < n_a + n_b ? rb[static_cast<size_t>(g - n_a) * d + i] : 0.0f);
        const __nv_bfloat16 hi = __float2bfloat16_rn(w);
        const float r1 = w - __bfloat162float(hi);
        const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
        const float r2 = r1 - __bfloat162float(mid);
        planes[q] = hi;
        planes[n + q] = mid;
        planes[2 * n + q] = __float2bfloat16_rn(r2);
    }
}

}  // namespace

void launch_split_rows(const float* ra, const float* rb, uint32_t n_a, uint32_t n_b, uint32_t d, uint32_t Npad,
                       void* planes, cudaStream_t s) {
    split_rows_kernel<<<592, 256, 0, s>>>(ra, rb, n_a, n_b, d, Npad, static_cast<__nv_bfloat16*>(planes));
}

size_t router_tc_partial_rows(uint32_t max_T, uint32_t d, uint32_t G, int num_sms) {
    size_t best = 0;
    for (uint32_t m = 1; (m - 1) * BM < max_T; ++m) {
        const uint32_t T = m * BM < max_T ? m * BM : max_T;
        const RouterTcPlan pl = plan_router_tc(T, d, G, num_sms);
        const size_t rows = static_cast<size_t>(pl.ks) * T;
        if (rows > best) best = rows;
    }
    return best;
}

// chunk depth x 2^-23 per unit of sum|x| max|W|, times 1.02 for the mid/lo
// accumulator (2 x depth additions of terms <= 2^-8 |x W|) and the fp32 |x|
// sums (relative error < 2^-16), and max|hi| <= max|W| (1 + 2^-9).
double router_guard_coef(uint32_t chunk_depth, float wmax) {
    return static_cast<double>(chunk_depth) * 0x1.0p-23 * 1.02 * static_cast<double>(wmax);
}

uint32_t router_tc_cols_per_cta(uint32_t G) {
    const uint32_t npad = ((G + 31) / 32) * 32;
    const uint32_t nsplit = (npad + 127) / 128;
    return ((npad / nsplit + 31) / 32) * 32;
}

RouterTcPlan plan_router_tc(uint32_t T, uint32_t d, uint32_t G, int num_sms) {
    RouterTcPlan pl{};
    pl.Npad = ((G + 31) / 32) * 32;
    // > 128 sub-experts (Qwen: 240): columns split over CTAs, so a stage of
    // the three weight planes stays <= 48 KB (3 stages instead of 1) and two
    // 256-deep chunks fit in TMEM (half the K splits and partials)
    pl.ncta = router_tc_cols_per_cta(G);
    pl.nsplit = (pl.Npad + pl.ncta - 1) / pl.ncta;
    pl.kb_total = (d + BK - 1) / BK;
    const uint32_t m_tiles = (T + BM - 1) / BM;
    const uint32_t mn_tiles = m_tiles * pl.nsplit;
    // few token tiles (decode): 64-deep chunks give 4x the K splits (CTAs),
    // cutting the per-CTA operand stream that bounds small-batch latency
    pl.chunk_kb = mn_tiles * ((pl.kb_total + kChunkKb - 1) / kChunkKb) < static_cast<uint32_t>(num_sms) / 2 ? 1
                                                                                                           : kChunkKb;
    const uint32_t n_chunks = (pl.kb_total + pl.chunk_kb - 1) / pl.chunk_kb;
    const uint32_t max_chunks_per_cta = 512 / (2 * pl.ncta);
    uint32_t ks = (static_cast<uint32_t>(num_sms) + mn_tiles - 1) / mn_tiles;
    ks = ks < 1 ? 1 : ks;
    ks = ks > n_chunks ? n_chunks : ks;
    const uint32_t ks_min = (n_chunks + max_chunks_per_cta - 1) / max_chunks_per_cta;
    if (ks < ks_min) ks = ks_min;
    const uint32_t chunks_per_split = (n_chunks + ks - 1) / ks;
    pl.kb_per_split = chunks_per_split * pl.chunk_kb;
    pl.ks = (pl.kb_total + pl.kb_per_split - 1) / pl.kb_per_split;
    pl.m_tiles = m_tiles;
    const uint32_t stage_bytes = BM * BK * 2 + 3 * pl.ncta * BK * 2;
    uint32_t stages = (200u * 1024u) / stage_bytes;
    pl.stages = stages > kMaxStages ? kMaxStages : stages;
    pl.smem = 1024 + pl.stages * stage_bytes + 256;
    return pl;
}

void launch_split_router(const float* wr, uint32_t d, uint32_t G, uint32_t Npad, void* planes, cudaStream_t s) {
    split_router_kernel<<<592, 256, 0, s>>>(wr, d, G, Npad, static_cast<__nv_bfloat16*>(planes));
}

void launch_router_tc(const CUtensorMap* tmX, const CUtensorMap* tmW, const RouterTcPlan& pl, uint32_t T,
                      void* partial, cudaStream_t s, bool out_f32) {
    RouterTcParams p{T,       pl.Npad,   pl.kb_total, pl.kb_per_split, pl.stages, pl.chunk_kb, pl.ncta, pl.nsplit,
                     partial, out_f32 ? 1u : 0u};
    func_attr_once(reinterpret_cast<const void*>(router_tc_kernel), 227 * 1024);
    launch_k(router_tc_kernel, dim3(pl.m_tiles, pl.ks * pl.nsplit), dim3(kThreads), pl.smem, s, *tmX, *tmW, p);
}

}  // namespace mp
