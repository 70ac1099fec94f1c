// gemm_tc2.cu -- grouped GEMM with 256-row tiles on one SM: two M=128
// tcgen05 accumulators (rows 0-127 / 128-255 of the tile, TMEM columns
// [0,256) / [256,512)) share every 256-wide B k-slice.  Operand bytes per MMA
// cycle drop by a third versus 128x256 tiles (A 32 KB + B 32 KB feed 1024
// MMA cycles per 64-deep k-block), so the 3-stage smem ring covers 3072
// cycles of TMA latency instead of 2048 -- the ring-depth sweep showed the
// 128-row kernel is latency-limited.  The price: TMEM holds one tile, so the
// epilogue (8 warps, one per 32 rows x accumulator) is not overlapped with
// the next tile's MMAs.  Tiles whose last rows fit in 128 issue only the first
// accumulator's MMAs, so the M-tail waste stays at 128-row granularity.
// Same data layout, tile order and epilogues as gemm_tc.cu.
#include "mp_common.cuh"
#include "mp_kernels.h"

namespace mp {

namespace {

constexpr uint32_t BM = 256, HM = 128, BN = 256, BK = 64, STAGES = 3;
constexpr uint32_t A_BYTES = BM * BK * 2, AH_BYTES = HM * BK * 2, B_BYTES = BN * BK * 2;
constexpr uint32_t kThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue
constexpr size_t kSmemBytes = 1024 + STAGES * (A_BYTES + B_BYTES) + 256;

struct Tc2Params {
    uint32_t G, K, N_group, n_valid, ld_out, NT;
    const uint32_t* offsets;
    const uint32_t* mprefix;  // prefix of ceil(count_g / 256)
    __nv_bfloat16* out;
};

__device__ __forceinline__ void map_tile(uint32_t tile, const uint32_t* s_prefix, uint32_t G, uint32_t NT,
                                         uint32_t& g, uint32_t& m, uint32_t& n) {
    uint32_t lo = 0, hi = G;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_prefix[mid] * NT <= tile)
            lo = mid + 1;
        else
            hi = mid;
    }
    g = lo - 1;
    const uint32_t local = tile - s_prefix[g] * NT;
    const uint32_t mt = s_prefix[g + 1] - s_prefix[g];
    n = local / mt;
    m = local - n * mt;
}

template <bool SWIGLU>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Tc2Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint32_t s_prefix[kMaxG + 1];
    __shared__ uint32_t s_off[kMaxG + 1];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = base;
    uint8_t* sB = base + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 256);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    for (uint32_t q = threadIdx.x; q <= p.G; q += kThreads) {
        s_prefix[q] = p.mprefix[q];
        s_off[q] = p.offsets[q];
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t total = s_prefix[p.G] * p.NT;
    const uint32_t nkb = p.K / BK;

    if (warp == 0) {
        if (lane == 0) {
            uint32_t it = 0;
            for (uint32_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
                uint32_t g, m, n;
                map_tile(tile, s_prefix, p.G, p.NT, g, m, n);
                const uint32_t rows = min(BM, s_off[g + 1] - s_off[g] - m * BM);
                const bool two = rows > HM;
                const int32_t arow = static_cast<int32_t>(s_off[g] + m * BM);
                const int32_t brow = static_cast<int32_t>(g * p.N_group + n * BN);
                for (uint32_t kb = 0; kb < nkb; ++kb, ++it) {
                    const uint32_t s = it % STAGES, ph = (it / STAGES) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    mbar_expect_tx(&full[s], (two ? 2 : 1) * AH_BYTES + B_BYTES);
                    uint8_t* a = sA + s * A_BYTES;
                    tma_load_2d(a, &tmA, &full[s], static_cast<int32_t>(kb * BK), arow);
                    if (two) tma_load_2d(a + AH_BYTES, &tmA, &full[s], static_cast<int32_t>(kb * BK), arow + HM);
                    tma_load_2d(sB + s * B_BYTES, &tmB, &full[s], static_cast<int32_t>(kb * BK), brow);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(HM, BN);
            uint32_t it = 0, tc = 0;
            for (uint32_t tile = blockIdx.x; tile < total; tile += gridDim.x, ++tc) {
                uint32_t g, m, n;
                map_tile(tile, s_prefix, p.G, p.NT, g, m, n);
                const bool two = min(BM, s_off[g + 1] - s_off[g] - m * BM) > HM;
                mbar_wait(tempty, (tc & 1u) ^ 1u);
                tc_fence_after();
                for (uint32_t kb = 0; kb < nkb; ++kb, ++it) {
                    const uint32_t s = it % STAGES, ph = (it / STAGES) & 1u;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + s * A_BYTES);
                    const uint32_t b0 = smem_u32(sB + s * B_BYTES);
#pragma unroll
                    for (uint32_t k = 0; k < BK / 16; ++k) {
                        const uint64_t bd = umma_desc_sw128(b0 + k * 32);
                        umma_bf16(tmem_base, umma_desc_sw128(a0 + k * 32), bd, idesc, (kb | k) != 0u);
                        if (two)
                            umma_bf16(tmem_base + BN, umma_desc_sw128(a0 + AH_BYTES + k * 32), bd, idesc,
                                      (kb | k) != 0u);
                    }
                    umma_commit(&empty[s]);
                }
                umma_commit(tfull);
            }
        }
        __syncwarp();
    } else {
        const uint32_t q = warp & 3u;          // TMEM lane quarter
        const uint32_t h = (warp - 2) >> 2;    // accumulator (tile half)
        uint32_t tc = 0;
        for (uint32_t tile = blockIdx.x; tile < total; tile += gridDim.x, ++tc) {
            uint32_t g, m, n;
            map_tile(tile, s_prefix, p.G, p.NT, g, m, n);
            const uint32_t cnt = s_off[g + 1] - s_off[g];
            const bool two = min(BM, cnt - m * BM) > HM;
            mbar_wait(tfull, tc & 1u);
            tc_fence_after();
            if (h == 0 || two) {
                const uint32_t row_local = m * BM + h * HM + q * 32 + lane;
                const bool valid = row_local < cnt;
                __nv_bfloat16* orow = p.out + static_cast<size_t>(s_off[g] + row_local) * p.ld_out;
                const uint32_t taddr = tmem_base + ((q * 32u) << 16) + h * BN;
                if constexpr (SWIGLU) {
#pragma unroll 1
                    for (uint32_t c = 0; c < 4; ++c) {
                        uint32_t gr[32], ur[32];
                        tmem_ld32(taddr + c * 32, gr);
                        tmem_ld32(taddr + 128 + c * 32, ur);
                        tmem_ld_wait();
                        uint32_t pk[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const float g0 = __uint_as_float(gr[2 * i]), g1 = __uint_as_float(gr[2 * i + 1]);
                            const float u0 = __uint_as_float(ur[2 * i]), u1 = __uint_as_float(ur[2 * i + 1]);
                            pk[i] = pack_bf16x2(silu_f32(g0) * u0, silu_f32(g1) * u1);
                        }
                        if (valid) {
                            __nv_bfloat16* dst = orow + n * 128 + c * 32;
#pragma unroll
                            for (int v = 0; v < 4; ++v)
                                st_global_v4(dst + v * 8,
                                             make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]));
                        }
                    }
                } else {
#pragma unroll 1
                    for (uint32_t c = 0; c < BN / 32; ++c) {
                        uint32_t r[32];
                        tmem_ld32(taddr + c * 32, r);
                        tmem_ld_wait();
                        const uint32_t col = n * BN + c * 32;
                        if (valid && col < p.n_valid) {
                            uint32_t pk[16];
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                pk[i] = pack_bf16x2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
                            __nv_bfloat16* dst = orow + col;
#pragma unroll
                            for (int v = 0; v < 4; ++v)
                                st_global_v4(dst + v * 8,
                                             make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]));
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(tempty);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

}  // namespace

void launch_gemm_tc2(bool swiglu, const CUtensorMap* tmA, const CUtensorMap* tmB, void* out, const GemmShape& sh,
                     const uint32_t* offsets, const uint32_t* mprefix256, int num_sms, cudaStream_t s) {
    Tc2Params p{sh.G, sh.K, sh.N_group, sh.n_valid, sh.ld_out, (sh.N_group + BN - 1) / BN, offsets, mprefix256,
                static_cast<__nv_bfloat16*>(out)};
    const uint32_t max_tiles = (sh.max_rows / BM + sh.G) * p.NT;
    const uint32_t grid = max_tiles < (uint32_t)num_sms ? max_tiles : (uint32_t)num_sms;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(gemm_tc2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
        cudaFuncSetAttribute(gemm_tc2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
        attr_set = true;
    }
    if (swiglu)
        gemm_tc2_kernel<true><<<grid, kThreads, kSmemBytes, s>>>(*tmA, *tmB, p);
    else
        gemm_tc2_kernel<false><<<grid, kThreads, kSmemBytes, s>>>(*tmA, *tmB, p);
}

}  // namespace mp
