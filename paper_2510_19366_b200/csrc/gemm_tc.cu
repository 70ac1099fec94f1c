// gemm_tc.cu -- grouped GEMMs of the sub-expert SwiGLU FFN on the 5th-gen
// tensor cores (tcgen05.mma, accumulators in TMEM, operands staged by TMA).
//
//   gemm1 (SWIGLU=true):  H[r][n*128 + h*64 + c] = silu(acc[r][h*128 + c]) * acc[r][h*128 + 64 + c]
//       A = x_perm (rows x d_pad), B = W1[g] rows n*256 .. n*256+255
//       (blocks of 64 gate rows then the 64 up rows of the same neurons,
//       packed by pack.cu, kIlv), so one 128x256 TMEM accumulator holds both
//       halves of the SwiGLU for 128 neurons and the activation is fused in
//       the epilogue.
//   gemm2 (SWIGLU=false): O[r][n*256 + c] = acc[r][c]
//   calibration epilogues (kEpiActAbs, kEpiCount): see TcParams.
//       A = H (rows x w_pad), B = W2[g] (d_pad x w_pad).
// Variable-size groups: sub-expert g owns rows [offsets[g], offsets[g+1])
// (written by the bucket scan on the device); tiles are enumerated (g, n, m)
// from the device prefix of ceil(count_g / 128) by a persistent grid of one
// CTA per SM, m fastest so the CTAs sharing one weight tile run together and
// the tile is fetched from HBM once.  Rows of a partial M tile that belong to
// the next group are computed and discarded (masked stores).
//
// Warp roles (192 threads): warp 0 = TMA producer (one lane), warp 1 = TMEM
// allocator + MMA issuer (one lane), warps 2..5 = epilogue (TMEM lane quarter
// = warp % 4).  Operand rings: A and B have SEPARATE smem rings (NA x 16 KB,
// NB x 32 KB), each slot refilled the moment the MMAs reading it complete.
// Measured with the MMA-issuer trace (MOEPRISM_TC_TRACE,
// tests/probes/gemm_trace.py + ring_ab.sh): split 4+4 rings take 6% fewer
// cycles than one 4 x 48 KB ring; 3+5, 4+3, 3+4 are 9-17% slower, 5+4 equal
// -- both operands stream from HBM/L2 and need >= 4 k-blocks of lookahead.
// 2 TMEM accumulators of 256 columns (tmem_full / tmem_empty) let the
// epilogue of tile i overlap the MMAs of tile i+1.
// Measured and dropped (tests/probes, profiles/r01_mma_cost.csv): swapped
// tail tiles (D^T = W . X^T with N = rows rounded to 16: slower, k=8 gemm1
// 0.98 -> 1.21 ms), two N=128 MMAs per k-step (slower: A is read from smem
// twice), two K-interleaved accumulator chains (MMA issue at the floor, but
// the epilogue is exposed).  The limiter of this kernel is the operand feed
// (48 KB of A+B per SM per k-block); gemm_tc2.cu (CTA pairs) halves B.
#include <cstdio>
#include <cstdlib>

#include "mp_common.cuh"
#include "mp_kernels.h"

#ifndef MP_TC_NA
#define MP_TC_NA 4
#endif
#ifndef MP_TC_NB
#define MP_TC_NB 4
#endif

namespace mp {

namespace {

constexpr uint32_t BM = kTcBM;  // 128
constexpr uint32_t BN = 256;
#ifndef MP_TC_KSUB
// 64-deep TMA sub-blocks per pipeline stage.  2 (with MP_TC_NA=2 MP_TC_NB=2)
// measured slower: 2 stages expose the load latency (profiles/r02ag_1sm_kblock128_ab.txt).
// The shared expert's decode split count (layer.cu) assumes 64-deep k-blocks.
#define MP_TC_KSUB 1
#endif
constexpr uint32_t KSUB = MP_TC_KSUB;
constexpr uint32_t BK = 64 * KSUB;  // k-block depth: KSUB 128-byte swizzle rows of bf16
constexpr uint32_t NA = MP_TC_NA, NB = MP_TC_NB;

constexpr uint32_t A_BYTES = BM * BK * 2;
constexpr uint32_t B_BYTES = BN * BK * 2;
constexpr uint32_t SUBA = BM * 64 * 2;  // one 64-deep sub-block of the A / B stage
constexpr uint32_t SUBB = BN * 64 * 2;
constexpr uint32_t kThreads = 192;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kEpiStage = 32 * 32 * 2;  // one 32-row x 32-column bf16 box of a warp's output slab
constexpr size_t kSmemBytes = 1024 + NA * A_BYTES + NB * B_BYTES + 256 + 4 * 2 * kEpiStage;
constexpr uint32_t kTileCache = 256;  // decoded tiles per CTA kept in shared memory

struct TcParams {
    uint32_t G, K, N_group, n_valid, ld_out, NT;
    const uint32_t* offsets;
    const uint32_t* mprefix;
    __nv_bfloat16* out;
    uint64_t* trace;  // [grid][4] MMA-issuer timing (diagnostics) or null
    uint32_t b_row0;  // first B row (calibration: one expert of the packed W1)
    const uint32_t* gmap;  // nullable: B group of group g (sub-expert offload cache slot), else g
    const uint32_t* starts;  // nullable: group g's rows are [starts[g], offsets[g+1]) (split-schedule tails)
    // kEpiActAbs: fp32 |SwiGLU| of packed neuron q to column colmap[q] (< 0: padding)
    // kEpiCount:  uint32(acc) (exact 0/1 co-activation counts)
    const int32_t* colmap;
    void* out32;
    // split-K (kEpiF32Part): K is cut into ksplit ranges of kps k-blocks; the
    // tile of split s writes its fp32 partial to out32 + s * split_stride
    uint32_t ksplit, kps;
    size_t split_stride;
    uint32_t small_a;  // the short-box A maps are valid
    uint32_t tma_out;  // plain epilogue: tmO is valid (full warp slabs leave through TMA stores)
    // gemm1 B tail (0: off): valid neurons per group; the 64-neuron blocks
    // past them are not loaded, the partial one through b_tail_rows-row boxes
    // (tmBt) -- the padding rows of the packed W1 never leave HBM.  Their smem
    // rows hold stale data, so the matching h columns are garbage: gemm2 reads
    // h and W2 through maps whose K extent stops at the valid neurons.
    uint32_t b_valid, b_tail_rows;
    // gemm1 A gather (nullable): token id of every permuted row; A rows are
    // then gathered from the token matrix x (tmA: box {64 cols, 1 row}) by
    // TMA gather4 -- no materialised x_perm (dispatch writes tables only)
    const uint32_t* gather_tok;
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

// (tile, k-block) cursor of one operand stream of a CTA
struct Cursor {
    uint32_t tile, kb, kb1;  // current k-block, end of the tile's k range
    uint32_t n;              // N tile
    int32_t row;             // A row (arow) or B row (brow) of the current tile
    uint32_t rows;           // A: valid rows of the tile (<= BM)
    uint32_t i;              // index of the tile among this CTA's tiles
};

// tmA16 / tmA32 / tmA64: the A operand with 16- / 32- / 64-row boxes.  A tile
// with at most that many valid rows (decode batches: a few rows per
// sub-expert) loads only those rows; the rest of the 128-row slot keeps stale
// rows whose outputs are discarded (masked stores), so the L2 -> SM feed
// carries the weight tile and little else.  SW128 swizzle repeats every 8
// rows, so a short box lands exactly like the first rows of a full one.
template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmA16, const __grid_constant__ CUtensorMap tmA32,
                   const __grid_constant__ CUtensorMap tmA64, const __grid_constant__ CUtensorMap tmO,
                   const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBt, TcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint32_t s_prefix[kMaxG + 1];
    __shared__ uint32_t s_off[kMaxG + 1];
    __shared__ uint32_t s_gmap[kMaxG];
    __shared__ uint32_t s_start[kMaxG];
    // this CTA's tiles decoded once (g | n << 8 | split << 20, m): the
    // binary search + divisions of map_tile were ~13% of the warp samples of
    // short-K GEMMs (Qwen's K = 384 down projection, ncu source page)
    __shared__ uint2 s_tiles[kTileCache];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sB = base;                 // NB x 32 KB (1024-aligned)
    uint8_t* sA = base + NB * B_BYTES;  // NA x 16 KB
    uint64_t* fullA = reinterpret_cast<uint64_t*>(sA + NA * A_BYTES);
    uint64_t* emptyA = fullA + NA;
    uint64_t* fullB = emptyA + NA;
    uint64_t* emptyB = fullB + NB;
    uint64_t* tfull = emptyB + NB;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    // plain-epilogue staging: 2 boxes per epilogue warp (after the barriers)
    uint8_t* sEpi = reinterpret_cast<uint8_t*>(reinterpret_cast<uintptr_t>(sA + NA * A_BYTES + 256 + 127) & ~uintptr_t(127));

    const uint32_t warp = threadIdx.x / 32;
    const uint32_t lane = threadIdx.x % 32;

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < NA; ++s) {
            mbar_init(&fullA[s], 1);
            mbar_init(&emptyA[s], 1);
        }
        for (uint32_t s = 0; s < NB; ++s) {
            mbar_init(&fullB[s], 1);
            mbar_init(&emptyB[s], 1);
        }
        for (uint32_t a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 128);
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        if (p.tma_out) tma_prefetch_desc(&tmO);
        if (p.b_valid) {
            tma_prefetch_desc(&tmBh);
            tma_prefetch_desc(&tmBt);
        }
        if (p.small_a) {
            tma_prefetch_desc(&tmA16);
            tma_prefetch_desc(&tmA32);
            tma_prefetch_desc(&tmA64);
        }
    }
    if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
    griddep_wait();  // group metadata comes from the routing epilogue
    griddep_launch();
    for (uint32_t q = threadIdx.x; q <= p.G; q += blockDim.x) {
        s_prefix[q] = p.mprefix[q];
        s_off[q] = p.offsets[q];
        if (q < p.G) s_gmap[q] = p.gmap ? p.gmap[q] : q;
        if (q < p.G) s_start[q] = p.starts ? p.starts[q] : p.offsets[q];
    }
    __syncthreads();
    const uint32_t base_total = s_prefix[p.G] * p.NT;
    const uint32_t total = base_total * p.ksplit;
    const uint32_t nkb = (p.K + BK - 1) / BK;  // a partial last k-block is zero-filled by the TMA
    // balanced rounds: with R = ceil(total / grid) tiles per CTA, only
    // ceil(total / R) CTAs take tiles, every one exactly R or R - 1 (no last
    // round on a fraction of the SMs: Qwen decode gemm1, 630 tiles, 106.5 ->
    // 102 us on 126 instead of 148 CTAs under ncu)
    const uint32_t per_cta = (total + gridDim.x - 1) / gridDim.x;
    const uint32_t nact = per_cta ? (total + per_cta - 1) / per_cta : gridDim.x;
    const uint32_t first = blockIdx.x < nact ? blockIdx.x : total;  // idle CTAs start past the end
    for (uint32_t i = threadIdx.x; i < kTileCache; i += blockDim.x) {
        const uint32_t tile = first + i * nact;
        if (tile >= total) break;
        uint32_t g, m, n;
        const uint32_t split = tile / base_total;
        map_tile(tile - split * base_total, s_prefix, p.G, p.NT, g, m, n);
        s_tiles[i] = make_uint2(g | (n << 8) | (split << 20), m);
    }
    // (tile index of this CTA, i) -> g, m, n, split
    auto decode = [&](uint32_t tile, uint32_t i, uint32_t& g, uint32_t& m, uint32_t& n, uint32_t& split) {
        if (i < kTileCache) {
            const uint2 v = s_tiles[i];
            g = v.x & 0xFFu;
            n = (v.x >> 8) & 0xFFFu;
            split = v.x >> 20;
            m = v.y;
        } else {
            split = tile / base_total;
            map_tile(tile - split * base_total, s_prefix, p.G, p.NT, g, m, n);
        }
    };
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // one B stage: the 256-row weight tile, or (gemm1 B tail) its valid blocks
    auto load_b = [&](uint32_t s, uint32_t ph, uint32_t kb, int32_t row, uint32_t n) {
        mbar_wait(&emptyB[s], ph ^ 1u);
        const uint32_t nb = n * 2;  // first 64-neuron block of the tile (128 rows: gate, up)
        if (!p.b_valid || p.b_valid >= (nb + 2) * 64) {
            mbar_expect_tx(&fullB[s], B_BYTES);
            for (uint32_t sb = 0; sb < KSUB; ++sb)
                tma_load_2d(sB + s * B_BYTES + sb * SUBB, &tmB, &fullB[s], static_cast<int32_t>(kb * BK + sb * 64), row);
        } else {
            uint32_t v[2], bytes = 0;
#pragma unroll
            for (uint32_t hb = 0; hb < 2; ++hb) {
                const uint32_t lo = (nb + hb) * 64;
                v[hb] = p.b_valid > lo ? min(64u, p.b_valid - lo) : 0u;
                bytes += v[hb] == 64 ? 128 * 64 * 2 : v[hb] ? 2 * p.b_tail_rows * 64 * 2 : 0;
            }
            mbar_expect_tx(&fullB[s], bytes * KSUB);
            for (uint32_t sb = 0; sb < KSUB; ++sb) {
                const int32_t kc = static_cast<int32_t>(kb * BK + sb * 64);
#pragma unroll
                for (uint32_t hb = 0; hb < 2; ++hb) {
                    uint8_t* dst = sB + s * B_BYTES + sb * SUBB + hb * (128 * 64 * 2);
                    const int32_t r = row + static_cast<int32_t>(hb * 128);
                    if (v[hb] == 64) {
                        tma_load_2d(dst, &tmBh, &fullB[s], kc, r);
                    } else if (v[hb]) {  // gate rows, then the up rows of the same neurons
                        tma_load_2d(dst, &tmBt, &fullB[s], kc, r);
                        tma_load_2d(dst + kIlv * 64 * 2, &tmBt, &fullB[s], kc, r + static_cast<int32_t>(kIlv));
                    }
                }
            }
        }
    };
    if (warp == 0 && p.gather_tok) {
        // Gather producer: the whole warp.  Lane 0 streams B and arms the A
        // barriers; for A, lane q gathers rows 4q..4q+3 of the tile with one
        // TMA gather4 per k-block (token ids of the tile held in registers).
        int32_t tok[4] = {0, 0, 0, 0};
        auto set_rows = [&](Cursor& c, bool is_a) {
            if (c.tile >= total) return;
            uint32_t g, m, n, split;
            decode(c.tile, c.i, g, m, n, split);
            c.row = is_a ? static_cast<int32_t>(s_start[g] + m * BM)
                         : static_cast<int32_t>(p.b_row0 + s_gmap[g] * p.N_group + n * BN);
            c.rows = min(BM, s_off[g + 1] - s_start[g] - m * BM);
            c.n = n;
            c.kb = split * p.kps;
            c.kb1 = min(nkb, c.kb + p.kps);
            if (is_a) {
                const uint32_t first = __ldg(p.gather_tok + c.row);  // padding rows repeat a valid token
#pragma unroll
                for (uint32_t r = 0; r < 4; ++r) {
                    const uint32_t rr = lane * 4 + r;
                    tok[r] = static_cast<int32_t>(rr < c.rows ? __ldg(p.gather_tok + c.row + rr) : first);
                }
            }
        };
        auto advance = [&](Cursor& c, bool is_a) {
            if (++c.kb == c.kb1) {
                c.tile += nact;
                ++c.i;
                set_rows(c, is_a);
            }
        };
        Cursor cb{first, 0, 0, 0, 0, 0, 0}, ca{first, 0, 0, 0, 0, 0, 0};
        set_rows(cb, false);
        set_rows(ca, true);
        uint32_t ib = 0, ia = 0;
        while (cb.tile < total || ca.tile < total) {
            if (cb.tile < total) {
                if (lane == 0) load_b(ib % NB, (ib / NB) & 1u, cb.kb, cb.row, cb.n);
                advance(cb, false);
                ++ib;
            }
            if (ca.tile < total && (ib >= ia + (NB - NA) || cb.tile >= total)) {
                const uint32_t s = ia % NA, ph = (ia / NA) & 1u;
                const uint32_t ng = (ca.rows + 3) / 4;
                if (lane == 0) {
                    mbar_wait(&emptyA[s], ph ^ 1u);
                    mbar_expect_tx(&fullA[s], ng * 4 * BK * 2);  // KSUB sub-blocks of ng x 4 rows
                }
                __syncwarp();
                if (lane < ng)
                    for (uint32_t sb = 0; sb < KSUB; ++sb)
                        tma_gather4(sA + s * A_BYTES + sb * SUBA + lane * (4 * 64 * 2), &tmA, &fullA[s],
                                    static_cast<int32_t>(ca.kb * BK + sb * 64), tok);
                advance(ca, true);
                ++ia;
            }
        }
    } else if (warp == 0) {
        if (lane == 0) {
            // one ordered issue stream: B(j) then A(j - (NB - NA)), each behind
            // its own empty barrier
            auto set_rows = [&](Cursor& c, bool is_a) {
                if (c.tile >= total) return;
                uint32_t g, m, n, split;
                decode(c.tile, c.i, g, m, n, split);
                c.row = is_a ? static_cast<int32_t>(s_start[g] + m * BM)
                             : static_cast<int32_t>(p.b_row0 + s_gmap[g] * p.N_group + n * BN);
                c.rows = min(BM, s_off[g + 1] - s_start[g] - m * BM);
                c.n = n;
                c.kb = split * p.kps;
                c.kb1 = min(nkb, c.kb + p.kps);
            };
            auto advance = [&](Cursor& c, bool is_a) {
                if (++c.kb == c.kb1) {
                    c.tile += nact;
                    ++c.i;
                    set_rows(c, is_a);
                }
            };
            Cursor cb{first, 0, 0, 0, 0, 0, 0}, ca{first, 0, 0, 0, 0, 0, 0};
            set_rows(cb, false);
            set_rows(ca, true);
            uint32_t ib = 0, ia = 0;  // loads issued per stream
            auto issue_b = [&]() {
                load_b(ib % NB, (ib / NB) & 1u, cb.kb, cb.row, cb.n);
                advance(cb, false);
                ++ib;
            };
            auto issue_a = [&]() {
                const uint32_t s = ia % NA, ph = (ia / NA) & 1u;
                mbar_wait(&emptyA[s], ph ^ 1u);
                const uint32_t box = !p.small_a ? BM : ca.rows <= 16 ? 16u : ca.rows <= 32 ? 32u : ca.rows <= 64 ? 64u : BM;
                const CUtensorMap* tA = box == 16 ? &tmA16 : box == 32 ? &tmA32 : box == 64 ? &tmA64 : &tmA;
                mbar_expect_tx(&fullA[s], box * BK * 2);
                for (uint32_t sb = 0; sb < KSUB; ++sb)
                    tma_load_2d(sA + s * A_BYTES + sb * SUBA, tA, &fullA[s], static_cast<int32_t>(ca.kb * BK + sb * 64),
                                ca.row);
                advance(ca, true);
                ++ia;
            };
            // the deeper ring's stream runs |NA - NB| loads ahead of the other
            // one; each load waits only for its own slot to drain
            while (cb.tile < total || ca.tile < total) {
                if (NB >= NA) {
                    if (cb.tile < total) issue_b();
                    if (ca.tile < total && ib >= ia + (NB - NA)) issue_a();
                    else if (cb.tile >= total && ca.tile < total) issue_a();
                } else {
                    if (ca.tile < total) issue_a();
                    if (cb.tile < total && ia >= ib + (NA - NB)) issue_b();
                    else if (ca.tile >= total && cb.tile < total) issue_b();
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
            uint32_t it = 0, tc = 0;
            // optional timing trace (MOEPRISM_TC_TRACE): cycles the MMA issuer
            // waits for accumulators (epilogue) and for operand stages (loads)
            const uint64_t t_start = p.trace ? clock64() : 0;
            uint64_t w_acc = 0, w_full = 0;
            for (uint32_t tile = first; tile < total; tile += nact, ++tc) {
                const uint32_t acc = tc & 1u, aph = (tc >> 1) & 1u;
                uint64_t t0 = p.trace ? clock64() : 0;
                mbar_wait(&tempty[acc], aph ^ 1u);
                if (p.trace) w_acc += clock64() - t0;
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                const uint32_t kb_lo = (p.ksplit > 1 ? tile / base_total : 0u) * p.kps, kb_hi = min(nkb, kb_lo + p.kps);
                for (uint32_t kb = kb_lo; kb < kb_hi; ++kb, ++it) {
                    const uint32_t sa = it % NA, pa = (it / NA) & 1u;
                    const uint32_t sb = it % NB, pb = (it / NB) & 1u;
                    t0 = p.trace ? clock64() : 0;
                    mbar_wait(&fullB[sb], pb);
                    mbar_wait(&fullA[sa], pa);
                    if (p.trace) w_full += clock64() - t0;
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + sa * A_BYTES);
                    const uint32_t b0 = smem_u32(sB + sb * B_BYTES);
#pragma unroll
                    for (uint32_t k = 0; k < BK / 16; ++k)
                        umma_bf16(d_tmem, umma_desc_sw128(a0 + (k >> 2) * SUBA + (k & 3u) * 32),
                                  umma_desc_sw128(b0 + (k >> 2) * SUBB + (k & 3u) * 32), idesc,
                                  (kb != kb_lo || k != 0) ? 1u : 0u);
                    umma_commit(&emptyA[sa]);
                    umma_commit(&emptyB[sb]);
                }
                umma_commit(&tfull[acc]);
            }
            if (p.trace) {
                uint64_t* tr = p.trace + blockIdx.x * 4;
                tr[0] = clock64() - t_start;
                tr[1] = w_acc;
                tr[2] = w_full;
                tr[3] = tc;
            }
        }
        __syncwarp();
    } else {
        const uint32_t q = warp & 3u;  // TMEM lane quarter this warp may access
        uint32_t tc = 0;
        uint32_t epi_it = 0;  // TMA-stored chunks of this warp (staging buffer parity)
        for (uint32_t tile = first; tile < total; tile += nact, ++tc) {
            uint32_t g, m, n, split;
            decode(tile, tc, g, m, n, split);
            const uint32_t acc = tc & 1u, aph = (tc >> 1) & 1u;
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            const uint32_t row_local = m * BM + q * 32 + lane;
            const bool valid = row_local < s_off[g + 1] - s_start[g];
            __nv_bfloat16* orow = p.out + static_cast<size_t>(s_start[g] + row_local) * p.ld_out;
            const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * BN;
            if constexpr (EPI == kEpiActAbs) {
                // calibration profiler: |a| in the original neuron order
                float* arow = static_cast<float*>(p.out32) + static_cast<size_t>(s_start[g] + row_local) * p.ld_out;
#pragma unroll 1
                for (uint32_t c = 0; c < 4; ++c) {
                    const uint32_t gcol = (c >> 1) * 128 + (c & 1u) * 32;
                    uint32_t gr[32], ur[32];
                    tmem_ld32(taddr + gcol, gr);
                    tmem_ld32(taddr + gcol + kIlv, ur);
                    tmem_ld_wait();
                    if (valid) {
                        const int32_t* cm = p.colmap + n * 128 + c * 32;
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const int32_t j = __ldg(cm + i);
                            if (j >= 0) arow[j] = fabsf(silu_f32(__uint_as_float(gr[i])) * __uint_as_float(ur[i]));
                        }
                    }
                }
            } else if constexpr (EPI == kEpiF32Part) {
                // split-K partial: fp32, 16-byte stores; the consumer sums the splits in order
                float* prow = static_cast<float*>(p.out32) + split * p.split_stride +
                              static_cast<size_t>(s_start[g] + row_local) * p.ld_out;
#pragma unroll 1
                for (uint32_t c = 0; c < BN / 32; ++c) {
                    uint32_t r[32];
                    tmem_ld32(taddr + c * 32, r);
                    tmem_ld_wait();
                    const uint32_t col = n * BN + c * 32;
                    if (valid && col < p.n_valid) {
#pragma unroll
                        for (int i = 0; i < 32; i += 4)
                            st_global_v4(prow + col + i, make_uint4(r[i], r[i + 1], r[i + 2], r[i + 3]));
                    }
                }
            } else if constexpr (EPI == kEpiCount) {
                uint32_t* crow = static_cast<uint32_t*>(p.out32) + static_cast<size_t>(s_start[g] + row_local) * p.ld_out;
#pragma unroll 1
                for (uint32_t c = 0; c < BN / 32; ++c) {
                    uint32_t r[32];
                    tmem_ld32(taddr + c * 32, r);
                    tmem_ld_wait();
                    const uint32_t col = n * BN + c * 32;
                    if (valid && col < p.n_valid) {
#pragma unroll
                        for (int i = 0; i < 32; i += 4) {
                            if (col + i + 3 < p.n_valid && (p.ld_out & 3u) == 0) {
                                st_global_v4(crow + col + i,
                                             make_uint4(__float2uint_rn(__uint_as_float(r[i])),
                                                        __float2uint_rn(__uint_as_float(r[i + 1])),
                                                        __float2uint_rn(__uint_as_float(r[i + 2])),
                                                        __float2uint_rn(__uint_as_float(r[i + 3]))));
                            } else {
                                for (int u = 0; u < 4; ++u)
                                    if (col + i + u < p.n_valid) crow[col + i + u] = __float2uint_rn(__uint_as_float(r[i + u]));
                            }
                        }
                    }
                }
            } else if constexpr (EPI == kEpiSwiglu) {
#pragma unroll 1
                for (uint32_t c = 0; c < 4; ++c) {
                    // neurons n*128 + c*32 .. +31: gate columns (c/2)*128 + (c%2)*32, up + 64
                    const uint32_t gcol = (c >> 1) * 128 + (c & 1u) * 32;
                    uint32_t gr[32], ur[32];
                    tmem_ld32(taddr + gcol, gr);
                    tmem_ld32(taddr + gcol + kIlv, ur);
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
                            st_global_v4(dst + v * 8, make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]));
                    }
                }
            } else {
                // two register sets: the TMEM load of chunk c + 1 is in flight
                // while chunk c is converted and stored (short-K GEMMs, e.g.
                // Qwen's K = 384 down projection, are epilogue-bound).
                // A warp whose 32 rows are all valid stages each 32 x 32 chunk
                // in shared memory and writes it with one TMA store (2 KB of
                // whole 64-byte row segments) instead of 4 vector stores per
                // lane that each touch 32 rows; ragged slabs store directly.
                const bool slab = p.tma_out && m * BM + q * 32 + 32 <= s_off[g + 1] - s_start[g];
                const int32_t slab_row = static_cast<int32_t>(s_start[g] + m * BM + q * 32);
                auto store = [&](uint32_t c, const uint32_t* r) {
                    const uint32_t col = n * BN + c * 32;
                    if (col >= p.n_valid) return;
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        pk[i] = pack_bf16x2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
                    if (slab) {
                        uint8_t* buf = sEpi + (q * 2 + (epi_it & 1u)) * kEpiStage;
                        if (epi_it >= 2) {  // the store issued from this buffer two chunks ago has read it
                            if (lane == 0) bulk_wait_read<1>();
                            __syncwarp();
                        }
                        uint4* dst = reinterpret_cast<uint4*>(buf + lane * 64);
#pragma unroll
                        for (int v = 0; v < 4; ++v) dst[v] = make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_2d(&tmO, buf, static_cast<int32_t>(col), slab_row);
                            bulk_commit();
                        }
                        ++epi_it;
                    } else if (valid) {
                        __nv_bfloat16* dst = orow + col;
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            st_global_v4(dst + v * 8, make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]));
                    }
                };
                uint32_t ra[32], rb[32];
                tmem_ld32(taddr, ra);
                tmem_ld_wait();
#pragma unroll 1
                for (uint32_t c = 0; c < BN / 32; c += 2) {
                    tmem_ld32(taddr + (c + 1) * 32, rb);
                    store(c, ra);
                    tmem_ld_wait();
                    if (c + 2 < BN / 32) tmem_ld32(taddr + (c + 2) * 32, ra);
                    store(c + 1, rb);
                    tmem_ld_wait();
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
        }
        if (epi_it && lane == 0) bulk_wait0();  // the TMA stores are complete before the CTA retires
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem_base);
    }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
    return fn;
}

uint64_t* g_trace[2] = {nullptr, nullptr};

}  // namespace

size_t gemm_tc_smem_bytes() { return kSmemBytes; }

// MOEPRISM_TC_TRACE=1: per-CTA MMA-issuer timing of the last gemm1 / gemm2
// launch, readable with mp_debug_gemm_trace (diagnostics only).
uint64_t* gemm_trace_buffer(bool swiglu) {
    static const bool on = [] {
        const char* e = std::getenv("MOEPRISM_TC_TRACE");
        return e && e[0] == '1';
    }();
    if (!on) return nullptr;
    uint64_t*& b = g_trace[swiglu ? 0 : 1];
    if (!b) cudaMalloc(&b, (4096 + 128 * 128 * 4) * sizeof(uint64_t));  // + per-tile records (pair kernel)
    return b;
}
uint64_t* gemm_trace_ptr(int which) { return g_trace[which & 1]; }

bool make_tmap_bf16_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                       uint32_t box_cols) {
    return make_tmap_bf16_2d_ex(m, base, rows, cols, cols, box_rows, box_cols, true);
}

bool make_tmap_bf16_2d_ex(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t pitch,
                          uint32_t box_rows, uint32_t box_cols, bool swizzle128, uint32_t l2_promo) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    const cuuint64_t gdim[2] = {cols, rows};
    const cuuint64_t gstride[1] = {pitch * 2};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estride[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride, box, estride,
               CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
               l2_promo == 0    ? CU_TENSOR_MAP_L2_PROMOTION_NONE
               : l2_promo == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
               : l2_promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                 : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void launch_gemm_tc(bool swiglu, const CUtensorMap* tmA, const CUtensorMap* tmB, void* out, const GemmShape& sh,
                    const uint32_t* offsets, const uint32_t* mprefix, int num_sms, cudaStream_t s,
                    const uint32_t* gmap, const uint32_t* starts, const CUtensorMap* tmA_small,
                    const CUtensorMap* tmO, const GemmBTail* btail, const uint32_t* gather_tok) {
    launch_gemm_tc_epi(swiglu ? kEpiSwiglu : kEpiPlain, tmA, tmB, out, sh, offsets, mprefix, num_sms, s, 0, nullptr,
                       gmap, starts, 1, tmA_small, tmO, btail, gather_tok);
}

void launch_gemm_tc_epi(int epi, const CUtensorMap* tmA, const CUtensorMap* tmB, void* out, const GemmShape& sh,
                        const uint32_t* offsets, const uint32_t* mprefix, int num_sms, cudaStream_t s,
                        uint32_t b_row0, const int32_t* colmap, const uint32_t* gmap, const uint32_t* starts,
                        uint32_t ksplit, const CUtensorMap* tmA_small, const CUtensorMap* tmO,
                        const GemmBTail* btail, const uint32_t* gather_tok) {
    const bool swiglu = epi == kEpiSwiglu;
    TcParams p;
    p.G = sh.G;
    p.K = sh.K;
    p.N_group = sh.N_group;
    p.n_valid = sh.n_valid;
    p.ld_out = sh.ld_out;
    p.NT = (sh.N_group + BN - 1) / BN;
    p.offsets = offsets;
    p.mprefix = mprefix;
    p.out = static_cast<__nv_bfloat16*>(out);
    p.trace = (epi == kEpiSwiglu || epi == kEpiPlain) ? gemm_trace_buffer(swiglu) : nullptr;
    p.b_row0 = b_row0;
    p.gmap = gmap;
    p.starts = starts;
    p.colmap = colmap;
    p.out32 = out;
    const uint32_t nkb = (sh.K + BK - 1) / BK;
    p.ksplit = epi == kEpiF32Part ? (ksplit < 1 ? 1u : ksplit > nkb ? nkb : ksplit) : 1u;
    p.kps = (nkb + p.ksplit - 1) / p.ksplit;
    p.ksplit = (nkb + p.kps - 1) / p.kps;  // no empty splits
    p.split_stride = static_cast<size_t>(sh.max_rows) * sh.ld_out;
    p.small_a = tmA_small ? 1u : 0u;
    const CUtensorMap& a16 = tmA_small ? tmA_small[0] : *tmA;
    const CUtensorMap& a32 = tmA_small ? tmA_small[1] : *tmA;
    const CUtensorMap& a64 = tmA_small ? tmA_small[2] : *tmA;
    static const bool epi_tma = [] {  // MOEPRISM_EPI_TMA=0: direct vector stores only (A/B)
        const char* e = std::getenv("MOEPRISM_EPI_TMA");
        return !(e && e[0] == '0');
    }();
    p.tma_out = (epi == kEpiPlain && tmO && epi_tma) ? 1u : 0u;
    p.gather_tok = epi == kEpiSwiglu ? gather_tok : nullptr;
    const CUtensorMap& o_map = p.tma_out ? *tmO : *tmA;
    const bool tail = btail && btail->valid && epi == kEpiSwiglu && btail->valid < sh.N_group / 2;
    p.b_valid = tail ? btail->valid : 0u;
    p.b_tail_rows = tail ? btail->tail_rows : 0u;
    const CUtensorMap& bh_map = tail ? btail->half : *tmB;
    const CUtensorMap& bt_map = tail ? btail->part : *tmB;

    // upper bound on tiles; the kernel reads the exact count from the device
    const uint32_t max_tiles = (sh.max_rows / BM + sh.G) * p.NT * p.ksplit;
    static const uint32_t grid_cap = [] {  // MOEPRISM_GEMM_GRID: cap on the 1-SM GEMM grid (diagnostics)
        const char* e = std::getenv("MOEPRISM_GEMM_GRID");
        return e ? static_cast<uint32_t>(std::atoi(e)) : 0u;
    }();
    uint32_t grid = max_tiles < (uint32_t)num_sms ? max_tiles : (uint32_t)num_sms;
    if (grid_cap && grid > grid_cap) grid = grid_cap;
    func_attr_once(reinterpret_cast<const void*>(gemm_tc_kernel<kEpiPlain>), (int)kSmemBytes);
    func_attr_once(reinterpret_cast<const void*>(gemm_tc_kernel<kEpiSwiglu>), (int)kSmemBytes);
    func_attr_once(reinterpret_cast<const void*>(gemm_tc_kernel<kEpiActAbs>), (int)kSmemBytes);
    func_attr_once(reinterpret_cast<const void*>(gemm_tc_kernel<kEpiCount>), (int)kSmemBytes);
    func_attr_once(reinterpret_cast<const void*>(gemm_tc_kernel<kEpiF32Part>), (int)kSmemBytes);
    switch (epi) {
        case kEpiF32Part: launch_k(gemm_tc_kernel<kEpiF32Part>, grid, dim3(kThreads), kSmemBytes, s, *tmA, *tmB, a16, a32, a64, o_map, bh_map, bt_map, p); break;
        case kEpiSwiglu: launch_k(gemm_tc_kernel<kEpiSwiglu>, grid, dim3(kThreads), kSmemBytes, s, *tmA, *tmB, a16, a32, a64, o_map, bh_map, bt_map, p); break;
        case kEpiActAbs: launch_k(gemm_tc_kernel<kEpiActAbs>, grid, dim3(kThreads), kSmemBytes, s, *tmA, *tmB, a16, a32, a64, o_map, bh_map, bt_map, p); break;
        case kEpiCount: launch_k(gemm_tc_kernel<kEpiCount>, grid, dim3(kThreads), kSmemBytes, s, *tmA, *tmB, a16, a32, a64, o_map, bh_map, bt_map, p); break;
        default: launch_k(gemm_tc_kernel<kEpiPlain>, grid, dim3(kThreads), kSmemBytes, s, *tmA, *tmB, a16, a32, a64, o_map, bh_map, bt_map, p); break;
    }
}

}  // namespace mp
