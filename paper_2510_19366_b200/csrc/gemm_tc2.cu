// gemm_tc2.cu -- grouped GEMMs on CTA PAIRS (tcgen05.mma.cta_group::2): a
// cluster of two CTAs on the two SMs of one TPC computes a 256 x 256 tile,
// each CTA holding 128 rows of A and 128 of the 256 B rows in its own shared
// memory; the MMA (issued by the leader CTA only) reads both halves and
// writes each CTA's 128 rows x 256 columns into that CTA's TMEM.
//
// Why (measured, gemm_tc.cu trace + tests/probes/mma_cost.cu): the 1-SM
// 128 x 256 kernel runs its MMAs at ~95% of the N/2-cycle floor while fed,
// but waits 17-19% of the time for operand stages at k >= 8 -- every SM
// pulls 48 KB of A+B per 64-deep k-block from L2 (~26 TB/s chip-wide at the
// MMA floor).  A pair shares B: 32 KB per SM per k-block, one third less L2
// -> SM traffic and shared-memory fill bandwidth for the same MMA work.
//
// Layout / semantics are gemm_tc.cu's (same packed weights, same epilogues):
//   gemm1 (SWIGLU): B tile = W1 rows n*256 .. +255 = [64 gate | 64 up] for
//     neurons n*128 + 0..63, then the same for + 64..127; CTA r loads rows
//     n*256 + 128 r .. +127 (accumulator columns [128 r, 128 r + 128)).
//   gemm2: B tile = W2 rows n*256 .. +255 = output columns; CTA r loads its half.
// Tiles are (g, n, m) with 256-row m tiles (prefix of ceil(count_g / 256)),
// m fastest, handed to the clusters of a persistent grid in balanced rounds
// walked in snake order (tile_at below).
//
// Remainder tiles (round 2) run with SWAPPED operands: a group's last tile of
// r < 256 rows computes D^T = W_tile . X_r^T as an M=256 (weight rows) x
// N=Nt (tokens, Nt = r rounded up to 32) pair MMA.  The weight tile becomes
// the A operand (each CTA's own 128 rows, read only by its own tensor core)
// and the r token rows the B operand (Nt/2 per CTA, loaded through 16 / 32 /
// 64-row TMA boxes).  Per CTA and 64-deep k-block a plain remainder tile moves
// 32 KB into shared memory and 48 KB out of it (its B half is read by both
// tensor cores) whatever r is; the swapped one moves 16 KB + 64 Nt in and
// 16 KB + 128 Nt out (0.47 of that at Nt = 32).  Measured (per-tile trace,
// profiles/r02k_pair_tile_trace.txt): a swapped Nt = 32 tile still takes a
// full tile's ~610 cycles per k-block (an M=256 pair MMA costs >= 96 cycles
// whatever N is, profiles/r02k_mma_cost.csv, and spreading its k-steps over
// 4 accumulators changed nothing), but it issues 1/8 of the MMA work: under
// the 1000 W cap the energy saved is clock gained (Mixtral k = 4..16 5-10%
// faster than plain remainders, profiles/r02k_swap_ab.txt).  The
// accumulator then holds weight rows in TMEM lanes and tokens
// in columns: the epilogue transposes 32 x 32 blocks through shared memory
// (16-byte row stores), and for gemm1 the up rows (lanes 64..127 of a CTA in
// the [64 gate | 64 up] layout) cross to the gate warps through shared
// memory before SiLU(gate) * up.
//
// Remainder schedules measured and dropped (round 1):
// M=128 tail tiles (a tail tile costs the same ~580 cycles per k-block as a
// full one -- the pipeline is bound by the operand feed, ~510 cycles of MMA
// issue + ~70 of waits), a merged remainder riding on the previous tile as an
// extra M=128 MMA (its accumulator takes the other TMEM buffer and exposes an
// epilogue), a remainder spread over two N tiles (two M=128 MMAs re-reading A
// from shared memory), and tails on the 1-SM kernel after the pair kernel
// (+0.9 GB of weight re-reads).  Every scheme re-reads an operand or a weight
// tile; under the 1000 W cap the step lands within ~3% either way, so the pair
// kernel runs plain 256-row tiles only.
//
// Barriers: full[s] lives in the leader CTA (both CTAs' TMA loads complete_tx
// on it; the leader's expect_tx covers both); empty[s], tfull[a] are signalled
// in both CTAs by a multicast tcgen05.commit; tempty[a] lives in the leader and
// counts one arrival per epilogue warp of both CTAs (remote arrive for the
// peer).  TMEM: 2 accumulators x 256 columns per CTA (epilogue of tile i
// overlaps the MMAs of tile i+1), allocated with cta_group::2 by both CTAs.
#include <cstdio>
#include <cstdlib>

#include "mp_common.cuh"
#include "mp_kernels.h"

#ifndef MP_PAIR_TRACE  // 1: MMA-issuer timing into the trace buffer (diagnostic builds only)
#define MP_PAIR_TRACE 0
#endif
// L2 policies on the operand loads (diagnostic builds): bit 0 B evict_first,
// bit 1 A evict_last.  Measured (ncu DRAM bytes, k=8/16): evict_first on the
// weights raises DRAM reads 28-68% (concurrent m-tile pairs reuse them),
// evict_last on A saves 2-4%: both off.
#ifndef MP_PAIR_HINTS
#define MP_PAIR_HINTS 0
#endif
// Pipeline: 3 stages of 128-deep k-blocks (two 64-deep TMA sub-blocks per
// operand).  Measured against 6 stages of 64-deep k-blocks (the same bytes in
// flight): the per-k-block barrier round trip and issue overhead halves --
// leader cycles -14% (gemm1) / -16% (gemm2) at Mixtral k=8, steps -2..-7% at
// k = 6..16 (profiles/r02ac_kblock128_ab.txt).
#ifndef MP_PAIR_STAGES
#define MP_PAIR_STAGES 3
#endif

namespace mp {

namespace {

constexpr uint32_t BM = 256;  // rows per pair tile (128 per CTA)
constexpr uint32_t HM = 128;
constexpr uint32_t BN = 256;
#ifndef MP_PAIR_KSUB
#define MP_PAIR_KSUB 2  // 64-deep TMA sub-blocks per pipeline stage (1: 64-deep k-blocks, with 6 stages)
#endif
constexpr uint32_t KSUB = MP_PAIR_KSUB;
constexpr uint32_t BK = 64 * KSUB;
constexpr uint32_t SUB_A = HM * 64 * 2;   // one 64-deep sub-block of A / of the B half: 16 KB
constexpr uint32_t SUB_B = 128 * 64 * 2;
constexpr uint32_t NSP = MP_PAIR_STAGES;
constexpr uint32_t A_BYTES = HM * BK * 2;   // per CTA and stage: 128 A rows x BK (32 KB)
constexpr uint32_t B_BYTES = 128 * BK * 2;  // per CTA and stage: half of the 256-row B tile (32 KB)
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
#ifndef MP_PAIR_EPI_WARPS
#define MP_PAIR_EPI_WARPS 4
#endif
// warp 0 TMA, warp 1 TMEM alloc + MMA (leader), warps 2..5 epilogue (one per
// TMEM lane quarter).  Measured (round 1, tile_trace.py, k=8): 8 epilogue
// warps halve the SwiGLU epilogue (13.7k -> 6.1k cycles per tile) but it is
// hidden behind the next tile's MMAs anyway, and the extra polling warps slow
// gemm2 by 9%; round 2's 8-warp variant for the short-K Qwen down projection
// was no faster either.  The swapped-remainder epilogue assumes 4.
constexpr uint32_t kEpiWarps = MP_PAIR_EPI_WARPS;
constexpr uint32_t kThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kXchBytes = 64 * 33 * 4;         // gemm1 swapped tiles: up rows -> gate warps (fp32, padded)
constexpr uint32_t kStgBytes = 4 * 2 * 32 * 32 * 2;  // per epilogue warp: two 32 x 32 bf16 blocks (TMA-store
                                                    // staging, double-buffered; swapped tiles' transposes)
constexpr size_t kSmemBytes = 1024 + NSP * STAGE_BYTES + 256 + kXchBytes + kStgBytes;
static_assert(kSmemBytes + 4096 <= 232448, "pair GEMM shared memory");
static_assert(kEpiWarps == 4, "the swapped-tail epilogue pairs lane quarters 0/1 with 2/3 (4 epilogue warps)");

struct PairParams {
    uint32_t G, K, N_group, n_valid, ld_out, NT;
    const uint32_t* offsets;
    const uint32_t* mprefix;  // prefix of ceil(count_g / 256)
    __nv_bfloat16* out;
    uint64_t* trace;  // [grid][4] MMA-issuer timing of the leaders (diagnostics) or null
    const uint32_t* gmap;  // nullable: B group of group g (sub-expert offload cache slot), else g
    uint32_t swap_tail;    // remainder tiles with swapped operands (needs the short A maps)
    uint32_t tma_out;      // plain epilogue: tmO valid (whole 32-row warp slabs leave through TMA stores)
};

// remainder tile: rows r < 256 of the group's last m tile; Nt = tokens per
// swapped MMA (r rounded up to 32 -> each CTA loads Nt / 2, a multiple of 16)
MP_DEV uint32_t swap_cols(uint32_t swap, uint32_t cnt, uint32_t m) {
    const uint32_t r = cnt - m * BM;
    return (swap && r < BM) ? ((r + 31u) & ~31u) : 0u;
}
// Tile order: round i hands tiles i*npairs .. +npairs-1 to the pairs, walked
// in reverse on odd rounds, so a pair alternates its position inside the
// (g, n) blocks of [full..., remainder] tiles instead of always drawing the
// same kind (with 2-tile blocks and an even pair count, plain striding gave
// half the pairs every full tile and the other half every remainder).
MP_DEV uint32_t tile_at(uint32_t i, uint32_t pair, uint32_t npairs) {
    return i * npairs + ((i & 1u) ? npairs - 1u - pair : pair);
}
MP_DEV void named_bar(uint32_t id, uint32_t n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

MP_DEV uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
MP_DEV void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` (own smem offset) in CTA `rank` of the cluster
MP_DEV uint32_t mapa(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
MP_DEV void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
MP_DEV bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
MP_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait_cluster(bar, parity)) {
    }
}
// TMA 2D tile load into own smem, completion signalled on an mbarrier that
// may live in the peer CTA (cluster address)
MP_DEV void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar_cluster)
        : "memory");
}
MP_DEV void tma_load_2d_pair_hint(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int32_t c0, int32_t c1,
                                  uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.cta_group::2.L2::cache_hint "
        "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar_cluster), "l"(policy)
        : "memory");
}
MP_DEV void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// arrive (once) on the barrier at this smem offset in both CTAs of the pair
// when all prior tcgen05 ops of this thread complete
MP_DEV void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}
MP_DEV void tmem_alloc_pair(uint32_t* smem_dst) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
MP_DEV void tmem_dealloc_pair(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kTmemCols) : "memory");
}

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
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmA16, const __grid_constant__ CUtensorMap tmA32,
                     const __grid_constant__ CUtensorMap tmA64, const __grid_constant__ CUtensorMap tmO,
                     PairParams p) {
    constexpr uint32_t NS = NSP;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint32_t s_prefix[kMaxG + 1];
    __shared__ uint32_t s_off[kMaxG + 1];
    __shared__ uint32_t s_gmap[kMaxG];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // identical offsets in both CTAs (same dynamic smem layout)
    uint8_t* sA = base;                // NS x 16 KB
    uint8_t* sB = base + NS * A_BYTES;  // NS x 16 KB
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + NS * B_BYTES);
    uint64_t* empty = full + NS;
    uint64_t* tfull = empty + NS;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* xch = reinterpret_cast<float*>(base + NS * STAGE_BYTES + 256);
    uint16_t* stg_all = reinterpret_cast<uint16_t*>(base + NS * STAGE_BYTES + 256 + kXchBytes);

    const uint32_t warp = threadIdx.x / 32;
    const uint32_t lane = threadIdx.x % 32;
    const uint32_t rank = cluster_rank();
    const uint32_t pair = blockIdx.x >> 1, npairs_grid = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (uint32_t a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * kEpiWarps);  // epilogue warps x 2 CTAs
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        if (p.tma_out) tma_prefetch_desc(&tmO);
        if (p.swap_tail) {
            tma_prefetch_desc(&tmA16);
            tma_prefetch_desc(&tmA32);
            tma_prefetch_desc(&tmA64);
        }
    }
    if (warp == 1) tmem_alloc_pair(tmem_slot);
    griddep_wait();  // group metadata comes from the routing epilogue
    griddep_launch();
    for (uint32_t q = threadIdx.x; q <= p.G; q += blockDim.x) {
        s_prefix[q] = p.mprefix[q];
        s_off[q] = p.offsets[q];
        if (q < p.G) s_gmap[q] = p.gmap ? p.gmap[q] : q;
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // peer barriers initialised before any remote signal
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t total = s_prefix[p.G] * p.NT;
    // balanced rounds (as in gemm_tc.cu): only ceil(total / R) pairs take
    // tiles, R = ceil(total / pairs) each
    const uint32_t rounds = (total + npairs_grid - 1) / npairs_grid;
    const uint32_t npairs = rounds ? (total + rounds - 1) / rounds : npairs_grid;
    const uint32_t my_rounds = pair < npairs ? rounds : 0u;  // idle pairs take no tiles
    const uint32_t nkb = (p.K + BK - 1) / BK;  // a partial last k-block is zero-filled by the TMA

    if (warp == 0) {
        if (lane == 0) {
            const uint32_t full_leader = mapa(&full[0], 0);  // full[s] of the leader: + 8 s
#if MP_PAIR_HINTS
            const uint64_t pol_b = l2_policy_evict_first(), pol_a = l2_policy_evict_last();
            (void)pol_a;
            (void)pol_b;
#endif
            uint32_t it = 0;
            for (uint32_t i = 0; i < my_rounds; ++i) {
                const uint32_t tile = tile_at(i, pair, npairs);
                if (tile >= total) continue;
                uint32_t g, m, n;
                map_tile(tile, s_prefix, p.G, p.NT, g, m, n);
                const uint32_t nt = swap_cols(p.swap_tail, s_off[g + 1] - s_off[g], m);
                const uint32_t half = nt / 2;  // swapped: token rows per CTA
                const int32_t arow = static_cast<int32_t>(s_off[g] + m * BM + rank * (nt ? half : HM));
                const int32_t brow = static_cast<int32_t>(s_gmap[g] * p.N_group + n * BN + rank * 128);
                for (uint32_t kb = 0; kb < nkb; ++kb, ++it) {
                    const uint32_t s = it % NS, ph = (it / NS) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    if (rank == 0) mbar_expect_tx(&full[s], 2 * KSUB * (SUB_B + (nt ? half * 128u : SUB_A)));
                    const uint32_t fb = full_leader + s * 8;
                    for (uint32_t sb = 0; sb < KSUB; ++sb) {
                    const int32_t kc = static_cast<int32_t>(kb * BK + sb * 64);
                    uint8_t* dA = sA + s * A_BYTES + sb * SUB_A;
                    uint8_t* dB = sB + s * B_BYTES + sb * SUB_B;
                    if (nt && half < HM) {
                        // token rows through 64 / 32 / 16-row boxes (half is a multiple of 16)
                        uint32_t done = 0;
                        if (half & 64u) {
                            tma_load_2d_pair(dA, &tmA64, fb, kc, arow);
                            done = 64;
                        }
                        if (half & 32u) {
                            tma_load_2d_pair(dA + done * 128u, &tmA32, fb, kc, arow + (int32_t)done);
                            done += 32;
                        }
                        if (half & 16u)
                            tma_load_2d_pair(dA + done * 128u, &tmA16, fb, kc, arow + (int32_t)done);
                    } else {
#if MP_PAIR_HINTS & 2
                        tma_load_2d_pair_hint(dA, &tmA, fb, kc, arow, pol_a);
#else
                        tma_load_2d_pair(dA, &tmA, fb, kc, arow);
#endif
                    }
#if MP_PAIR_HINTS & 1
                    tma_load_2d_pair_hint(dB, &tmB, fb, kc, brow, pol_b);
#else
                    tma_load_2d_pair(dB, &tmB, fb, kc, brow);
#endif
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0 && lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
            uint32_t it = 0, tc = 0;
#if MP_PAIR_TRACE
            const uint64_t t_start = clock64();
            uint64_t w_acc = 0, w_full = 0;
#endif
            for (uint32_t i = 0; i < my_rounds; ++i) {
                const uint32_t tile = tile_at(i, pair, npairs);
                if (tile >= total) continue;
                const uint32_t acc = tc & 1u;
#if MP_PAIR_TRACE
                uint64_t t0 = clock64();
#endif
                // acquisition tc of the buffer waits for its release tc - 2
                mbar_wait_cluster(&tempty[acc], ((tc >> 1) & 1u) ^ 1u);
#if MP_PAIR_TRACE
                w_acc += clock64() - t0;
                const uint64_t t_tile = clock64(), wf0 = w_full;
#endif
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                uint32_t g, m, n;
                map_tile(tile, s_prefix, p.G, p.NT, g, m, n);
                const uint32_t nt = swap_cols(p.swap_tail, s_off[g + 1] - s_off[g], m);
                const uint32_t id = nt ? umma_idesc_bf16(BM, nt) : idesc;
                for (uint32_t kb = 0; kb < nkb; ++kb, ++it) {
                    const uint32_t s = it % NS, ph = (it / NS) & 1u;
#if MP_PAIR_TRACE
                    t0 = clock64();
#endif
                    mbar_wait(&full[s], ph);
#if MP_PAIR_TRACE
                    w_full += clock64() - t0;
#endif
                    tc_fence_after();
                    // swapped remainder: the weight tile is the A operand, the tokens B
                    const uint32_t a0 = smem_u32(nt ? sB + s * B_BYTES : sA + s * A_BYTES);
                    const uint32_t b0 = smem_u32(nt ? sA + s * A_BYTES : sB + s * B_BYTES);
#pragma unroll
                    for (uint32_t k = 0; k < BK / 16; ++k) {
                        // k-step k: sub-block k / 4 (16 KB apart in both operand slots), 32 bytes per step
                        const uint32_t off = (k >> 2) * SUB_A + (k & 3u) * 32;
                        umma_bf16_pair(d_tmem, umma_desc_sw128(a0 + off), umma_desc_sw128(b0 + off), id,
                                       (kb | k) != 0u);
                    }
                    umma_commit_pair(&empty[s]);
                }
                umma_commit_pair(&tfull[acc]);
#if MP_PAIR_TRACE
                if (p.trace && tc < 128) {  // per-tile record: tile, operand waits, MMA-phase cycles, tail
                    uint64_t* r = p.trace + 4096 + ((size_t)pair * 128 + tc) * 4;
                    r[0] = tile;
                    r[1] = w_full - wf0;
                    r[2] = clock64() - t_tile;
                    r[3] = nt;  // 0 full tile, else the swapped remainder's token columns
                }
#endif
                ++tc;
            }
#if MP_PAIR_TRACE
            if (p.trace) {
                uint64_t* tr = p.trace + blockIdx.x * 4;
                tr[0] = clock64() - t_start;
                tr[1] = w_acc;
                tr[2] = w_full;
                tr[3] = tc;
            }
#endif
        }
        __syncwarp();
    } else {
        const uint32_t q = warp & 3u;  // TMEM lane quarter this warp may access
        const uint32_t part = (warp - 2) / 4, nparts = kEpiWarps / 4;  // column share of this warp
        const uint32_t tempty_leader = mapa(&tempty[0], 0);
        uint16_t* stg = stg_all + (warp - 2) * 2048;  // this warp's two 32 x 32 bf16 staging blocks
        uint32_t epi_it = 0;                          // TMA-store chunks issued by this warp
        // One accumulator to bf16 rows of the group: lane = row rank*128 +
        // q*32 + lane, all 256 D columns.
        auto emit = [&](uint32_t buf, uint32_t row0, uint32_t g, uint32_t n, uint32_t cnt) {
            const uint32_t row_local = row0 + rank * HM + q * 32 + lane;
            constexpr uint32_t nchunk = 8;  // 32-column chunks of D held by the lane
            const bool valid = row_local < cnt;
            const bool any = (row_local - lane) < cnt;  // warp has a valid row
            __nv_bfloat16* orow = p.out + static_cast<size_t>(s_off[g] + row_local) * p.ld_out;
            const uint32_t taddr = tmem_base + ((q * 32u) << 16) + buf * BN;
            if (!any) return;
            if constexpr (SWIGLU) {
                // D chunk pair (gate, up) = columns (h*128 + c2*32, + 64) for
                // neurons n*128 + h*64 + c2*32 .. +31
#pragma unroll 1
                for (uint32_t c = part; c < nchunk / 2; c += nparts) {
                    const uint32_t h = c >> 1, c2 = c & 1u;
                    const uint32_t tcol = h * 128 + c2 * 32;
                    uint32_t gr[32], ur[32];
                    tmem_ld32(taddr + tcol, gr);
                    tmem_ld32(taddr + tcol + kIlv, ur);
                    tmem_ld_wait();
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float g0 = __uint_as_float(gr[2 * i]), g1 = __uint_as_float(gr[2 * i + 1]);
                        const float u0 = __uint_as_float(ur[2 * i]), u1 = __uint_as_float(ur[2 * i + 1]);
                        pk[i] = pack_bf16x2(silu_f32(g0) * u0, silu_f32(g1) * u1);
                    }
                    if (valid) {
                        __nv_bfloat16* dst = orow + n * 128 + h * 64 + c2 * 32;
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            st_global_v4(dst + v * 8, make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]));
                    }
                }
            } else {
                // A warp whose 32 rows are all valid stages each 32 x 32 chunk
                // in shared memory and writes it with one TMA store (whole
                // 64-byte row segments; short-K GEMMs such as Qwen's K = 384
                // down projection are epilogue-bound); ragged slabs store directly.
                const bool slab = p.tma_out && row0 + rank * HM + q * 32 + 32 <= cnt;
                const int32_t slab_row = static_cast<int32_t>(s_off[g] + row0 + rank * HM + q * 32);
                auto store = [&](uint32_t c, const uint32_t* r) {
                    const uint32_t col = n * BN + c * 32;
                    if (col >= p.n_valid) return;
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        pk[i] = pack_bf16x2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
                    if (slab) {
                        uint16_t* buf = stg + (epi_it & 1u) * 1024;
                        if (epi_it >= 2) {  // the store issued from this buffer two chunks ago has read it
                            if (lane == 0) bulk_wait_read<1>();
                            __syncwarp();
                        }
                        uint4* dst = reinterpret_cast<uint4*>(buf + lane * 32);
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
                // the TMEM load of the next chunk overlaps this chunk's stores
                uint32_t ra[32], rb[32];
                tmem_ld32(taddr + part * 32, ra);
                tmem_ld_wait();
#pragma unroll 1
                for (uint32_t c = part; c < nchunk; c += 2 * nparts) {
                    const bool more = c + nparts < nchunk;
                    if (more) tmem_ld32(taddr + (c + nparts) * 32, rb);
                    store(c, ra);
                    tmem_ld_wait();
                    if (!more) break;
                    if (c + 2 * nparts < nchunk) tmem_ld32(taddr + (c + 2 * nparts) * 32, ra);
                    store(c + nparts, rb);
                    tmem_ld_wait();
                }
            }
        };
        // Swapped remainder tile: TMEM lane = weight row (CTA rank's 128 of the
        // 256-row N tile), column j = token row0 + j (j < nt).  32 x 32 blocks
        // go through a per-warp transpose buffer and leave as 16-byte row
        // segments (4 per thread per block).
        auto put_block = [&](uint32_t row0, uint32_t g, uint32_t cnt, uint32_t c, uint32_t col0, bool col_ok) {
            __syncwarp();
#pragma unroll
            for (uint32_t i = 0; i < 4; ++i) {
                const uint32_t idx = i * 32 + lane, j = idx >> 2, seg = idx & 3u;
                const uint32_t row = row0 + c * 32 + j;
                const uint4 v = *reinterpret_cast<const uint4*>(stg + j * 32 + seg * 8);
                if (row < cnt && col_ok)
                    st_global_v4(p.out + static_cast<size_t>(s_off[g] + row) * p.ld_out + col0 + seg * 8, v);
            }
            __syncwarp();
        };
        auto emit_swapped = [&](uint32_t buf, uint32_t row0, uint32_t g, uint32_t n, uint32_t cnt, uint32_t nt) {
            const uint32_t taddr = tmem_base + ((q * 32u) << 16) + buf * BN;
            if (epi_it) {  // staged TMA stores of earlier tiles have read the buffer
                if (lane == 0) bulk_wait_read<0>();
                __syncwarp();
            }
            const uint32_t nch = nt / 32;
            uint32_t r[32];
            auto load_chunk = [&](uint32_t c) {
                tmem_ld32(taddr + c * 32, r);
                tmem_ld_wait();
            };
            if constexpr (SWIGLU) {
                // lanes 0..63 gate, 64..127 up of neurons n*128 + rank*64 + 0..63
                float* xrow = xch + ((q & 1u) * 32 + lane) * 33;
#pragma unroll 1
                for (uint32_t c = 0; c < nch; ++c) {
                    load_chunk(c);
                    if (q >= 2) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) xrow[j] = __uint_as_float(r[j]);
                    }
                    named_bar(1, 128);
                    if (q < 2) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float hv = silu_f32(__uint_as_float(r[j])) * xrow[j];
                            stg[j * 32 + lane] = __bfloat16_as_ushort(__float2bfloat16_rn(hv));
                        }
                        put_block(row0, g, cnt, c, n * 128 + rank * 64 + q * 32, true);
                    }
                    named_bar(2, 128);
                }
            } else {
                const uint32_t col0 = n * BN + rank * HM + q * 32;
#pragma unroll 1
                for (uint32_t c = 0; c < nch; ++c) {
                    load_chunk(c);
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        stg[j * 32 + lane] = __bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(r[j])));
                    put_block(row0, g, cnt, c, col0, col0 < p.n_valid);
                }
            }
        };
        auto release = [&](uint32_t buf) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader + buf * 8);
        };
        uint32_t tc = 0;
#if MP_PAIR_TRACE
        uint64_t e_busy = 0, e_ext = 0, e_wait = 0;
#endif
        for (uint32_t i = 0; i < my_rounds; ++i) {
            const uint32_t tile = tile_at(i, pair, npairs);
            if (tile >= total) continue;
            uint32_t g, m, n;
            map_tile(tile, s_prefix, p.G, p.NT, g, m, n);
            const uint32_t acc = tc & 1u;
#if MP_PAIR_TRACE
            const uint64_t e0 = clock64();
#endif
            mbar_wait(&tfull[acc], (tc >> 1) & 1u);  // one commit per tile on its buffer
            tc_fence_after();
#if MP_PAIR_TRACE
            const uint64_t e1 = clock64();
            e_wait += e1 - e0;
#endif
            const uint32_t cnt = s_off[g + 1] - s_off[g];
            const uint32_t nt = swap_cols(p.swap_tail, cnt, m);
            if (nt)
                emit_swapped(acc, m * BM, g, n, cnt, nt);
            else
                emit(acc, m * BM, g, n, cnt);
            release(acc);
#if MP_PAIR_TRACE
            e_busy += clock64() - e1;
#endif
            ++tc;
        }
#if MP_PAIR_TRACE
        if (p.trace && warp == 2 && lane == 0) {  // epilogue timing of one warp per CTA
            uint64_t* tr = p.trace + 2048 + blockIdx.x * 4;
            tr[0] = e_busy;
            tr[1] = e_ext;
            tr[2] = e_wait;
            tr[3] = tc;
        }
#endif
        if (epi_it && lane == 0) bulk_wait0();  // the TMA stores are complete before the CTA retires
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // the leader's last MMAs / the peer's last TMEM reads are done
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(tmem_base);
    }
}

}  // namespace

size_t gemm_pair_smem_bytes() { return kSmemBytes; }

bool pair_swap_enabled() {
    static const bool on = [] {  // MOEPRISM_PAIR_SWAP=0: plain 256-row remainder tiles (A/B)
        const char* e = std::getenv("MOEPRISM_PAIR_SWAP");
        return !(e && e[0] == '0');
    }();
    return on;
}

// tmB: box of 128 rows (each CTA loads half of the 256-row B tile); mprefix256:
// prefix of ceil(count_g / 256) over the groups; tmA_small (nullable): [3]
// maps of A with 16 / 32 / 64-row boxes -- remainder tiles run swapped.
void launch_gemm_tc2(bool swiglu, const CUtensorMap* tmA, const CUtensorMap* tmB, void* out, const GemmShape& sh,
                     const uint32_t* offsets, const uint32_t* mprefix256, int num_sms, cudaStream_t s,
                     const uint32_t* gmap, const CUtensorMap* tmA_small, const CUtensorMap* tmO) {
    const bool swap = tmA_small != nullptr && pair_swap_enabled();
    PairParams p{sh.G, sh.K, sh.N_group, sh.n_valid, sh.ld_out, (sh.N_group + BN - 1) / BN, offsets, mprefix256,
                 static_cast<__nv_bfloat16*>(out), gemm_trace_buffer(swiglu), gmap, swap ? 1u : 0u,
                 (!swiglu && tmO) ? 1u : 0u};
    const CUtensorMap* o_map = p.tma_out ? tmO : tmA;
    const CUtensorMap* s16 = swap ? &tmA_small[0] : tmA;
    const CUtensorMap* s32 = swap ? &tmA_small[1] : tmA;
    const CUtensorMap* s64 = swap ? &tmA_small[2] : tmA;
    if (p.trace) cudaMemsetAsync(p.trace, 0, (4096 + 128 * 128 * 4) * sizeof(uint64_t), s);
    const uint32_t max_tiles = (sh.max_rows / BM + sh.G) * p.NT;
    static const uint32_t grid_cap = [] {  // MOEPRISM_PAIR_GRID: cap on the pairs of the grid (diagnostics)
        const char* e = std::getenv("MOEPRISM_PAIR_GRID");
        return e ? static_cast<uint32_t>(std::atoi(e)) : 0u;
    }();
    uint32_t pairs = static_cast<uint32_t>(num_sms) / 2;
    if (grid_cap && pairs > grid_cap) pairs = grid_cap;
    if (max_tiles < pairs) pairs = max_tiles;
    if (pairs == 0) pairs = 1;
    func_attr_once(reinterpret_cast<const void*>(gemm_pair_kernel<true>), (int)kSmemBytes);
    func_attr_once(reinterpret_cast<const void*>(gemm_pair_kernel<false>), (int)kSmemBytes);
    const dim3 grid(2 * pairs), block(kThreads);
    if (swiglu)
        launch_k(gemm_pair_kernel<true>, grid, block, kSmemBytes, s, *tmA, *tmB, *s16, *s32, *s64, *o_map, p);
    else
        launch_k(gemm_pair_kernel<false>, grid, block, kSmemBytes, s, *tmA, *tmB, *s16, *s32, *s64, *o_map, p);
}

}  // namespace mp
