// mp_kernels.h -- host-side launchers for the sm_100a kernels (internal).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace mp {

constexpr uint32_t kRouteTokensPerBlock = 32;  // tokens per router / bucket CTA
constexpr uint32_t kTcBM = 128;                // tcgen05 grouped GEMM tile M
constexpr uint32_t kSimtBM = 64;               // SIMT grouped GEMM tile M
constexpr uint32_t kMaxG = 256;                // max E*S sub-experts (Qwen: 240)
// W1 gate/up interleave: rows in blocks of 2*kIlv = kIlv gate rows then the
// kIlv up rows of the same neurons (pack.cu).  64 puts gate and up of a
// neuron in the same TMEM lane for both the 256-row and the 128-row (tail)
// CTA-pair MMA shapes (gemm_tc2.cu).
constexpr uint32_t kIlv = 64;

// Device scratch for the bucketing of one forward.
struct BucketWs {
    uint32_t* lrank;         // [T][k_max] rank inside (block, bucket)
    uint32_t* block_counts;  // [nblk][G]
    uint32_t* block_base;    // [nblk][G]
    uint32_t* offsets;       // [G+1]
    uint32_t* mprefix_tc;    // [G+1] prefix of ceil(count/128)
    uint32_t* mprefix_simt;  // [G+1] prefix of ceil(count/64)
    uint32_t* mprefix_tc2;   // [G+1] prefix of ceil(count/256) (CTA-pair tiles)
    uint32_t* perm_tok;      // [rows]
    float* perm_w;           // [rows]
    uint32_t* slot_row;      // [T][k_max]
    int* err;                // device error flags (bit 0: bad k / selection, bit 1: non-finite x)
};

// Certification bound of the tensor-core router logits for token t:
//   guard_t = coef * sum_i |x_ti| + 2^-23 * max_g |logit_tg| + floor_abs
// coef = chunk depth * 2^-23 * max|W_r| * (1 + margin) (router_guard_coef);
// sum |x_t| is formed by the consumer kernels from the bf16 row (L2-resident).
struct RouterGuard {
    double coef;
    double floor_abs;  // MOEPRISM_ROUTER_GUARD (tests widen the window), else 0
};
// dtype: 0 f32, 1 bf16
void launch_router_linear(int dtype, const void* x, uint32_t T, uint32_t d, const float* wrT, uint32_t G,
                          uint32_t k_max, const uint32_t* kpt, uint32_t k, int weight_mode, uint32_t* sel, float* w,
                          int* err, uint32_t* stats, cudaStream_t s);
// stats (nullable): stats[1] += near ties (k-th/(k+1)-th gap < 1e-6)
void launch_router_scores_topk(const float* scores, uint32_t T, uint32_t G, uint32_t k_max, const uint32_t* kpt,
                               uint32_t k, int weight_mode, uint32_t* sel, float* w, int* err, uint32_t* stats,
                               cudaStream_t s);
// Proxy router (proxy.cu).  Exact path: fp64 gate activations in the
// reference's order -> scores [T][G] (double, at the front of `scores`).
void launch_proxy_scores(int dtype, const void* x, uint32_t T, uint32_t d, const float* gate_w, const float* up_w,
                         const uint32_t* gate_off, uint32_t n_gate_rows, uint32_t G, float* scores, cudaStream_t s);
// Tensor-core path: after launch_router_tc over the [gate; up] planes (fp32
// partials), scores + per-sub-expert bounds + certified top-k; uncertain
// tokens to flagged[2..] with their scores in pscore [T][G] and per-sub-expert
// classes in pclass [T][G], re-selected by launch_proxy_fixup from fp64 gate
// activations.
void launch_proxy_tc_topk(const float* partial, uint32_t ks, uint32_t T, uint32_t NR, uint32_t Npad,
                          const uint32_t* gate_off, uint32_t G, uint32_t k_max, const uint32_t* kpt, uint32_t k,
                          int weight_mode, uint32_t* sel, float* w, int* err, const RouterGuard& rg, const void* x,
                          uint32_t d, double* pscore, int8_t* pclass, uint32_t* flagged, cudaStream_t s);
void launch_proxy_fixup(const void* x, uint32_t d, const float* gate_w, const float* up_w, const uint32_t* gate_off,
                        uint32_t G, uint32_t k_max, const uint32_t* kpt, uint32_t k, int weight_mode, uint32_t* sel,
                        float* w, int* err, const double* pscore, const int8_t* pclass, uint32_t* flagged,
                        int num_sms, cudaStream_t s);
void launch_bucket_local(const uint32_t* sel, uint32_t T, uint32_t k_max, uint32_t G, BucketWs& ws,
                         cudaStream_t s);
void launch_bucket_scan(uint32_t T, uint32_t G, BucketWs& ws, cudaStream_t s);
// x_perm == null: permutation tables only (the GEMM gathers the rows itself)
// check_finite: also scan x for non-finite values (err bit 2)
// tb: tokens per bucketing block of the ranks / bases (kRouteTokensPerBlock,
// or the fused router's smaller blocks for small batches)
void launch_dispatch(int dtype, const void* x, uint32_t T, uint32_t d, uint32_t d_pad, const uint32_t* sel,
                     const float* w, uint32_t k_max, uint32_t G, BucketWs& ws, void* x_perm, cudaStream_t s,
                     bool check_finite = true, uint32_t tb = kRouteTokensPerBlock);
// group_S > 0: unit-weight semantics, round once per parent expert (fp32 mode)
// o_sh / w_sh (bf16 only, nullable): shared-expert output rows [T][d_pad] and
// per-token weights, added after the routed sub-experts -- or, with
// sh_splits > 0, fp32 split-K partials [sh_splits][sh_stride] summed in split
// order; x_res (bf16 only, nullable): residual input [T][d], y = x_res + sum
// (accumulator start value)
void launch_combine(int dtype, const void* o, uint32_t d, uint32_t d_pad, const uint32_t* slot_row,
                    const uint32_t* sel, const float* w, uint32_t k_max, uint32_t group_S, uint32_t T, void* y,
                    cudaStream_t s, const void* o_sh = nullptr, const float* w_sh = nullptr,
                    const void* x_res = nullptr, uint32_t sh_splits = 0, size_t sh_stride = 0, uint32_t k_hint = 0, int num_sms = 148);
void launch_shared_gate(const void* x, uint32_t T, uint32_t d, const float* gate, float* w_sh, uint32_t* sh_off,
                        uint32_t* sh_mprefix, cudaStream_t s);

// Tensor-core linear router (router_tc.cu): plan, weight split, launch, and
// the fixed-order fp64 reduction of the K-split partials + top-k (route.cu).
struct RouterTcPlan {
    uint32_t Npad, kb_total, kb_per_split, ks, m_tiles, stages, chunk_kb, ncta, nsplit;
    size_t smem;
};
RouterTcPlan plan_router_tc(uint32_t T, uint32_t d, uint32_t G, int num_sms);
// rows ([ks][T] products) of the K-split partial buffers over every T <= max_T
size_t router_tc_partial_rows(uint32_t max_T, uint32_t d, uint32_t G, int num_sms);
uint32_t router_tc_cols_per_cta(uint32_t G);  // TMA box rows of the weight-plane tensor map
void launch_split_router(const float* wr, uint32_t d, uint32_t G, uint32_t Npad, void* planes, cudaStream_t s);
// rows [n_a][d] ++ [n_b][d] (fp32) -> three bf16 planes [3][Npad][d]
void launch_split_rows(const float* ra, const float* rb, uint32_t n_a, uint32_t n_b, uint32_t d, uint32_t Npad,
                       void* planes, cudaStream_t s);
// out_f32: partials rounded to fp32 once per K split (the proxy router's
// 2*E*S*r gate/up columns; the rounding adds <= 2^-24 sum|x||W| to the bound)
void launch_router_tc(const CUtensorMap* tmX, const CUtensorMap* tmW, const RouterTcPlan& pl, uint32_t T,
                      void* partial, cudaStream_t s, bool out_f32 = false);
double router_guard_coef(uint32_t chunk_depth, float wmax);
// Routing statistics of a forward (stats / flagged, zeroed by the caller):
// [0] tokens re-selected from exact fp64 logits, [1] near ties (exact
// k-th/(k+1)-th gap < 1e-6), then (non-fused path) the re-selected tokens.
// rg: per-token tensor-core logit error bound; tokens whose k-th/(k+1)-th gap is below
// 2*guard_t + 1e-6 are appended to flagged[2..] (count in flagged[0]) and
// re-selected from exact fp64 logits by launch_router_fixup.
void launch_partials_topk(const double* partial, uint32_t ks, uint32_t T, uint32_t G, uint32_t Npad, uint32_t k_max,
                          const uint32_t* kpt, uint32_t k, int weight_mode, uint32_t* sel, float* w, int* err,
                          const RouterGuard& rg, const void* x, uint32_t d, uint32_t* flagged, cudaStream_t s);
// Fused routing epilogue of the tensor-core router (bf16 x, d % 4 == 0):
// partials -> top-k -> exact re-selection of near-tie tokens (count added to
// *n_fixed) -> bucket ranks -> device-wide scans (last CTA; *ticket must be
// 0 on entry and is left 0).  Replaces partials_topk + router_fixup +
// bucket_local + bucket_scan.  Returns whether it also wrote the permutation
// tables (tables requested and the grid-barrier path taken).
bool launch_route_bucket(const double* partial, uint32_t ks, uint32_t T, uint32_t G, uint32_t Npad, uint32_t k_max,
                         const uint32_t* kpt, uint32_t k, int weight_mode, uint32_t* sel, float* w,
                         const RouterGuard& rg, const void* x, uint32_t d, const float* wrT, uint32_t* ticket,
                         uint32_t* stats, BucketWs& ws, cudaStream_t s, uint32_t tb = kRouteTokensPerBlock,
                         int num_sms = 0, bool tables = false);  // tables: also write perm_tok / perm_w / slot_row
// tokens per CTA of the fused routing epilogue: fewer for small batches (more
// CTAs; measured: one or two 32-token CTAs at T = 64 are slower)
inline uint32_t route_tokens_per_block(uint32_t T) {
    return T <= 256 ? 2u : T <= 1024 ? 8u : kRouteTokensPerBlock;
}
// ticket: 3 zeroed words (last-CTA ticket; grid-barrier arrive / depart
// counters), left zero.  More than 8 K splits are summed CTA-wide in the
// kernel.  num_sms: a grid of <= num_sms CTAs forms its bucket bases after a
// grid barrier.
// in-place fixed-order sum of the K-split router partials into plane 0
void launch_partials_reduce(double* partial, uint32_t ks, uint32_t T, uint32_t G, uint32_t Npad, cudaStream_t s);
void launch_router_fixup(int dtype, const void* x, uint32_t d, const float* wrT, uint32_t G, uint32_t k_max,
                         const uint32_t* kpt, uint32_t k, int weight_mode, uint32_t* sel, float* w, int* err,
                         uint32_t* flagged, int num_sms, cudaStream_t s);

// Packing (load time).
void launch_pack_w1(int dtype, const float* wg, const float* wu, uint32_t d, uint32_t ff, const int32_t* nmap,
                    uint32_t S, uint32_t w_pad, uint32_t d_pad, void* W1_e, cudaStream_t s);
void launch_pack_w2(int dtype, const float* wd, uint32_t d, uint32_t ff, const int32_t* nmap, uint32_t S,
                    uint32_t w_pad, uint32_t d_pad, void* W2_e, cudaStream_t s);
void launch_transpose_router(const float* wr, uint32_t d, uint32_t G, uint32_t G_pad, float* wrT, cudaStream_t s);
void launch_pack_gate_rows(const float* wg, const float* wu, uint32_t d, uint32_t ff, const uint32_t* neurons,
                           uint32_t n, float* gate_rows, float* up_rows, cudaStream_t s);
void launch_finite_check(const float* p, size_t n, int* flag, cudaStream_t s);
void launch_synth_fill(void* dst, int dtype, size_t n, uint64_t seed, uint64_t first, double scale, cudaStream_t s);

// Grouped GEMMs.  Rows of group g live at [offsets[g], offsets[g+1]) of the
// permuted row space; weights of group g at W + g * (rows per group).
struct GemmShape {
    uint32_t G, K, N_group;  // per group: N_group output rows of W (gate/up interleaved for gemm1)
    uint32_t max_rows;       // row capacity of A / out
    uint32_t ld_out;         // elements per output row
    uint32_t n_valid;        // columns < n_valid are stored (gemm2: d_pad) -- gemm1 stores all
};
void launch_gemm1_simt(int dtype, const void* A, const void* W1, void* H, const GemmShape& sh,
                       const uint32_t* offsets, const uint32_t* mprefix, cudaStream_t s);
void launch_gemm2_simt(int dtype, const void* Hm, const void* W2, void* O, const GemmShape& sh,
                       const uint32_t* offsets, const uint32_t* mprefix, cudaStream_t s);
// gmap (nullable): group g's weights are B group gmap[g] (offload cache slots)
// starts (nullable): group g's rows are [starts[g], offsets[g+1])
// tmA_small (nullable): [3] maps of A with 16 / 32 / 64-row boxes (short tiles load only their rows)
// gather_tok (nullable, SwiGLU epilogue): A rows gathered from the token
//   matrix by TMA gather4 (tmA = map of x with {64, 1} boxes), token id of
//   permuted row r = gather_tok[r]; no x_perm
// tmO (nullable, plain epilogue): map of the output with 32 x 32 boxes, no swizzle
//   (make_tmap_bf16_2d_ex): full 32-row warp slabs leave through TMA stores
// gemm1 B tail: the packed W1 rows past `valid` neurons per group (padding to
// the 128-row tile) are not read; half = 128-row-box map, part = map with
// tail_rows-row boxes (valid % 64 rounded up to 8) of the packed W1.
struct GemmBTail {
    CUtensorMap half, part;
    uint32_t valid, tail_rows;
};
void launch_gemm_tc(bool swiglu, const CUtensorMap* tmA, const CUtensorMap* tmB, void* out, const GemmShape& sh,
                    const uint32_t* offsets, const uint32_t* mprefix, int num_sms, cudaStream_t s,
                    const uint32_t* gmap = nullptr, const uint32_t* starts = nullptr,
                    const CUtensorMap* tmA_small = nullptr, const CUtensorMap* tmO = nullptr,
                    const GemmBTail* btail = nullptr, const uint32_t* gather_tok = nullptr);
size_t gemm_tc_smem_bytes();
// Epilogue modes of the 1-SM tensor-core GEMM (gemm_tc.cu).
constexpr int kEpiPlain = 0;   // bf16 acc
constexpr int kEpiSwiglu = 1;  // bf16 silu(gate) * up (fused SwiGLU)
constexpr int kEpiActAbs = 2;  // fp32 |silu(gate) * up| scattered to colmap[packed neuron] (calibration)
constexpr int kEpiCount = 3;   // uint32 counts (co-activation of 0/1 operands)
constexpr int kEpiF32Part = 4; // fp32 split-K partials: out + split * max_rows * ld_out (ksplit of launch_gemm_tc_epi)
// b_row0: first B row; colmap: kEpiActAbs column map; out: bf16 / f32 / u32 per mode
void launch_gemm_tc_epi(int epi, const CUtensorMap* tmA, const CUtensorMap* tmB, void* out, const GemmShape& sh,
                        const uint32_t* offsets, const uint32_t* mprefix, int num_sms, cudaStream_t s,
                        uint32_t b_row0 = 0, const int32_t* colmap = nullptr, const uint32_t* gmap = nullptr,
                        const uint32_t* starts = nullptr, uint32_t ksplit = 1,
                        const CUtensorMap* tmA_small = nullptr, const CUtensorMap* tmO = nullptr,
                        const GemmBTail* btail = nullptr, const uint32_t* gather_tok = nullptr);
uint64_t* gemm_trace_buffer(bool swiglu);
uint64_t* gemm_trace_ptr(int which);
// CTA-pair (cta_group::2) 256 x 256 tiles; tmB box of 128 rows (gemm_tc2.cu);
// tmA_small (nullable): [3] maps of A with 16 / 32 / 64-row boxes -> remainder
// tiles run with swapped operands; tmO (nullable, plain epilogue): 32 x 32-box
// map of the output (whole warp slabs leave through TMA stores)
bool pair_swap_enabled();  // MOEPRISM_PAIR_SWAP (default on)
void launch_gemm_tc2(bool swiglu, const CUtensorMap* tmA, const CUtensorMap* tmB, void* out, const GemmShape& sh,
                     const uint32_t* offsets, const uint32_t* mprefix256, int num_sms, cudaStream_t s,
                     const uint32_t* gmap = nullptr, const CUtensorMap* tmA_small = nullptr,
                     const CUtensorMap* tmO = nullptr);

// Calibration (calib.cu).
void launch_binarize_topk(const float* act, uint32_t rows, uint32_t cols, uint32_t k_a, uint8_t* bits,
                          cudaStream_t s);
void launch_bits_to_bf16_t(const uint8_t* bits, uint32_t rows, uint32_t cols, uint32_t ld, void* out, cudaStream_t s);
void launch_centrality(const uint32_t* co, uint32_t dim, const uint32_t* label, const uint32_t* mem_off,
                       const uint32_t* members, unsigned long long* score, cudaStream_t s);
void launch_gate_select(const unsigned long long* score, const uint32_t* mem_off, const uint32_t* members,
                        uint32_t n_sub, uint32_t r, const uint32_t* out_off, uint32_t* out, cudaStream_t s);
void launch_fidelity(const float* act, uint32_t rows, uint32_t cols, uint32_t n_sub, const uint32_t* mem_off,
                     const uint32_t* members, const uint32_t* gate_off, const uint32_t* gate_ids, uint32_t k,
                     double* norm, double* proxy, double* recall, cudaStream_t s);
// meta = {0, rows, 0, ceil(rows / 128)}: offsets + 128-row tile prefix of one group
void launch_set_group_meta(uint32_t* meta, uint32_t rows, cudaStream_t s);

// One-time (per kernel, per device) dynamic shared-memory attribute; thread-safe
// (layer.cu).  max_carveout: also prefer the maximum shared-memory carveout.
void func_attr_once(const void* func, int max_dyn_smem, bool max_carveout = false);
// L2 prefetch of [p, p + bytes) with bulk prefetches (no data movement to SMs)
void launch_l2_prefetch(const void* p, size_t bytes, cudaStream_t s);
// max |p[i]| over n floats into *out (device, must be zeroed; atomic max on the bits)
void launch_absmax(const float* p, size_t n, float* out, cudaStream_t s);

// cuTensorMapEncodeTiled through the runtime's driver entry point.
bool make_tmap_bf16_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                       uint32_t box_cols);
// Same with a row pitch (elements) >= cols -- columns >= cols read as zeros /
// are not written --, a choice of 128-byte swizzle or none, and the L2
// promotion of the loads' misses (0 / 64 / 128 / 256 bytes; 256 re-reads
// up to 192 bytes of padding past a trimmed row end).
bool make_tmap_bf16_2d_ex(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t pitch,
                          uint32_t box_rows, uint32_t box_cols, bool swizzle128, uint32_t l2_promo = 256);

}  // namespace mp

namespace mp {
// Expert-parallel dispatch / combine (ep.cu).
void launch_ep_dest(const uint32_t* sel, uint32_t T, uint32_t k_max, uint32_t per_rank, uint32_t world, uint32_t* dest,
                    cudaStream_t s);
void launch_ep_slot(const uint32_t* dest, const uint32_t* lrank, const uint32_t* block_base, uint32_t T, uint32_t world,
                    uint32_t* slot_row, cudaStream_t s);
// dst_tables: device [3][world] destination pointers (x rows, sel, w); rows of
// rank r land at base[r] + (send position - send_off[r])
void launch_ep_pack(int dtype, const void* x, const uint32_t* sel, const float* w, uint32_t T, uint32_t d,
                    uint32_t k_max, uint32_t per_rank, uint32_t S, uint32_t world, const uint32_t* dest,
                    const uint32_t* slot_row, void* const* dst_tables, const uint32_t* base, const uint32_t* send_off,
                    cudaStream_t s);
void launch_ep_return(int dtype, const void* part, uint32_t n_recv, uint32_t d, uint32_t world, const uint32_t* roff,
                      const uint32_t* dbase, void* const* back, cudaStream_t s);
void launch_ep_combine(int dtype, const void* back, uint32_t T, uint32_t d, uint32_t world, const uint32_t* slot_row,
                       void* y, cudaStream_t s, const void* x_res = nullptr);
}  // namespace mp
