/*
 * moe_layer.h -- C-ABI of the B200-native MoE-Prism sub-expert MoE layer.
 *
 * The reference (MoE-Prism, /root/reference/proj) exposes its hot path only
 * as header-only C++ free functions; it has no FFI.  This header is the thin
 * C boundary a binding (ctypes / cgo / JNI / N-API) would load, and the C++
 * wrapper moe_layer.hpp sits on top of it with the reference's own
 * signatures.  Each entry point names the reference interface it replaces:
 *
 *   mp_layer_forward           <- per-token loop of partitioned_forward
 *                                 (inc/expert.hpp:101-135) composed over the
 *                                 selected sub-experts, plus the router
 *
 *   mp_layer_forward_selected  <- partitioned_forward with an explicit active
 *                                 set per token (inc/expert.hpp:101-135)
 *   mp_layer_route             <- select_topk_subexperts over router scores
 *                                 (inc/gating.hpp:129-145), linear or proxy
 *                                 (proxy_scores, inc/gating.hpp:107-125)
 *   mp_layer_load_expert[_file]<- ToyExpert / load_toy_expert
 *                                 (inc/expert.hpp:17-39, inc/io.hpp:225-251)
 *   mp_layer_set_partition     <- Partition + validate (inc/partition.hpp:15-46)
 *   mp_layer_load_partition_map<- read_ndjson + partition_doc_from_json
 *                                 (inc/serde.hpp:113-151, gates :160-168)
 *   mp_layer_set_gates         <- GateSet + validate (inc/gating.hpp:19-43)
 *
 * Conventions (mirroring inc/error.hpp:8-16):
 *   status 0 ok; 1 validation error (ValidationError); 2 I/O error (IoError);
 *   3 CUDA error.  mp_last_error() returns the calling thread's message.
 * Ownership: the layer owns its (packed, device-resident) weights; the caller
 * owns activations.  Device pointers are CUDA global memory on the layer's
 * device.  `stream` is a cudaStream_t (NULL = legacy default stream).
 * Threading: one handle per stream; forward is stream-ordered and not
 * re-entrant on one handle; distinct handles are independent.
 * There is no CPU fallback: every compute entry point launches CUDA kernels
 * and fails with status 3 when no sm_100a device is usable.
 */
#ifndef MOEPRISM_MOE_LAYER_H
#define MOEPRISM_MOE_LAYER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MP_OK 0
#define MP_ERR_VALIDATION 1
#define MP_ERR_IO 2
#define MP_ERR_CUDA 3

#define MP_DTYPE_F32 0  /* fp32 end to end: SIMT FFMA grouped GEMMs (1e-5 mode) */
#define MP_DTYPE_BF16 1 /* bf16 activations/weights, fp32 accumulate: tcgen05 */

#define MP_ROUTER_LINEAR 0 /* logits = x . W_r (fp32) */
#define MP_ROUTER_PROXY 1  /* proxy gate neurons, inc/gating.hpp:107-125 */

#define MP_WEIGHT_UNIT 0           /* y = sum of selected sub-expert outputs (reference) */
#define MP_WEIGHT_SOFTMAX_RENORM 1 /* y = sum p_g / sum_sel p * o_g */

#define MP_SEL_NONE 0xFFFFFFFFu /* padding in [T x k_max] selection arrays */
#define MP_MAX_SUBEXPERTS 256u  /* max E*S sub-experts of one layer (Qwen: 240) */

typedef int mp_status;
typedef struct mp_layer_s* mp_layer_t;

typedef struct {
    uint32_t n_experts;    /* E parent experts */
    uint32_t n_subexperts; /* S sub-experts per expert (Partition::n_subexperts) */
    uint32_t d_model;      /* d */
    uint32_t d_ff;         /* ffn neurons per expert */
    uint32_t dtype;        /* MP_DTYPE_* of x, y and the packed weights */
    uint32_t router_mode;  /* MP_ROUTER_* */
    uint32_t weight_mode;  /* MP_WEIGHT_* */
    uint32_t k_max;        /* max active sub-experts per token (<= E*S) */
    uint32_t max_tokens;   /* workspace capacity, tokens per forward */
    int32_t device;        /* CUDA device ordinal */
    uint32_t flags;        /* MP_LAYER_* role flags (0 = full layer) */
} mp_layer_desc;

/* Role flags for expert parallelism: a replicated router-only
 * layer routes every local token over all E*S sub-experts; an experts-only
 * layer holds this rank's E_local experts and runs mp_layer_forward_selected
 * on the tokens received from all ranks. */
#define MP_LAYER_ROUTER_ONLY 1u  /* no expert storage; mp_layer_route only */
#define MP_LAYER_EXPERTS_ONLY 2u /* no router; mp_layer_forward_selected only */
/* The per-forward token scratch (permuted rows, SwiGLU activations, expert
 * outputs: GBs at serving sizes) comes from a per-device pool shared by every
 * layer with this flag and the same shapes -- for layer stacks whose layers
 * run one after the other on one stream (32 layers). */
#define MP_LAYER_SHARED_SCRATCH 4u

/* Library / device info.  mp_device_check fails (3) unless device `dev` is an
 * sm_100 part this build has code for. */
const char* mp_version(void);
const char* mp_last_error(void);
mp_status mp_device_check(int32_t dev);

mp_status mp_layer_create(const mp_layer_desc* desc, mp_layer_t* out);
mp_status mp_layer_destroy(mp_layer_t h);
mp_status mp_layer_get_desc(mp_layer_t h, mp_layer_desc* out);

/* Expert e's weights in the MPEX layout (inc/io.hpp:210-223): w_gate, w_up
 * d_model x d_ff row-major fp32, w_down d_ff x d_model row-major fp32.
 * Host or device pointers.  Rejects non-finite weights (inc/expert.hpp:34).
 * The packer (neurons grouped per sub-expert, gate/up interleaved, zero
 * padded, cast to dtype) runs on the GPU once both the weights and the
 * partition of expert e are known. */
mp_status mp_layer_load_expert(mp_layer_t h, uint32_t e, const float* w_gate, const float* w_up, const float* w_down);
mp_status mp_layer_load_expert_file(mp_layer_t h, uint32_t e, const char* mpex_path);

/* Partition of expert e (inc/partition.hpp:15-46): assignment[j] = label of
 * neuron j, n == d_ff, balanced, all labels < n_sub == desc.n_subexperts. */
mp_status mp_layer_set_partition(mp_layer_t h, uint32_t e, uint32_t n_sub, const uint32_t* assignment, size_t n);
/* NDJSON partition map (inc/serde.hpp:100-151): one document per expert,
 * "expert_id" selects e.  Documents carrying "r"/"gates" also set the gate
 * set of that expert (inc/serde.hpp:156-168). */
mp_status mp_layer_load_partition_map(mp_layer_t h, const char* ndjson_path);

/* Linear router: w_r is d_model x (E*S) row-major fp32, host or device. */
mp_status mp_layer_set_router(mp_layer_t h, const float* w_r);
/* Shared (always-on) expert, Qwen1.5-MoE style (no
 * reference counterpart, restated in the oracle): every token adds
 * sigmoid(x . shared_gate) * toy_ffn_forward(shared, x) (inc/expert.hpp:79-96)
 * after its routed sub-experts.  MPEX layout (d_model x d_ff_shared w_gate /
 * w_up, d_ff_shared x d_model w_down), fp32, host or device; shared_gate is
 * d_model fp32 or NULL (weight 1).  bf16 full layers only; applied by
 * mp_layer_forward / mp_layer_forward_host (not by forward_selected, whose
 * semantics are partitioned_forward's explicit active sets). */
mp_status mp_layer_set_shared_expert(mp_layer_t h, uint32_t d_ff_shared, const float* w_gate, const float* w_up,
                                     const float* w_down, const float* shared_gate);

/* Fused residual (bf16 layers): mp_layer_forward / _host write
 * y = x + MoE(x) (the x_{l+1} = x_l + MoE_l(x_l) step of a layer stack,
 * SURVEY 8(d) C3), the residual being the combine's accumulator start value.
 * y must not alias x.  Off by default. */
mp_status mp_layer_set_residual(mp_layer_t h, int on);

/* Proxy router gate set of expert e (inc/gating.hpp:19-43) in CSR form:
 * ids[offsets[s] .. offsets[s+1]) are the ascending gate neurons of s. */
mp_status mp_layer_set_gates(mp_layer_t h, uint32_t e, uint32_t r, const uint32_t* offsets, const uint32_t* ids);

/* Layer forward on device buffers.  x, y: T x d_model of desc.dtype.
 * k_per_token (device, nullable): per-token active count, each in
 * [1, k_max]; when NULL every token uses k.  Optional device outputs:
 * sel_out T x k_max (ascending ids, MP_SEL_NONE padded), w_out T x k_max
 * combine weights, offsets_out E*S+1 bucket offsets. */
mp_status mp_layer_forward(mp_layer_t h, const void* x, uint32_t n_tokens, const uint32_t* k_per_token, uint32_t k,
                           void* y, uint32_t* sel_out, float* w_out, uint32_t* offsets_out, void* stream);

/* Same, on HOST buffers (pinned or pageable): copies x (and k_per_token) in,
 * runs, copies y (and the optional outputs) out, synchronises the stream. */
mp_status mp_layer_forward_host(mp_layer_t h, const void* x, uint32_t n_tokens, const uint32_t* k_per_token,
                                uint32_t k, void* y, uint32_t* sel_out, float* w_out, uint32_t* offsets_out,
                                void* stream);

/* A sequence of forwards on HOST buffers with the copies pipelined against
 * the compute: batch i's upload (own stream) and download (own stream)
 * overlap the compute of its neighbours through two device staging slots.
 * xs[i], ys[i]: host n_tokens[i] x d_model buffers of the layer dtype (pinned
 * for the copies to overlap); one k for every token.  Synchronises before
 * returning; device validation flags raise like mp_layer_forward_host. */
mp_status mp_layer_forward_host_batches(mp_layer_t h, uint32_t n_batches, const void* const* xs,
                                        const uint32_t* n_tokens, uint32_t k, void* const* ys, void* stream);

/* Forward with an explicit selection (device, T x k_max, ascending global
 * sub-expert ids e*S+s, MP_SEL_NONE padded; duplicates rejected on the
 * host path).  w (device, nullable): per-slot weights; NULL = unit weights,
 * i.e. partitioned_forward semantics summed over experts. */
mp_status mp_layer_forward_selected(mp_layer_t h, const void* x, uint32_t n_tokens, const uint32_t* sel,
                                    const float* w, void* y, uint32_t* offsets_out, void* stream);
/* Same on HOST buffers (sel / w host too); validates the selection on the
 * host first (range, duplicates: inc/expert.hpp:111-118), synchronises. */
mp_status mp_layer_forward_selected_host(mp_layer_t h, const void* x, uint32_t n_tokens, const uint32_t* sel,
                                         const float* w, void* y, void* stream);

/* Router only: selection + weights (device outputs, T x k_max). */
mp_status mp_layer_route(mp_layer_t h, const void* x, uint32_t n_tokens, const uint32_t* k_per_token, uint32_t k,
                         uint32_t* sel_out, float* w_out, void* stream);

/* Routing statistics of the last mp_layer_forward / mp_layer_route on this
 * handle (synchronises `stream`): reselected = tokens whose tensor-core
 * selection was not certified by the per-token error bound (or that may be a
 * near tie) and were re-selected from exact fp64 logits; near_ties = tokens
 * whose exact k-th/(k+1)-th logit gap is < 1e-6 (the routing contract's
 * near-tie window, reported separately).  Either pointer may be NULL. */
mp_status mp_layer_route_stats(mp_layer_t h, uint32_t* reselected, uint32_t* near_ties, void* stream);

/* Device-side validation flags raised by forwards on device buffers (k out of
 * range, duplicate / out-of-range selection, non-finite input): synchronises
 * `stream`, returns 1 with the message if any were raised, then clears them.
 * (mp_layer_forward_host checks them itself.) */
mp_status mp_layer_check_errors(mp_layer_t h, void* stream);

/* Per-stage device timing with CUDA events on the forward's stream.
 * names: comma-separated stage list; ms/launches: per stage accumulated
 * since the last reset.  Returns the number of stages in *n. */
mp_status mp_layer_set_profiling(mp_layer_t h, int on);
mp_status mp_layer_stage_times(mp_layer_t h, char* names, size_t names_len, double* ms, uint64_t* launches,
                               uint32_t* n, uint32_t cap);
mp_status mp_layer_reset_stage_times(mp_layer_t h);
/* Kernels launched by this handle since creation. */
uint64_t mp_layer_launch_count(mp_layer_t h);

/* Counter-based synthetic data (the generator of oracle/moe_oracle.c
 * orc_synth_fill, bit-identical): dst[j] = dtype(float((u*2-1)*scale)),
 * u = stream(seed) element first+j.  Device dst. */
mp_status mp_synth_fill(void* dst, uint32_t dtype, size_t n, uint64_t seed, uint64_t first, double scale,
                        void* stream);

/* ---- expert parallelism: token dispatch / combine across ranks ----
 * Sub-experts are sharded by parent expert: rank r owns the global ids
 * [r * experts_per_rank * S, (r + 1) * experts_per_rank * S).  For one layer:
 *   mp_layer_route (router-only layer) -> sel, w  [T x k_max], global ids
 *   mp_ep_plan:    destination ranks per token (deduplicated, ascending),
 *                  per-rank send counts (host), stable order by token
 *   mp_ep_pack:    send rows x[t] once per destination rank, with the
 *                  selection re-expressed in that rank's local ids + weights
 *   -- all-to-all of rows / metadata (NCCL, by the host runtime) --
 *   mp_layer_forward_selected (experts-only layer) on the received rows
 *   -- all-to-all of the per-(token, rank) partial outputs back --
 *   mp_ep_combine: y[t] = sum over destination ranks in ascending order
 *                  (deterministic; fp32 accumulate).
 * send_sel / send_w are [rows x k_max]; rows are grouped by destination rank
 * in rank order, tokens ascending inside a group. */
typedef struct mp_ep_s* mp_ep_t;
mp_status mp_ep_create(uint32_t world, uint32_t rank, uint32_t experts_per_rank, uint32_t n_subexperts,
                       uint32_t d_model, uint32_t k_max, uint32_t max_tokens, uint32_t dtype, int32_t device,
                       mp_ep_t* out);
/* Sub-expert-granularity sharding (SURVEY 8(e), E not divisible by the world
 * size, e.g. Qwen 240 sub-experts over 8 GPUs): rank r owns global ids
 * [r*per_rank, (r+1)*per_rank); its experts-only layer holds parent experts
 * floor(r*per_rank/S) .. floor(((r+1)*per_rank-1)/S) and receives selections
 * in local ids g - floor(r*per_rank/S)*S.  mp_ep_create == per_rank = epr*S. */
mp_status mp_ep_create_subexpert(uint32_t world, uint32_t rank, uint32_t per_rank, uint32_t S, uint32_t d,
                                 uint32_t k_max, uint32_t max_tokens, uint32_t dtype, int32_t device, mp_ep_t* out);
mp_status mp_ep_destroy(mp_ep_t ep);
/* sel: device [T x k_max] global ids.  send_counts: HOST [world] (synchronises). */
mp_status mp_ep_plan(mp_ep_t ep, const uint32_t* sel, uint32_t n_tokens, uint32_t* send_counts, void* stream);
/* x: device [T x d] of dtype; outputs device [sum(send_counts) x ...]. */
mp_status mp_ep_pack(mp_ep_t ep, const void* x, const uint32_t* sel, const float* w, uint32_t n_tokens,
                     void* send_x, uint32_t* send_sel, float* send_w, void* stream);
/* back: device [sum(send_counts) x d] partial outputs (dtype), in send order. */
mp_status mp_ep_combine(mp_ep_t ep, const void* back, uint32_t n_tokens, void* y, void* stream);

/* ---- expert-parallel layer forward with an NCCL transport (C++ host) ----
 * The whole layer on this rank's tokens in one call, no Python on the path:
 *   mp_layer_route (router: a MP_LAYER_ROUTER_ONLY layer, replicated) ->
 *   plan (destination ranks per token, deduplicated) -> count matrix
 *   (ncclAllGather; the layer's one host synchronisation -- NCCL needs the
 *   all-to-allv sizes on the host) -> pack -> rows + selections + weights by
 *   grouped ncclSend/ncclRecv (all-to-allv over NVLink/NVSwitch) ->
 *   mp_layer_forward_selected (experts: this rank's MP_LAYER_EXPERTS_ONLY
 *   layer, max_tokens >= world * ep max_tokens) -> partials returned the same
 *   way -> combine in ascending rank order (deterministic).
 * The communicator: rank 0 calls mp_ep_nccl_unique_id, the host runtime
 * broadcasts the 128 bytes (MPI, a TCP store, torch.distributed), every rank
 * calls mp_ep_nccl_init (collective).  NCCL is loaded at run time
 * (libnccl.so.2; the process's own copy when one is loaded).
 * flags: MP_EP_RESIDUAL -> y = x + MoE(x) (layer stacks).
 * x, y: device [n_tokens x d_model] of the ep dtype; k_per_token: device or
 * NULL.  mp_ep_last_counts: rows sent to / received from each rank by the
 * last mp_ep_forward (host arrays of `world` entries, either may be NULL). */
#define MP_EP_NCCL_ID_BYTES 128
#define MP_EP_RESIDUAL 1u
mp_status mp_ep_nccl_unique_id(uint8_t* id);
mp_status mp_ep_nccl_init(mp_ep_t ep, const uint8_t* id);
mp_status mp_ep_forward(mp_ep_t ep, mp_layer_t router, mp_layer_t experts, const void* x, uint32_t n_tokens,
                        const uint32_t* k_per_token, uint32_t k, void* y, uint32_t flags, void* stream);
mp_status mp_ep_last_counts(mp_ep_t ep, uint32_t* send_rows, uint32_t* recv_rows);

/* ---- Sub-expert offload cache (the reference simulates it:
 * cache_step / run_offload_sim, inc/offload.hpp:202-290). ----
 * mp_layer_enable_offload moves the packed weights to pinned host memory and
 * keeps a device cache of cache_units units (unit_subexperts = 1: one
 * sub-expert, "fine"; = S: a whole expert, "monolithic").  Every forward then
 * reads its bucket sizes back (the stream is synchronised), runs one
 * cache_step with the reference's LRU policy over the units that received
 * tokens, copies the misses host->device and computes from the cache.
 * Outputs are bit-identical to the resident layer.  Fails if one forward
 * needs more units than the cache holds (the reference's ValidationError).
 * mp_layer_offload_stats: cumulative hits / misses / bytes, and the last
 * forward's requested units (ascending) and miss count. */
mp_status mp_layer_enable_offload(mp_layer_t h, uint32_t unit_subexperts, uint32_t cache_units);
mp_status mp_layer_offload_stats(mp_layer_t h, uint64_t* hits, uint64_t* misses, uint64_t* bytes_h2d,
                                 uint32_t* last_units, uint32_t cap, uint32_t* n_last, uint32_t* last_misses);

/* ---- Calibration: the activation profile the offline
 * refactoring engine partitions experts with, computed on the GPU. ----
 * mp_layer_collect_activations <- collect_activation_matrix
 *   (inc/expert.hpp:137-151): act[b][j] = |a_j(x_b)| of expert e, fp32,
 *   B x d_ff row-major in the ORIGINAL neuron order; x device B x d_model of
 *   the layer dtype (bf16 layers: the fused SwiGLU GEMM with an |a|
 *   epilogue, bf16 operands / fp32 accumulation).
 * mp_binarize_topk <- binarize_topk (inc/activation.hpp:213-240): per row
 *   the k_a largest magnitudes -> 1, ties to the lower column; device
 *   act [rows x cols] fp32 -> bits [rows x cols] u8.  Exact.
 * mp_coactivation <- coactivation (inc/activation.hpp:242-266):
 *   co[i][j] = #rows with bits i and j set; device bits -> co [cols x cols]
 *   u32, a tensor-core GEMM over the 0/1 matrix (exact, rows <= 2^24). */
mp_status mp_layer_collect_activations(mp_layer_t h, uint32_t e, const void* x, uint32_t B, float* act,
                                       void* stream);
mp_status mp_binarize_topk(const float* act, uint32_t rows, uint32_t cols, uint32_t k_a, uint8_t* bits,
                           void* stream);
mp_status mp_coactivation(const uint8_t* bits, uint32_t rows, uint32_t cols, uint32_t* co, void* stream);
/* select_gate_neurons (inc/gating.hpp:72-103) on a device co-activation
 * matrix: per sub-expert the r most central members (co-activation with the
 * other members, diagonal excluded, ties to the lower neuron), ascending; host
 * outputs gate_offsets[n_sub+1], gate_ids[...] (capacity <= dim). Exact. */
mp_status mp_select_gate_neurons(const uint32_t* co, uint32_t dim, uint32_t n_sub, const uint32_t* assignment,
                                 uint32_t r, uint32_t* gate_offsets, uint32_t* gate_ids, void* stream);
/* gating_fidelity (inc/gating.hpp:149-174): mean top-k recall of the proxy
 * selection against the true sub-expert norms over the rows of a device
 * activation matrix; partition and gate set (CSR) on the host. */
mp_status mp_gating_fidelity(const float* act, uint32_t rows, uint32_t cols, uint32_t n_sub,
                             const uint32_t* assignment, const uint32_t* gate_offsets, const uint32_t* gate_ids,
                             uint32_t k, double* out, void* stream);

/* Peer-memory exchange (the all-to-alls as direct stores into the peers'
 * buffers: CUDA IPC handles, NVLink between the GPUs of a node).
 * setup: allocates this rank's receive (x rows, selection, weights) and
 *   return buffers and writes their 4 IPC handles (4 x 64 bytes) to `handles`;
 * open: all_handles = every rank's 4 handles, rank-major (world x 256 bytes);
 * p2p_pack: after mp_ep_plan, with counts = the all-gathered plan
 *   (world x world, counts[s*world + d] = rows s sends to d): writes this
 *   rank's rows straight into each destination's receive buffer; *n_recv =
 *   rows this rank will receive.  The caller then makes every rank's pack
 *   complete (stream sync + a host barrier) before the expert layers read;
 * recv_buffers: the receive buffers (rows grouped by source rank, ascending);
 * p2p_return: the expert partials (n_recv x d) go straight back into the
 *   sources' return buffers; barrier again; p2p_combine: as mp_ep_combine
 *   from this rank's return buffer. */
mp_status mp_ep_p2p_setup(mp_ep_t ep, uint32_t max_recv_rows, uint8_t* handles);
mp_status mp_ep_p2p_open(mp_ep_t ep, const uint8_t* all_handles);
mp_status mp_ep_p2p_pack(mp_ep_t ep, const void* x, const uint32_t* sel, const float* w, uint32_t n_tokens,
                         const uint32_t* counts, uint32_t* n_recv, void* stream);
mp_status mp_ep_p2p_recv_buffers(mp_ep_t ep, void** recv_x, uint32_t** recv_sel, float** recv_w);
mp_status mp_ep_p2p_return(mp_ep_t ep, const void* part, uint32_t n_recv, void* stream);
mp_status mp_ep_p2p_combine(mp_ep_t ep, uint32_t n_tokens, void* y, void* stream);

/* Host-only readers (no GPU touched), format-compatible with the reference.
 * mp_format_read_mpex <- load_toy_expert (inc/io.hpp:225-251): call with
 * null weight pointers to learn the dims, then with d_model*d_ff buffers.
 * mp_format_read_partition_doc <- read_ndjson + partition_doc_from_json +
 * gate_set_from_json (inc/serde.hpp:113-168): document `index`; null output
 * pointers are skipped (two-phase like the MPEX reader).
 * mp_validate_partition <- validate(Partition) (inc/partition.hpp:34-46). */
mp_status mp_format_read_mpex(const char* path, uint32_t* d_model, uint32_t* d_ff, float* w_gate, float* w_up,
                              float* w_down);
mp_status mp_format_read_partition_doc(const char* path, size_t index, size_t* n_docs, uint64_t* expert_id,
                                       uint32_t* n_sub, size_t* n, uint32_t* assignment, uint32_t* r,
                                       size_t* n_gate_ids, uint32_t* gate_offsets, uint32_t* gate_ids);
mp_status mp_validate_partition(uint32_t n_sub, const uint32_t* assignment, size_t n);
/* MPAM activation matrix <- save_activation_matrix / load_activation_matrix
 * (inc/io.hpp:147-200, binary): the reader rectifies |v|, rejects trailing
 * bytes and non-finite values; two-phase (data NULL -> dims only). */
mp_status mp_format_write_mpam(const char* path, uint32_t rows, uint32_t cols, const float* data);
mp_status mp_format_read_mpam(const char* path, uint32_t* rows, uint32_t* cols, float* data);

#ifdef __cplusplus
}
#endif
#endif /* MOEPRISM_MOE_LAYER_H */
