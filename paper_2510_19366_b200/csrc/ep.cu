// ep.cu -- expert-parallel token dispatch / combine.
//
// Sub-experts are sharded in contiguous global-id ranges: rank r owns
// [r*per_rank, (r+1)*per_rank) -- whole parent experts when per_rank is a
// multiple of S, else sub-expert granularity (Qwen: 240 / 8 = 30 per rank,
// SURVEY 8(e)); a rank's experts-only layer then holds the parent experts its
// range touches and numbers sub-experts from base(r) = floor(r*per_rank/S)*S.  A token is sent ONCE to every rank owning at least
// one of its selected sub-experts (dedup), together with its selection
// re-expressed in that rank's local ids and the combine weights; the owner
// returns one weighted partial per (token, rank) and the source sums them in
// ascending rank order (deterministic).  The per-destination ordering reuses
// the layer's bucketing kernels (buckets = ranks, stable by token), so send
// rows are grouped by rank, tokens ascending -- the layout an NCCL
// all-to-allv (grouped ncclSend/ncclRecv) consumes directly.
#include <cstring>
#include <exception>
#include <new>
#include <string>
#include <vector>

#include "moeprism/moe_layer.h"
#include "mp_common.cuh"
#include "mp_kernels.h"

#define MP_API extern "C" __attribute__((visibility("default")))

namespace mp {
namespace {

// dest[t][0..world): ascending destination ranks of token t, MP_SEL_NONE padded
__global__ void ep_dest_kernel(const uint32_t* __restrict__ sel, uint32_t T, uint32_t k_max, uint32_t per_rank,
                               uint32_t world, uint32_t* __restrict__ dest) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    uint32_t mask = 0;  // world <= 32
    for (uint32_t j = 0; j < k_max; ++j) {
        const uint32_t g = sel[(size_t)t * k_max + j];
        if (g != kSelNone) mask |= 1u << min(g / per_rank, 31u);
    }
    uint32_t n = 0;
    for (uint32_t r = 0; r < world; ++r)
        if ((mask >> r) & 1u) dest[(size_t)t * world + n++] = r;
    for (; n < world; ++n) dest[(size_t)t * world + n] = kSelNone;
}

// slot_row[t][j] = position of (token t, its j-th destination rank) in the
// rank-grouped send buffer = bucket base of (t's CTA block, rank) + local rank
__global__ void ep_slot_kernel(const uint32_t* __restrict__ dest, const uint32_t* __restrict__ lrank,
                               const uint32_t* __restrict__ block_base, uint32_t T, uint32_t world,
                               uint32_t* __restrict__ slot_row) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= T * world) return;
    const uint32_t t = q / world;
    const uint32_t r = dest[q];
    slot_row[q] = r == kSelNone ? kSelNone
                                : block_base[(size_t)(t / kRouteTokensPerBlock) * world + r] + lrank[q];
}

// Destinations of the packed rows: with P2P, rank r's rows go straight into
// rank r's receive buffers (CUDA IPC / NVLink peer pointers) at row
// base[r] + (pos - send_off[r]); locally (NCCL path) every destination is the
// one send buffer with base[r] = send_off[r], i.e. row = pos.
struct EpDest {
    void* const* x;           // [world] row buffers
    uint32_t* const* sel;     // [world] selection buffers
    float* const* w;          // [world] weight buffers
    const uint32_t* base;     // [world] first row of this rank's segment in the destination
    const uint32_t* send_off; // [world + 1] send-order offsets (bucket offsets, buckets = ranks)
};

template <typename Tx>
__global__ void __launch_bounds__(256) ep_pack_kernel(const Tx* __restrict__ x, const uint32_t* __restrict__ sel,
                                                      const float* __restrict__ w, uint32_t T, uint32_t d,
                                                      uint32_t k_max, uint32_t per_rank, uint32_t S, uint32_t world,
                                                      const uint32_t* __restrict__ dest,
                                                      const uint32_t* __restrict__ slot_row, EpDest D) {
    const uint32_t t = blockIdx.x * 8 + threadIdx.x / 32;
    const uint32_t lane = threadIdx.x & 31;
    if (t >= T) return;
    for (uint32_t j = 0; j < world; ++j) {
        const uint32_t r = dest[(size_t)t * world + j];
        if (r == kSelNone) break;
        const uint32_t pos = D.base[r] + slot_row[(size_t)t * world + j] - D.send_off[r];
        Tx* send_x = static_cast<Tx*>(D.x[r]);
        uint32_t* send_sel = D.sel[r];
        float* send_w = D.w[r];
        // metadata: the token's selection restricted to rank r, local ids
        if (lane == 0) {
            uint32_t n = 0;
            for (uint32_t q = 0; q < k_max; ++q) {
                const uint32_t g = sel[(size_t)t * k_max + q];
                if (g != kSelNone && g / per_rank == r) {
                    send_sel[(size_t)pos * k_max + n] = g - (r * per_rank / S) * S;  // local id on rank r
                    send_w[(size_t)pos * k_max + n] = w ? w[(size_t)t * k_max + q] : 1.0f;
                    ++n;
                }
            }
            for (; n < k_max; ++n) {
                send_sel[(size_t)pos * k_max + n] = kSelNone;
                send_w[(size_t)pos * k_max + n] = 0.0f;
            }
        }
        // the row itself, 16-byte vectors when aligned
        constexpr uint32_t VE = 16 / sizeof(Tx);
        const Tx* src = x + (size_t)t * d;
        Tx* dst = send_x + (size_t)pos * d;
        if ((d % VE) == 0) {
            for (uint32_t c = lane * VE; c < d; c += 32 * VE)
                *reinterpret_cast<uint4*>(dst + c) = __ldg(reinterpret_cast<const uint4*>(src + c));
        } else {
            for (uint32_t c = lane; c < d; c += 32) dst[c] = src[c];
        }
    }
}

// y[t] = (x_res[t] +) sum of the token's partials in ascending rank order
template <typename Tx>
__global__ void __launch_bounds__(256) ep_combine_kernel(const Tx* __restrict__ back, uint32_t T, uint32_t d,
                                                         uint32_t world, const uint32_t* __restrict__ slot_row,
                                                         const Tx* __restrict__ x_res, Tx* __restrict__ y) {
    __shared__ uint32_t rows[32];
    const uint32_t t = blockIdx.x;
    if (threadIdx.x < world) rows[threadIdx.x] = slot_row[(size_t)t * world + threadIdx.x];
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < d; c += blockDim.x) {
        float acc = x_res ? to_f32(x_res[(size_t)t * d + c]) : 0.0f;  // fused residual: the start value
        for (uint32_t j = 0; j < world; ++j) {
            const uint32_t r = rows[j];
            if (r == kSelNone) break;
            acc += to_f32(back[(size_t)r * d + c]);
        }
        y[(size_t)t * d + c] = from_f32<Tx>(acc);
    }
}

// P2P return: received row q (from source s = segment of q in roff) goes back
// into source s's back buffer at row dbase[s] + (q - roff[s]) -- the source's
// send position, so its combine reads it like the NCCL path's return.
template <typename Tx>
__global__ void __launch_bounds__(256) ep_return_kernel(const Tx* __restrict__ part, uint32_t n_recv, uint32_t d,
                                                        uint32_t world, const uint32_t* __restrict__ roff,
                                                        const uint32_t* __restrict__ dbase, void* const* back) {
    const uint32_t q = blockIdx.x * 8 + threadIdx.x / 32;
    const uint32_t lane = threadIdx.x & 31;
    if (q >= n_recv) return;
    uint32_t s = 0;
    while (s + 1 < world && roff[s + 1] <= q) ++s;
    Tx* dst = static_cast<Tx*>(back[s]) + (size_t)(dbase[s] + q - roff[s]) * d;
    const Tx* src = part + (size_t)q * d;
    constexpr uint32_t VE = 16 / sizeof(Tx);
    if ((d % VE) == 0) {
        for (uint32_t c = lane * VE; c < d; c += 32 * VE)
            *reinterpret_cast<uint4*>(dst + c) = __ldg(reinterpret_cast<const uint4*>(src + c));
    } else {
        for (uint32_t c = lane; c < d; c += 32) dst[c] = src[c];
    }
}

}  // namespace
}  // namespace mp

#include "mp_ep_impl.h"

namespace {
thread_local std::string g_ep_err;
struct EpErr {
    int code;
    std::string msg;
};
[[noreturn]] void ep_fail(int code, const std::string& m) { throw EpErr{code, m}; }
void ep_ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) ep_fail(MP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
template <class F>
int ep_guarded(F&& f);
void ep_free(mp_ep_s* E) {
    if (E->nccl) mp_ep_nccl_free(E);
    for (void* p : E->opened) cudaIpcCloseMemHandle(p);
    void* ptrs[] = {E->dest, E->ws.lrank, E->ws.block_counts, E->ws.block_base, E->ws.offsets, E->ws.mprefix_tc,
                    E->ws.mprefix_simt, E->ws.mprefix_tc2, E->ws.perm_tok, E->ws.perm_w, E->ws.slot_row, E->ws.err,
                    E->recv_x, E->recv_sel, E->recv_w, E->back, E->d_px, E->d_meta};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    delete E;
}
template <class T>
T* ep_alloc(size_t n) {
    void* p = nullptr;
    ep_ck(cudaMalloc(&p, (n ? n : 1) * sizeof(T)), "ep alloc");
    return static_cast<T*>(p);
}
}  // namespace

// Errors surface through mp_last_error(); layer.cu owns that buffer, so the
// EP entry points report through a setter it exports.
extern "C" void mp_internal_set_error(const char* msg);

namespace {
template <class F>
int ep_guarded(F&& f) {
    try {
        f();
        return MP_OK;
    } catch (const EpErr& e) {
        mp_internal_set_error(e.msg.c_str());
        return e.code;
    } catch (const std::bad_alloc&) {
        mp_internal_set_error("host out of memory");
        return MP_ERR_CUDA;
    } catch (const std::exception& e) {
        mp_internal_set_error(e.what());
        return MP_ERR_CUDA;
    }
}

// Every entry point runs on the handle's device and restores the caller's.
struct EpDeviceGuard {
    int prev = -1;
    explicit EpDeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) ep_ck(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~EpDeviceGuard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};
}  // namespace

namespace {
// device pointer tables: [0, 4w) peers (x, sel, w, back), [4w, 7w) local send
// destinations; meta [4][w+1]
void ensure_tables(mp_ep_s* E) {
    if (!E->d_px) E->d_px = ep_alloc<void*>(8 * (size_t)E->world);
    if (!E->d_meta) E->d_meta = ep_alloc<uint32_t>(4 * ((size_t)E->world + 1));
}
}  // namespace

MP_API mp_status mp_ep_create_subexpert(uint32_t world, uint32_t rank, uint32_t per_rank, uint32_t S, uint32_t d,
                                        uint32_t k_max, uint32_t max_tokens, uint32_t dtype, int32_t device,
                                        mp_ep_t* out) {
    return ep_guarded([&] {
        if (!out) ep_fail(MP_ERR_VALIDATION, "null argument");
        if (world < 1 || world > 32 || rank >= world) ep_fail(MP_ERR_VALIDATION, "bad world / rank");
        if (per_rank < 1 || S < 1 || d < 1 || k_max < 1 || k_max > 256 || max_tokens < 1)
            ep_fail(MP_ERR_VALIDATION, "bad expert-parallel shape");
        if (dtype != MP_DTYPE_F32 && dtype != MP_DTYPE_BF16) ep_fail(MP_ERR_VALIDATION, "unknown dtype");
        EpDeviceGuard dg(device);
        auto* E = new mp_ep_s{world, rank, per_rank, S, d, k_max, max_tokens, dtype, device};
        try {
            const size_t tw = (size_t)max_tokens * world;
            const uint32_t nblk = (max_tokens + mp::kRouteTokensPerBlock - 1) / mp::kRouteTokensPerBlock;
            E->dest = ep_alloc<uint32_t>(tw);
            E->ws.lrank = ep_alloc<uint32_t>(tw);
            E->ws.block_counts = ep_alloc<uint32_t>((size_t)nblk * world);
            E->ws.block_base = ep_alloc<uint32_t>((size_t)nblk * world);
            E->ws.offsets = ep_alloc<uint32_t>(world + 1);
            E->ws.mprefix_tc = ep_alloc<uint32_t>(world + 1);
            E->ws.mprefix_simt = ep_alloc<uint32_t>(world + 1);
            E->ws.mprefix_tc2 = ep_alloc<uint32_t>(world + 1);
            E->ws.perm_tok = ep_alloc<uint32_t>(tw);
            E->ws.perm_w = ep_alloc<float>(tw);
            E->ws.slot_row = ep_alloc<uint32_t>(tw);
            E->ws.err = ep_alloc<int>(1);
            ep_ck(cudaMemset(E->ws.err, 0, sizeof(int)), "memset");
        } catch (...) {
            ep_free(E);
            throw;
        }
        *out = E;
    });
}

MP_API mp_status mp_ep_create(uint32_t world, uint32_t rank, uint32_t epr, uint32_t S, uint32_t d, uint32_t k_max,
                              uint32_t max_tokens, uint32_t dtype, int32_t device, mp_ep_t* out) {
    if (epr < 1 || S < 1) {
        mp_internal_set_error("bad expert-parallel shape");
        return MP_ERR_VALIDATION;
    }
    return mp_ep_create_subexpert(world, rank, epr * S, S, d, k_max, max_tokens, dtype, device, out);
}

MP_API mp_status mp_ep_destroy(mp_ep_t E) {
    return ep_guarded([&] {
        if (E) {
            EpDeviceGuard dg(E->device);
            cudaDeviceSynchronize();
            ep_free(E);
        }
    });
}

MP_API mp_status mp_ep_plan(mp_ep_t E, const uint32_t* sel, uint32_t T, uint32_t* send_counts, void* stream) {
    return ep_guarded([&] {
        if (!E || !send_counts || (T && !sel)) ep_fail(MP_ERR_VALIDATION, "null argument");
        EpDeviceGuard dg(E->device);
        if (T > E->max_tokens) ep_fail(MP_ERR_VALIDATION, "n_tokens exceeds max_tokens");
        E->last_T = T;
        if (T == 0) {
            for (uint32_t r = 0; r < E->world; ++r) send_counts[r] = 0;
            return;
        }
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        mp::launch_ep_dest(sel, T, E->k_max, E->per_rank, E->world, E->dest, s);
        mp::launch_bucket_local(E->dest, T, E->world, E->world, E->ws, s);
        mp::launch_bucket_scan(T, E->world, E->ws, s);
        mp::launch_ep_slot(E->dest, E->ws.lrank, E->ws.block_base, T, E->world, E->ws.slot_row, s);
        ep_ck(cudaGetLastError(), "ep plan");
        std::vector<uint32_t> off(E->world + 1);
        ep_ck(cudaMemcpyAsync(off.data(), E->ws.offsets, (E->world + 1) * 4, cudaMemcpyDeviceToHost, s), "counts");
        ep_ck(cudaStreamSynchronize(s), "ep plan sync");
        for (uint32_t r = 0; r < E->world; ++r) send_counts[r] = off[r + 1] - off[r];
    });
}

MP_API mp_status mp_ep_pack(mp_ep_t E, const void* x, const uint32_t* sel, const float* w, uint32_t T, void* send_x,
                            uint32_t* send_sel, float* send_w, void* stream) {
    return ep_guarded([&] {
        if (!E || (T && (!x || !sel || !send_x || !send_sel || !send_w))) ep_fail(MP_ERR_VALIDATION, "null argument");
        EpDeviceGuard dg(E->device);
        if (T != E->last_T) ep_fail(MP_ERR_VALIDATION, "mp_ep_pack must follow mp_ep_plan for the same tokens");
        if (T == 0) return;
        // identity destinations: every rank's segment of the one send buffer
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        ensure_tables(E);
        std::vector<void*> px(4 * (size_t)E->world);
        for (uint32_t r = 0; r < E->world; ++r) {
            px[r] = send_x;
            px[E->world + r] = send_sel;
            px[2 * E->world + r] = send_w;
        }
        ep_ck(cudaMemcpyAsync(E->d_px + 4 * E->world, px.data(), 3 * E->world * sizeof(void*), cudaMemcpyHostToDevice,
                              s),
              "ep tables");
        mp::launch_ep_pack(E->dtype, x, sel, w, T, E->d, E->k_max, E->per_rank, E->S, E->world, E->dest,
                           E->ws.slot_row, E->d_px + 4 * E->world, E->ws.offsets, E->ws.offsets, s);
        ep_ck(cudaGetLastError(), "ep pack");
    });
}

// ---- peer-memory exchange (CUDA IPC handles; NVLink peer stores between GPUs) ----

MP_API mp_status mp_ep_p2p_setup(mp_ep_t E, uint32_t max_recv_rows, uint8_t* handles) {
    return ep_guarded([&] {
        if (!E || !handles) ep_fail(MP_ERR_VALIDATION, "null argument");
        if (E->p2p || E->recv_x) ep_fail(MP_ERR_VALIDATION, "peer-memory exchange already set up");
        if (max_recv_rows < 1) ep_fail(MP_ERR_VALIDATION, "max_recv_rows must be >= 1");
        EpDeviceGuard dg(E->device);
        const size_t esz = E->dtype == MP_DTYPE_BF16 ? 2 : 4;
        E->max_recv = max_recv_rows;
        E->recv_x = ep_alloc<char>((size_t)max_recv_rows * E->d * esz);
        E->recv_sel = ep_alloc<uint32_t>((size_t)max_recv_rows * E->k_max);
        E->recv_w = ep_alloc<float>((size_t)max_recv_rows * E->k_max);
        E->back = ep_alloc<char>((size_t)E->max_tokens * E->world * E->d * esz);
        void* bufs[4] = {E->recv_x, E->recv_sel, E->recv_w, E->back};
        for (int i = 0; i < 4; ++i) {
            cudaIpcMemHandle_t h;
            ep_ck(cudaIpcGetMemHandle(&h, bufs[i]), "cudaIpcGetMemHandle");
            std::memcpy(handles + i * sizeof(cudaIpcMemHandle_t), &h, sizeof(h));
        }
        ensure_tables(E);
    });
}

MP_API mp_status mp_ep_p2p_open(mp_ep_t E, const uint8_t* all_handles) {
    return ep_guarded([&] {
        if (!E || !all_handles) ep_fail(MP_ERR_VALIDATION, "null argument");
        if (!E->recv_x) ep_fail(MP_ERR_VALIDATION, "mp_ep_p2p_setup first");
        EpDeviceGuard dg(E->device);
        const size_t hs = sizeof(cudaIpcMemHandle_t);
        std::vector<void*> px(4 * (size_t)E->world);
        void* own[4] = {E->recv_x, E->recv_sel, E->recv_w, E->back};
        for (uint32_t r = 0; r < E->world; ++r)
            for (int i = 0; i < 4; ++i) {
                void* p = own[i];
                if (r != E->rank) {
                    cudaIpcMemHandle_t h;
                    std::memcpy(&h, all_handles + (r * 4 + i) * hs, hs);
                    ep_ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
                    E->opened.push_back(p);
                }
                px[i * E->world + r] = p;
            }
        ep_ck(cudaMemcpy(E->d_px, px.data(), px.size() * sizeof(void*), cudaMemcpyHostToDevice), "peer table");
        E->p2p = true;
    });
}

namespace {
// counts[s * world + d] = rows rank s sends to rank d (the all-gathered plan)
void p2p_meta(mp_ep_s* E, const uint32_t* counts, cudaStream_t s, uint32_t& n_recv) {
    const uint32_t W = E->world, me = E->rank;
    std::vector<uint32_t> meta(4 * ((size_t)W + 1), 0);
    uint32_t* base = meta.data();           // my first row in rank r's receive buffer
    uint32_t* roff = base + (W + 1);        // my receive segments, per source
    uint32_t* dbase = roff + (W + 1);       // source s's send position of its rows for me
    for (uint32_t r = 0; r < W; ++r)
        for (uint32_t q = 0; q < me; ++q) base[r] += counts[(size_t)q * W + r];
    for (uint32_t q = 0; q < W; ++q) roff[q + 1] = roff[q] + counts[(size_t)q * W + me];
    for (uint32_t q = 0; q < W; ++q)
        for (uint32_t r = 0; r < me; ++r) dbase[q] += counts[(size_t)q * W + r];
    n_recv = roff[W];
    // every rank holds the whole plan: check EVERY destination's receive
    // count (all ranks use the same max_recv_rows), so all ranks fail the same
    // way before any peer store -- no rank writes past a peer's buffer and none
    // is left waiting in a barrier the others skip
    for (uint32_t r = 0; r < W; ++r) {
        uint64_t col = 0;
        for (uint32_t q = 0; q < W; ++q) col += counts[(size_t)q * W + r];
        if (col > E->max_recv)
            ep_fail(MP_ERR_VALIDATION, "rank " + std::to_string(r) + " would receive " + std::to_string(col) +
                                           " rows, more than max_recv_rows " + std::to_string(E->max_recv));
    }
    ep_ck(cudaMemcpyAsync(E->d_meta, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice, s), "p2p meta");
}
}  // namespace

MP_API mp_status mp_ep_p2p_pack(mp_ep_t E, const void* x, const uint32_t* sel, const float* w, uint32_t T,
                                const uint32_t* counts, uint32_t* n_recv, void* stream) {
    return ep_guarded([&] {
        if (!E || !counts || !n_recv || (T && (!x || !sel))) ep_fail(MP_ERR_VALIDATION, "null argument");
        EpDeviceGuard dg(E->device);
        if (!E->p2p) ep_fail(MP_ERR_VALIDATION, "mp_ep_p2p_open first");
        if (T != E->last_T) ep_fail(MP_ERR_VALIDATION, "mp_ep_p2p_pack must follow mp_ep_plan for the same tokens");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        uint32_t nr = 0;
        p2p_meta(E, counts, s, nr);
        *n_recv = nr;
        if (T == 0) return;
        mp::launch_ep_pack(E->dtype, x, sel, w, T, E->d, E->k_max, E->per_rank, E->S, E->world, E->dest,
                           E->ws.slot_row, E->d_px, E->d_meta, E->ws.offsets, s);
        ep_ck(cudaGetLastError(), "ep p2p pack");
    });
}

MP_API mp_status mp_ep_p2p_recv_buffers(mp_ep_t E, void** recv_x, uint32_t** recv_sel, float** recv_w) {
    return ep_guarded([&] {
        if (!E || !E->recv_x) ep_fail(MP_ERR_VALIDATION, "mp_ep_p2p_setup first");
        if (recv_x) *recv_x = E->recv_x;
        if (recv_sel) *recv_sel = E->recv_sel;
        if (recv_w) *recv_w = E->recv_w;
    });
}

MP_API mp_status mp_ep_p2p_return(mp_ep_t E, const void* part, uint32_t n_recv, void* stream) {
    return ep_guarded([&] {
        if (!E || (n_recv && !part)) ep_fail(MP_ERR_VALIDATION, "null argument");
        EpDeviceGuard dg(E->device);
        if (!E->p2p) ep_fail(MP_ERR_VALIDATION, "mp_ep_p2p_open first");
        const uint32_t W = E->world;
        mp::launch_ep_return(E->dtype, part, n_recv, E->d, W, E->d_meta + (W + 1), E->d_meta + 2 * (W + 1),
                             E->d_px + 3 * W, static_cast<cudaStream_t>(stream));
        ep_ck(cudaGetLastError(), "ep p2p return");
    });
}

MP_API mp_status mp_ep_p2p_combine(mp_ep_t E, uint32_t T, void* y, void* stream) {
    return ep_guarded([&] {
        if (!E || (T && !y)) ep_fail(MP_ERR_VALIDATION, "null argument");
        EpDeviceGuard dg(E->device);
        if (!E->p2p) ep_fail(MP_ERR_VALIDATION, "mp_ep_p2p_open first");
        if (T != E->last_T) ep_fail(MP_ERR_VALIDATION, "mp_ep_p2p_combine must follow mp_ep_plan for the same tokens");
        if (T == 0) return;
        mp::launch_ep_combine(E->dtype, E->back, T, E->d, E->world, E->ws.slot_row, y, static_cast<cudaStream_t>(stream));
        ep_ck(cudaGetLastError(), "ep p2p combine");
    });
}

MP_API mp_status mp_ep_combine(mp_ep_t E, const void* back, uint32_t T, void* y, void* stream) {
    return ep_guarded([&] {
        if (!E || (T && (!back || !y))) ep_fail(MP_ERR_VALIDATION, "null argument");
        EpDeviceGuard dg(E->device);
        if (T != E->last_T) ep_fail(MP_ERR_VALIDATION, "mp_ep_combine must follow mp_ep_plan for the same tokens");
        if (T == 0) return;
        mp::launch_ep_combine(E->dtype, back, T, E->d, E->world, E->ws.slot_row, y, static_cast<cudaStream_t>(stream));
        ep_ck(cudaGetLastError(), "ep combine");
    });
}

namespace mp {
void launch_ep_dest(const uint32_t* sel, uint32_t T, uint32_t k_max, uint32_t per_rank, uint32_t world, uint32_t* dest,
                    cudaStream_t s) {
    ep_dest_kernel<<<(T + 255) / 256, 256, 0, s>>>(sel, T, k_max, per_rank, world, dest);
}
void launch_ep_slot(const uint32_t* dest, const uint32_t* lrank, const uint32_t* block_base, uint32_t T, uint32_t world,
                    uint32_t* slot_row, cudaStream_t s) {
    ep_slot_kernel<<<(T * world + 255) / 256, 256, 0, s>>>(dest, lrank, block_base, T, world, slot_row);
}
void launch_ep_pack(int dtype, const void* x, const uint32_t* sel, const float* w, uint32_t T, uint32_t d,
                    uint32_t k_max, uint32_t per_rank, uint32_t S, uint32_t world, const uint32_t* dest,
                    const uint32_t* slot_row, void* const* dst_tables, const uint32_t* base, const uint32_t* send_off,
                    cudaStream_t s) {
    EpDest D{dst_tables, reinterpret_cast<uint32_t* const*>(dst_tables + world),
             reinterpret_cast<float* const*>(dst_tables + 2 * world), base, send_off};
    if (dtype == 1)
        ep_pack_kernel<__nv_bfloat16><<<(T + 7) / 8, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x), sel, w, T, d,
                                                                  k_max, per_rank, S, world, dest, slot_row, D);
    else
        ep_pack_kernel<float><<<(T + 7) / 8, 256, 0, s>>>(static_cast<const float*>(x), sel, w, T, d, k_max, per_rank,
                                                          S, world, dest, slot_row, D);
}
void launch_ep_return(int dtype, const void* part, uint32_t n_recv, uint32_t d, uint32_t world, const uint32_t* roff,
                      const uint32_t* dbase, void* const* back, cudaStream_t s) {
    if (n_recv == 0) return;
    if (dtype == 1)
        ep_return_kernel<__nv_bfloat16><<<(n_recv + 7) / 8, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(part),
                                                                         n_recv, d, world, roff, dbase, back);
    else
        ep_return_kernel<float><<<(n_recv + 7) / 8, 256, 0, s>>>(static_cast<const float*>(part), n_recv, d, world,
                                                                 roff, dbase, back);
}
void launch_ep_combine(int dtype, const void* back, uint32_t T, uint32_t d, uint32_t world, const uint32_t* slot_row,
                       void* y, cudaStream_t s, const void* x_res) {
    if (dtype == 1)
        ep_combine_kernel<__nv_bfloat16><<<T, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(back), T, d, world,
                                                           slot_row, static_cast<const __nv_bfloat16*>(x_res),
                                                           static_cast<__nv_bfloat16*>(y));
    else
        ep_combine_kernel<float><<<T, 256, 0, s>>>(static_cast<const float*>(back), T, d, world, slot_row,
                                                   static_cast<const float*>(x_res), static_cast<float*>(y));
}
}  // namespace mp
