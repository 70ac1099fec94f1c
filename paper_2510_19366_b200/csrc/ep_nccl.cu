// ep_nccl.cu -- the expert-parallel layer forward on the C++ host with an
// NCCL transport (north_star: "NCCL all-to-all over NVLink for
// token dispatch and combine", host code in C++):
//
//   mp_ep_forward: route (replicated router-only layer) -> plan (destination
//   ranks per token, deduplicated, rank-grouped send order) -> count matrix
//   (ncclAllGather of every rank's send counts; the ONE host synchronisation
//   of the layer: NCCL needs the all-to-allv sizes on the host) -> pack ->
//   token rows + selections + weights exchanged by grouped ncclSend/ncclRecv
//   (an all-to-allv; NVLink / NVSwitch between the GPUs of a node) -> experts
//   (experts-only layer, forward_selected on the received rows, one weighted
//   partial per (token, source rank)) -> partials returned by grouped
//   ncclSend/ncclRecv -> deterministic combine (ascending rank order,
//   optional fused residual).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, reusing the copy the
// process already loaded -- e.g. PyTorch's -- so communicators and calls come
// from one library); the product library has no link-time NCCL dependency.
// The communicator is created from a unique id the host runtime broadcasts
// (mp_ep_nccl_unique_id / mp_ep_nccl_init), the C-ABI carries no NCCL types.
#include <dlfcn.h>
#include <nccl.h>  // types only: every symbol is resolved with dlsym

#include <cstring>
#include <exception>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "moeprism/moe_layer.h"
#include "mp_common.cuh"
#include "mp_ep_impl.h"
#include "mp_kernels.h"

#define MP_API extern "C" __attribute__((visibility("default")))

extern "C" void mp_internal_set_error(const char* msg);

namespace {

struct NcclErr {
    int code;
    std::string msg;
};
[[noreturn]] void nfail(int code, const std::string& m) { throw NcclErr{code, m}; }
void nck_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) nfail(MP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL (PyTorch's)
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.error = std::string("NCCL not found (libnccl.so.2): ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && api.error.empty()) api.error = std::string("NCCL symbol missing: ") + name;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.AllGather, "ncclAllGather");
        sym(api.GetErrorString, "ncclGetErrorString");
    });
    if (!api.error.empty()) nfail(MP_ERR_CUDA, api.error);
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) nfail(MP_ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

template <class F>
int nguarded(F&& f) {
    try {
        f();
        return MP_OK;
    } catch (const NcclErr& e) {
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

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) nck_cuda(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DevGuard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

template <class T>
T* nalloc(size_t n, const char* what) {
    void* p = nullptr;
    nck_cuda(cudaMalloc(&p, (n ? n : 1) * sizeof(T)), what);
    return static_cast<T*>(p);
}

// counts[r] = offsets[r + 1] - offsets[r] (the rank-bucket sizes of the plan)
__global__ void ep_counts_kernel(const uint32_t* __restrict__ off, uint32_t world, uint32_t* __restrict__ counts) {
    const uint32_t r = threadIdx.x;
    if (r < world) counts[r] = off[r + 1] - off[r];
}

}  // namespace

struct mp_ep_nccl_s {
    ncclComm_t comm = nullptr;
    size_t send_cap = 0, recv_cap = 0;  // rows
    uint32_t* sel = nullptr;            // [max_tokens][k_max] routing of the local tokens
    float* w = nullptr;
    void* send_x = nullptr;             // [send_cap][d] rank-grouped
    uint32_t* send_sel = nullptr;       // [send_cap][k_max] (owner-local ids)
    float* send_w = nullptr;
    void* recv_x = nullptr;             // [recv_cap][d] grouped by source rank
    uint32_t* recv_sel = nullptr;
    float* recv_w = nullptr;
    void* part = nullptr;               // [recv_cap][d] expert partials
    void* back = nullptr;               // [send_cap][d] partials returned, send order
    uint32_t* cnt = nullptr;            // [world]
    uint32_t* cnt_all = nullptr;        // [world][world]
    uint32_t* cnt_host = nullptr;       // pinned [world][world]
    void** tables = nullptr;            // [3][world] pack destinations (the send buffers)
    std::vector<uint32_t> last_send, last_recv;
};

void mp_ep_nccl_free(mp_ep_s* E) {
    mp_ep_nccl_s* N = E->nccl;
    if (!N) return;
    if (N->comm) {
        try {
            nccl().CommDestroy(N->comm);
        } catch (...) {
        }
    }
    void* ptrs[] = {N->sel, N->w, N->send_x, N->send_sel, N->send_w, N->recv_x, N->recv_sel, N->recv_w,
                    N->part, N->back, N->cnt, N->cnt_all, N->tables};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (N->cnt_host) cudaFreeHost(N->cnt_host);
    delete N;
    E->nccl = nullptr;
}

MP_API mp_status mp_ep_nccl_unique_id(uint8_t* id) {
    return nguarded([&] {
        if (!id) nfail(MP_ERR_VALIDATION, "null argument");
        static_assert(sizeof(ncclUniqueId) == MP_EP_NCCL_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId u;
        nck(nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof(u));
    });
}

MP_API mp_status mp_ep_nccl_init(mp_ep_t E, const uint8_t* id) {
    return nguarded([&] {
        if (!E || !id) nfail(MP_ERR_VALIDATION, "null argument");
        if (E->nccl) nfail(MP_ERR_VALIDATION, "NCCL transport already initialised");
        DevGuard dg(E->device);
        const NcclApi& api = nccl();
        auto* N = new mp_ep_nccl_s;
        E->nccl = N;
        try {
            const size_t W = E->world, esz = E->dtype == MP_DTYPE_BF16 ? 2 : 4;
            // a token goes at most once to each rank: <= T * min(world, k_max) send rows
            N->send_cap = (size_t)E->max_tokens * std::min<size_t>(W, E->k_max);
            N->recv_cap = (size_t)E->max_tokens * W;
            N->sel = nalloc<uint32_t>((size_t)E->max_tokens * E->k_max, "ep routing");
            N->w = nalloc<float>((size_t)E->max_tokens * E->k_max, "ep routing");
            N->send_x = nalloc<char>(N->send_cap * E->d * esz, "ep send rows");
            N->send_sel = nalloc<uint32_t>(N->send_cap * E->k_max, "ep send selection");
            N->send_w = nalloc<float>(N->send_cap * E->k_max, "ep send weights");
            N->recv_x = nalloc<char>(N->recv_cap * E->d * esz, "ep receive rows");
            N->recv_sel = nalloc<uint32_t>(N->recv_cap * E->k_max, "ep receive selection");
            N->recv_w = nalloc<float>(N->recv_cap * E->k_max, "ep receive weights");
            N->part = nalloc<char>(N->recv_cap * E->d * esz, "ep partials");
            N->back = nalloc<char>(N->send_cap * E->d * esz, "ep returned partials");
            N->cnt = nalloc<uint32_t>(W, "ep counts");
            N->cnt_all = nalloc<uint32_t>(W * W, "ep count matrix");
            nck_cuda(cudaMallocHost(reinterpret_cast<void**>(&N->cnt_host), W * W * 4), "pinned counts");
            std::vector<void*> tab(3 * W);
            for (size_t r = 0; r < W; ++r) {
                tab[r] = N->send_x;
                tab[W + r] = N->send_sel;
                tab[2 * W + r] = N->send_w;
            }
            N->tables = nalloc<void*>(3 * W, "ep pack tables");
            nck_cuda(cudaMemcpy(N->tables, tab.data(), tab.size() * sizeof(void*), cudaMemcpyHostToDevice), "tables");
            ncclUniqueId u;
            std::memcpy(&u, id, sizeof(u));
            nck(api.CommInitRank(&N->comm, static_cast<int>(W), u, static_cast<int>(E->rank)), "ncclCommInitRank");
        } catch (...) {
            mp_ep_nccl_free(E);
            throw;
        }
    });
}

namespace {
// grouped all-to-allv of one buffer family: rank r's segment [soff[r], +scnt[r])
// rows of `send` to r, rows from r into [roff[r], +rcnt[r]) of `recv`
void alltoallv(const NcclApi& api, ncclComm_t comm, uint32_t W, const void* send, void* recv, size_t row_elems,
               size_t esz, ncclDataType_t ty, const std::vector<uint32_t>& scnt, const std::vector<uint32_t>& soff,
               const std::vector<uint32_t>& rcnt, const std::vector<uint32_t>& roff, cudaStream_t s) {
    for (uint32_t r = 0; r < W; ++r) {
        if (scnt[r])
            nck(api.Send(static_cast<const char*>(send) + (size_t)soff[r] * row_elems * esz, (size_t)scnt[r] * row_elems,
                         ty, static_cast<int>(r), comm, s),
                "ncclSend");
        if (rcnt[r])
            nck(api.Recv(static_cast<char*>(recv) + (size_t)roff[r] * row_elems * esz, (size_t)rcnt[r] * row_elems, ty,
                         static_cast<int>(r), comm, s),
                "ncclRecv");
    }
}
}  // namespace

MP_API mp_status mp_ep_forward(mp_ep_t E, mp_layer_t router, mp_layer_t experts, const void* x, uint32_t T,
                               const uint32_t* kpt, uint32_t k, void* y, uint32_t flags, void* stream) {
    return nguarded([&] {
        if (!E || !router || !experts || (T && (!x || !y))) nfail(MP_ERR_VALIDATION, "null argument");
        if (!E->nccl) nfail(MP_ERR_VALIDATION, "mp_ep_nccl_init first");
        if (T > E->max_tokens) nfail(MP_ERR_VALIDATION, "n_tokens exceeds the expert-parallel max_tokens");
        if (flags & ~MP_EP_RESIDUAL) nfail(MP_ERR_VALIDATION, "unknown mp_ep_forward flags");
        DevGuard dg(E->device);
        mp_ep_nccl_s* N = E->nccl;
        const NcclApi& api = nccl();
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const uint32_t W = E->world, me = E->rank;
        const size_t esz = E->dtype == MP_DTYPE_BF16 ? 2 : 4;
        const ncclDataType_t xty = E->dtype == MP_DTYPE_BF16 ? ncclBfloat16 : ncclFloat32;
        // 1. route (replicated router)
        int rc = mp_layer_route(router, x, T, kpt, k, N->sel, N->w, stream);
        if (rc) nfail(rc, mp_last_error());
        // 2. plan: destination ranks per token, rank-grouped send positions
        E->last_T = T;
        if (T) {
            mp::launch_ep_dest(N->sel, T, E->k_max, E->per_rank, W, E->dest, s);
            mp::launch_bucket_local(E->dest, T, W, W, E->ws, s);
            mp::launch_bucket_scan(T, W, E->ws, s);
            mp::launch_ep_slot(E->dest, E->ws.lrank, E->ws.block_base, T, W, E->ws.slot_row, s);
            ep_counts_kernel<<<1, 32, 0, s>>>(E->ws.offsets, W, N->cnt);
        } else {
            nck_cuda(cudaMemsetAsync(N->cnt, 0, W * 4, s), "counts");
        }
        nck_cuda(cudaGetLastError(), "ep plan");
        // 3. the count matrix on every rank (the layer's one host synchronisation)
        nck(api.AllGather(N->cnt, N->cnt_all, W, ncclUint32, N->comm, s), "ncclAllGather counts");
        nck_cuda(cudaMemcpyAsync(N->cnt_host, N->cnt_all, (size_t)W * W * 4, cudaMemcpyDeviceToHost, s), "counts");
        nck_cuda(cudaStreamSynchronize(s), "count exchange");
        std::vector<uint32_t> scnt(W), soff(W + 1, 0), rcnt(W), roff(W + 1, 0);
        for (uint32_t r = 0; r < W; ++r) {
            scnt[r] = N->cnt_host[(size_t)me * W + r];
            rcnt[r] = N->cnt_host[(size_t)r * W + me];
            soff[r + 1] = soff[r] + scnt[r];
            roff[r + 1] = roff[r] + rcnt[r];
        }
        const uint32_t n_send = soff[W], n_recv = roff[W];
        if (n_send > N->send_cap || n_recv > N->recv_cap) nfail(MP_ERR_VALIDATION, "expert-parallel buffers overflow");
        N->last_send = scnt;
        N->last_recv = rcnt;
        // 4. pack every token row once per destination rank (owner-local ids)
        if (T) {
            mp::launch_ep_pack(E->dtype, x, N->sel, N->w, T, E->d, E->k_max, E->per_rank, E->S, W, E->dest,
                               E->ws.slot_row, N->tables, E->ws.offsets, E->ws.offsets, s);
            nck_cuda(cudaGetLastError(), "ep pack");
        }
        // 5. dispatch: rows, selections, weights (one grouped all-to-allv)
        nck(api.GroupStart(), "ncclGroupStart");
        alltoallv(api, N->comm, W, N->send_x, N->recv_x, E->d, esz, xty, scnt, soff, rcnt, roff, s);
        alltoallv(api, N->comm, W, N->send_sel, N->recv_sel, E->k_max, 4, ncclUint32, scnt, soff, rcnt, roff, s);
        alltoallv(api, N->comm, W, N->send_w, N->recv_w, E->k_max, 4, ncclFloat32, scnt, soff, rcnt, roff, s);
        nck(api.GroupEnd(), "ncclGroupEnd");
        // 6. this rank's experts on the received rows: one weighted partial per row
        if (n_recv) {
            rc = mp_layer_forward_selected(experts, N->recv_x, n_recv, N->recv_sel, N->recv_w, N->part, nullptr,
                                           stream);
            if (rc) nfail(rc, mp_last_error());
        }
        // 7. return the partials to the token owners, in their send order
        nck(api.GroupStart(), "ncclGroupStart");
        alltoallv(api, N->comm, W, N->part, N->back, E->d, esz, xty, rcnt, roff, scnt, soff, s);
        nck(api.GroupEnd(), "ncclGroupEnd");
        // 8. deterministic combine (ascending rank order), optional residual
        if (T) {
            mp::launch_ep_combine(E->dtype, N->back, T, E->d, W, E->ws.slot_row, y, s,
                                  (flags & MP_EP_RESIDUAL) ? x : nullptr);
            nck_cuda(cudaGetLastError(), "ep combine");
        }
    });
}

MP_API mp_status mp_ep_last_counts(mp_ep_t E, uint32_t* send_rows, uint32_t* recv_rows) {
    return nguarded([&] {
        if (!E || !E->nccl) nfail(MP_ERR_VALIDATION, "no NCCL transport");
        for (uint32_t r = 0; r < E->world; ++r) {
            if (send_rows) send_rows[r] = r < E->nccl->last_send.size() ? E->nccl->last_send[r] : 0;
            if (recv_rows) recv_rows[r] = r < E->nccl->last_recv.size() ? E->nccl->last_recv[r] : 0;
        }
    });
}
