// layer.cu -- the C-ABI (include/moeprism/moe_layer.h): layer state, weight
// loading + packing, and the stream-ordered forward that chains the kernels
//   router -> bucket (histogram) -> bucket (scan) -> dispatch -> gemm1
//   (SwiGLU) -> gemm2 -> combine.
// Everything runs on the GPU; a missing / non-sm_100 device is a status-3
// error, never a CPU fallback.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "moeprism/moe_layer.h"
#include "mp_kernels.h"
#include "mp_layer_impl.h"

#define MP_API extern "C" __attribute__((visibility("default")))

#include <mutex>
#include <set>
#include <utility>

namespace mp {
// Function attributes belong to the current device's context: set them once
// per (kernel, device), under a lock (handles may live on several devices and
// be driven from several threads).
void func_attr_once(const void* func, int max_dyn_smem, bool max_carveout) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (!done.insert({func, dev}).second) return;
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn_smem);
    if (max_carveout)
        cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MOEPRISM_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}
}  // namespace mp

namespace {

thread_local std::string g_err;

struct Err {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Err{code, msg}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(MP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void ck_launch(const char* what) { ck(cudaGetLastError(), what); }

template <class F>
int guarded(F&& f) {
    try {
        f();
        return MP_OK;
    } catch (const Err& e) {
        g_err = e.msg;
        return e.code;
    } catch (const mp::Failure& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host out of memory";
        return MP_ERR_CUDA;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// Per-device pool of the big per-forward scratch buffers (x_perm, h, o) for
// layers created with MP_LAYER_SHARED_SCRATCH: layers that run one after the
// other on one stream (a layer stack) share one allocation of each exact size,
// reference counted.
struct ScratchPool {
    struct Ent {
        int dev;
        size_t bytes;
        void* p;
        int refs;
    };
    std::mutex mu;
    std::vector<Ent> ents;
};
ScratchPool& scratch_pool() {
    static ScratchPool pool;
    return pool;
}

void* scratch_acquire(size_t bytes, const char* what) {
    int dev = 0;
    cudaGetDevice(&dev);
    ScratchPool& P = scratch_pool();
    std::lock_guard<std::mutex> lk(P.mu);
    for (auto& e : P.ents)
        if (e.dev == dev && e.bytes == bytes) {
            ++e.refs;
            return e.p;
        }
    void* p = nullptr;
    ck(cudaMalloc(&p, bytes ? bytes : 1), what);
    P.ents.push_back({dev, bytes, p, 1});
    return p;
}
void scratch_release(void* p) {
    ScratchPool& P = scratch_pool();
    std::lock_guard<std::mutex> lk(P.mu);
    for (size_t i = 0; i < P.ents.size(); ++i)
        if (P.ents[i].p == p) {
            if (--P.ents[i].refs == 0) {
                cudaFree(p);
                P.ents.erase(P.ents.begin() + i);
            }
            return;
        }
}

template <class T>
T* dalloc(size_t n, const char* what) {
    void* p = nullptr;
    if (n == 0) n = 1;
    ck(cudaMalloc(&p, n * sizeof(T)), what);
    return static_cast<T*>(p);
}

uint32_t round_up(uint32_t v, uint32_t m) { return (v + m - 1) / m * m; }
// L2 promotion of the decode W2 map (MOEPRISM_W2D_PROMO, A/B only; default 64)
uint32_t w2d_promo() {
    const char* e = std::getenv("MOEPRISM_W2D_PROMO");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 64u;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// shared-expert split-K (decode batches): at most kShSplitRows tokens, kShSplitMax K splits
constexpr uint32_t kShSplitRows = 128, kShSplitMax = 12;

const char* kStageNames[] = {"router", "bucket", "dispatch", "gemm1", "gemm2", "combine"};
constexpr int kStages = 6;

}  // namespace

struct mp_layer_s {
    mp_layer_desc desc{};
    uint32_t E = 0, S = 0, G = 0, d = 0, ff = 0, dtype = 0, k_max = 0, max_tokens = 0;
    uint32_t w_pad = 0, d_pad = 0, G_pad = 0, rows_cap = 0, w2_rows = 0;
    uint32_t w_sub = 0;  // neurons per sub-expert (the packed width w_pad rounds it up to 128)
    size_t esz = 4;
    int num_sms = 0;
    bool use_tc = false;
    // grouped-GEMM kernel: 0 auto (CTA pairs, gemm_tc2, or 1-SM 128-row tiles,
    // gemm_tc, by rows per sub-expert); 1 1-SM, 2 pairs, 3 pairs with plain
    // (unswapped) remainder tiles; MOEPRISM_TC_TILE=128|256|256-plain forces
    int tile_mode = 0;
    bool tile256 = false, tile256_g2 = false;  // this forward's choice for gemm1 / gemm2
    bool r_tables = false;  // this forward's route_bucket also wrote the permutation tables (decode)
    bool has_experts = true, has_router = true;  // MP_LAYER_* role flags

    std::vector<std::vector<uint32_t>> assignment;
    std::vector<uint8_t> has_part, packed;
    std::vector<float*> raw;  // staged fp32 MPEX weights (wg | wu | wd) until packed
    bool router_set = false;

    // proxy router state
    std::vector<uint32_t> gate_r;
    std::vector<std::vector<std::vector<uint32_t>>> gates;  // [e][s] -> neurons
    std::vector<uint8_t> has_gates;
    float* gate_rows = nullptr;  // [n_gate][d] w_gate columns of the gate neurons
    float* up_rows = nullptr;
    uint32_t* gate_off = nullptr;  // [G+1] CSR over the gate rows
    uint32_t n_gate_rows = 0;
    bool gates_packed = false;
    double* scores = nullptr;  // [max_tokens][G]
    // tensor-core proxy path (bf16, d % 8 == 0): [gate; up] rows of the gate
    // neurons as three bf16 planes through router_tc, certified like the linear
    // router (proxy.cu); otherwise the exact fp64 path
    bool proxy_tc = false;
    uint32_t p_npad = 0;
    void* p_planes = nullptr;
    float* p_partial = nullptr;   // fp32 [ks][T][p_npad]
    int8_t* p_class = nullptr;    // [max_tokens][G] certification classes of flagged tokens
    float p_wmax = 0.0f;
    CUtensorMap tm_pplanes{};

    void* W1 = nullptr;
    void* W2 = nullptr;
    float* wrT = nullptr;
    // tensor-core router: W_r as three bf16 planes + fp64 K-split partials
    bool router_tc = false;
    uint32_t r_npad = 0, r_last_ks = 0, r_last_T = 0;
    void* wr_planes = nullptr;
    double* r_partial = nullptr;
    // routing statistics of the last forward: [0] tokens re-selected from exact
    // fp64 logits, [1] near ties (exact k-th/(k+1)-th gap < 1e-6), then the
    // re-selected tokens of the non-fused path
    uint32_t* r_flagged = nullptr;  // [2 + max_tokens]
    uint32_t* r_ticket = nullptr;   // last-CTA ticket of the fused routing epilogue (left 0)
    // Certification of the tensor-core logits (router_tc.cu): per token
    // guard_t = depth 2^-23 max|W_r| sum|x_t| + 2^-23 max|logit_t|; tokens whose
    // k-th/(k+1)-th gap is < 2 guard_t are re-selected from exact fp64 logits.
    float r_wmax = 0.0f;            // max |W_r|
    double r_guard_floor = 0.0;     // MOEPRISM_ROUTER_GUARD: extra absolute width (tests widen the window)
    CUtensorMap tm_wplanes{};
    int32_t* d_nmap = nullptr;
    int32_t* nmap_all = nullptr;  // [E][S*w_pad] packed neuron -> original neuron (-1 padding), calibration

    uint32_t* sel = nullptr;
    float* wsel = nullptr;
    uint32_t* kpt_dev = nullptr;
    mp::BucketWs ws{};
    void* x_perm = nullptr;
    void* h = nullptr;
    void* o = nullptr;
    bool shared_scratch = false;  // MP_LAYER_SHARED_SCRATCH: x_perm / h / o from the device pool
    void* x_stage = nullptr;
    void* y_stage = nullptr;
    CUtensorMap tm_xperm{}, tm_h{}, tm_w1{}, tm_w2{};
    CUtensorMap tm_o{};  // gemm2 output o, 32 x 32 boxes (TMA-store epilogue)
    CUtensorMap tm_w2d{};  // W2 with K trimmed to w_sub (decode batches)
    mp::GemmBTail w1_tail{};  // gemm1 reads only the w_sub valid neurons of each packed W1 group
    CUtensorMap tm_xperm_s[3]{}, tm_h_s[3]{};  // 16 / 32 / 64-row A boxes (short tiles of the 1-SM GEMM)
    CUtensorMap tm_w1h{}, tm_w2h{};  // 128-row boxes: each CTA of a pair loads half a B tile

    // shared (always-on) expert, Qwen-style: one dense group of sh_w_pad neurons
    uint32_t sh_ff = 0, sh_w_pad = 0, sh_w2_rows = 0;
    void* W1s = nullptr;
    void* W2s = nullptr;
    float* sh_gate = nullptr;  // [d] or null (weight 1)
    void* sh_h = nullptr;      // [max_tokens][sh_w_pad]
    void* sh_o = nullptr;      // [max_tokens][d_pad]
    float* sh_o32 = nullptr;   // [kShSplitMax][min(max_tokens, 128)][d_pad] fp32 split-K partials (decode)
    uint32_t sh_splits = 0;    // this forward's split count (0: sh_o holds bf16 rows)
    float* sh_w = nullptr;     // [max_tokens]
    uint32_t* sh_meta = nullptr;  // offsets {0, T}, tile prefixes {0, ceil(T/128)}, {0, ceil(T/256)}
    CUtensorMap tm_w1s{}, tm_w2s{}, tm_hs{}, tm_w1sh{}, tm_w2sh{};
    cudaStream_t sh_stream = nullptr;  // side stream of the shared expert
    cudaEvent_t sh_fork = nullptr, sh_join = nullptr;
    // decode batches: the routed weights the first gemm1 wave reads are
    // prefetched into L2 while the (latency-bound) routing chain runs
    cudaStream_t pf_stream = nullptr;
    cudaEvent_t pf_fork = nullptr, pf_join = nullptr;
    bool pf_pending = false;

    bool residual = false;  // mp_layer_set_residual: y = x + MoE(x), fused into the combine
    // pipelined host-buffer forwards (mp_layer_forward_host_batches): two
    // staging slots, copy streams and slot events
    void* px[2] = {nullptr, nullptr};
    void* py[2] = {nullptr, nullptr};
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_xready[2] = {}, ev_computed[2] = {}, ev_ydone[2] = {};
    uint32_t* cal_meta = nullptr;  // calibration GEMM group offsets / tile prefix

    // Sub-expert offload cache: the packed weights live in
    // pinned host memory; a device cache of `off_slots` units (a unit = 1
    // sub-expert "fine" or the S sub-experts of an expert "monolithic") is
    // managed with the reference's LRU policy (cache_step, inc/offload.hpp:
    // 202-255) and filled by real host->device copies.
    bool offload = false;
    uint32_t off_unit = 1, off_slots = 0;
    void* W1h = nullptr;  // pinned [G][2 w_pad][d_pad]
    void* W2h = nullptr;  // pinned [G][d_pad][w_pad]
    void* W1c = nullptr;  // device [slots * unit][2 w_pad][d_pad]
    void* W2c = nullptr;  // device [slots * unit][d_pad][w_pad] (+ TMA row padding)
    CUtensorMap tm_w1c{}, tm_w2c{}, tm_w1ch{}, tm_w2ch{};
    std::vector<uint32_t> lru;            // resident units, least recent first
    std::vector<int32_t> slot_of_unit;    // -1 when not resident
    std::vector<uint32_t> free_slots;
    uint32_t* gmap_dev = nullptr;         // [G] group -> cache group
    uint32_t* gmap_host = nullptr;        // pinned [G]
    uint32_t* off_host = nullptr;         // pinned [G + 1] bucket offsets
    uint64_t off_hits = 0, off_misses = 0, off_bytes = 0;
    std::vector<uint32_t> off_last_req;   // requested units of the last forward
    uint32_t off_last_misses = 0;

    bool profiling = false;
    struct EventSet {
        cudaEvent_t ev[kStages + 1];
        int order[kStages];
        int n = 0;
    };
    std::vector<EventSet*> ev_pool, ev_pending;
    double stage_ms[kStages] = {};
    uint64_t stage_launches[kStages] = {};
    uint64_t launches = 0;
};

namespace {

void free_layer(mp_layer_s* L) {
    for (float* p : L->raw)
        if (p) cudaFree(p);
    for (void* p : {L->x_perm, L->h, L->o})
        if (p) L->shared_scratch ? scratch_release(p) : (void)cudaFree(p);
    void* ptrs[] = {L->p_planes, L->p_partial, L->p_class, L->gate_rows, L->up_rows, L->gate_off, L->scores, L->W1, L->W2, L->wrT, L->wr_planes, L->r_partial, L->r_flagged, L->r_ticket, L->d_nmap, L->nmap_all, L->sel,
                    L->wsel, L->kpt_dev, L->ws.lrank, L->ws.block_counts, L->ws.block_base, L->ws.offsets,
                    L->ws.mprefix_tc, L->ws.mprefix_simt, L->ws.mprefix_tc2, L->ws.perm_tok, L->ws.perm_w, L->ws.slot_row, L->ws.err,
                    L->x_stage, L->y_stage, L->W1s, L->W2s, L->sh_gate, L->sh_h,
                    L->sh_o, L->sh_o32, L->sh_w, L->sh_meta, L->cal_meta};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (L->sh_stream) cudaStreamDestroy(L->sh_stream);
    for (cudaStream_t st : {L->h2d, L->d2h})
        if (st) cudaStreamDestroy(st);
    for (int i = 0; i < 2; ++i) {
        for (cudaEvent_t ev : {L->ev_xready[i], L->ev_computed[i], L->ev_ydone[i]})
            if (ev) cudaEventDestroy(ev);
        if (L->px[i] && L->px[i] != L->x_stage) cudaFree(L->px[i]);
        if (L->py[i] && L->py[i] != L->y_stage) cudaFree(L->py[i]);
    }
    if (L->sh_fork) cudaEventDestroy(L->sh_fork);
    if (L->sh_join) cudaEventDestroy(L->sh_join);
    if (L->pf_stream) cudaStreamDestroy(L->pf_stream);
    if (L->pf_fork) cudaEventDestroy(L->pf_fork);
    if (L->pf_join) cudaEventDestroy(L->pf_join);
    for (void* p : {L->W1c, L->W2c, static_cast<void*>(L->gmap_dev)})
        if (p) cudaFree(p);
    for (void* p : {L->W1h, L->W2h, static_cast<void*>(L->gmap_host), static_cast<void*>(L->off_host)})
        if (p) cudaFreeHost(p);
    for (auto* v : {&L->ev_pool, &L->ev_pending})
        for (auto* es : *v) {
            for (auto& e : es->ev) cudaEventDestroy(e);
            delete es;
        }
    delete L;
}

// Gathers sub-expert members (ascending, inc/partition.hpp:49-55) and packs
// expert e once both its weights and its partition are known.
void maybe_pack(mp_layer_s* L, uint32_t e) {
    if (L->packed[e] || !L->has_part[e] || !L->raw[e]) return;
    if (L->offload) fail(MP_ERR_VALIDATION, "the layer's weights are offloaded; reload requires a new layer");
    std::vector<int32_t> nmap(static_cast<size_t>(L->S) * L->w_pad, -1);
    std::vector<uint32_t> fill(L->S, 0);
    const auto& a = L->assignment[e];
    for (uint32_t j = 0; j < L->ff; ++j) {
        const uint32_t s = a[j];
        nmap[static_cast<size_t>(s) * L->w_pad + fill[s]++] = static_cast<int32_t>(j);
    }
    ck(cudaMemcpy(L->d_nmap, nmap.data(), nmap.size() * sizeof(int32_t), cudaMemcpyHostToDevice), "nmap upload");
    ck(cudaMemcpy(L->nmap_all + (size_t)e * nmap.size(), nmap.data(), nmap.size() * sizeof(int32_t),
                  cudaMemcpyHostToDevice),
       "nmap keep");
    const size_t n = static_cast<size_t>(L->d) * L->ff;
    const float* wg = L->raw[e];
    const float* wu = wg + n;
    const float* wd = wu + n;
    char* W1e = static_cast<char*>(L->W1) + static_cast<size_t>(e) * L->S * 2 * L->w_pad * L->d_pad * L->esz;
    char* W2e = static_cast<char*>(L->W2) + static_cast<size_t>(e) * L->S * L->d_pad * L->w_pad * L->esz;
    mp::launch_pack_w1(L->dtype, wg, wu, L->d, L->ff, L->d_nmap, L->S, L->w_pad, L->d_pad, W1e, 0);
    ck_launch("pack_w1");
    mp::launch_pack_w2(L->dtype, wd, L->d, L->ff, L->d_nmap, L->S, L->w_pad, L->d_pad, W2e, 0);
    ck_launch("pack_w2");
    ck(cudaDeviceSynchronize(), "pack");
    // proxy gate rows need the raw columns: keep raw only while gates are pending
    if (L->desc.router_mode != MP_ROUTER_PROXY) {
        cudaFree(L->raw[e]);
        L->raw[e] = nullptr;
    }
    L->packed[e] = 1;
    L->gates_packed = false;
}

void pack_gates(mp_layer_s* L) {
    if (L->gates_packed) return;
    for (uint32_t e = 0; e < L->E; ++e) {
        if (!L->has_gates[e]) fail(MP_ERR_VALIDATION, "proxy router: expert " + std::to_string(e) + " has no gate set");
        if (!L->raw[e]) fail(MP_ERR_VALIDATION, "proxy router: expert " + std::to_string(e) + " weights not loaded");
    }
    std::vector<uint32_t> off(L->G + 1, 0);
    for (uint32_t e = 0; e < L->E; ++e)
        for (uint32_t s = 0; s < L->S; ++s) off[e * L->S + s + 1] = off[e * L->S + s] + L->gates[e][s].size();
    L->n_gate_rows = off[L->G];
    if (L->scores) cudaFree(L->scores);
    // [T][G] double scores followed by the [T][n_gate_rows] |activation| scratch
    L->scores = reinterpret_cast<double*>(
        dalloc<char>((size_t)L->max_tokens * (L->G * sizeof(double) + L->n_gate_rows * sizeof(float)), "scores"));
    if (L->gate_rows) cudaFree(L->gate_rows);
    if (L->up_rows) cudaFree(L->up_rows);
    L->gate_rows = dalloc<float>(static_cast<size_t>(L->n_gate_rows) * L->d, "gate rows");
    L->up_rows = dalloc<float>(static_cast<size_t>(L->n_gate_rows) * L->d, "up rows");
    ck(cudaMemcpy(L->gate_off, off.data(), off.size() * 4, cudaMemcpyHostToDevice), "gate offsets");
    uint32_t* d_neur = dalloc<uint32_t>(L->n_gate_rows, "gate neuron ids");
    for (uint32_t e = 0; e < L->E; ++e) {
        std::vector<uint32_t> neur;
        for (uint32_t s = 0; s < L->S; ++s)
            for (uint32_t j : L->gates[e][s]) neur.push_back(j);
        if (neur.empty()) continue;
        ck(cudaMemcpy(d_neur, neur.data(), neur.size() * 4, cudaMemcpyHostToDevice), "gate neurons");
        const size_t n = static_cast<size_t>(L->d) * L->ff;
        const size_t row0 = off[e * L->S];
        mp::launch_pack_gate_rows(L->raw[e], L->raw[e] + n, L->d, L->ff, d_neur, static_cast<uint32_t>(neur.size()),
                                  L->gate_rows + row0 * L->d, L->up_rows + row0 * L->d, 0);
        ck_launch("pack_gate_rows");
        ck(cudaDeviceSynchronize(), "pack gates");
    }
    cudaFree(d_neur);
    // tensor-core path: planes of [gate rows; up rows], partial buffers, max |W|
    for (void* p : {L->p_planes, static_cast<void*>(L->p_partial), static_cast<void*>(L->p_class)})
        if (p) cudaFree(p);
    L->p_planes = nullptr;
    L->p_partial = nullptr;
    L->p_class = nullptr;
    uint32_t max_list = 0;
    for (uint32_t g = 0; g < L->G; ++g) max_list = std::max(max_list, off[g + 1] - off[g]);
    L->proxy_tc = L->dtype == MP_DTYPE_BF16 && (L->d % 8) == 0 && L->n_gate_rows <= 1024 && max_list <= 1024;
    if (const char* env = std::getenv("MOEPRISM_ROUTER"))
        if (std::string(env) == "simt") L->proxy_tc = false;  // diagnostics only
    if (L->proxy_tc) {
        const uint32_t nr2 = 2 * L->n_gate_rows;
        L->p_npad = round_up(nr2, 32);
        L->p_planes = dalloc<char>((size_t)3 * L->p_npad * L->d * 2, "proxy planes");
        mp::launch_split_rows(L->gate_rows, L->up_rows, L->n_gate_rows, L->n_gate_rows, L->d, L->p_npad, L->p_planes, 0);
        const size_t rows = mp::router_tc_partial_rows(L->max_tokens, L->d, nr2, L->num_sms);
        L->p_partial = dalloc<float>(rows * L->p_npad, "proxy partials");
        L->p_class = dalloc<int8_t>((size_t)L->max_tokens * L->G, "proxy classes");
        ck(cudaMemset(L->ws.err + 1, 0, sizeof(int)), "memset");
        mp::launch_absmax(L->gate_rows, (size_t)L->n_gate_rows * L->d, reinterpret_cast<float*>(L->ws.err + 1), 0);
        mp::launch_absmax(L->up_rows, (size_t)L->n_gate_rows * L->d, reinterpret_cast<float*>(L->ws.err + 1), 0);
        ck_launch("proxy planes");
        ck(cudaMemcpy(&L->p_wmax, L->ws.err + 1, sizeof(float), cudaMemcpyDeviceToHost), "proxy max |W|");
        ck(cudaMemset(L->ws.err + 1, 0, sizeof(int)), "memset");
        if (!mp::make_tmap_bf16_2d(&L->tm_pplanes, L->p_planes, 3ull * L->p_npad, L->d,
                                   mp::router_tc_cols_per_cta(nr2), 64))
            fail(MP_ERR_CUDA, "proxy planes tensor map");
    }
    L->gates_packed = true;
}

void check_ready(mp_layer_s* L) {
    if (!L->has_experts) fail(MP_ERR_VALIDATION, "router-only layer (MP_LAYER_ROUTER_ONLY) has no experts");
    for (uint32_t e = 0; e < L->E; ++e)
        if (!L->packed[e])
            fail(MP_ERR_VALIDATION, "expert " + std::to_string(e) + " is not ready (weights and partition required)");
}

// Per-stage device time: CUDA events recorded on the forward's stream and
// resolved lazily (no host sync inside a forward, so the CPU stays ahead and
// the events measure GPU time, not launch gaps).
struct StageTimer {
    mp_layer_s* L;
    cudaStream_t s;
    mp_layer_s::EventSet* es = nullptr;
    StageTimer(mp_layer_s* l, cudaStream_t st) : L(l), s(st) {}
    void begin(int stage) {
        (void)stage;
        if (!L->profiling || es) return;
        if (L->ev_pool.empty()) {
            auto* n = new mp_layer_s::EventSet;
            for (auto& e : n->ev) ck(cudaEventCreate(&e), "event");
            L->ev_pool.push_back(n);
        }
        es = L->ev_pool.back();
        L->ev_pool.pop_back();
        es->n = 0;
        cudaEventRecord(es->ev[0], s);
    }
    void end(int stage, int n_launch) {
        L->launches += n_launch;
        if (!L->profiling || !es) return;
        L->stage_launches[stage] += n_launch;
        cudaEventRecord(es->ev[stage + 1], s);
        es->order[es->n++] = stage;
    }
    void finish(const int*, int) {
        if (es) L->ev_pending.push_back(es);
        es = nullptr;
    }
};

void resolve_timings(mp_layer_s* L) {
    for (auto* es : L->ev_pending) {
        if (es->n) cudaEventSynchronize(es->ev[es->order[es->n - 1] + 1]);
        cudaEvent_t prev = es->ev[0];
        for (int q = 0; q < es->n; ++q) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, prev, es->ev[es->order[q] + 1]);
            L->stage_ms[es->order[q]] += ms;
            prev = es->ev[es->order[q] + 1];
        }
        L->ev_pool.push_back(es);
    }
    L->ev_pending.clear();
}

// One offload cache step (inc/offload.hpp:202-255 on real transfers): read the
// bucket sizes back (synchronises the stream), the requested units are those
// with tokens, misses are evicted-for and copied host->device on the stream,
// the group -> cache-slot map is uploaded.  LRU order, eviction and
// most-recent insertion (ascending unit id) follow cache_step exactly.
void offload_step(mp_layer_s* L, cudaStream_t s) {
    ck(cudaMemcpyAsync(L->off_host, L->ws.offsets, (size_t)(L->G + 1) * 4, cudaMemcpyDeviceToHost, s), "offsets");
    ck(cudaStreamSynchronize(s), "offload: bucket sizes");
    const uint32_t n_units = L->G / L->off_unit;
    std::vector<uint32_t> req;
    for (uint32_t u = 0; u < n_units; ++u) {
        bool any = false;
        for (uint32_t j = 0; j < L->off_unit; ++j) {
            const uint32_t g = u * L->off_unit + j;
            any |= L->off_host[g + 1] > L->off_host[g];
        }
        if (any) req.push_back(u);
    }
    if (req.size() > L->off_slots)
        fail(MP_ERR_VALIDATION, "request set of " + std::to_string(req.size()) +
                                    " units exceeds the cache capacity of " + std::to_string(L->off_slots));
    std::vector<uint8_t> requested(n_units, 0);
    uint32_t misses = 0;
    for (uint32_t u : req) {
        requested[u] = 1;
        misses += L->slot_of_unit[u] < 0;
    }
    // evict LRU units outside the request until the misses fit
    size_t need = L->lru.size() + misses;
    if (need > L->off_slots) {
        size_t to_evict = need - L->off_slots;
        std::vector<uint32_t> keep;
        for (uint32_t u : L->lru) {
            if (to_evict && !requested[u]) {
                L->free_slots.push_back(static_cast<uint32_t>(L->slot_of_unit[u]));
                L->slot_of_unit[u] = -1;
                --to_evict;
            } else {
                keep.push_back(u);
            }
        }
        L->lru.swap(keep);
    }
    // requested units become most recent, ascending id; misses take free slots
    std::vector<uint32_t> rest;
    for (uint32_t u : L->lru)
        if (!requested[u]) rest.push_back(u);
    const size_t b1 = (size_t)2 * L->w_pad * L->d_pad * L->esz;  // W1 bytes per sub-expert
    const size_t b2 = (size_t)L->d_pad * L->w_pad * L->esz;      // W2 bytes per sub-expert
    for (uint32_t u : req) {
        rest.push_back(u);
        if (L->slot_of_unit[u] >= 0) continue;
        const uint32_t slot = L->free_slots.back();
        L->free_slots.pop_back();
        L->slot_of_unit[u] = static_cast<int32_t>(slot);
        const size_t n1 = b1 * L->off_unit, n2 = b2 * L->off_unit;
        ck(cudaMemcpyAsync(static_cast<char*>(L->W1c) + slot * n1, static_cast<char*>(L->W1h) + u * n1, n1,
                           cudaMemcpyHostToDevice, s),
           "offload W1");
        ck(cudaMemcpyAsync(static_cast<char*>(L->W2c) + slot * n2, static_cast<char*>(L->W2h) + u * n2, n2,
                           cudaMemcpyHostToDevice, s),
           "offload W2");
        L->off_bytes += n1 + n2;
    }
    L->lru.swap(rest);
    for (uint32_t g = 0; g < L->G; ++g) {
        const int32_t sl = L->slot_of_unit[g / L->off_unit];
        L->gmap_host[g] = sl < 0 ? 0u : static_cast<uint32_t>(sl) * L->off_unit + g % L->off_unit;
    }
    ck(cudaMemcpyAsync(L->gmap_dev, L->gmap_host, (size_t)L->G * 4, cudaMemcpyHostToDevice, s), "gmap");
    L->off_misses += misses;
    L->off_hits += req.size() - misses;
    L->off_last_req = req;
    L->off_last_misses = misses;
}

// The shared expert does not depend on the routing: it runs on a side stream
// forked from the forward's stream (gate -> gemm1 -> gemm2), overlapping the
// router / bucketing / dispatch / routed GEMMs, and the combine joins it.
// Fork / join are events, so the forward stays graph-capturable.
void launch_shared_expert(mp_layer_s* L, const void* x, uint32_t T, cudaStream_t s, bool forked = false) {
    if (!forked) ck(cudaEventRecord(L->sh_fork, s), "fork shared expert");
    ck(cudaStreamWaitEvent(L->sh_stream, L->sh_fork, 0), "fork shared expert");
    cudaStream_t ss = L->sh_stream;
    mp::launch_shared_gate(x, T, L->d, L->sh_gate, L->sh_w, L->sh_meta, L->sh_meta + 2, ss);
    CUtensorMap tmX;
    if (!mp::make_tmap_bf16_2d(&tmX, x, T, L->d, 128, 64)) fail(MP_ERR_CUDA, "shared expert tensor map");
    // one group of T rows: CTA pairs from 192 rows (the tile mode knobs steer the routed GEMMs only)
    const bool sh_pair = T >= 192;
    const int sh_sms = L->num_sms;  // (capping it to leave SMs to the routing chain measured slower)
    mp::GemmShape s1{1, L->d_pad, 2 * L->sh_w_pad, T, L->sh_w_pad, 2 * L->sh_w_pad};
    mp::GemmShape s2{1, L->sh_w_pad, L->d_pad, T, L->d_pad, L->d_pad};
    // small batches: the down projection has d_pad / 256 output tiles (8 CTAs
    // at Qwen's d = 2048) over a long K (5632): split K over the idle SMs, fp32
    // partials summed in split order by the combine
    const uint32_t n_tiles = ((T + mp::kTcBM - 1) / mp::kTcBM) * (L->d_pad / 256);
    L->sh_splits = 0;
    if (!sh_pair && T <= kShSplitRows && n_tiles * 4 <= static_cast<uint32_t>(L->num_sms)) {
        const uint32_t nkb = L->sh_w_pad / 64;
        uint32_t want = std::min<uint32_t>(kShSplitMax, static_cast<uint32_t>(L->num_sms) / n_tiles);
        want = std::max<uint32_t>(1, std::min(want, nkb));
        const uint32_t kps = (nkb + want - 1) / want;
        L->sh_splits = (nkb + kps - 1) / kps;
    }
    if (L->sh_splits) {
        mp::launch_gemm_tc(true, &tmX, &L->tm_w1s, L->sh_h, s1, L->sh_meta, L->sh_meta + 2, sh_sms, ss);
        mp::launch_gemm_tc_epi(mp::kEpiF32Part, &L->tm_hs, &L->tm_w2s, L->sh_o32, s2, L->sh_meta, L->sh_meta + 2,
                               sh_sms, ss, 0, nullptr, nullptr, nullptr, L->sh_splits);
    } else if (sh_pair) {
        mp::launch_gemm_tc2(true, &tmX, &L->tm_w1sh, L->sh_h, s1, L->sh_meta, L->sh_meta + 4, sh_sms, ss, nullptr);
        mp::launch_gemm_tc2(false, &L->tm_hs, &L->tm_w2sh, L->sh_o, s2, L->sh_meta, L->sh_meta + 4, sh_sms, ss,
                            nullptr);
    } else {
        mp::launch_gemm_tc(true, &tmX, &L->tm_w1s, L->sh_h, s1, L->sh_meta, L->sh_meta + 2, sh_sms, ss);
        mp::launch_gemm_tc(false, &L->tm_hs, &L->tm_w2s, L->sh_o, s2, L->sh_meta, L->sh_meta + 2, sh_sms, ss);
    }
    ck_launch("shared expert");
    ck(cudaEventRecord(L->sh_join, ss), "join shared expert");
    L->launches += 3;
}

// Decode batches (T * k_max <= 8 rows per sub-expert on average): nearly every
// sub-expert receives a token, gemm1 reads its weights group by group in tile
// order, and the routing chain before it leaves HBM idle.  Optionally
// (MOEPRISM_DECODE_PF_MB > 0) prefetch the W1 tiles of the first groups into
// L2 on a side stream meanwhile; joined before the combine (graph-capturable).
// Off by default: measured 3-5% slower at Qwen decode (the prefetch competes
// with the routing chain; profiles/r02e_pf_sweep.txt).
void prefetch_routed_weights(mp_layer_s* L, uint32_t T, cudaStream_t s) {
    L->pf_pending = false;
    if (!L->use_tc || L->offload || !L->has_experts || (size_t)T * L->k_max > (size_t)8 * L->G) return;
    if (!L->pf_stream) {
        ck(cudaStreamCreateWithFlags(&L->pf_stream, cudaStreamNonBlocking), "prefetch stream");
        ck(cudaEventCreateWithFlags(&L->pf_fork, cudaEventDisableTiming), "prefetch event");
        ck(cudaEventCreateWithFlags(&L->pf_join, cudaEventDisableTiming), "prefetch event");
    }
    const size_t w1_group = (size_t)2 * L->w_pad * L->d_pad * L->esz;
    static const size_t cap = [] {  // MOEPRISM_DECODE_PF_MB: prefetch size (A/B)
        const char* e = std::getenv("MOEPRISM_DECODE_PF_MB");
        return (size_t)(e ? std::atoi(e) : 0) << 20;
    }();
    const size_t bytes = std::min<size_t>((size_t)L->G * w1_group, cap);
    if (!bytes) return;
    ck(cudaEventRecord(L->pf_fork, s), "prefetch fork");
    ck(cudaStreamWaitEvent(L->pf_stream, L->pf_fork, 0), "prefetch fork");
    mp::launch_l2_prefetch(L->W1, bytes, L->pf_stream);
    ck_launch("l2 prefetch");
    ck(cudaEventRecord(L->pf_join, L->pf_stream), "prefetch join");
    L->pf_pending = true;
    L->launches += 1;
}

// Small batches (<= 16 rows per sub-expert on average): the 1-SM gemm1
// gathers its A rows from x itself (TMA gather4, one per 4 rows and k-block)
// and dispatch writes only the permutation tables -- no x_perm.  Large
// batches materialise x_perm: gather4 moves ~5 B/cycle per SM, so a gathered
// 128-row A operand left gemm1 2.2-2.7x slower at 4096 Mixtral tokens
// (profiles/r02g_gather_ab.txt); decode batches gain 2-3%.
bool gather_batch(const mp_layer_s* L, const void* x, uint32_t T, uint32_t k_eff) {
    static const int gather_env = [] {  // MOEPRISM_GATHER=0 never / 1 always (A/B)
        const char* e = std::getenv("MOEPRISM_GATHER");
        return e ? std::atoi(e) : -1;
    }();
    const bool shape = gather_env == 1 || (gather_env < 0 && (size_t)T * k_eff <= (size_t)16 * L->G);
    return shape && L->use_tc && (L->d % 8) == 0 && (reinterpret_cast<uintptr_t>(x) % 16) == 0;
}

// bucket -> dispatch -> gemm1 -> gemm2 -> combine, given sel / w on the device.
void run_experts(mp_layer_s* L, const void* x, uint32_t T, const uint32_t* sel, const float* w, bool unit, void* y,
                 cudaStream_t s, StageTimer& tm, bool check_finite = false, bool with_shared = false,
                 uint32_t kscalar = 0, bool bucketed = false) {
    // Kernel choice (auto): the kernel with the lower expected SM time per
    // (sub-expert, 256-column N tile) over bucket sizes M +- sqrt(M), M = T k /
    // G (per-token k: k_max), in units of a 1-SM 128-row tile (a partial last
    // tile of r rows loads only its rows: 0.5 + 0.5 r / 128).  A CTA-pair
    // tile (256 rows; with swapped remainder tiles, gemm_tc2.cu, a remainder
    // tile costs about a full one) costs 1.25 of those (2 SMs; round-2
    // 128-deep pair k-blocks) plus a per-tile overhead that matters at short
    // K (the pair epilogue is twice the SM time of a 1-SM one): + 2 / (64-deep
    // k-blocks of the shorter GEMM).  In-process A/B (tests/probes/tile_ab_k.py,
    // profiles/r02ae_tile_ab.txt): pairs ahead at the Mixtral shape for k >= 3
    // (4-13%), 1.6% at k = 2 (the model keeps 1-SM tiles there); 1-SM tiles
    // ahead at Qwen prefill (K = 384 down projection) for k = 8 and 16 by
    // 6% / 3%, ties at k = 4 and 12.  Without the swapped remainders (A/B) the
    // round-1 rule: pairs credited 5% on padded rows.
    {
        const double rows = double(T) * (kscalar ? kscalar : L->k_max) / L->G;
        const double sd = std::sqrt(rows > 1.0 ? rows : 1.0);
        double c128 = 0.0, c256 = 0.0, pad128 = 0.0, pad256 = 0.0;
        for (double m : {rows - sd, rows, rows + sd}) {
            const double mm = m < 1.0 ? 1.0 : m;
            const double full = std::floor(mm / 128.0), r = mm - 128.0 * full;
            c128 += full + (r > 0.0 ? 0.5 + 0.5 * r / 128.0 : 0.0);
            c256 += std::ceil(mm / 256.0);
            pad128 += std::ceil(mm / 128.0) * 128.0;
            pad256 += std::ceil(mm / 256.0) * 256.0;
        }
        static const double pair_cost = [] {  // MOEPRISM_PAIR_COST: SM time of a pair tile / a 1-SM tile (A/B)
            const char* e = std::getenv("MOEPRISM_PAIR_COST");
            return e ? std::atof(e) : 1.25;
        }();
        // per GEMM: its own K (gemm1 d_pad, gemm2 w_pad) in the short-K term
        auto pairs_for = [&](uint32_t K) {
            const double nkb = std::max(1.0, K / 64.0);
            return mp::pair_swap_enabled() ? c256 * (pair_cost + 2.0 / nkb) < c128
                                           : (rows >= 192.0 && pad256 / 1.05 < pad128);
        };
        static const bool per_gemm = [] {  // MOEPRISM_TILE_PER_GEMM=0: one choice for both GEMMs (A/B)
            const char* e = std::getenv("MOEPRISM_TILE_PER_GEMM");
            return !(e && e[0] == '0');
        }();
        const bool p1 = per_gemm ? pairs_for(L->d_pad) : pairs_for(std::min(L->d_pad, L->w_pad));
        const bool p2 = per_gemm ? pairs_for(L->w_pad) : p1;
        L->tile256 = L->tile_mode >= 2 || (L->tile_mode == 0 && p1);
        L->tile256_g2 = L->tile_mode >= 2 || (L->tile_mode == 0 && p2);
    }
    if (!bucketed) {
        tm.begin(1);
        mp::launch_bucket_local(sel, T, L->k_max, L->G, L->ws, s);
        mp::launch_bucket_scan(T, L->G, L->ws, s);
        ck_launch("bucket");
        tm.end(1, 2);
    }
    const bool gather = !L->tile256 && gather_batch(L, x, T, kscalar ? kscalar : L->k_max);
    CUtensorMap tmXg;
    if (gather && !mp::make_tmap_bf16_2d(&tmXg, x, T, L->d, 1, 64)) fail(MP_ERR_CUDA, "gather tensor map");
    tm.begin(2);
    if (L->offload) offload_step(L, s);  // transfers counted in the dispatch stage
    // the fused routing kernel already flagged non-finite input rows (sum |x|),
    // and at decode batches wrote the permutation tables too
    const bool tables_done = bucketed && L->r_tables && gather;
    L->r_tables = false;
    if (!tables_done) {
        mp::launch_dispatch(L->dtype, x, T, L->d, L->d_pad, sel, w, L->k_max, L->G, L->ws,
                            gather ? nullptr : L->x_perm, s, !bucketed,
                            bucketed ? mp::route_tokens_per_block(T) : mp::kRouteTokensPerBlock);
        ck_launch("dispatch");
    }
    tm.end(2, tables_done ? 0 : 1);
    mp::GemmShape g1{L->G, L->d_pad, 2 * L->w_pad, T * L->k_max, L->w_pad, 2 * L->w_pad};
    mp::GemmShape g2{L->G, L->w_pad, L->d_pad, T * L->k_max, L->d_pad, L->d_pad};
    tm.begin(3);
    const uint32_t* gmap = L->offload ? L->gmap_dev : nullptr;
    static const bool tail_env = [] {  // MOEPRISM_W1_TAIL=0: gemm1 reads the padded W1 rows too (A/B)
        const char* e = std::getenv("MOEPRISM_W1_TAIL");
        return !(e && e[0] == '0');
    }();
    // decode batches (a few rows per sub-expert: HBM-bound on the weights)
    // skip the W1 / W2 padding of w_sub -> w_pad; measured slower for large
    // buckets (the tail tile's split B loads), so only there
    const bool trim = tail_env && !L->offload && L->w_sub < L->w_pad &&
                      (size_t)T * (kscalar ? kscalar : L->k_max) <= (size_t)64 * L->G;
    if (L->use_tc && L->tile256)
        mp::launch_gemm_tc2(true, &L->tm_xperm, L->offload ? &L->tm_w1ch : &L->tm_w1h, L->h, g1, L->ws.offsets,
                            L->ws.mprefix_tc2, L->num_sms, s, gmap, L->tile_mode == 3 ? nullptr : L->tm_xperm_s);
    else if (L->use_tc)
        mp::launch_gemm_tc(true, gather ? &tmXg : &L->tm_xperm, L->offload ? &L->tm_w1c : &L->tm_w1, L->h, g1,
                           L->ws.offsets, L->ws.mprefix_tc, L->num_sms, s, gmap, nullptr,
                           gather ? nullptr : L->tm_xperm_s, nullptr, trim ? &L->w1_tail : nullptr,
                           gather ? L->ws.perm_tok : nullptr);
    else
        mp::launch_gemm1_simt(L->dtype, L->x_perm, L->W1, L->h, g1, L->ws.offsets, L->ws.mprefix_simt, s);
    ck_launch("gemm1");
    const bool shared = with_shared && L->sh_ff;
    tm.end(3, 1);
    tm.begin(4);
    if (L->use_tc && L->tile256_g2)
        mp::launch_gemm_tc2(false, &L->tm_h, L->offload ? &L->tm_w2ch : &L->tm_w2h, L->o, g2, L->ws.offsets,
                            L->ws.mprefix_tc2, L->num_sms, s, gmap, L->tile_mode == 3 ? nullptr : L->tm_h_s,
                            &L->tm_o);
    else if (L->use_tc)
        mp::launch_gemm_tc(false, &L->tm_h, L->offload ? &L->tm_w2c : trim ? &L->tm_w2d : &L->tm_w2, L->o, g2,
                           L->ws.offsets,
                           L->ws.mprefix_tc, L->num_sms, s, gmap, nullptr, L->tm_h_s, &L->tm_o);
    else
        mp::launch_gemm2_simt(L->dtype, L->h, L->W2, L->o, g2, L->ws.offsets, L->ws.mprefix_simt, s);
    ck_launch("gemm2");
    tm.end(4, 1);
    if (shared) ck(cudaStreamWaitEvent(s, L->sh_join, 0), "join shared expert");
    if (L->pf_pending) {
        ck(cudaStreamWaitEvent(s, L->pf_join, 0), "join prefetch");
        L->pf_pending = false;
    }
    tm.begin(5);
    const uint32_t group_S = unit ? L->S : 0;
    mp::launch_combine(L->dtype, L->o, L->d, L->d_pad, L->ws.slot_row, sel, w, L->k_max, group_S, T, y, s,
                       shared ? (L->sh_splits ? static_cast<const void*>(L->sh_o32) : L->sh_o) : nullptr,
                       shared ? L->sh_w : nullptr, (with_shared && L->residual) ? x : nullptr,
                       shared ? L->sh_splits : 0u, static_cast<size_t>(T) * L->d_pad, kscalar, L->num_sms);
    ck_launch("combine");
    tm.end(5, 1);
}

// Returns true when the bucketing of this forward already ran (fused into the
// tensor-core router's epilogue; requested by fuse_bucket).
bool route(mp_layer_s* L, const void* x, uint32_t T, const uint32_t* kpt, uint32_t k, cudaStream_t s,
           StageTimer& tm, bool with_shared = false, bool fuse_bucket = false) {
    bool bucketed = false;
    if (!kpt && (k < 1 || k > L->k_max || k > L->G))
        fail(MP_ERR_VALIDATION, "k_active = " + std::to_string(k) + " out of range [1, " +
                                    std::to_string(std::min(L->k_max, L->G)) + "]");
    tm.begin(0);
    // zeroed before the router so the router -> routing-epilogue boundary is
    // kernel to kernel (programmatic dependent launch)
    if (L->has_router) ck(cudaMemsetAsync(L->r_flagged, 0, 2 * sizeof(uint32_t), s), "memset routing stats");
    // The shared expert forks here (it depends on x only) but its kernels are
    // enqueued after the routing chain's, so the routing CTAs reach the SMs
    // first (Qwen prefill: 4-5% at k = 16, <= 1% elsewhere;
    // profiles/r02u_shared_order_ab.txt).  MOEPRISM_SH_ORDER=0: enqueued first.
    static const int sh_order = [] {
        const char* e = std::getenv("MOEPRISM_SH_ORDER");
        return e ? std::atoi(e) : 1;
    }();
    bool sh_deferred = false;
    if (with_shared && L->sh_ff) {
        if (reinterpret_cast<uintptr_t>(x) % 16) fail(MP_ERR_VALIDATION, "shared expert needs 16-byte aligned x");
        if (sh_order == 1) {
            ck(cudaEventRecord(L->sh_fork, s), "fork shared expert");
            sh_deferred = true;
        } else {
            launch_shared_expert(L, x, T, s);
        }
    }
    if (with_shared) prefetch_routed_weights(L, T, s);
    if (L->desc.router_mode == MP_ROUTER_PROXY) {
        pack_gates(L);
        if (L->proxy_tc && (reinterpret_cast<uintptr_t>(x) % 16) == 0) {
            const uint32_t nr2 = 2 * L->n_gate_rows;
            const mp::RouterTcPlan pl = mp::plan_router_tc(T, L->d, nr2, L->num_sms);
            CUtensorMap tmX;
            if (!mp::make_tmap_bf16_2d(&tmX, x, T, L->d, 128, 64)) fail(MP_ERR_CUDA, "proxy router tensor map");
            mp::launch_router_tc(&tmX, &L->tm_pplanes, pl, T, L->p_partial, s, true);
            // fp32 partials: one more rounding of <= 2^-24 sum|x||W| per token
            const mp::RouterGuard rg{mp::router_guard_coef(pl.chunk_kb * 64, L->p_wmax) + 0x1.0p-24 * L->p_wmax,
                                     L->r_guard_floor};
            mp::launch_proxy_tc_topk(L->p_partial, pl.ks, T, L->n_gate_rows, L->p_npad, L->gate_off, L->G, L->k_max,
                                     kpt, k, L->desc.weight_mode, L->sel, L->wsel, L->ws.err, rg, x, L->d, L->scores,
                                     L->p_class,
                                     L->r_flagged, s);
            mp::launch_proxy_fixup(x, L->d, L->gate_rows, L->up_rows, L->gate_off, L->G, L->k_max, kpt, k,
                                   L->desc.weight_mode, L->sel, L->wsel, L->ws.err, L->scores, L->p_class, L->r_flagged,
                                   L->num_sms, s);
            ck_launch("router(proxy, tensor core)");
            tm.end(0, 3);
        } else {
            mp::launch_proxy_scores(L->dtype, x, T, L->d, L->gate_rows, L->up_rows, L->gate_off, L->n_gate_rows, L->G,
                                    reinterpret_cast<float*>(L->scores), s);
            mp::launch_router_scores_topk(reinterpret_cast<const float*>(L->scores), T, L->G, L->k_max, kpt, k,
                                          L->desc.weight_mode, L->sel, L->wsel, L->ws.err, L->r_flagged, s);
            ck_launch("router(proxy)");
            tm.end(0, 3);
        }
    } else {
        if (!L->has_router) fail(MP_ERR_VALIDATION, "experts-only layer (MP_LAYER_EXPERTS_ONLY) has no router");
        if (!L->router_set) fail(MP_ERR_VALIDATION, "router weights not set (mp_layer_set_router)");
        if (L->router_tc && (reinterpret_cast<uintptr_t>(x) % 16) == 0) {
            const mp::RouterTcPlan pl = mp::plan_router_tc(T, L->d, L->G, L->num_sms);
            CUtensorMap tmX;
            if (!mp::make_tmap_bf16_2d(&tmX, x, T, L->d, 128, 64)) fail(MP_ERR_CUDA, "router tensor map");
            mp::launch_router_tc(&tmX, &L->tm_wplanes, pl, T, L->r_partial, s);
            const mp::RouterGuard rg{mp::router_guard_coef(pl.chunk_kb * 64, L->r_wmax), L->r_guard_floor};
            L->r_last_ks = pl.ks;
            L->r_last_T = T;
            static const bool fuse_env = [] {  // MOEPRISM_FUSE_BUCKET=0: separate top-k / fixup / bucketing (A/B)
                const char* e = std::getenv("MOEPRISM_FUSE_BUCKET");
                return !(e && e[0] == '0');
            }();
            if (fuse_bucket && fuse_env && L->has_experts && (L->d % 4) == 0) {
                // routing epilogue + exact near-tie re-selection + bucketing in one kernel
                // (many K splits -- small batches -- are summed CTA-wide inside it)
                uint32_t ks = pl.ks;
                static const uint32_t reduce_above = [] {  // MOEPRISM_PARTIALS_REDUCE_ABOVE: separate reduce (A/B)
                    const char* e = std::getenv("MOEPRISM_PARTIALS_REDUCE_ABOVE");
                    return e ? static_cast<uint32_t>(std::atoi(e)) : 0xFFFFFFFFu;
                }();
                if (ks > reduce_above) {
                    mp::launch_partials_reduce(L->r_partial, ks, T, L->G, pl.Npad, s);
                    ks = 1;
                    L->r_last_ks = 1;  // plane 0 now holds the logits
                    L->launches += 1;
                }
                // decode batches (gemm1 gathers its rows from x): the permutation
                // tables come out of the routing kernel and dispatch is skipped
                L->r_tables = mp::launch_route_bucket(L->r_partial, ks, T, L->G, pl.Npad, L->k_max, kpt, k, L->desc.weight_mode,
                                        L->sel, L->wsel, rg, x, L->d, L->wrT, L->r_ticket, L->r_flagged,
                                        L->ws, s, mp::route_tokens_per_block(T), L->num_sms,
                                        gather_batch(L, x, T, kpt ? L->k_max : k));
                bucketed = true;
                ck_launch("router(tc)+bucket");
                tm.end(0, 2);
            } else {
                mp::launch_partials_topk(L->r_partial, pl.ks, T, L->G, pl.Npad, L->k_max, kpt, k, L->desc.weight_mode,
                                         L->sel, L->wsel, L->ws.err, rg, x, L->d, L->r_flagged, s);
                mp::launch_router_fixup(L->dtype, x, L->d, L->wrT, L->G, L->k_max, kpt, k, L->desc.weight_mode,
                                        L->sel, L->wsel, L->ws.err, L->r_flagged, L->num_sms, s);
                ck_launch("router(tc)");
                tm.end(0, 3);
            }
        } else {
            mp::launch_router_linear(L->dtype, x, T, L->d, L->wrT, L->G, L->k_max, kpt, k, L->desc.weight_mode,
                                     L->sel, L->wsel, L->ws.err, L->r_flagged, s);
            ck_launch("router");
            tm.end(0, 1);
        }
    }
    if (sh_deferred) launch_shared_expert(L, x, T, s, true);
    return bucketed;
}

void copy_outputs(mp_layer_s* L, uint32_t T, uint32_t* sel_out, float* w_out, uint32_t* off_out, cudaStream_t s,
                  cudaMemcpyKind kind) {
    if (sel_out) ck(cudaMemcpyAsync(sel_out, L->sel, (size_t)T * L->k_max * 4, kind, s), "sel_out");
    if (w_out) ck(cudaMemcpyAsync(w_out, L->wsel, (size_t)T * L->k_max * 4, kind, s), "w_out");
    if (off_out) ck(cudaMemcpyAsync(off_out, L->ws.offsets, (size_t)(L->G + 1) * 4, kind, s), "offsets_out");
}

void check_tokens(mp_layer_s* L, uint32_t T) {
    if (T > L->max_tokens)
        fail(MP_ERR_VALIDATION,
             "n_tokens " + std::to_string(T) + " exceeds max_tokens " + std::to_string(L->max_tokens));
}

void raise_device_errors(int flags) {
    if (flags & 2) fail(MP_ERR_VALIDATION, "input vector is not finite");
    if (flags & 1) fail(MP_ERR_VALIDATION, "selection out of range or duplicated (k_active / active sub-expert)");
}

}  // namespace

// ============================================================== C-ABI

MP_API const char* mp_version(void) { return "moeprism-b200 0.1 (sm_100a)"; }
MP_API const char* mp_last_error(void) { return g_err.c_str(); }

MP_API mp_status mp_device_check(int32_t dev) {
    return guarded([&] {
        int n = 0;
        ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (dev < 0 || dev >= n) fail(MP_ERR_CUDA, "no CUDA device " + std::to_string(dev));
        cudaDeviceProp p;
        ck(cudaGetDeviceProperties(&p, dev), "cudaGetDeviceProperties");
        if (p.major != 10 || p.minor != 0)
            fail(MP_ERR_CUDA, std::string("device ") + p.name + " is sm_" + std::to_string(p.major) +
                                  std::to_string(p.minor) + "; this library carries sm_100a code only");
    });
}

MP_API mp_status mp_layer_create(const mp_layer_desc* desc, mp_layer_t* out) {
    return guarded([&] {
        if (!desc || !out) fail(MP_ERR_VALIDATION, "null argument");
        const mp_layer_desc& D = *desc;
        if (D.n_experts < 1 || D.n_subexperts < 1) fail(MP_ERR_VALIDATION, "need n_experts >= 1 and n_subexperts >= 1");
        if (D.d_model < 1 || D.d_ff < 1) fail(MP_ERR_VALIDATION, "toy expert needs d_model >= 1 and d_ff >= 1");
        if (D.d_ff < D.n_subexperts) fail(MP_ERR_VALIDATION, "partition needs at least as many neurons as sub-experts");
        const uint64_t G = (uint64_t)D.n_experts * D.n_subexperts;
        if (G > mp::kMaxG) fail(MP_ERR_VALIDATION, "E*S = " + std::to_string(G) + " exceeds " + std::to_string(mp::kMaxG));
        if (D.k_max < 1 || D.k_max > G) fail(MP_ERR_VALIDATION, "k_max must be in [1, E*S]");
        if (D.dtype != MP_DTYPE_F32 && D.dtype != MP_DTYPE_BF16) fail(MP_ERR_VALIDATION, "unknown dtype");
        if (D.router_mode > MP_ROUTER_PROXY || D.weight_mode > MP_WEIGHT_SOFTMAX_RENORM)
            fail(MP_ERR_VALIDATION, "unknown router / weight mode");
        if (D.max_tokens < 1) fail(MP_ERR_VALIDATION, "max_tokens must be >= 1");
        if (D.flags & ~(MP_LAYER_ROUTER_ONLY | MP_LAYER_EXPERTS_ONLY | MP_LAYER_SHARED_SCRATCH) ||
            (D.flags & (MP_LAYER_ROUTER_ONLY | MP_LAYER_EXPERTS_ONLY)) == (MP_LAYER_ROUTER_ONLY | MP_LAYER_EXPERTS_ONLY))
            fail(MP_ERR_VALIDATION, "invalid layer role flags");
        {
            int rc = mp_device_check(D.device);
            if (rc) fail(rc, g_err);
        }
        DeviceGuard dg(D.device);
        auto* L = new mp_layer_s;
        try {
            L->desc = D;
            L->E = D.n_experts;
            L->S = D.n_subexperts;
            L->G = static_cast<uint32_t>(G);
            L->d = D.d_model;
            L->ff = D.d_ff;
            L->dtype = D.dtype;
            L->k_max = D.k_max;
            L->max_tokens = D.max_tokens;
            L->esz = D.dtype == MP_DTYPE_BF16 ? 2 : 4;
            L->use_tc = D.dtype == MP_DTYPE_BF16;
            if (const char* env = std::getenv("MOEPRISM_BF16_GEMM"))
                if (std::string(env) == "simt") L->use_tc = false;  // diagnostics only
            if (const char* env = std::getenv("MOEPRISM_TC_TILE"))
                L->tile_mode = std::string(env) == "256"         ? 2
                               : std::string(env) == "128"       ? 1
                               : std::string(env) == "256-plain" ? 3
                                                                 : 0;
            const uint32_t w_sub = (L->ff + L->S - 1) / L->S;
            L->w_pad = round_up(w_sub, 128);
            L->w_sub = w_sub;
            L->d_pad = round_up(L->d, 64);
            L->G_pad = round_up(L->G, 64);
            L->rows_cap = round_up(std::max<uint32_t>(L->max_tokens * L->k_max, 1), 128);
            L->w2_rows = round_up(L->G * L->d_pad, 256);
            int dev = D.device;
            ck(cudaDeviceGetAttribute(&L->num_sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
            L->assignment.resize(L->E);
            L->has_part.assign(L->E, 0);
            L->packed.assign(L->E, 0);
            L->raw.assign(L->E, nullptr);
            L->gate_r.assign(L->E, 0);
            L->gates.resize(L->E);
            L->has_gates.assign(L->E, 0);
            const bool experts = !(D.flags & MP_LAYER_ROUTER_ONLY);
            const bool router = !(D.flags & MP_LAYER_EXPERTS_ONLY);
            L->has_experts = experts;
            L->has_router = router;
            if (experts) {
                const size_t w1 = (size_t)L->G * 2 * L->w_pad * L->d_pad;
                const size_t w2 = (size_t)L->w2_rows * L->w_pad;
                L->W1 = dalloc<char>(w1 * L->esz, "W1");
                L->W2 = dalloc<char>(w2 * L->esz, "W2");
                ck(cudaMemset(L->W2, 0, w2 * L->esz), "memset W2");
                L->d_nmap = dalloc<int32_t>((size_t)L->S * L->w_pad, "nmap");
                L->nmap_all = dalloc<int32_t>((size_t)L->E * L->S * L->w_pad, "nmap (all experts)");
            }
            if (router) {
                L->wrT = dalloc<float>((size_t)L->G_pad * L->d, "router");
                L->router_tc = D.dtype == MP_DTYPE_BF16 && (L->d % 8) == 0 && D.router_mode == MP_ROUTER_LINEAR;
                if (const char* env = std::getenv("MOEPRISM_ROUTER"))
                    if (std::string(env) == "simt") L->router_tc = false;  // diagnostics only
                if (L->router_tc) {
                    L->r_npad = round_up(L->G, 32);
                    // K-split partials [ks][T][Npad]: 256-deep splits, or 64-deep ones
                    // when few token tiles (plan_router_tc) -- size for both
                    const size_t n_part = mp::router_tc_partial_rows(L->max_tokens, L->d, L->G, L->num_sms);
                    L->wr_planes = dalloc<char>((size_t)3 * L->r_npad * L->d * 2, "router planes");
                    L->r_partial = dalloc<double>(n_part * L->r_npad, "router partials");
                    L->r_ticket = dalloc<uint32_t>(4, "router ticket");
                    ck(cudaMemset(L->r_ticket, 0, 4 * sizeof(uint32_t)), "memset ticket");
                    if (!mp::make_tmap_bf16_2d(&L->tm_wplanes, L->wr_planes, 3ull * L->r_npad, L->d,
                                               mp::router_tc_cols_per_cta(L->G), 64))
                        fail(MP_ERR_CUDA, "router planes tensor map");
                }
                if (D.router_mode == MP_ROUTER_PROXY) L->gate_off = dalloc<uint32_t>(L->G + 1, "gate offsets");
                if (const char* env = std::getenv("MOEPRISM_ROUTER_GUARD")) L->r_guard_floor = std::atof(env);
                L->r_flagged = dalloc<uint32_t>((size_t)L->max_tokens + 2, "routing stats");
                ck(cudaMemset(L->r_flagged, 0, 2 * sizeof(uint32_t)), "memset routing stats");
            }
            const size_t tk = (size_t)L->max_tokens * L->k_max;
            // bucketing blocks: 32 tokens, or 8 / 2 in the fused router for small batches
            const uint32_t nblk = std::max({(L->max_tokens + mp::kRouteTokensPerBlock - 1) / mp::kRouteTokensPerBlock,
                                            (std::min<uint32_t>(L->max_tokens, 1024) + 7) / 8,
                                            (std::min<uint32_t>(L->max_tokens, 256) + 1) / 2});
            L->sel = dalloc<uint32_t>(tk, "sel");
            L->wsel = dalloc<float>(tk, "w");
            L->kpt_dev = dalloc<uint32_t>(L->max_tokens, "k per token");
            L->ws.err = dalloc<int>(2, "err");  // [0] flags, [1] scratch (router max |W|)
            ck(cudaMemset(L->ws.err, 0, 2 * sizeof(int)), "memset err");
            L->x_stage = dalloc<char>((size_t)L->max_tokens * L->d * L->esz, "x stage");
            if (experts) {
                L->ws.lrank = dalloc<uint32_t>(tk, "lrank");
                L->ws.block_counts = dalloc<uint32_t>((size_t)nblk * L->G, "block counts");
                L->ws.block_base = dalloc<uint32_t>((size_t)nblk * L->G, "block base");
                L->ws.offsets = dalloc<uint32_t>(L->G + 1, "offsets");
                L->ws.mprefix_tc = dalloc<uint32_t>(L->G + 1, "mprefix");
                L->ws.mprefix_simt = dalloc<uint32_t>(L->G + 1, "mprefix");
                L->ws.mprefix_tc2 = dalloc<uint32_t>(L->G + 1, "mprefix");
                L->ws.perm_tok = dalloc<uint32_t>(L->rows_cap, "perm");
                L->ws.perm_w = dalloc<float>(L->rows_cap, "perm w");
                L->ws.slot_row = dalloc<uint32_t>(tk, "slot row");
                const size_t bx = (size_t)L->rows_cap * L->d_pad * L->esz, bh = (size_t)L->rows_cap * L->w_pad * L->esz;
                // fp32 mode keeps sub-expert outputs in double until the combine rounds them
                const size_t bo = (size_t)L->rows_cap * L->d_pad * (L->dtype == MP_DTYPE_F32 ? 8 : L->esz);
                L->shared_scratch = (D.flags & MP_LAYER_SHARED_SCRATCH) != 0;
                if (L->shared_scratch) {
                    L->x_perm = scratch_acquire(bx, "x_perm (shared)");
                    L->h = scratch_acquire(bh, "h (shared)");
                    L->o = scratch_acquire(bo, "o (shared)");
                } else {
                    L->x_perm = dalloc<char>(bx, "x_perm");
                    L->h = dalloc<char>(bh, "h");
                    L->o = dalloc<char>(bo, "o");
                }
                L->y_stage = dalloc<char>((size_t)L->max_tokens * L->d * L->esz, "y stage");
                if (L->use_tc) {
                    bool ok =
                        mp::make_tmap_bf16_2d(&L->tm_xperm, L->x_perm, L->rows_cap, L->d_pad, 128, 64) &&
                        mp::make_tmap_bf16_2d(&L->tm_w1, L->W1, (uint64_t)L->G * 2 * L->w_pad, L->d_pad, 256, 64) &&
                        // gemm2's A (h) stops at the w_sub valid neurons: its padding columns
                        // are zero-filled by the TMA, not read (they hold garbage when gemm1
                        // skipped the padding rows of W1, w1_tail)
                        mp::make_tmap_bf16_2d_ex(&L->tm_h, L->h, L->rows_cap, L->w_sub, L->w_pad, 128, 64, true) &&
                        mp::make_tmap_bf16_2d(&L->tm_w2, L->W2, L->w2_rows, L->w_pad, 256, 64) &&
                        // decode batches (HBM-bound): W2 read up to w_sub only, 64-byte L2
                        // promotion so the trimmed row end does not fetch the padding
                        mp::make_tmap_bf16_2d_ex(&L->tm_w2d, L->W2, L->w2_rows, L->w_sub, L->w_pad, 256, 64, true, w2d_promo()) &&
                        mp::make_tmap_bf16_2d(&L->tm_w1h, L->W1, (uint64_t)L->G * 2 * L->w_pad, L->d_pad, 128, 64) &&
                        mp::make_tmap_bf16_2d(&L->tm_w2h, L->W2, L->w2_rows, L->w_pad, 128, 64) &&
                        mp::make_tmap_bf16_2d_ex(&L->tm_o, L->o, L->rows_cap, L->d, L->d_pad, 32, 32, false);
                    for (int b = 0; b < 3 && ok; ++b)
                        ok = mp::make_tmap_bf16_2d(&L->tm_xperm_s[b], L->x_perm, L->rows_cap, L->d_pad, 16u << b, 64) &&
                             mp::make_tmap_bf16_2d_ex(&L->tm_h_s[b], L->h, L->rows_cap, L->w_sub, L->w_pad, 16u << b, 64,
                                                      true);
                    if (ok && L->w_sub < L->w_pad) {  // gemm1: the padding rows of each W1 group are not read
                        L->w1_tail.valid = L->w_sub;
                        L->w1_tail.tail_rows = round_up(L->w_sub % mp::kIlv ? L->w_sub % mp::kIlv : mp::kIlv, 8);
                        ok = mp::make_tmap_bf16_2d(&L->w1_tail.half, L->W1, (uint64_t)L->G * 2 * L->w_pad, L->d_pad, 128,
                                                   64) &&
                             mp::make_tmap_bf16_2d(&L->w1_tail.part, L->W1, (uint64_t)L->G * 2 * L->w_pad, L->d_pad,
                                                   L->w1_tail.tail_rows, 64);
                    }
                    if (!ok) fail(MP_ERR_CUDA, "cuTensorMapEncodeTiled failed");
                }
            }
        } catch (...) {
            free_layer(L);
            throw;
        }
        *out = L;
    });
}

MP_API mp_status mp_layer_destroy(mp_layer_t h) {
    return guarded([&] {
        if (!h) return;
        DeviceGuard dg(h->desc.device);
        cudaDeviceSynchronize();
        free_layer(h);
    });
}

MP_API mp_status mp_layer_get_desc(mp_layer_t h, mp_layer_desc* out) {
    return guarded([&] {
        if (!h || !out) fail(MP_ERR_VALIDATION, "null argument");
        *out = h->desc;
    });
}

MP_API mp_status mp_layer_load_expert(mp_layer_t L, uint32_t e, const float* wg, const float* wu, const float* wd) {
    return guarded([&] {
        if (!L || !wg || !wu || !wd) fail(MP_ERR_VALIDATION, "null argument");
        if (e >= L->E) fail(MP_ERR_VALIDATION, "expert " + std::to_string(e) + " out of range");
        if (!L->has_experts) fail(MP_ERR_VALIDATION, "router-only layer holds no expert weights");
        DeviceGuard dg(L->desc.device);
        const size_t n = (size_t)L->d * L->ff;
        if (!L->raw[e]) L->raw[e] = dalloc<float>(3 * n, "expert staging");
        float* dst = L->raw[e];
        const float* srcs[3] = {wg, wu, wd};
        for (int m = 0; m < 3; ++m)
            ck(cudaMemcpy(dst + m * n, srcs[m], n * sizeof(float), cudaMemcpyDefault), "expert upload");
        // validate(ToyExpert): every weight finite (inc/expert.hpp:34-37)
        ck(cudaMemset(L->ws.err, 0, sizeof(int)), "memset");
        mp::launch_finite_check(dst, 3 * n, L->ws.err, 0);
        ck_launch("finite check");
        int flag = 0;
        ck(cudaMemcpy(&flag, L->ws.err, sizeof(int), cudaMemcpyDeviceToHost), "flag");
        if (flag) {
            cudaFree(L->raw[e]);
            L->raw[e] = nullptr;
            fail(MP_ERR_VALIDATION, "toy expert weight is not finite");
        }
        L->packed[e] = 0;
        maybe_pack(L, e);
    });
}

MP_API mp_status mp_layer_load_expert_file(mp_layer_t L, uint32_t e, const char* path) {
    return guarded([&] {
        if (!L || !path) fail(MP_ERR_VALIDATION, "null argument");
        mp::MpexData m = mp::read_mpex(path);
        if (m.d_model != L->d || m.d_ff != L->ff)
            fail(MP_ERR_VALIDATION, std::string(path) + " holds a " + std::to_string(m.d_model) + "x" +
                                        std::to_string(m.d_ff) + " expert; the layer expects " +
                                        std::to_string(L->d) + "x" + std::to_string(L->ff));
        int rc = mp_layer_load_expert(L, e, m.w_gate.data(), m.w_up.data(), m.w_down.data());
        if (rc) fail(rc, g_err);
    });
}

MP_API mp_status mp_layer_set_partition(mp_layer_t L, uint32_t e, uint32_t n_sub, const uint32_t* a, size_t n) {
    return guarded([&] {
        if (!L || !a) fail(MP_ERR_VALIDATION, "null argument");
        if (e >= L->E) fail(MP_ERR_VALIDATION, "expert " + std::to_string(e) + " out of range");
        mp::validate_partition(n_sub, a, n);
        if (n_sub != L->S)
            fail(MP_ERR_VALIDATION, "partition has " + std::to_string(n_sub) + " sub-experts; the layer expects " +
                                        std::to_string(L->S));
        if (n != L->ff)
            fail(MP_ERR_VALIDATION, "partition covers " + std::to_string(n) + " neurons but the expert has d_ff " +
                                        std::to_string(L->ff));
        DeviceGuard dg(L->desc.device);
        if (L->packed[e] && !L->raw[e])
            fail(MP_ERR_VALIDATION, "expert " + std::to_string(e) +
                                        " is already packed; reload its weights to change the partition");
        L->assignment[e].assign(a, a + n);
        L->has_part[e] = 1;
        L->packed[e] = 0;
        maybe_pack(L, e);
    });
}

MP_API mp_status mp_layer_load_partition_map(mp_layer_t L, const char* path) {
    return guarded([&] {
        if (!L || !path) fail(MP_ERR_VALIDATION, "null argument");
        auto docs = mp::read_partition_map(path);
        for (const auto& d : docs) {
            if (d.expert_id >= L->E)
                fail(MP_ERR_VALIDATION, "partition map expert_id " + std::to_string(d.expert_id) + " out of range");
            int rc = mp_layer_set_partition(L, static_cast<uint32_t>(d.expert_id), d.n_subexperts,
                                            d.assignment.data(), d.assignment.size());
            if (rc) fail(rc, g_err);
            if (d.has_gates) {
                std::vector<uint32_t> off(1, 0), ids;
                for (const auto& l : d.gates) {
                    ids.insert(ids.end(), l.begin(), l.end());
                    off.push_back(static_cast<uint32_t>(ids.size()));
                }
                rc = mp_layer_set_gates(L, static_cast<uint32_t>(d.expert_id), d.r, off.data(), ids.data());
                if (rc) fail(rc, g_err);
            }
        }
    });
}

MP_API mp_status mp_layer_set_router(mp_layer_t L, const float* w_r) {
    return guarded([&] {
        if (!L || !w_r) fail(MP_ERR_VALIDATION, "null argument");
        if (!L->has_router) fail(MP_ERR_VALIDATION, "experts-only layer has no router");
        DeviceGuard dg(L->desc.device);
        const size_t n = (size_t)L->d * L->G;
        float* tmp = dalloc<float>(n, "router staging");
        cudaError_t e1 = cudaMemcpy(tmp, w_r, n * sizeof(float), cudaMemcpyDefault);
        if (e1 != cudaSuccess) {
            cudaFree(tmp);
            ck(e1, "router upload");
        }
        ck(cudaMemset(L->ws.err, 0, 2 * sizeof(int)), "memset");
        mp::launch_finite_check(tmp, n, L->ws.err, 0);
        // max |W_r| (the router's certification bound); ws.err[1] as scratch
        mp::launch_absmax(tmp, n, reinterpret_cast<float*>(L->ws.err + 1), 0);
        mp::launch_transpose_router(tmp, L->d, L->G, L->G_pad, L->wrT, 0);
        if (L->router_tc) mp::launch_split_router(tmp, L->d, L->G, L->r_npad, L->wr_planes, 0);
        ck_launch("router transpose");
        int flag[2] = {0, 0};
        ck(cudaMemcpy(flag, L->ws.err, 2 * sizeof(int), cudaMemcpyDeviceToHost), "flag");
        ck(cudaMemset(L->ws.err, 0, 2 * sizeof(int)), "memset");
        cudaFree(tmp);
        if (flag[0]) fail(MP_ERR_VALIDATION, "router weight is not finite");
        std::memcpy(&L->r_wmax, &flag[1], sizeof(float));
        L->router_set = true;
    });
}

MP_API mp_status mp_layer_set_shared_expert(mp_layer_t L, uint32_t ff_sh, const float* wg, const float* wu,
                                            const float* wd, const float* gate) {
    return guarded([&] {
        if (!L || !wg || !wu || !wd) fail(MP_ERR_VALIDATION, "null argument");
        if (!L->has_experts || !L->has_router)
            fail(MP_ERR_VALIDATION, "the shared expert belongs to a full layer (no EP role flags)");
        if (L->dtype != MP_DTYPE_BF16 || !L->use_tc) fail(MP_ERR_VALIDATION, "the shared expert needs the bf16 dtype");
        if (ff_sh < 1) fail(MP_ERR_VALIDATION, "shared expert needs d_ff >= 1");
        if (L->d % 8) fail(MP_ERR_VALIDATION, "shared expert needs d_model % 8 == 0 (16-byte rows for TMA)");
        if (L->sh_ff) fail(MP_ERR_VALIDATION, "shared expert already set");
        DeviceGuard dg(L->desc.device);
        const uint32_t w_pad = round_up(ff_sh, 128);
        const uint32_t w2_rows = round_up(L->d_pad, 256);
        const size_t n = (size_t)L->d * ff_sh;
        float* raw = dalloc<float>(3 * n, "shared staging");
        int32_t* nmap = nullptr;
        try {
            const float* srcs[3] = {wg, wu, wd};
            for (int m = 0; m < 3; ++m)
                ck(cudaMemcpy(raw + m * n, srcs[m], n * sizeof(float), cudaMemcpyDefault), "shared upload");
            ck(cudaMemset(L->ws.err, 0, sizeof(int)), "memset");
            mp::launch_finite_check(raw, 3 * n, L->ws.err, 0);
            int flag = 0;
            ck(cudaMemcpy(&flag, L->ws.err, sizeof(int), cudaMemcpyDeviceToHost), "flag");
            if (flag) fail(MP_ERR_VALIDATION, "shared expert weight is not finite");
            std::vector<int32_t> id(w_pad, -1);
            for (uint32_t j = 0; j < ff_sh; ++j) id[j] = static_cast<int32_t>(j);
            nmap = dalloc<int32_t>(w_pad, "shared nmap");
            ck(cudaMemcpy(nmap, id.data(), w_pad * 4, cudaMemcpyHostToDevice), "nmap");
            L->W1s = dalloc<char>((size_t)2 * w_pad * L->d_pad * 2, "W1 shared");
            L->W2s = dalloc<char>((size_t)w2_rows * w_pad * 2, "W2 shared");
            ck(cudaMemset(L->W2s, 0, (size_t)w2_rows * w_pad * 2), "memset");
            mp::launch_pack_w1(L->dtype, raw, raw + n, L->d, ff_sh, nmap, 1, w_pad, L->d_pad, L->W1s, 0);
            mp::launch_pack_w2(L->dtype, raw + 2 * n, L->d, ff_sh, nmap, 1, w_pad, L->d_pad, L->W2s, 0);
            ck_launch("shared pack");
            if (gate) {
                L->sh_gate = dalloc<float>(L->d, "shared gate");
                ck(cudaMemcpy(L->sh_gate, gate, L->d * sizeof(float), cudaMemcpyDefault), "shared gate");
                ck(cudaMemset(L->ws.err, 0, sizeof(int)), "memset");
                mp::launch_finite_check(L->sh_gate, L->d, L->ws.err, 0);
                ck(cudaMemcpy(&flag, L->ws.err, sizeof(int), cudaMemcpyDeviceToHost), "flag");
                if (flag) fail(MP_ERR_VALIDATION, "shared expert gate is not finite");
            }
            L->sh_h = dalloc<char>((size_t)L->max_tokens * w_pad * 2, "shared h");
            L->sh_o = dalloc<char>((size_t)L->max_tokens * L->d_pad * 2, "shared o");
            L->sh_o32 = dalloc<float>((size_t)kShSplitMax * std::min(L->max_tokens, kShSplitRows) * L->d_pad,
                                      "shared split-K partials");
            L->sh_w = dalloc<float>(L->max_tokens, "shared w");
            L->sh_meta = dalloc<uint32_t>(6, "shared meta");
            bool ok = mp::make_tmap_bf16_2d(&L->tm_w1s, L->W1s, 2ull * w_pad, L->d_pad, 256, 64) &&
                      mp::make_tmap_bf16_2d(&L->tm_w2s, L->W2s, w2_rows, w_pad, 256, 64) &&
                      mp::make_tmap_bf16_2d(&L->tm_hs, L->sh_h, L->max_tokens, w_pad, 128, 64) &&
                      mp::make_tmap_bf16_2d(&L->tm_w1sh, L->W1s, 2ull * w_pad, L->d_pad, 128, 64) &&
                      mp::make_tmap_bf16_2d(&L->tm_w2sh, L->W2s, w2_rows, w_pad, 128, 64);
            if (!ok) fail(MP_ERR_CUDA, "shared expert tensor maps");
            ck(cudaStreamCreateWithFlags(&L->sh_stream, cudaStreamNonBlocking), "shared expert stream");
            ck(cudaEventCreateWithFlags(&L->sh_fork, cudaEventDisableTiming), "shared expert event");
            ck(cudaEventCreateWithFlags(&L->sh_join, cudaEventDisableTiming), "shared expert event");
            ck(cudaDeviceSynchronize(), "shared pack");
        } catch (...) {
            cudaFree(raw);
            if (nmap) cudaFree(nmap);
            for (void** p : {&L->W1s, &L->W2s, reinterpret_cast<void**>(&L->sh_gate), &L->sh_h, &L->sh_o,
                             reinterpret_cast<void**>(&L->sh_o32),
                             reinterpret_cast<void**>(&L->sh_w), reinterpret_cast<void**>(&L->sh_meta)}) {
                if (*p) cudaFree(*p);
                *p = nullptr;
            }
            throw;
        }
        cudaFree(raw);
        cudaFree(nmap);
        L->sh_ff = ff_sh;
        L->sh_w_pad = w_pad;
        L->sh_w2_rows = w2_rows;
    });
}

MP_API mp_status mp_layer_set_residual(mp_layer_t L, int on) {
    return guarded([&] {
        if (!L) fail(MP_ERR_VALIDATION, "null argument");
        if (on && L->dtype != MP_DTYPE_BF16) fail(MP_ERR_VALIDATION, "the fused residual needs the bf16 dtype");
        L->residual = on != 0;
    });
}

MP_API mp_status mp_layer_set_gates(mp_layer_t L, uint32_t e, uint32_t r, const uint32_t* off, const uint32_t* ids) {
    return guarded([&] {
        if (!L || !off || !ids) fail(MP_ERR_VALIDATION, "null argument");
        if (e >= L->E) fail(MP_ERR_VALIDATION, "expert " + std::to_string(e) + " out of range");
        // validate(GateSet), inc/gating.hpp:33-43
        if (r < 1) fail(MP_ERR_VALIDATION, "gate set shape is inconsistent");
        std::vector<std::vector<uint32_t>> g(L->S);
        for (uint32_t s = 0; s < L->S; ++s) {
            if (off[s + 1] <= off[s]) fail(MP_ERR_VALIDATION, "every sub-expert needs at least one gate neuron");
            g[s].assign(ids + off[s], ids + off[s + 1]);
            for (size_t q = 0; q < g[s].size(); ++q) {
                if (q && g[s][q] < g[s][q - 1]) fail(MP_ERR_VALIDATION, "gate neuron lists must be ascending");
                if (g[s][q] >= L->ff)
                    fail(MP_ERR_VALIDATION, "gate neuron " + std::to_string(g[s][q]) + " out of range for d_ff " +
                                                std::to_string(L->ff));
            }
        }
        L->gates[e] = std::move(g);
        L->gate_r[e] = r;
        L->has_gates[e] = 1;
        L->gates_packed = false;
    });
}

MP_API mp_status mp_layer_forward(mp_layer_t L, const void* x, uint32_t T, const uint32_t* kpt, uint32_t k, void* y,
                                  uint32_t* sel_out, float* w_out, uint32_t* offsets_out, void* stream) {
    return guarded([&] {
        if (!L || (T && (!x || !y))) fail(MP_ERR_VALIDATION, "null argument");
        check_tokens(L, T);
        check_ready(L);
        if (T == 0) return;
        DeviceGuard dg(L->desc.device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        StageTimer tm(L, s);
        const bool bucketed = route(L, x, T, kpt, k, s, tm, true, true);
        run_experts(L, x, T, L->sel, L->wsel, L->desc.weight_mode == MP_WEIGHT_UNIT, y, s, tm, false, true,
                    kpt ? 0 : k, bucketed);
        copy_outputs(L, T, sel_out, w_out, offsets_out, s, cudaMemcpyDeviceToDevice);
        static const int order[] = {0, 1, 2, 3, 4, 5};
        tm.finish(order, 6);
    });
}

MP_API mp_status mp_layer_forward_host(mp_layer_t L, const void* x, uint32_t T, const uint32_t* kpt, uint32_t k,
                                       void* y, uint32_t* sel_out, float* w_out, uint32_t* offsets_out, void* stream) {
    return guarded([&] {
        if (!L || (T && (!x || !y))) fail(MP_ERR_VALIDATION, "null argument");
        check_tokens(L, T);
        check_ready(L);
        if (T == 0) return;
        if (kpt)
            for (uint32_t t = 0; t < T; ++t)
                if (kpt[t] < 1 || kpt[t] > L->k_max || kpt[t] > L->G)
                    fail(MP_ERR_VALIDATION, "k_active = " + std::to_string(kpt[t]) + " out of range [1, " +
                                                std::to_string(std::min(L->k_max, L->G)) + "]");
        DeviceGuard dg(L->desc.device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const size_t xbytes = (size_t)T * L->d * L->esz;
        ck(cudaMemsetAsync(L->ws.err, 0, sizeof(int), s), "memset err");
        ck(cudaMemcpyAsync(L->x_stage, x, xbytes, cudaMemcpyHostToDevice, s), "x upload");
        const uint32_t* kd = nullptr;
        if (kpt) {
            ck(cudaMemcpyAsync(L->kpt_dev, kpt, (size_t)T * 4, cudaMemcpyHostToDevice, s), "k upload");
            kd = L->kpt_dev;
        }
        StageTimer tm(L, s);
        const bool bucketed = route(L, L->x_stage, T, kd, k, s, tm, true, true);
        run_experts(L, L->x_stage, T, L->sel, L->wsel, L->desc.weight_mode == MP_WEIGHT_UNIT, L->y_stage, s, tm, true,
                    true, kpt ? 0 : k, bucketed);
        ck(cudaMemcpyAsync(y, L->y_stage, xbytes, cudaMemcpyDeviceToHost, s), "y download");
        copy_outputs(L, T, sel_out, w_out, offsets_out, s, cudaMemcpyDeviceToHost);
        int flags = 0;
        ck(cudaMemcpyAsync(&flags, L->ws.err, sizeof(int), cudaMemcpyDeviceToHost, s), "flags");
        ck(cudaStreamSynchronize(s), "forward");
        static const int order[] = {0, 1, 2, 3, 4, 5};
        tm.finish(order, 6);
        raise_device_errors(flags);
    });
}

// Pipelined host-buffer forwards: batch i's host->device copy (H2D stream),
// compute (the caller's stream) and device->host copy (D2H stream) run
// concurrently with batches i-1 / i+1 through two staging slots, ordered by
// events: a slot's x is not overwritten before the compute that reads it is
// done, its y not before the previous download of that slot completed.
MP_API mp_status mp_layer_forward_host_batches(mp_layer_t L, uint32_t n, const void* const* xs,
                                               const uint32_t* n_tokens, uint32_t k, void* const* ys,
                                               void* stream) {
    return guarded([&] {
        if (!L || (n && (!xs || !ys || !n_tokens))) fail(MP_ERR_VALIDATION, "null argument");
        check_ready(L);
        if (k < 1 || k > L->k_max || k > L->G)
            fail(MP_ERR_VALIDATION, "k_active = " + std::to_string(k) + " out of range [1, " +
                                        std::to_string(std::min(L->k_max, L->G)) + "]");
        for (uint32_t i = 0; i < n; ++i) {
            check_tokens(L, n_tokens[i]);
            if (n_tokens[i] && (!xs[i] || !ys[i])) fail(MP_ERR_VALIDATION, "null batch buffer");
        }
        if (n == 0) return;
        DeviceGuard dg(L->desc.device);
        if (!L->h2d) {
            ck(cudaStreamCreateWithFlags(&L->h2d, cudaStreamNonBlocking), "h2d stream");
            ck(cudaStreamCreateWithFlags(&L->d2h, cudaStreamNonBlocking), "d2h stream");
            for (int i = 0; i < 2; ++i) {
                ck(cudaEventCreateWithFlags(&L->ev_xready[i], cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&L->ev_computed[i], cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&L->ev_ydone[i], cudaEventDisableTiming), "event");
            }
            const size_t bytes = (size_t)L->max_tokens * L->d * L->esz;
            L->px[0] = L->x_stage;
            L->py[0] = L->y_stage;
            L->px[1] = dalloc<char>(bytes, "x stage 2");
            L->py[1] = dalloc<char>(bytes, "y stage 2");
        }
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        ck(cudaMemsetAsync(L->ws.err, 0, sizeof(int), s), "memset err");
        // the slots may still be in use by an earlier call's copies
        ck(cudaStreamSynchronize(L->d2h), "d2h");
        StageTimer tm(L, s);
        for (uint32_t i = 0; i < n; ++i) {
            const uint32_t T = n_tokens[i], sl = i & 1u;
            if (T == 0) continue;
            const size_t bytes = (size_t)T * L->d * L->esz;
            if (i >= 2) ck(cudaStreamWaitEvent(L->h2d, L->ev_computed[sl], 0), "wait compute");
            ck(cudaMemcpyAsync(L->px[sl], xs[i], bytes, cudaMemcpyHostToDevice, L->h2d), "x upload");
            ck(cudaEventRecord(L->ev_xready[sl], L->h2d), "event");
            ck(cudaStreamWaitEvent(s, L->ev_xready[sl], 0), "wait x");
            if (i >= 2) ck(cudaStreamWaitEvent(s, L->ev_ydone[sl], 0), "wait y");
            const bool bucketed = route(L, L->px[sl], T, nullptr, k, s, tm, true, true);
            run_experts(L, L->px[sl], T, L->sel, L->wsel, L->desc.weight_mode == MP_WEIGHT_UNIT, L->py[sl], s, tm,
                        true, true, k, bucketed);
            ck(cudaEventRecord(L->ev_computed[sl], s), "event");
            ck(cudaStreamWaitEvent(L->d2h, L->ev_computed[sl], 0), "wait compute");
            ck(cudaMemcpyAsync(ys[i], L->py[sl], bytes, cudaMemcpyDeviceToHost, L->d2h), "y download");
            ck(cudaEventRecord(L->ev_ydone[sl], L->d2h), "event");
        }
        int flags = 0;
        ck(cudaMemcpyAsync(&flags, L->ws.err, sizeof(int), cudaMemcpyDeviceToHost, s), "flags");
        ck(cudaStreamSynchronize(s), "forward");
        ck(cudaStreamSynchronize(L->d2h), "download");
        static const int order[] = {0, 1, 2, 3, 4, 5};
        tm.finish(order, 6);
        raise_device_errors(flags);
    });
}

MP_API mp_status mp_layer_forward_selected(mp_layer_t L, const void* x, uint32_t T, const uint32_t* sel,
                                           const float* w, void* y, uint32_t* offsets_out, void* stream) {
    return guarded([&] {
        if (!L || (T && (!x || !y || !sel))) fail(MP_ERR_VALIDATION, "null argument");
        check_tokens(L, T);
        check_ready(L);
        if (T == 0) return;
        DeviceGuard dg(L->desc.device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        StageTimer tm(L, s);
        run_experts(L, x, T, sel, w, w == nullptr, y, s, tm);
        if (offsets_out)
            ck(cudaMemcpyAsync(offsets_out, L->ws.offsets, (size_t)(L->G + 1) * 4, cudaMemcpyDeviceToDevice, s),
               "offsets_out");
        static const int order[] = {1, 2, 3, 4, 5};
        tm.finish(order, 5);
    });
}

MP_API mp_status mp_layer_route(mp_layer_t L, const void* x, uint32_t T, const uint32_t* kpt, uint32_t k,
                                uint32_t* sel_out, float* w_out, void* stream) {
    return guarded([&] {
        if (!L || (T && (!x || !sel_out || !w_out))) fail(MP_ERR_VALIDATION, "null argument");
        check_tokens(L, T);
        if (T == 0) return;
        DeviceGuard dg(L->desc.device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        StageTimer tm(L, s);
        route(L, x, T, kpt, k, s, tm);
        copy_outputs(L, T, sel_out, w_out, nullptr, s, cudaMemcpyDeviceToDevice);
        static const int order[] = {0};
        tm.finish(order, 1);
    });
}

MP_API mp_status mp_layer_route_stats(mp_layer_t L, uint32_t* reselected, uint32_t* near_ties, void* stream) {
    return guarded([&] {
        if (!L) fail(MP_ERR_VALIDATION, "null argument");
        if (!L->has_router) fail(MP_ERR_VALIDATION, "experts-only layer has no router");
        DeviceGuard dg(L->desc.device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        uint32_t st[2] = {0, 0};
        ck(cudaMemcpyAsync(st, L->r_flagged, sizeof(st), cudaMemcpyDeviceToHost, s), "routing stats");
        ck(cudaStreamSynchronize(s), "sync");
        if (reselected) *reselected = st[0];
        if (near_ties) *near_ties = st[1];
    });
}

MP_API mp_status mp_layer_check_errors(mp_layer_t L, void* stream) {
    return guarded([&] {
        if (!L) fail(MP_ERR_VALIDATION, "null argument");
        DeviceGuard dg(L->desc.device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        int flags = 0;
        ck(cudaMemcpyAsync(&flags, L->ws.err, sizeof(int), cudaMemcpyDeviceToHost, s), "flags");
        ck(cudaStreamSynchronize(s), "sync");
        ck(cudaMemsetAsync(L->ws.err, 0, sizeof(int), s), "memset err");
        raise_device_errors(flags);
    });
}

MP_API mp_status mp_layer_set_profiling(mp_layer_t L, int on) {
    return guarded([&] {
        if (!L) fail(MP_ERR_VALIDATION, "null argument");
        L->profiling = on != 0;
    });
}

MP_API mp_status mp_layer_stage_times(mp_layer_t L, char* names, size_t names_len, double* ms, uint64_t* launches,
                                      uint32_t* n, uint32_t cap) {
    return guarded([&] {
        if (!L) fail(MP_ERR_VALIDATION, "null argument");
        resolve_timings(L);
        std::string all;
        for (int q = 0; q < kStages; ++q) {
            if (q) all += ",";
            all += kStageNames[q];
            if (ms && (uint32_t)q < cap) ms[q] = L->stage_ms[q];
            if (launches && (uint32_t)q < cap) launches[q] = L->stage_launches[q];
        }
        if (names && names_len) {
            std::strncpy(names, all.c_str(), names_len - 1);
            names[names_len - 1] = 0;
        }
        if (n) *n = kStages;
    });
}

MP_API mp_status mp_layer_reset_stage_times(mp_layer_t L) {
    return guarded([&] {
        if (!L) fail(MP_ERR_VALIDATION, "null argument");
        resolve_timings(L);
        for (int q = 0; q < kStages; ++q) L->stage_ms[q] = 0, L->stage_launches[q] = 0;
    });
}

MP_API uint64_t mp_layer_launch_count(mp_layer_t L) { return L ? L->launches : 0; }

MP_API mp_status mp_synth_fill(void* dst, uint32_t dtype, size_t n, uint64_t seed, uint64_t first, double scale,
                               void* stream) {
    return guarded([&] {
        if (!dst) fail(MP_ERR_VALIDATION, "null argument");
        if (dtype != MP_DTYPE_F32 && dtype != MP_DTYPE_BF16) fail(MP_ERR_VALIDATION, "unknown dtype");
        if (!is_device_ptr(dst)) fail(MP_ERR_VALIDATION, "mp_synth_fill needs a device pointer");
        mp::launch_synth_fill(dst, (int)dtype, n, seed, first, scale, static_cast<cudaStream_t>(stream));
        ck_launch("synth fill");
    });
}

// ---- host-only format readers (no GPU needed) ----

MP_API mp_status mp_format_read_mpex(const char* path, uint32_t* d_model, uint32_t* d_ff, float* w_gate, float* w_up,
                                     float* w_down) {
    return guarded([&] {
        if (!path || !d_model || !d_ff) fail(MP_ERR_VALIDATION, "null argument");
        mp::MpexData m = mp::read_mpex(path);
        *d_model = m.d_model;
        *d_ff = m.d_ff;
        const size_t n = (size_t)m.d_model * m.d_ff;
        if (w_gate) std::memcpy(w_gate, m.w_gate.data(), n * 4);
        if (w_up) std::memcpy(w_up, m.w_up.data(), n * 4);
        if (w_down) std::memcpy(w_down, m.w_down.data(), n * 4);
    });
}

MP_API mp_status mp_format_read_partition_doc(const char* path, size_t index, size_t* n_docs, uint64_t* expert_id,
                                              uint32_t* n_sub, size_t* n, uint32_t* assignment, uint32_t* r,
                                              size_t* n_gate_ids, uint32_t* gate_offsets, uint32_t* gate_ids) {
    return guarded([&] {
        if (!path || !n_docs) fail(MP_ERR_VALIDATION, "null argument");
        auto docs = mp::read_partition_map(path);
        *n_docs = docs.size();
        if (index >= docs.size()) fail(MP_ERR_VALIDATION, "document index out of range");
        const auto& d = docs[index];
        if (expert_id) *expert_id = d.expert_id;
        if (n_sub) *n_sub = d.n_subexperts;
        if (n) *n = d.assignment.size();
        if (assignment) std::memcpy(assignment, d.assignment.data(), d.assignment.size() * 4);
        if (r) *r = d.has_gates ? d.r : 0;
        size_t tot = 0;
        if (d.has_gates) {
            if (gate_offsets) gate_offsets[0] = 0;
            for (size_t s = 0; s < d.gates.size(); ++s) {
                if (gate_ids) std::memcpy(gate_ids + tot, d.gates[s].data(), d.gates[s].size() * 4);
                tot += d.gates[s].size();
                if (gate_offsets) gate_offsets[s + 1] = static_cast<uint32_t>(tot);
            }
        }
        if (n_gate_ids) *n_gate_ids = tot;
    });
}

MP_API mp_status mp_validate_partition(uint32_t n_sub, const uint32_t* a, size_t n) {
    return guarded([&] {
        if (!a && n) fail(MP_ERR_VALIDATION, "null argument");
        mp::validate_partition(n_sub, a, n);
    });
}

// ---- debugging aid (not part of the public header): internal buffers ----
MP_API mp_status mp_debug_buffers(mp_layer_t L, void** x_perm, void** h, void** o, void** W1, void** W2,
                                  uint32_t* dims /* w_pad, d_pad, rows_cap, use_tc */) {
    return guarded([&] {
        if (!L) fail(MP_ERR_VALIDATION, "null argument");
        if (x_perm) *x_perm = L->x_perm;
        if (h) *h = L->h;
        if (o) *o = L->o;
        if (W1) *W1 = L->W1;
        if (W2) *W2 = L->W2;
        if (dims) {
            dims[0] = L->w_pad;
            dims[1] = L->d_pad;
            dims[2] = L->rows_cap;
            dims[3] = L->use_tc ? 1u : 0u;
        }
    });
}

// debugging aid: fp64 K-split partials of the last tensor-core router call,
// [ks][T][npad]; logits = sum over ks (fixed order).
MP_API mp_status mp_debug_router_partials(mp_layer_t L, void** partial, uint32_t* ks, uint32_t* T, uint32_t* npad,
                                          uint32_t* n_flagged) {
    return guarded([&] {
        if (!L || !L->router_tc) fail(MP_ERR_VALIDATION, "no tensor-core router on this layer");
        ck(cudaMemcpy(n_flagged, L->r_flagged, sizeof(uint32_t), cudaMemcpyDeviceToHost), "flagged");
        *partial = L->r_partial;
        *ks = L->r_last_ks;
        *T = L->r_last_T;
        *npad = L->r_npad;
    });
}

MP_API mp_status mp_layer_forward_selected_host(mp_layer_t L, const void* x, uint32_t T, const uint32_t* sel,
                                                const float* w, void* y, void* stream) {
    return guarded([&] {
        if (!L || (T && (!x || !y || !sel))) fail(MP_ERR_VALIDATION, "null argument");
        check_tokens(L, T);
        check_ready(L);
        if (T == 0) return;
        // host validation with the reference's verdicts (inc/expert.hpp:111-118)
        std::vector<uint8_t> seen(L->G);
        for (uint32_t t = 0; t < T; ++t) {
            std::fill(seen.begin(), seen.end(), 0);
            for (uint32_t j = 0; j < L->k_max; ++j) {
                const uint32_t g = sel[(size_t)t * L->k_max + j];
                if (g == MP_SEL_NONE) continue;
                if (g >= L->G)
                    fail(MP_ERR_VALIDATION, "active sub-expert " + std::to_string(g % L->S) + " out of range for N=" +
                                                std::to_string(L->S));
                if (seen[g]) fail(MP_ERR_VALIDATION, "active sub-expert list has duplicates");
                seen[g] = 1;
            }
        }
        DeviceGuard dg(L->desc.device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const size_t xbytes = (size_t)T * L->d * L->esz;
        const size_t sbytes = (size_t)T * L->k_max * 4;
        ck(cudaMemsetAsync(L->ws.err, 0, sizeof(int), s), "memset err");
        ck(cudaMemcpyAsync(L->x_stage, x, xbytes, cudaMemcpyHostToDevice, s), "x upload");
        ck(cudaMemcpyAsync(L->sel, sel, sbytes, cudaMemcpyHostToDevice, s), "sel upload");
        if (w) ck(cudaMemcpyAsync(L->wsel, w, sbytes, cudaMemcpyHostToDevice, s), "w upload");
        StageTimer tm(L, s);
        run_experts(L, L->x_stage, T, L->sel, w ? L->wsel : nullptr, w == nullptr, L->y_stage, s, tm, true);
        ck(cudaMemcpyAsync(y, L->y_stage, xbytes, cudaMemcpyDeviceToHost, s), "y download");
        int flags = 0;
        ck(cudaMemcpyAsync(&flags, L->ws.err, sizeof(int), cudaMemcpyDeviceToHost, s), "flags");
        ck(cudaStreamSynchronize(s), "forward");
        tm.finish(nullptr, 0);
        raise_device_errors(flags);
    });
}

// error channel shared with the other C-ABI translation units (ep.cu)
extern "C" void mp_internal_set_error(const char* msg) { g_err = msg ? msg : ""; }

// debugging aid: MMA-issuer timing of the last gemm1 (which=0) / gemm2 (1)
// launch when MOEPRISM_TC_TRACE=1: per CTA {total cycles, waiting for the
// accumulator (epilogue), waiting for smem stages (loads), tiles}.
MP_API mp_status mp_debug_gemm_trace(int which, uint64_t* out, uint32_t n_ctas) {
    return guarded([&] {
        uint64_t* p = mp::gemm_trace_ptr(which);
        if (!p) fail(MP_ERR_VALIDATION, "trace off (MOEPRISM_TC_TRACE=1)");
        ck(cudaMemcpy(out, p, (size_t)n_ctas * 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost), "trace");
    });
}

// Diagnostics (not in the public header): grouped-GEMM kernel choice of a
// layer at run time, 0 auto / 1 one-SM 128-row tiles / 2 CTA-pair 256-row
// tiles, for A/B timing (tests/probes/tile_ab.py).  The remainder schedules
// measured and dropped in round 1 (M=128 pair tails, the split schedule,
// merged and wide remainders) are described in gemm_tc2.cu and DESIGN.md.
MP_API mp_status mp_debug_set_tile_mode(mp_layer_t L, int mode) {
    return guarded([&] {
        if (!L || mode < 0 || mode > 3) fail(MP_ERR_VALIDATION, "bad argument");
        L->tile_mode = mode;
    });
}

// ============================================================== calibration
// the activation profile the offline refactoring engine
// partitions experts with, on the GPU.

MP_API mp_status mp_layer_collect_activations(mp_layer_t L, uint32_t e, const void* x, uint32_t B, float* act,
                                              void* stream) {
    return guarded([&] {
        if (!L || (B && (!x || !act))) fail(MP_ERR_VALIDATION, "null argument");
        if (e >= L->E) fail(MP_ERR_VALIDATION, "expert " + std::to_string(e) + " out of range");
        if (!L->has_experts) fail(MP_ERR_VALIDATION, "router-only layer holds no expert weights");
        if (!L->packed[e]) fail(MP_ERR_VALIDATION, "expert " + std::to_string(e) + " is not ready");
        if (!L->use_tc) fail(MP_ERR_VALIDATION, "the activation profiler runs on the bf16 tensor-core layout");
        if (L->offload) fail(MP_ERR_VALIDATION, "the activation profiler needs device-resident weights (offload on)");
        if (L->d % 8) fail(MP_ERR_VALIDATION, "the activation profiler needs d_model % 8 == 0");
        // inc/expert.hpp:141: an empty calibration list is a ValidationError
        if (B == 0) fail(MP_ERR_VALIDATION, "calibration input list is empty");
        if (reinterpret_cast<uintptr_t>(x) % 16) fail(MP_ERR_VALIDATION, "x must be 16-byte aligned");
        DeviceGuard dg(L->desc.device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (!L->cal_meta) L->cal_meta = dalloc<uint32_t>(4, "calibration meta");
        CUtensorMap tmX;
        if (!mp::make_tmap_bf16_2d(&tmX, x, B, L->d, 128, 64)) fail(MP_ERR_CUDA, "calibration tensor map");
        mp::launch_set_group_meta(L->cal_meta, B, s);
        // one group: all S sub-experts of expert e (S * 2 * w_pad rows of W1), A = x
        const uint32_t n_rows = L->S * 2 * L->w_pad;
        mp::GemmShape sh{1, L->d_pad, n_rows, B, L->ff, n_rows};
        mp::launch_gemm_tc_epi(mp::kEpiActAbs, &tmX, &L->tm_w1, act, sh, L->cal_meta, L->cal_meta + 2, L->num_sms, s,
                               e * n_rows, L->nmap_all + (size_t)e * L->S * L->w_pad);
        ck_launch("collect activations");
        L->launches += 2;
    });
}

MP_API mp_status mp_binarize_topk(const float* act, uint32_t rows, uint32_t cols, uint32_t k_a, uint8_t* bits,
                                  void* stream) {
    return guarded([&] {
        if (!act || !bits) fail(MP_ERR_VALIDATION, "null argument");
        if (rows < 1 || cols < 1)
            fail(MP_ERR_VALIDATION, "activation matrix must have at least one row and one column");
        if (k_a < 1 || k_a > cols)
            fail(MP_ERR_VALIDATION, "k_a = " + std::to_string(k_a) + " out of range [1, " + std::to_string(cols) + "]");
        mp::launch_binarize_topk(act, rows, cols, k_a, bits, static_cast<cudaStream_t>(stream));
        ck_launch("binarize_topk");
    });
}

MP_API mp_status mp_coactivation(const uint8_t* bits, uint32_t rows, uint32_t cols, uint32_t* co, void* stream) {
    return guarded([&] {
        if (!bits || !co) fail(MP_ERR_VALIDATION, "null argument");
        if (rows < 1 || cols < 1) fail(MP_ERR_VALIDATION, "binary activation shape is inconsistent");
        if (rows > (1u << 24)) fail(MP_ERR_VALIDATION, "co-activation counts are exact for at most 2^24 rows");
        int dev = 0, sms = 0;
        ck(cudaGetDevice(&dev), "device");
        ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const uint32_t ld = round_up(rows, 64);
        void* bt = nullptr;
        uint32_t* meta = nullptr;
        ck(cudaMallocAsync(&bt, (size_t)cols * ld * 2, s), "co-activation scratch");
        cudaError_t e2 = cudaMallocAsync(reinterpret_cast<void**>(&meta), 4 * sizeof(uint32_t), s);
        if (e2 != cudaSuccess) {
            cudaFreeAsync(bt, s);
            ck(e2, "co-activation meta");
        }
        mp::launch_bits_to_bf16_t(bits, rows, cols, ld, bt, s);
        mp::launch_set_group_meta(meta, cols, s);
        CUtensorMap tA, tB;
        const bool ok = mp::make_tmap_bf16_2d(&tA, bt, cols, ld, 128, 64) && mp::make_tmap_bf16_2d(&tB, bt, cols, ld, 256, 64);
        if (ok) {
            // C[i][j] = sum_r B[r][i] B[r][j]: A = B^T (cols x rows), B operand = B^T
            mp::GemmShape sh{1, ld, cols, cols, cols, cols};
            mp::launch_gemm_tc_epi(mp::kEpiCount, &tA, &tB, co, sh, meta, meta + 2, sms, s);
        }
        cudaError_t le = cudaGetLastError();
        cudaFreeAsync(bt, s);
        cudaFreeAsync(meta, s);
        if (!ok) fail(MP_ERR_CUDA, "co-activation tensor maps");
        ck(le, "coactivation");
    });
}

MP_API mp_status mp_format_write_mpam(const char* path, uint32_t rows, uint32_t cols, const float* data) {
    return guarded([&] {
        if (!path || !data) fail(MP_ERR_VALIDATION, "null argument");
        mp::write_mpam(path, rows, cols, data);
    });
}

MP_API mp_status mp_format_read_mpam(const char* path, uint32_t* rows, uint32_t* cols, float* data) {
    return guarded([&] {
        if (!path || !rows || !cols) fail(MP_ERR_VALIDATION, "null argument");
        uint32_t r = 0, c = 0;
        std::vector<float> d = mp::read_mpam(path, r, c);
        *rows = r;
        *cols = c;
        if (data) std::memcpy(data, d.data(), d.size() * 4);
    });
}

// ============================================================== offload
MP_API mp_status mp_layer_enable_offload(mp_layer_t L, uint32_t unit_subexperts, uint32_t cache_units) {
    return guarded([&] {
        if (!L) fail(MP_ERR_VALIDATION, "null argument");
        if (L->offload) fail(MP_ERR_VALIDATION, "offload already enabled");
        if (!L->use_tc || !L->has_experts || !L->has_router)
            fail(MP_ERR_VALIDATION, "offload needs a full bf16 tensor-core layer");
        if (unit_subexperts != 1 && unit_subexperts != L->S)
            fail(MP_ERR_VALIDATION, "unit must be 1 sub-expert (fine) or S (monolithic expert)");
        const uint32_t n_units = L->G / unit_subexperts;
        if (cache_units < 1 || cache_units > n_units)
            fail(MP_ERR_VALIDATION, "cache capacity must be in [1, " + std::to_string(n_units) + "] units");
        check_ready(L);
        DeviceGuard dg(L->desc.device);
        ck(cudaDeviceSynchronize(), "sync");
        const size_t w1 = (size_t)L->G * 2 * L->w_pad * L->d_pad * L->esz;
        const size_t w2 = (size_t)L->G * L->d_pad * L->w_pad * L->esz;
        const uint32_t cg = cache_units * unit_subexperts;  // cache groups
        const size_t c1 = (size_t)cg * 2 * L->w_pad * L->d_pad * L->esz;
        const uint32_t c2_rows = round_up(cg * L->d_pad, 256);
        const size_t c2 = (size_t)c2_rows * L->w_pad * L->esz;
        ck(cudaMallocHost(&L->W1h, w1), "pinned W1");
        ck(cudaMallocHost(&L->W2h, w2), "pinned W2");
        ck(cudaMemcpy(L->W1h, L->W1, w1, cudaMemcpyDeviceToHost), "W1 to host");
        ck(cudaMemcpy(L->W2h, L->W2, w2, cudaMemcpyDeviceToHost), "W2 to host");
        cudaFree(L->W1);
        cudaFree(L->W2);
        L->W1 = L->W2 = nullptr;  // the device now holds only the cache
        L->W1c = dalloc<char>(c1, "W1 cache");
        L->W2c = dalloc<char>(c2, "W2 cache");
        ck(cudaMemset(L->W2c, 0, c2), "memset W2 cache");
        L->gmap_dev = dalloc<uint32_t>(L->G, "gmap");
        ck(cudaMallocHost(reinterpret_cast<void**>(&L->gmap_host), L->G * 4), "pinned gmap");
        ck(cudaMallocHost(reinterpret_cast<void**>(&L->off_host), (L->G + 1) * 4), "pinned offsets");
        const bool ok = mp::make_tmap_bf16_2d(&L->tm_w1c, L->W1c, (uint64_t)cg * 2 * L->w_pad, L->d_pad, 256, 64) &&
                        mp::make_tmap_bf16_2d(&L->tm_w1ch, L->W1c, (uint64_t)cg * 2 * L->w_pad, L->d_pad, 128, 64) &&
                        mp::make_tmap_bf16_2d(&L->tm_w2c, L->W2c, c2_rows, L->w_pad, 256, 64) &&
                        mp::make_tmap_bf16_2d(&L->tm_w2ch, L->W2c, c2_rows, L->w_pad, 128, 64);
        if (!ok) fail(MP_ERR_CUDA, "offload cache tensor maps");
        L->off_unit = unit_subexperts;
        L->off_slots = cache_units;
        L->slot_of_unit.assign(n_units, -1);
        L->free_slots.clear();
        for (uint32_t sl = cache_units; sl-- > 0;) L->free_slots.push_back(sl);  // slot 0 first
        L->lru.clear();
        L->off_hits = L->off_misses = L->off_bytes = 0;
        L->offload = true;
    });
}

MP_API mp_status mp_layer_offload_stats(mp_layer_t L, uint64_t* hits, uint64_t* misses, uint64_t* bytes_h2d,
                                        uint32_t* last_units, uint32_t cap, uint32_t* n_last, uint32_t* last_misses) {
    return guarded([&] {
        if (!L) fail(MP_ERR_VALIDATION, "null argument");
        if (!L->offload) fail(MP_ERR_VALIDATION, "offload is not enabled");
        if (hits) *hits = L->off_hits;
        if (misses) *misses = L->off_misses;
        if (bytes_h2d) *bytes_h2d = L->off_bytes;
        if (n_last) *n_last = static_cast<uint32_t>(L->off_last_req.size());
        if (last_misses) *last_misses = L->off_last_misses;
        if (last_units)
            for (size_t i = 0; i < L->off_last_req.size() && i < cap; ++i) last_units[i] = L->off_last_req[i];
    });
}

// ---- proxy-gate construction and its fidelity (inc/gating.hpp:47-174) ----
namespace {
// ascending member lists of a partition as CSR (subexpert_members, inc/partition.hpp:49-55)
void members_csr(uint32_t n_sub, const uint32_t* a, uint32_t n, std::vector<uint32_t>& off,
                 std::vector<uint32_t>& mem) {
    off.assign(n_sub + 1, 0);
    for (uint32_t c = 0; c < n; ++c) ++off[a[c] + 1];
    for (uint32_t s = 0; s < n_sub; ++s) off[s + 1] += off[s];
    mem.assign(n, 0);
    std::vector<uint32_t> fill(off.begin(), off.end() - 1);
    for (uint32_t c = 0; c < n; ++c) mem[fill[a[c]]++] = c;
}
template <class T>
T* upload_async(const std::vector<T>& v, cudaStream_t s, std::vector<void*>& owned) {
    void* p = nullptr;
    ck(cudaMallocAsync(&p, std::max<size_t>(v.size(), 1) * sizeof(T), s), "calibration scratch");
    owned.push_back(p);
    if (!v.empty()) ck(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s), "upload");
    return static_cast<T*>(p);
}
void* scratch_async(size_t bytes, cudaStream_t s, std::vector<void*>& owned) {
    void* p = nullptr;
    ck(cudaMallocAsync(&p, std::max<size_t>(bytes, 1), s), "calibration scratch");
    owned.push_back(p);
    return p;
}
struct ScratchGuard {
    std::vector<void*> owned;
    cudaStream_t s;
    ~ScratchGuard() {
        for (void* p : owned) cudaFreeAsync(p, s);
    }
};
}  // namespace

// select_gate_neurons (inc/gating.hpp:72-103) over a device co-activation
// matrix [dim][dim] u32: per sub-expert the r most central members (centrality
// = co-activation with the other members, diagonal excluded; ties to the lower
// neuron), ascending.  Outputs on the host: gate_offsets[n_sub + 1] and
// gate_ids[gate_offsets[n_sub]] (capacity sum_s min(r, |group s|) <= dim).
MP_API mp_status mp_select_gate_neurons(const uint32_t* co, uint32_t dim, uint32_t n_sub, const uint32_t* assignment,
                                        uint32_t r, uint32_t* gate_offsets, uint32_t* gate_ids, void* stream) {
    return guarded([&] {
        if (!co || !assignment || !gate_offsets || !gate_ids) fail(MP_ERR_VALIDATION, "null argument");
        mp::validate_partition(n_sub, assignment, dim);
        if (r < 1) fail(MP_ERR_VALIDATION, "gate neuron count r must be >= 1");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        std::vector<uint32_t> off, mem, label(assignment, assignment + dim), out_off(n_sub + 1, 0);
        members_csr(n_sub, assignment, dim, off, mem);
        for (uint32_t q = 0; q < n_sub; ++q) out_off[q + 1] = out_off[q] + std::min(r, off[q + 1] - off[q]);
        ScratchGuard sg{{}, s};
        uint32_t* d_label = upload_async(label, s, sg.owned);
        uint32_t* d_off = upload_async(off, s, sg.owned);
        uint32_t* d_mem = upload_async(mem, s, sg.owned);
        uint32_t* d_oo = upload_async(out_off, s, sg.owned);
        auto* d_score = static_cast<unsigned long long*>(scratch_async((size_t)dim * 8, s, sg.owned));
        auto* d_out = static_cast<uint32_t*>(scratch_async((size_t)out_off[n_sub] * 4, s, sg.owned));
        mp::launch_centrality(co, dim, d_label, d_off, d_mem, d_score, s);
        mp::launch_gate_select(d_score, d_off, d_mem, n_sub, r, d_oo, d_out, s);
        ck_launch("select_gate_neurons");
        ck(cudaMemcpyAsync(gate_ids, d_out, (size_t)out_off[n_sub] * 4, cudaMemcpyDeviceToHost, s), "gate ids");
        ck(cudaStreamSynchronize(s), "select_gate_neurons");
        std::copy(out_off.begin(), out_off.end(), gate_offsets);
    });
}

// gating_fidelity (inc/gating.hpp:149-174): mean over rows of the top-k recall
// of the proxy selection (mean |a| over each sub-expert's gate neurons)
// against the selection on the true sub-expert norms (subexpert_norms,
// inc/partition.hpp:78-95).  act: device [rows][cols] fp32; the partition and
// the gate set (CSR, ascending ids) on the host.  Same double sums in the
// same order as the reference; the row recalls are summed in row order.
MP_API mp_status mp_gating_fidelity(const float* act, uint32_t rows, uint32_t cols, uint32_t n_sub,
                                    const uint32_t* assignment, const uint32_t* gate_offsets,
                                    const uint32_t* gate_ids, uint32_t k, double* out, void* stream) {
    return guarded([&] {
        if (!act || !assignment || !gate_offsets || !gate_ids || !out) fail(MP_ERR_VALIDATION, "null argument");
        if (rows < 1 || cols < 1)
            fail(MP_ERR_VALIDATION, "activation matrix must have at least one row and one column");
        mp::validate_partition(n_sub, assignment, cols);
        if (n_sub > 256) fail(MP_ERR_VALIDATION, "at most 256 sub-experts per expert");
        for (uint32_t q = 0; q < n_sub; ++q) {  // validate(GateSet), inc/gating.hpp:33-43
            if (gate_offsets[q + 1] <= gate_offsets[q])
                fail(MP_ERR_VALIDATION, "every sub-expert needs at least one gate neuron");
            for (uint32_t g = gate_offsets[q]; g < gate_offsets[q + 1]; ++g) {
                if (gate_ids[g] >= cols)
                    fail(MP_ERR_VALIDATION, "gate neuron " + std::to_string(gate_ids[g]) +
                                                " out of range for activation vector of length " +
                                                std::to_string(cols));
                if (g > gate_offsets[q] && gate_ids[g] < gate_ids[g - 1])
                    fail(MP_ERR_VALIDATION, "gate neuron lists must be ascending");
            }
        }
        if (k < 1 || k > n_sub)
            fail(MP_ERR_VALIDATION,
                 "k_active = " + std::to_string(k) + " out of range [1, " + std::to_string(n_sub) + "]");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        std::vector<uint32_t> off, mem;
        members_csr(n_sub, assignment, cols, off, mem);
        std::vector<uint32_t> goff(gate_offsets, gate_offsets + n_sub + 1), gids(gate_ids, gate_ids + goff[n_sub]);
        ScratchGuard sg{{}, s};
        uint32_t* d_off = upload_async(off, s, sg.owned);
        uint32_t* d_mem = upload_async(mem, s, sg.owned);
        uint32_t* d_goff = upload_async(goff, s, sg.owned);
        uint32_t* d_gids = upload_async(gids, s, sg.owned);
        auto* d_norm = static_cast<double*>(scratch_async((size_t)rows * n_sub * 8, s, sg.owned));
        auto* d_proxy = static_cast<double*>(scratch_async((size_t)rows * n_sub * 8, s, sg.owned));
        auto* d_recall = static_cast<double*>(scratch_async((size_t)rows * 8, s, sg.owned));
        mp::launch_fidelity(act, rows, cols, n_sub, d_off, d_mem, d_goff, d_gids, k, d_norm, d_proxy, d_recall, s);
        ck_launch("gating_fidelity");
        std::vector<double> recall(rows);
        ck(cudaMemcpyAsync(recall.data(), d_recall, (size_t)rows * 8, cudaMemcpyDeviceToHost, s), "recall");
        ck(cudaStreamSynchronize(s), "gating_fidelity");
        double total = 0.0;
        for (double v : recall) total += v;
        *out = total / static_cast<double>(rows);
    });
}
