// moe_layer.hpp -- C++ host API of the B200-native MoE-Prism sub-expert layer,
// in the reference's style (value types, std::span inputs, ValidationError /
// IoError exceptions; inc/error.hpp:8-16), over the C-ABI in moe_layer.h.
//
//   moeprism::b200::MoeLayer      the layer: weights / partitions / router or
//                                 gates loaded from the offline engine's
//                                 artefacts, forward(tokens, k) -> hidden.
//   moeprism::b200::moe_forward   free-function form of MoeLayer::forward.
//   moeprism::b200::partitioned_forward
//                                 drop-in for inc/expert.hpp:101-135 with the
//                                 reference's exact signature and validation
//                                 verdicts, computed on the GPU.
//
// Coexistence with the reference headers (proj/include/moeprism/*.hpp):
//   * when they are on the include path (detected by <moeprism/partition.hpp>,
//     or forced with -DMOEPRISM_WITH_REFERENCE_HEADERS), this header includes
//     them and uses their ToyExpert / Partition / GateSet / validate /
//     ValidationError / IoError -- one set of value types, no redefinitions;
//   * otherwise it defines the same types itself, field for field, and
//     exports the b200 API into namespace moeprism (moeprism::MoeLayer,
//     moeprism::partitioned_forward, ...);
//   * include/moeprism/dropin/moeprism/expert.hpp shadows the reference's
//     expert.hpp so that code written against the reference (its own test
//     suites: tests/cpp/ref_expert_suite.cpp) calls the GPU partitioned_forward
//     unchanged.
// Header-only; link libmoeprism_b200.so.  No CPU fallback: compute calls
// throw std::runtime_error (status 3) when no sm_100a device is usable.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <numeric>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "moeprism/moe_layer.h"

#if !defined(MOEPRISM_WITH_REFERENCE_HEADERS) && defined(__has_include)
#if __has_include(<moeprism/partition.hpp>)
#define MOEPRISM_WITH_REFERENCE_HEADERS 1
#endif
#endif

#ifdef MOEPRISM_WITH_REFERENCE_HEADERS
#include <moeprism/error.hpp>
#include <moeprism/expert.hpp>
#include <moeprism/gating.hpp>
#include <moeprism/partition.hpp>
#else
namespace moeprism {

// Same taxonomy as the reference (inc/error.hpp:9-16).
struct ValidationError : std::runtime_error {
    explicit ValidationError(const std::string& what) : std::runtime_error(what) {}
};
struct IoError : std::runtime_error {
    explicit IoError(const std::string& what) : std::runtime_error(what) {}
};

// The reference's value types (inc/expert.hpp:17-23, inc/partition.hpp:15-20,
// inc/gating.hpp:19-23), field for field.
struct ToyExpert {
    std::size_t d_model = 0;
    std::size_t d_ff = 0;
    std::vector<float> w_gate;  // d_model x d_ff, row-major
    std::vector<float> w_up;    // d_model x d_ff, row-major
    std::vector<float> w_down;  // d_ff x d_model, row-major
};

struct Partition {
    std::uint32_t n_subexperts = 0;
    std::vector<std::uint32_t> assignment;  // neuron index -> sub-expert label
    std::size_t n_neurons() const { return assignment.size(); }
};

struct GateSet {
    std::uint32_t n_subexperts = 0;
    std::uint32_t r = 0;
    std::vector<std::vector<std::uint32_t>> gate_neurons;
};

// validate(ToyExpert), inc/expert.hpp:25-39 -- same verdicts and messages.
inline void validate(const ToyExpert& e) {
    if (e.d_model < 1 || e.d_ff < 1) throw ValidationError("toy expert needs d_model >= 1 and d_ff >= 1");
    if (e.w_gate.size() != e.d_model * e.d_ff || e.w_up.size() != e.d_model * e.d_ff ||
        e.w_down.size() != e.d_ff * e.d_model)
        throw ValidationError("toy expert weight shapes do not match d_model=" + std::to_string(e.d_model) +
                              ", d_ff=" + std::to_string(e.d_ff));
    for (const auto* w : {&e.w_gate, &e.w_up, &e.w_down})
        for (float v : *w)
            if (!std::isfinite(v)) throw ValidationError("toy expert weight is not finite");
}

// validate(Partition), inc/partition.hpp:34-46 (the library's own checker).
inline void validate(const Partition& p) {
    const mp_status rc = mp_validate_partition(p.n_subexperts, p.assignment.data(), p.assignment.size());
    if (rc == MP_ERR_VALIDATION) throw ValidationError(mp_last_error());
    if (rc != MP_OK) throw std::runtime_error(mp_last_error());
}

}  // namespace moeprism
#endif

namespace moeprism::b200 {

using ::moeprism::GateSet;
using ::moeprism::IoError;
using ::moeprism::Partition;
using ::moeprism::ToyExpert;
using ::moeprism::ValidationError;

enum class Dtype : std::uint32_t { f32 = MP_DTYPE_F32, bf16 = MP_DTYPE_BF16 };
enum class RouterMode : std::uint32_t { linear = MP_ROUTER_LINEAR, proxy = MP_ROUTER_PROXY };
enum class WeightMode : std::uint32_t { unit = MP_WEIGHT_UNIT, softmax_renorm = MP_WEIGHT_SOFTMAX_RENORM };

struct LayerConfig {
    std::uint32_t n_experts = 8;
    std::uint32_t n_subexperts = 8;
    std::uint32_t d_model = 4096;
    std::uint32_t d_ff = 14336;
    Dtype dtype = Dtype::bf16;
    RouterMode router = RouterMode::linear;
    WeightMode weights = WeightMode::softmax_renorm;
    std::uint32_t k_max = 16;
    std::uint32_t max_tokens = 4096;
    int device = 0;
    std::uint32_t flags = 0;  // MP_LAYER_ROUTER_ONLY / MP_LAYER_EXPERTS_ONLY (expert parallelism)
};

namespace detail {

inline void check(mp_status rc) {
    if (rc == MP_OK) return;
    const std::string msg = mp_last_error();
    if (rc == MP_ERR_VALIDATION) throw ValidationError(msg);
    if (rc == MP_ERR_IO) throw IoError(msg);
    throw std::runtime_error(msg);
}

// round-to-nearest-even fp32 -> bf16 bits (finite inputs)
inline std::uint16_t to_bf16(float f) {
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<std::uint16_t>(u >> 16);
}
inline float from_bf16(std::uint16_t h) {
    const std::uint32_t u = static_cast<std::uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

}  // namespace detail

class MoeLayer {
public:
    explicit MoeLayer(const LayerConfig& c) : cfg_(c) {
        const mp_layer_desc d{c.n_experts, c.n_subexperts, c.d_model, c.d_ff, static_cast<std::uint32_t>(c.dtype),
                              static_cast<std::uint32_t>(c.router), static_cast<std::uint32_t>(c.weights), c.k_max,
                              c.max_tokens, c.device, c.flags};
        detail::check(mp_layer_create(&d, &h_));
    }
    ~MoeLayer() {
        if (h_) mp_layer_destroy(h_);
    }
    MoeLayer(const MoeLayer&) = delete;
    MoeLayer& operator=(const MoeLayer&) = delete;
    MoeLayer(MoeLayer&& o) noexcept : cfg_(o.cfg_), h_(std::exchange(o.h_, nullptr)) {}
    MoeLayer& operator=(MoeLayer&& o) noexcept {
        std::swap(h_, o.h_);
        cfg_ = o.cfg_;
        return *this;
    }

    const LayerConfig& config() const { return cfg_; }
    mp_layer_t handle() const { return h_; }

    void load_expert(std::uint32_t e, const ToyExpert& x) {
        validate(x);
        if (x.d_model != cfg_.d_model || x.d_ff != cfg_.d_ff)
            throw ValidationError("expert shape does not match the layer");
        detail::check(mp_layer_load_expert(h_, e, x.w_gate.data(), x.w_up.data(), x.w_down.data()));
    }
    void load_expert_file(std::uint32_t e, const std::filesystem::path& p) {
        detail::check(mp_layer_load_expert_file(h_, e, p.c_str()));
    }
    void set_partition(std::uint32_t e, const Partition& p) {
        detail::check(mp_layer_set_partition(h_, e, p.n_subexperts, p.assignment.data(), p.assignment.size()));
    }
    void load_partition_map(const std::filesystem::path& p) { detail::check(mp_layer_load_partition_map(h_, p.c_str())); }
    void set_router(std::span<const float> w_r) {
        if (w_r.size() != static_cast<std::size_t>(cfg_.d_model) * cfg_.n_experts * cfg_.n_subexperts)
            throw ValidationError("router weight must be d_model x (E*S)");
        detail::check(mp_layer_set_router(h_, w_r.data()));
    }
    void set_residual(bool on) { detail::check(mp_layer_set_residual(h_, on ? 1 : 0)); }
    // Qwen-style always-on shared expert; gate empty = weight 1 (moe_layer.h).
    void set_shared_expert(const ToyExpert& x, std::span<const float> gate = {}) {
        validate(x);
        if (x.d_model != cfg_.d_model) throw ValidationError("shared expert d_model does not match the layer");
        if (!gate.empty() && gate.size() != cfg_.d_model) throw ValidationError("shared gate must have d_model entries");
        detail::check(mp_layer_set_shared_expert(h_, x.d_ff, x.w_gate.data(), x.w_up.data(), x.w_down.data(),
                                                 gate.empty() ? nullptr : gate.data()));
    }
    void set_gates(std::uint32_t e, const GateSet& g) {
        std::vector<std::uint32_t> off(1, 0), ids;
        for (const auto& l : g.gate_neurons) {
            ids.insert(ids.end(), l.begin(), l.end());
            off.push_back(static_cast<std::uint32_t>(ids.size()));
        }
        if (g.gate_neurons.size() != g.n_subexperts || g.n_subexperts != cfg_.n_subexperts)
            throw ValidationError("gate set shape is inconsistent");
        detail::check(mp_layer_set_gates(h_, e, g.r, off.data(), ids.data()));
    }

    // Host API: x is T x d_model fp32 row-major; one k for every token.
    std::vector<float> forward(std::span<const float> x, std::uint32_t k) const { return run(x, nullptr, k); }
    // Per-token elastic k (the QoS knob, inc/scheduler.hpp:26 k_min per request).
    std::vector<float> forward(std::span<const float> x, std::span<const std::uint32_t> k_per_token) const {
        if (k_per_token.size() != x.size() / cfg_.d_model)
            throw ValidationError("k_per_token needs one entry per token");
        return run(x, k_per_token.data(), 0);
    }
    // Explicit active sets (T x k_max global ids, MP_SEL_NONE padded), unit
    // weights: the partitioned_forward semantics summed over experts.
    std::vector<float> forward_selected(std::span<const float> x, std::span<const std::uint32_t> sel) const {
        const std::uint32_t T = tokens(x);
        if (sel.size() != static_cast<std::size_t>(T) * cfg_.k_max)
            throw ValidationError("selection must be T x k_max");
        if (cfg_.dtype == Dtype::f32) {
            std::vector<float> y(x.size());
            detail::check(mp_layer_forward_selected_host(h_, x.data(), T, sel.data(), nullptr, y.data(), nullptr));
            return y;
        }
        std::vector<std::uint16_t> xb(x.size()), yb(x.size());
        for (std::size_t i = 0; i < x.size(); ++i) xb[i] = detail::to_bf16(x[i]);
        detail::check(mp_layer_forward_selected_host(h_, xb.data(), T, sel.data(), nullptr, yb.data(), nullptr));
        std::vector<float> y(x.size());
        for (std::size_t i = 0; i < y.size(); ++i) y[i] = detail::from_bf16(yb[i]);
        return y;
    }
    // Device API: x, y device buffers of the layer dtype; stream = cudaStream_t.
    void forward_device(const void* x, std::uint32_t T, std::uint32_t k, void* y, void* stream = nullptr,
                        const std::uint32_t* k_per_token_dev = nullptr) const {
        detail::check(mp_layer_forward(h_, x, T, k_per_token_dev, k, y, nullptr, nullptr, nullptr, stream));
    }

private:
    std::uint32_t tokens(std::span<const float> x) const {
        if (x.size() % cfg_.d_model != 0)
            throw ValidationError("input length " + std::to_string(x.size()) + " is not a multiple of d_model " +
                                  std::to_string(cfg_.d_model));
        return static_cast<std::uint32_t>(x.size() / cfg_.d_model);
    }
    std::vector<float> run(std::span<const float> x, const std::uint32_t* kpt, std::uint32_t k) const {
        const std::uint32_t T = tokens(x);
        for (float v : x)
            if (!std::isfinite(v)) throw ValidationError("input vector is not finite");
        if (cfg_.dtype == Dtype::f32) {
            std::vector<float> y(x.size());
            detail::check(
                mp_layer_forward_host(h_, x.data(), T, kpt, k, y.data(), nullptr, nullptr, nullptr, nullptr));
            return y;
        }
        std::vector<std::uint16_t> xb(x.size()), yb(x.size());
        for (std::size_t i = 0; i < x.size(); ++i) xb[i] = detail::to_bf16(x[i]);
        detail::check(mp_layer_forward_host(h_, xb.data(), T, kpt, k, yb.data(), nullptr, nullptr, nullptr, nullptr));
        std::vector<float> y(x.size());
        for (std::size_t i = 0; i < y.size(); ++i) y[i] = detail::from_bf16(yb[i]);
        return y;
    }

    LayerConfig cfg_;
    mp_layer_t h_ = nullptr;
};

// One rank of an expert-parallel layer on the C++ host: the
// replicated router, this rank's contiguous range of sub-experts, and the
// NCCL transport (moe_layer.h mp_ep_forward).  Rank r of `world` owns global
// sub-experts [r * G / world, (r + 1) * G / world) -- whole experts when
// world divides E, else sub-expert granularity.  Typical use:
//   ExpertParallelLayer ep(cfg, world, rank);
//   std::array<std::uint8_t, MP_EP_NCCL_ID_BYTES> id{};
//   if (rank == 0) id = ExpertParallelLayer::unique_id();
//   broadcast(id);                  // MPI_Bcast / a TCP store / ...
//   ep.connect(id);                 // collective
//   for e owned: ep.load_expert(e, ...); ep.set_partition(e, ...);
//   ep.set_router(w_r);
//   ep.forward_device(x, T, k, y, stream);
class ExpertParallelLayer {
public:
    ExpertParallelLayer(const LayerConfig& c, std::uint32_t world, std::uint32_t rank)
        : cfg_(c), world_(world), rank_(rank), per_rank_(shard(c, world, rank)),
          first_e_(per_rank_ * rank / c.n_subexperts), last_e_((per_rank_ * (rank + 1) - 1) / c.n_subexperts),
          router_(role(c, MP_LAYER_ROUTER_ONLY, 0, 0)), experts_(role(c, MP_LAYER_EXPERTS_ONLY, first_e_, last_e_)) {
        detail::check(mp_ep_create_subexpert(world, rank, per_rank_, c.n_subexperts, c.d_model, c.k_max, c.max_tokens,
                                             static_cast<std::uint32_t>(c.dtype), c.device, &ep_));
    }
    ~ExpertParallelLayer() {
        if (ep_) mp_ep_destroy(ep_);
    }
    ExpertParallelLayer(const ExpertParallelLayer&) = delete;
    ExpertParallelLayer& operator=(const ExpertParallelLayer&) = delete;

    static std::vector<std::uint8_t> unique_id() {
        std::vector<std::uint8_t> id(MP_EP_NCCL_ID_BYTES);
        detail::check(mp_ep_nccl_unique_id(id.data()));
        return id;
    }
    void connect(std::span<const std::uint8_t> id) {
        if (id.size() != MP_EP_NCCL_ID_BYTES) throw ValidationError("NCCL unique id must be 128 bytes");
        detail::check(mp_ep_nccl_init(ep_, id.data()));
    }
    bool owns(std::uint32_t e) const { return e >= first_e_ && e <= last_e_; }
    void load_expert(std::uint32_t e, const ToyExpert& x) {
        if (owns(e)) experts_.load_expert(e - first_e_, x);
    }
    void set_partition(std::uint32_t e, const Partition& p) {
        if (owns(e)) experts_.set_partition(e - first_e_, p);
    }
    void set_router(std::span<const float> w_r) { router_.set_router(w_r); }
    // x, y: device [T x d_model] of the layer dtype; residual: y = x + MoE(x)
    void forward_device(const void* x, std::uint32_t T, std::uint32_t k, void* y, void* stream = nullptr,
                        const std::uint32_t* k_per_token_dev = nullptr, bool residual = false) {
        detail::check(mp_ep_forward(ep_, router_.handle(), experts_.handle(), x, T, k_per_token_dev, k, y,
                                    residual ? MP_EP_RESIDUAL : 0u, stream));
    }
    mp_ep_t handle() const { return ep_; }

private:
    static std::uint32_t shard(const LayerConfig& c, std::uint32_t world, std::uint32_t rank) {
        const std::uint32_t G = c.n_experts * c.n_subexperts;
        if (world < 1 || rank >= world || G % world)
            throw ValidationError("the E*S sub-experts must shard evenly over the ranks");
        return G / world;
    }
    LayerConfig role(const LayerConfig& c, std::uint32_t flags, std::uint32_t first, std::uint32_t last) const {
        LayerConfig r = c;
        r.flags = flags;
        if (flags == MP_LAYER_EXPERTS_ONLY) {
            r.n_experts = last - first + 1;
            r.weights = WeightMode::softmax_renorm;  // the owner applies the routing weights
            r.max_tokens = c.max_tokens * world_;    // rows from every rank
        }
        return r;
    }

    LayerConfig cfg_;
    std::uint32_t world_, rank_, per_rank_, first_e_, last_e_;
    MoeLayer router_, experts_;
    mp_ep_t ep_ = nullptr;
};

inline std::vector<float> moe_forward(const MoeLayer& layer, std::span<const float> x,
                                      std::span<const std::uint32_t> k_per_token) {
    return layer.forward(x, k_per_token);
}

// Drop-in for partitioned_forward (inc/expert.hpp:101-135): same signature,
// same ValidationError verdicts in the same order, unweighted sum over the
// active sub-experts, computed by the fp32 (fp64-accumulating) GPU path --
// within 1e-5 * (1 + |y|) of the reference.  One single-expert layer per call
// (weights uploaded and packed each time): a compatibility entry point, not
// the serving path.  Any reference-valid partition is accepted: up to
// MP_MAX_SUBEXPERTS sub-experts the layer holds the partition itself; beyond
// that the active neurons (ascending, the reference's summation order) are
// gathered into one sub-expert of a one-expert layer.
inline std::vector<float> partitioned_forward(const ToyExpert& e, const Partition& p, std::span<const float> x,
                                              std::span<const std::uint32_t> active) {
    validate(e);
    validate(p);
    if (x.size() != e.d_model)
        throw ValidationError("input length " + std::to_string(x.size()) + " does not match d_model " +
                              std::to_string(e.d_model));
    for (float v : x)
        if (!std::isfinite(v)) throw ValidationError("input vector is not finite");
    if (p.assignment.size() != e.d_ff)
        throw ValidationError("partition covers " + std::to_string(p.assignment.size()) +
                              " neurons but the expert has d_ff " + std::to_string(e.d_ff));
    std::vector<std::uint8_t> is_active(p.n_subexperts, 0);
    for (std::uint32_t n : active) {
        if (n >= p.n_subexperts)
            throw ValidationError("active sub-expert " + std::to_string(n) + " out of range for N=" +
                                  std::to_string(p.n_subexperts));
        if (is_active[n]) throw ValidationError("active sub-expert list has duplicates");
        is_active[n] = 1;
    }
    if (active.empty()) return std::vector<float>(e.d_model, 0.0f);
    LayerConfig c;
    c.n_experts = 1;
    c.d_model = static_cast<std::uint32_t>(e.d_model);
    c.dtype = Dtype::f32;
    c.weights = WeightMode::unit;
    c.max_tokens = 1;
    if (p.n_subexperts <= MP_MAX_SUBEXPERTS) {
        c.n_subexperts = p.n_subexperts;
        c.d_ff = static_cast<std::uint32_t>(e.d_ff);
        c.k_max = static_cast<std::uint32_t>(active.size());
        MoeLayer layer(c);
        layer.set_partition(0, p);
        layer.load_expert(0, e);
        std::vector<std::uint32_t> sel(active.begin(), active.end());
        std::sort(sel.begin(), sel.end());
        return layer.forward_selected(x, sel);
    }
    ToyExpert g;  // the active neurons in ascending order
    g.d_model = e.d_model;
    for (std::size_t j = 0; j < e.d_ff; ++j) g.d_ff += is_active[p.assignment[j]];
    g.w_gate.resize(g.d_model * g.d_ff);
    g.w_up.resize(g.d_model * g.d_ff);
    g.w_down.reserve(g.d_ff * g.d_model);
    for (std::size_t j = 0, q = 0; j < e.d_ff; ++j) {
        if (!is_active[p.assignment[j]]) continue;
        for (std::size_t i = 0; i < e.d_model; ++i) {
            g.w_gate[i * g.d_ff + q] = e.w_gate[i * e.d_ff + j];
            g.w_up[i * g.d_ff + q] = e.w_up[i * e.d_ff + j];
        }
        g.w_down.insert(g.w_down.end(), e.w_down.begin() + j * e.d_model, e.w_down.begin() + (j + 1) * e.d_model);
        ++q;
    }
    c.n_subexperts = 1;
    c.d_ff = static_cast<std::uint32_t>(g.d_ff);
    c.k_max = 1;
    MoeLayer layer(c);
    Partition one;
    one.n_subexperts = 1;
    one.assignment.assign(g.d_ff, 0u);
    layer.set_partition(0, one);
    layer.load_expert(0, g);
    const std::vector<std::uint32_t> sel{0u};
    return layer.forward_selected(x, sel);
}

}  // namespace moeprism::b200

#ifndef MOEPRISM_WITH_REFERENCE_HEADERS
// Without the reference headers the GPU API is the moeprism API.
namespace moeprism {
using b200::Dtype;
using b200::ExpertParallelLayer;
using b200::LayerConfig;
using b200::moe_forward;
using b200::MoeLayer;
using b200::partitioned_forward;
using b200::RouterMode;
using b200::WeightMode;
}  // namespace moeprism
#endif
