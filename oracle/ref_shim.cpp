// ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference headers.
// TEST INFRASTRUCTURE ONLY (see oracle/moe_oracle.c header for who may load it).
//
// Compiled by oracle/Makefile directly against the sources where they lie
// (-I/root/reference/proj/include -I/root/reference/proj/tests); nothing from
// the reference is copied into this repository.  The output goes to
// oracle/_ref/libmoeprism_ref.so (git-ignored; it travels to the GPU box with
// the gpurun snapshot).  It exposes the reference's own functions verbatim so
// that (1) the C restatement in moe_oracle.c can be pinned bit for bit, and
// (2) bench.py --impl reference can time the reference CPU path.
//
// The only code here that is not a direct call is the multi-expert layer
// composition (the reference has no layer): per token, the
// router logits are formed with the accumulation rule of
// inc/expert.hpp:64-71, select_topk_subexperts picks the sub-experts, and the
// output is a sum of verbatim partitioned_forward calls.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "moeprism/activation.hpp"
#include "moeprism/error.hpp"
#include "moeprism/expert.hpp"
#include "moeprism/gating.hpp"
#include "moeprism/io.hpp"
#include "moeprism/offload.hpp"
#include "moeprism/partition.hpp"
#include "moeprism/perfmodel.hpp"
#include "moeprism/rng.hpp"
#include "moeprism/serde.hpp"
#include "support.hpp"

using namespace moeprism;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 1;
    } catch (const IoError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

ToyExpert make_expert(std::size_t d, std::size_t ff, const float* wg, const float* wu, const float* wd) {
    ToyExpert e;
    e.d_model = d;
    e.d_ff = ff;
    e.w_gate.assign(wg, wg + d * ff);
    e.w_up.assign(wu, wu + d * ff);
    e.w_down.assign(wd, wd + d * ff);
    return e;
}

Partition make_partition(std::uint32_t n_sub, std::size_t n, const std::uint32_t* a) {
    Partition p;
    p.n_subexperts = n_sub;
    p.assignment.assign(a, a + n);
    return p;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_mt64_draw(std::uint64_t seed, std::size_t n, std::uint64_t* out) {
    std::mt19937_64 rng(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = rng();
}

void ref_uniform01(std::uint64_t seed, std::size_t n, double* out) {
    std::mt19937_64 rng(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = uniform01(rng);
}

int ref_random_expert(std::size_t d, std::size_t ff, std::uint64_t seed, float* wg, float* wu, float* wd) {
    return guarded([&] {
        const ToyExpert e = testsupport::random_expert(d, ff, seed);
        std::memcpy(wg, e.w_gate.data(), d * ff * sizeof(float));
        std::memcpy(wu, e.w_up.data(), d * ff * sizeof(float));
        std::memcpy(wd, e.w_down.data(), d * ff * sizeof(float));
    });
}

int ref_random_balanced_partition(std::size_t n, std::uint32_t n_sub, std::uint64_t seed, std::uint32_t* out) {
    return guarded([&] {
        const Partition p = testsupport::random_balanced_partition(n, n_sub, seed);
        std::memcpy(out, p.assignment.data(), n * sizeof(std::uint32_t));
    });
}

int ref_contiguous_partition(std::size_t n, std::uint32_t n_sub, std::uint32_t* out) {
    return guarded([&] {
        const Partition p = contiguous_partition(n, n_sub);
        std::memcpy(out, p.assignment.data(), n * sizeof(std::uint32_t));
    });
}

int ref_validate_partition(std::uint32_t n_sub, std::size_t n, const std::uint32_t* a) {
    return guarded([&] { validate(make_partition(n_sub, n, a)); });
}

int ref_toy_ffn_forward(std::size_t d, std::size_t ff, const float* wg, const float* wu, const float* wd,
                        const float* x, std::size_t nx, float* y, float* a) {
    return guarded([&] {
        const ToyExpert e = make_expert(d, ff, wg, wu, wd);
        const ForwardResult r = toy_ffn_forward(e, std::span<const float>(x, nx));
        std::memcpy(y, r.y.data(), d * sizeof(float));
        std::memcpy(a, r.a.data(), ff * sizeof(float));
    });
}

int ref_partitioned_forward(std::size_t d, std::size_t ff, const float* wg, const float* wu, const float* wd,
                            std::uint32_t n_sub, std::size_t n_assign, const std::uint32_t* assignment,
                            const float* x, std::size_t nx, const std::uint32_t* active, std::size_t n_active,
                            float* y) {
    return guarded([&] {
        const ToyExpert e = make_expert(d, ff, wg, wu, wd);
        const Partition p = make_partition(n_sub, n_assign, assignment);
        const std::vector<float> out = partitioned_forward(
            e, p, std::span<const float>(x, nx), std::span<const std::uint32_t>(active, n_active));
        std::memcpy(y, out.data(), out.size() * sizeof(float));
    });
}

int ref_proxy_scores(const float* act, std::size_t n_act, std::uint32_t n_sub, std::uint32_t r,
                     const std::uint32_t* off, const std::uint32_t* ids, double* scores) {
    return guarded([&] {
        GateSet g;
        g.n_subexperts = n_sub;
        g.r = r;
        g.gate_neurons.resize(n_sub);
        for (std::uint32_t n = 0; n < n_sub; ++n) g.gate_neurons[n].assign(ids + off[n], ids + off[n + 1]);
        const auto s = proxy_scores(std::span<const float>(act, n_act), g);
        std::memcpy(scores, s.data(), n_sub * sizeof(double));
    });
}

int ref_select_topk(const double* scores, std::size_t n, std::uint32_t k, std::uint32_t* out) {
    return guarded([&] {
        const auto sel = select_topk_subexperts(std::span<const double>(scores, n), k);
        std::memcpy(out, sel.data(), sel.size() * sizeof(std::uint32_t));
    });
}

// ---- formats (inc/io.hpp:210-251, inc/serde.hpp:100-168) ----

int ref_save_toy_expert(const char* path, std::size_t d, std::size_t ff, const float* wg, const float* wu,
                        const float* wd) {
    return guarded([&] { save_toy_expert(make_expert(d, ff, wg, wu, wd), path); });
}

// Two-phase load: call with null weight pointers to learn d/ff, then again.
int ref_load_toy_expert(const char* path, std::size_t* d, std::size_t* ff, float* wg, float* wu, float* wd) {
    return guarded([&] {
        const ToyExpert e = load_toy_expert(path);
        *d = e.d_model;
        *ff = e.d_ff;
        if (wg) std::memcpy(wg, e.w_gate.data(), e.w_gate.size() * sizeof(float));
        if (wu) std::memcpy(wu, e.w_up.data(), e.w_up.size() * sizeof(float));
        if (wd) std::memcpy(wd, e.w_down.data(), e.w_down.size() * sizeof(float));
    });
}

int ref_append_partition_doc(const char* path, std::uint64_t expert_id, std::uint32_t n_sub, std::size_t n,
                             const std::uint32_t* assignment, double cost, std::uint64_t seed, int truncate) {
    return guarded([&] {
        PartitionDoc doc;
        doc.expert_id = expert_id;
        doc.result.partition = make_partition(n_sub, n, assignment);
        doc.result.cost = cost;
        doc.result.config = default_solver_config(n_sub);
        doc.result.config.seed = seed;
        append_ndjson(path, partition_doc_to_json(doc), truncate != 0);
    });
}

// Appends a partition doc that also carries a gate set (the gates stage
// output, proj/README.md:112-117): partition json merged with gate_set_to_json.
int ref_append_partition_gates_doc(const char* path, std::uint64_t expert_id, std::uint32_t n_sub,
                                   std::size_t n, const std::uint32_t* assignment, std::uint32_t r,
                                   const std::uint32_t* off, const std::uint32_t* ids, int truncate) {
    return guarded([&] {
        PartitionDoc doc;
        doc.expert_id = expert_id;
        doc.result.partition = make_partition(n_sub, n, assignment);
        doc.result.config = default_solver_config(n_sub < 2 ? 2 : n_sub);
        json j = partition_doc_to_json(doc);
        GateSet g;
        g.n_subexperts = n_sub;
        g.r = r;
        g.gate_neurons.resize(n_sub);
        for (std::uint32_t s = 0; s < n_sub; ++s) g.gate_neurons[s].assign(ids + off[s], ids + off[s + 1]);
        json gj = gate_set_to_json(g);
        j["r"] = gj["r"];
        j["gates"] = gj["gates"];
        append_ndjson(path, j, truncate != 0);
    });
}

// Reads document `index` of an NDJSON partition map through
// read_ndjson + partition_doc_from_json.  Two-phase like the loader.
int ref_read_partition_doc(const char* path, std::size_t index, std::uint64_t* expert_id, std::uint32_t* n_sub,
                           std::size_t* n, std::uint32_t* assignment, std::size_t* n_docs) {
    return guarded([&] {
        const auto docs = read_ndjson(path);
        *n_docs = docs.size();
        if (index >= docs.size()) throw ValidationError("document index out of range");
        const PartitionDoc doc = partition_doc_from_json(docs[index]);
        *expert_id = doc.expert_id;
        *n_sub = doc.result.partition.n_subexperts;
        *n = doc.result.partition.assignment.size();
        if (assignment)
            std::memcpy(assignment, doc.result.partition.assignment.data(), *n * sizeof(std::uint32_t));
    });
}

// ---- reference CPU layer (the --impl reference arm of bench.py) ----

struct RefLayer {
    std::vector<ToyExpert> experts;
    std::vector<Partition> partitions;
    std::size_t S = 0;
};

void* ref_layer_create(std::size_t E, std::size_t S, std::size_t d, std::size_t ff, const float* const* wg,
                       const float* const* wu, const float* const* wd, const std::uint32_t* const* assignment) {
    auto* L = new RefLayer;
    L->S = S;
    for (std::size_t e = 0; e < E; ++e) {
        L->experts.push_back(make_expert(d, ff, wg[e], wu[e], wd[e]));
        L->partitions.push_back(make_partition(static_cast<std::uint32_t>(S), ff, assignment[e]));
    }
    return L;
}

void ref_layer_destroy(void* h) { delete static_cast<RefLayer*>(h); }

// Routing: logits in double (rule of inc/expert.hpp:64-71), selection through
// select_topk_subexperts verbatim, softmax renormalisation in double.
int ref_layer_route(void* h, std::size_t T, const float* x, const float* wr, const std::uint32_t* k_per_token,
                    std::uint32_t k_scalar, std::uint32_t k_max, int weight_mode, std::uint32_t* sel, float* w) {
    auto* L = static_cast<RefLayer*>(h);
    return guarded([&] {
        const std::size_t d = L->experts[0].d_model;
        const std::size_t G = L->experts.size() * L->S;
        std::vector<double> logit(G);
        for (std::size_t t = 0; t < T; ++t) {
            std::fill(logit.begin(), logit.end(), 0.0);
            for (std::size_t i = 0; i < d; ++i) {
                const double xi = x[t * d + i];
                for (std::size_t g = 0; g < G; ++g) logit[g] += xi * static_cast<double>(wr[i * G + g]);
            }
            const std::uint32_t k = k_per_token ? k_per_token[t] : k_scalar;
            const auto s = select_topk_subexperts(logit, k);
            const double mx = *std::max_element(logit.begin(), logit.end());
            double z = 0.0;
            for (auto g : s) z += std::exp(logit[g] - mx);
            for (std::uint32_t j = 0; j < k_max; ++j) {
                sel[t * k_max + j] = j < k ? s[j] : 0xFFFFFFFFu;
                w[t * k_max + j] =
                    j < k ? (weight_mode == 1 ? static_cast<float>(std::exp(logit[s[j]] - mx) / z) : 1.0f) : 0.0f;
            }
        }
    });
}

// y_t = sum over verbatim partitioned_forward calls (one per selected
// sub-expert in weighted mode, one per parent expert in unit mode).
// std::thread over tokens: the functions are pure (proj/README.md:167-168).
int ref_layer_forward(void* h, std::size_t T, const float* x, std::uint32_t k_max, const std::uint32_t* sel,
                      const float* w, int weight_mode, float* y, int nthreads) {
    auto* L = static_cast<RefLayer*>(h);
    const std::size_t d = L->experts[0].d_model;
    const std::size_t S = L->S;
    std::vector<int> rcs(nthreads > 0 ? nthreads : 1, 0);
    auto work = [&](std::size_t t0, std::size_t t1, int* rc) {
        *rc = guarded([&] {
            std::vector<double> acc(d);
            for (std::size_t t = t0; t < t1; ++t) {
                std::fill(acc.begin(), acc.end(), 0.0);
                const std::span<const float> xt(x + t * d, d);
                for (std::size_t e = 0; e < L->experts.size(); ++e) {
                    std::vector<std::uint32_t> active;
                    std::vector<float> wts;
                    for (std::uint32_t j = 0; j < k_max; ++j) {
                        const std::uint32_t g = sel[t * k_max + j];
                        if (g != 0xFFFFFFFFu && g / S == e) {
                            active.push_back(static_cast<std::uint32_t>(g % S));
                            wts.push_back(w[t * k_max + j]);
                        }
                    }
                    if (active.empty()) continue;
                    if (weight_mode == 0) {
                        const auto part = partitioned_forward(L->experts[e], L->partitions[e], xt, active);
                        for (std::size_t i = 0; i < d; ++i) acc[i] += static_cast<double>(part[i]);
                    } else {
                        for (std::size_t q = 0; q < active.size(); ++q) {
                            const std::uint32_t one[1] = {active[q]};
                            const auto part = partitioned_forward(L->experts[e], L->partitions[e], xt, one);
                            for (std::size_t i = 0; i < d; ++i)
                                acc[i] += static_cast<double>(wts[q]) * static_cast<double>(part[i]);
                        }
                    }
                }
                for (std::size_t i = 0; i < d; ++i) y[t * d + i] = static_cast<float>(acc[i]);
            }
        });
    };
    const int nt = static_cast<int>(std::min<std::size_t>(rcs.size(), T ? T : 1));
    std::vector<std::thread> th;
    for (int q = 0; q < nt; ++q) th.emplace_back(work, T * q / nt, T * (q + 1) / nt, &rcs[q]);
    for (auto& t : th) t.join();
    for (int rc : rcs)
        if (rc) return rc;
    return 0;
}


// ---- calibration side, verbatim reference calls ----
int ref_collect_activation_matrix(std::size_t d, std::size_t ff, const float* wg, const float* wu, const float* wd,
                                  std::size_t B, const float* x, float* out) {
    return guarded([&] {
        ToyExpert e = make_expert(d, ff, wg, wu, wd);
        std::vector<std::vector<float>> in(B);
        for (std::size_t b = 0; b < B; ++b) in[b].assign(x + b * d, x + (b + 1) * d);
        ActivationMatrix m = collect_activation_matrix(e, in);
        std::memcpy(out, m.data.data(), m.data.size() * sizeof(float));
    });
}

int ref_binarize_topk(const float* act, std::size_t rows, std::size_t cols, std::size_t k_a, std::uint8_t* bits) {
    return guarded([&] {
        ActivationMatrix m = make_activation_matrix(rows, cols);
        m.data.assign(act, act + rows * cols);
        BinaryActivation b = binarize_topk(m, k_a);
        std::memcpy(bits, b.bits.data(), b.bits.size());
    });
}

int ref_coactivation(const std::uint8_t* bits, std::size_t rows, std::size_t cols, std::size_t k_a,
                     std::uint32_t* co) {
    return guarded([&] {
        BinaryActivation b;
        b.rows = rows;
        b.cols = cols;
        b.k_a = k_a;
        b.bits.assign(bits, bits + rows * cols);
        CoActivationMatrix c = coactivation(b);
        std::memcpy(co, c.data.data(), c.data.size() * sizeof(std::uint32_t));
    });
}

int ref_save_activation_matrix(const char* path, std::size_t rows, std::size_t cols, const float* data) {
    return guarded([&] {
        ActivationMatrix m = make_activation_matrix(rows, cols);
        m.data.assign(data, data + rows * cols);
        save_activation_matrix(m, path);
    });
}

int ref_load_activation_matrix(const char* path, std::size_t* rows, std::size_t* cols, float* data) {
    return guarded([&] {
        ActivationMatrix m = load_activation_matrix(path, MatrixFormat::binary);
        *rows = m.rows;
        *cols = m.cols;
        if (data) std::memcpy(data, m.data.data(), m.data.size() * sizeof(float));
    });
}

// load_perf_table (validates the grid) + eval_cost at (batch, k)
int ref_perf_table_eval(const char* path, std::uint64_t batch, std::uint32_t k, double* cost, std::size_t* n_batch,
                        std::size_t* n_k) {
    return guarded([&] {
        PerfTable t = load_perf_table(path);
        *cost = eval_cost(t, batch, k);
        *n_batch = t.batch_axis.size();
        *n_k = t.k_axis.size();
    });
}

// cache_step (inc/offload.hpp:202-255) folded over a request sequence, fine
// granularity, unit bytes 1: the per-step miss counts of the reference LRU.
int ref_offload_replay(std::uint32_t n_units, std::uint32_t capacity, std::size_t n_steps,
                       const std::uint32_t* step_off, const std::uint32_t* ids, std::uint64_t* misses) {
    return guarded([&] {
        OffloadConfig cfg;
        cfg.n_experts = n_units;
        cfg.subexperts_per_expert = 1;
        cfg.expert_bytes = 1;
        cfg.vram_bytes = capacity;
        cfg.pcie_bytes_per_s = 1.0;
        cfg.compute_s_per_subexpert = 1.0;
        cfg.granularity = Granularity::fine;
        CacheState c = make_cache(cfg);
        for (std::size_t t = 0; t < n_steps; ++t) {
            std::vector<std::uint32_t> req(ids + step_off[t], ids + step_off[t + 1]);
            misses[t] = cache_step(c, req, cfg).miss_count;
        }
    });
}

// ---- gate construction / fidelity (inc/gating.hpp:28-174) and the C4 fixtures ----
std::size_t ref_default_binarize_count(std::size_t cols) { return default_binarize_count(cols); }

int ref_random_matrix(std::size_t rows, std::size_t cols, std::uint64_t seed, float* out) {
    return guarded([&] {
        ActivationMatrix m = testsupport::random_matrix(rows, cols, seed);
        std::memcpy(out, m.data.data(), m.data.size() * sizeof(float));
    });
}

int ref_planted_cluster(std::size_t tokens, std::uint32_t n_sub, std::size_t group, std::uint64_t seed, float* matrix,
                        std::uint32_t* assignment) {
    return guarded([&] {
        auto pc = testsupport::planted_cluster(tokens, n_sub, group, seed);
        std::memcpy(matrix, pc.matrix.data.data(), pc.matrix.data.size() * sizeof(float));
        std::memcpy(assignment, pc.partition.assignment.data(), pc.partition.assignment.size() * 4);
    });
}

int ref_select_gate_neurons(const std::uint32_t* co, std::size_t dim, std::uint32_t n_sub,
                            const std::uint32_t* assignment, std::uint32_t r, std::uint32_t* offsets,
                            std::uint32_t* ids) {
    return guarded([&] {
        CoActivationMatrix c;
        c.dim = dim;
        c.data.assign(co, co + dim * dim);
        GateSet g = select_gate_neurons(c, make_partition(n_sub, dim, assignment), r);
        offsets[0] = 0;
        for (std::uint32_t q = 0; q < n_sub; ++q) {
            offsets[q + 1] = offsets[q] + static_cast<std::uint32_t>(g.gate_neurons[q].size());
            std::copy(g.gate_neurons[q].begin(), g.gate_neurons[q].end(), ids + offsets[q]);
        }
    });
}

int ref_gating_fidelity(const float* act, std::size_t rows, std::size_t cols, std::uint32_t n_sub,
                        const std::uint32_t* assignment, std::uint32_t r, const std::uint32_t* offsets,
                        const std::uint32_t* ids, std::uint32_t k, double* out) {
    return guarded([&] {
        ActivationMatrix m = make_activation_matrix(rows, cols);
        m.data.assign(act, act + rows * cols);
        GateSet g;
        g.n_subexperts = n_sub;
        g.r = r;
        g.gate_neurons.resize(n_sub);
        for (std::uint32_t q = 0; q < n_sub; ++q) g.gate_neurons[q].assign(ids + offsets[q], ids + offsets[q + 1]);
        *out = gating_fidelity(m, make_partition(n_sub, cols, assignment), g, k);
    });
}
}  // extern "C"
