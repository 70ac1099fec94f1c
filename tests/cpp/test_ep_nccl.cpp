// The expert-parallel layer on the C++ host (moe_layer.hpp ExpertParallelLayer
// over mp_ep_forward: NCCL all-to-allv dispatch / return, deterministic
// combine) against the single-GPU MoeLayer on the same weights, in a 1-rank
// NCCL communicator (the pool gives one GPU per call; the exchange, counts and
// combine code paths are the multi-rank ones).  Outputs must be bit-identical
// for scalar and per-token k; with the residual the expert-parallel combine
// adds x to each rank's bf16 partial, so the reference is bf16(x + y).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "moeprism/moe_layer.hpp"

using namespace moeprism;

static int g_fail = 0;
#define CHECK(c)                                                    \
    do {                                                            \
        if (!(c)) {                                                 \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++g_fail;                                               \
        }                                                           \
    } while (0)

int main() {
    const std::uint32_t E = 4, S = 4, d = 256, ff = 512, T = 96, K = 4;
    LayerConfig c;
    c.n_experts = E;
    c.n_subexperts = S;
    c.d_model = d;
    c.d_ff = ff;
    c.k_max = 8;
    c.max_tokens = T;
    std::mt19937_64 rng(5);
    std::uniform_real_distribution<float> U(-1.f, 1.f);
    MoeLayer full(c);
    ExpertParallelLayer ep(c, 1, 0);
    ep.connect(ExpertParallelLayer::unique_id());
    for (std::uint32_t e = 0; e < E; ++e) {
        ToyExpert x;
        x.d_model = d;
        x.d_ff = ff;
        for (auto* w : {&x.w_gate, &x.w_up, &x.w_down}) {
            w->resize(d * ff);
            for (auto& v : *w) v = U(rng) * 0.0625f;
        }
        Partition p;
        p.n_subexperts = S;
        for (std::uint32_t j = 0; j < ff; ++j) p.assignment.push_back((j * 7 + e) % S);
        full.set_partition(e, p);
        full.load_expert(e, x);
        ep.set_partition(e, p);
        ep.load_expert(e, x);
    }
    std::vector<float> wr(d * E * S);
    for (auto& v : wr) v = U(rng) * 0.0625f;
    full.set_router(wr);
    ep.set_router(wr);
    std::vector<std::uint16_t> xh(T * d);
    for (auto& v : xh) v = b200::detail::to_bf16(U(rng));
    std::vector<std::uint32_t> kpt(T);
    for (auto& v : kpt) v = 1 + static_cast<std::uint32_t>(rng() % 8);
    void *x = nullptr, *y1 = nullptr, *y2 = nullptr, *kd = nullptr;
    cudaMalloc(&x, T * d * 2);
    cudaMalloc(&y1, T * d * 2);
    cudaMalloc(&y2, T * d * 2);
    cudaMalloc(&kd, T * 4);
    cudaMemcpy(x, xh.data(), T * d * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(kd, kpt.data(), T * 4, cudaMemcpyHostToDevice);
    std::vector<std::uint16_t> a(T * d), b(T * d);
    for (int mode = 0; mode < 3; ++mode) {
        const bool residual = mode == 1;
        const std::uint32_t* kp = mode == 2 ? static_cast<const std::uint32_t*>(kd) : nullptr;
        full.forward_device(x, T, K, y1, nullptr, kp);
        ep.forward_device(x, T, K, y2, nullptr, kp, residual);
        cudaDeviceSynchronize();
        cudaMemcpy(a.data(), y1, T * d * 2, cudaMemcpyDeviceToHost);
        cudaMemcpy(b.data(), y2, T * d * 2, cudaMemcpyDeviceToHost);
        if (residual)
            for (std::size_t i = 0; i < a.size(); ++i)
                a[i] = b200::detail::to_bf16(b200::detail::from_bf16(xh[i]) + b200::detail::from_bf16(a[i]));
        CHECK(std::memcmp(a.data(), b.data(), a.size() * 2) == 0);
        std::printf("%s mode %d (%s)\n", std::memcmp(a.data(), b.data(), a.size() * 2) == 0 ? "PASS" : "FAIL", mode,
                    mode == 0 ? "scalar k" : mode == 1 ? "fused residual" : "per-token k");
    }
    std::uint32_t sent = 0, recv = 0;
    mp_ep_last_counts(ep.handle(), &sent, &recv);
    CHECK(sent == T && recv == T);  // one rank: every token once to itself
    cudaFree(x);
    cudaFree(y1);
    cudaFree(y2);
    cudaFree(kd);
    std::printf(g_fail ? "FAILED %d checks\n" : "ALL PASSED\n", g_fail);
    return g_fail ? 1 : 0;
}
