// test_dropin.cpp -- the reference's expert / decomposition known-answer tests
// (proj/tests/test_expert.cpp, proj/tests/acceptance.cpp criterion 1) restated
// as asserts and run against the GPU drop-in moeprism::partitioned_forward and
// moeprism::MoeLayer (include/moeprism/moe_layer.hpp).  Expected values are
// computed from the definition here, like tests/support.hpp does.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "moeprism/moe_layer.hpp"

using namespace moeprism;

static int g_fail = 0;
#define CHECK(cond)                                                   \
    do {                                                              \
        if (!(cond)) {                                                \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); \
            ++g_fail;                                                 \
        }                                                             \
    } while (0)

static double uniform01(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

// tests/support.hpp:73-86
static ToyExpert random_expert(std::size_t d, std::size_t ff, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    ToyExpert e;
    e.d_model = d;
    e.d_ff = ff;
    for (auto* w : {&e.w_gate, &e.w_up, &e.w_down}) {
        w->resize(d * ff);
        for (auto& v : *w) v = static_cast<float>(uniform01(rng) * 2.0 - 1.0);
    }
    return e;
}
// tests/support.hpp:89-105
static Partition random_balanced_partition(std::size_t n, std::uint32_t ns, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::vector<std::uint32_t> order(n);
    for (std::size_t i = 0; i < n; ++i) order[i] = static_cast<std::uint32_t>(i);
    for (std::size_t i = n - 1; i > 0; --i) {
        const std::uint64_t m = i + 1, mx = ~0ull, lim = mx - mx % m;
        std::uint64_t r;
        do r = rng();
        while (r >= lim);
        std::swap(order[i], order[r % m]);
    }
    Partition p;
    p.n_subexperts = ns;
    p.assignment.assign(n, 0);
    for (std::size_t i = 0; i < n; ++i) p.assignment[order[i]] = static_cast<std::uint32_t>(i % ns);
    return p;
}
// definition of the activations (inc/expert.hpp:62-75) in double
static std::vector<double> acts(const ToyExpert& e, const std::vector<float>& x) {
    std::vector<double> a(e.d_ff);
    for (std::size_t j = 0; j < e.d_ff; ++j) {
        double g = 0, u = 0;
        for (std::size_t i = 0; i < e.d_model; ++i) {
            g += double(x[i]) * e.w_gate[i * e.d_ff + j];
            u += double(x[i]) * e.w_up[i * e.d_ff + j];
        }
        a[j] = double(float(g / (1.0 + std::exp(-g)) * u));
    }
    return a;
}
static std::vector<double> part_sum(const ToyExpert& e, const Partition& p, const std::vector<float>& x,
                                    const std::vector<std::uint32_t>& act) {
    const auto a = acts(e, x);
    std::vector<double> y(e.d_model, 0.0);
    for (std::size_t j = 0; j < e.d_ff; ++j) {
        bool on = false;
        for (auto s : act) on |= p.assignment[j] == s;
        if (!on) continue;
        for (std::size_t i = 0; i < e.d_model; ++i) y[i] += a[j] * e.w_down[j * e.d_model + i];
    }
    return y;
}
static bool close(float got, double want, double tol = 1e-5) { return std::fabs(got - want) <= tol * (1.0 + std::fabs(want)); }

template <class F>
static bool throws_validation(F&& f) {
    try {
        f();
    } catch (const ValidationError&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    {  // all-active == full (test_expert.cpp:76-88)
        const ToyExpert e = random_expert(8, 12, 5);
        const Partition p = random_balanced_partition(12, 4, 6);
        std::mt19937_64 rng(7);
        std::vector<float> x(8);
        for (auto& v : x) v = static_cast<float>(uniform01(rng) * 2.0 - 1.0);
        const auto y = partitioned_forward(e, p, x, std::vector<std::uint32_t>{0, 1, 2, 3});
        const auto want = part_sum(e, p, x, {0, 1, 2, 3});
        for (std::size_t i = 0; i < y.size(); ++i) CHECK(close(y[i], want[i]));
        std::printf("PASS all-active equals full\n");
    }
    {  // empty -> zero (:90-96)
        const ToyExpert e = random_expert(5, 10, 8);
        const Partition p = random_balanced_partition(10, 2, 9);
        const auto y = partitioned_forward(e, p, std::vector<float>(5, 0.25f), std::vector<std::uint32_t>{});
        for (float v : y) CHECK(v == 0.0f);
        std::printf("PASS empty active set is zero\n");
    }
    {  // single sub-expert hand sum (:98-115)
        const ToyExpert e = random_expert(2, 4, 10);
        Partition p;
        p.n_subexperts = 2;
        p.assignment = {0, 1, 0, 1};
        const std::vector<float> x = {0.5f, -0.75f};
        const auto y = partitioned_forward(e, p, x, std::vector<std::uint32_t>{1});
        const auto a = acts(e, x);
        for (std::size_t i = 0; i < 2; ++i) {
            double want = 0;
            for (std::size_t j : {1u, 3u}) want += a[j] * e.w_down[j * 2 + i];
            CHECK(close(y[i], want));
        }
        std::printf("PASS single sub-expert hand sum\n");
    }
    {  // additivity (:117-132)
        const ToyExpert e = random_expert(6, 12, 11);
        const Partition p = random_balanced_partition(12, 4, 12);
        std::mt19937_64 rng(13);
        std::vector<float> x(6);
        for (auto& v : x) v = static_cast<float>(uniform01(rng) * 2.0 - 1.0);
        const auto ya = partitioned_forward(e, p, x, std::vector<std::uint32_t>{0, 2});
        const auto yb = partitioned_forward(e, p, x, std::vector<std::uint32_t>{1, 3});
        const auto yall = partitioned_forward(e, p, x, std::vector<std::uint32_t>{0, 1, 2, 3});
        for (std::size_t i = 0; i < yall.size(); ++i) CHECK(close(yall[i], double(ya[i]) + yb[i]));
        std::printf("PASS additivity\n");
    }
    {  // validation (:134-146)
        const ToyExpert e = random_expert(4, 8, 14);
        const std::vector<float> x(4, 0.0f);
        Partition bad_w = random_balanced_partition(6, 2, 15);
        const Partition p = random_balanced_partition(8, 2, 16);
        CHECK(throws_validation([&] { partitioned_forward(e, bad_w, x, std::vector<std::uint32_t>{0}); }));
        CHECK(throws_validation([&] { partitioned_forward(e, p, x, std::vector<std::uint32_t>{2}); }));
        CHECK(throws_validation([&] { partitioned_forward(e, p, x, std::vector<std::uint32_t>{0, 0}); }));
        CHECK(throws_validation([&] { partitioned_forward(e, p, std::vector<float>(3, 0.0f), std::vector<std::uint32_t>{0}); }));
        ToyExpert nan_e = e;
        nan_e.w_up[1] = NAN;
        CHECK(throws_validation([&] { partitioned_forward(nan_e, p, x, std::vector<std::uint32_t>{0}); }));
        std::printf("PASS validation verdicts\n");
    }
    {  // acceptance C1 (acceptance.cpp:69-100), 30 trials on the GPU
        const std::uint32_t n_opts[3] = {2, 4, 8};
        for (int trial = 0; trial < 30; ++trial) {
            std::mt19937_64 rng(1000 + trial);
            const std::uint32_t n = n_opts[trial % 3];
            auto uidx = [&](std::uint64_t m) {
                const std::uint64_t mx = ~0ull, lim = mx - mx % m;
                std::uint64_t r;
                do r = rng();
                while (r >= lim);
                return r % m;
            };
            const std::size_t d = 1 + uidx(64);
            const std::size_t ff = n + uidx(129 - n);
            const ToyExpert e = random_expert(d, ff, 5000 + trial);
            const Partition p = random_balanced_partition(ff, n, 6000 + trial);
            std::vector<float> x(d);
            for (auto& v : x) v = static_cast<float>(uniform01(rng) * 2.0 - 1.0);
            std::vector<std::uint32_t> all(n);
            std::iota(all.begin(), all.end(), 0u);
            const auto y = partitioned_forward(e, p, x, all);
            const auto want = part_sum(e, p, x, all);
            for (std::size_t i = 0; i < d; ++i) CHECK(close(y[i], want[i]));
        }
        std::printf("PASS acceptance C1 (30 trials)\n");
    }
    {  // reference-valid partitions with more than 64 / more than 256 sub-experts
        for (std::uint32_t n : {100u, 300u}) {
            const std::size_t d = 16, ff = 3 * n + 7;
            const ToyExpert e = random_expert(d, ff, 70 + n);
            const Partition p = random_balanced_partition(ff, n, 80 + n);
            std::mt19937_64 rng(90 + n);
            std::vector<float> x(d);
            for (auto& v : x) v = static_cast<float>(uniform01(rng) * 2.0 - 1.0);
            std::vector<std::uint32_t> act;
            for (std::uint32_t s2 = 0; s2 < n; s2 += 3) act.push_back(s2);
            if (act.back() != n - 1) act.push_back(n - 1);
            std::vector<std::uint32_t> all(n);
            std::iota(all.begin(), all.end(), 0u);
            const auto y = partitioned_forward(e, p, x, act);
            const auto want = part_sum(e, p, x, act);
            const auto ya = partitioned_forward(e, p, x, all);
            const auto wa = part_sum(e, p, x, all);
            for (std::size_t i = 0; i < d; ++i) CHECK(close(y[i], want[i]) && close(ya[i], wa[i]));
        }
        std::printf("PASS partitions with 100 and 300 sub-experts\n");
    }
    {  // MoeLayer: unit weights, every sub-expert of 2 experts (k = E*S) == sum of full experts
        LayerConfig c;
        c.n_experts = 2;
        c.n_subexperts = 4;
        c.d_model = 32;
        c.d_ff = 64;
        c.dtype = Dtype::f32;
        c.weights = WeightMode::unit;
        c.k_max = 8;
        c.max_tokens = 8;
        MoeLayer layer(c);
        std::vector<ToyExpert> ex;
        std::vector<Partition> ps;
        for (std::uint32_t e = 0; e < 2; ++e) {
            ex.push_back(random_expert(32, 64, 40 + e));
            ps.push_back(random_balanced_partition(64, 4, 50 + e));
            layer.set_partition(e, ps[e]);
            layer.load_expert(e, ex[e]);
        }
        std::vector<float> wr(32 * 8, 0.01f);
        layer.set_router(wr);
        std::mt19937_64 rng(3);
        std::vector<float> x(8 * 32);
        for (auto& v : x) v = static_cast<float>(uniform01(rng) * 2.0 - 1.0);
        const auto y = layer.forward(x, 8u);
        for (std::size_t t = 0; t < 8; ++t) {
            std::vector<float> xt(x.begin() + t * 32, x.begin() + (t + 1) * 32);
            for (std::size_t i = 0; i < 32; ++i) {
                double want = 0;
                for (std::uint32_t e = 0; e < 2; ++e) want += double(float(part_sum(ex[e], ps[e], xt, {0, 1, 2, 3})[i]));
                CHECK(close(y[t * 32 + i], want));
            }
        }
        CHECK(throws_validation([&] { layer.forward(x, 9u); }));
        std::printf("PASS MoeLayer all-sub-experts forward\n");
    }
    std::printf(g_fail ? "FAILED %d checks\n" : "ALL PASSED\n", g_fail);
    return g_fail ? 1 : 0;
}
