/*
 * moe_oracle.c -- CPU restatement of MoE-Prism's online sub-expert layer
 * forward.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the parity oracle for the B200 path.  It is imported only by
 * tests/, by __graft_entry__.smoke() (as the checker) and by bench.py's
 * cpu_baseline / --impl reference legs.  The product path
 * (paper_2510_19366_b200/ + include/) never links, loads or calls it.
 *
 * Every function restates a reference function (file:line under
 * /root/reference/proj/include/moeprism/, cited as inc/X.hpp:N) or, where the
 * reference has no code (linear router, softmax renormalisation, bucketing,
 * multi-expert composition), the restatement SURVEY.md section 8(c) fixes as the
 * contract.  Parity of the restated reference functions is PINNED against the
 * reference itself: oracle/ref_shim.cpp compiles the reference headers
 * verbatim into oracle/_ref/libmoeprism_ref.so and tests/test_oracle.py
 * checks this file against it bit for bit (plus the reference's own KATs
 * restated as asserts, and the committed golden vectors in tests/golden/).
 *
 * Arithmetic rules copied from the reference: double accumulators, i (or j)
 * ascending, products of float operands formed in double, results cast to
 * float.  Compile with -ffp-contract=off so no FMA contraction changes the
 * rounding relative to the reference's x86-64 -O3 build.
 *
 * Status codes: 0 ok, 1 validation error (ValidationError), 2 I/O (IoError).
 */
#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_VALIDATION 1
#define ORC_IO 2

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* mt19937_64 (the generator inc/rng.hpp draws through; the standard 64-bit
 * Mersenne Twister with std::mt19937_64's default seeding).                 */

typedef struct {
    uint64_t mt[312];
    int idx;
} orc_mt64;

static void mt_seed(orc_mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

static uint64_t mt_next(orc_mt64* s) {
    static const uint64_t MAG[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (s->idx >= 312) {
        int i;
        uint64_t x;
        for (i = 0; i < 312 - 156; ++i) {
            x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ MAG[x & 1ULL];
        }
        for (; i < 311; ++i) {
            x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ MAG[x & 1ULL];
        }
        x = (s->mt[311] & UM) | (s->mt[0] & LM);
        s->mt[311] = s->mt[155] ^ (x >> 1) ^ MAG[x & 1ULL];
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

/* inc/rng.hpp:15-17 */
static double uniform01(orc_mt64* s) { return (double)(mt_next(s) >> 11) * 0x1.0p-53; }

/* inc/rng.hpp:20-28 */
static uint64_t uniform_index(orc_mt64* s, uint64_t n) {
    const uint64_t max = UINT64_MAX;
    const uint64_t limit = max - max % n;
    uint64_t x;
    do {
        x = mt_next(s);
    } while (x >= limit);
    return x % n;
}

/* Raw draws, for pinning the generator against std::mt19937_64. */
void orc_mt64_draw(uint64_t seed, size_t n, uint64_t* out) {
    orc_mt64 s;
    mt_seed(&s, seed);
    for (size_t i = 0; i < n; ++i) out[i] = mt_next(&s);
}

/* n draws of float(uniform01*2-1) * scale from one stream: the fill used by
 * tests/support.hpp:80 (random_expert) and by the layer configs of SURVEY
 * 8(d) for inputs x and the router W_r (scale = 1/sqrt(d) there).          */
void orc_mt_uniform_pm1(uint64_t seed, size_t n, double scale, float* out) {
    orc_mt64 s;
    mt_seed(&s, seed);
    for (size_t i = 0; i < n; ++i) out[i] = (float)((uniform01(&s) * 2.0 - 1.0) * scale);
}

/* tests/support.hpp:73-86 */
int orc_random_expert(size_t d, size_t ff, uint64_t seed, float* wg, float* wu, float* wd) {
    orc_mt64 s;
    mt_seed(&s, seed);
    for (size_t i = 0; i < d * ff; ++i) wg[i] = (float)(uniform01(&s) * 2.0 - 1.0);
    for (size_t i = 0; i < d * ff; ++i) wu[i] = (float)(uniform01(&s) * 2.0 - 1.0);
    for (size_t i = 0; i < d * ff; ++i) wd[i] = (float)(uniform01(&s) * 2.0 - 1.0);
    return ORC_OK;
}

/* tests/support.hpp:89-105 */
int orc_random_balanced_partition(size_t n, uint32_t n_sub, uint64_t seed, uint32_t* assignment) {
    if (n == 0) return fail(ORC_VALIDATION, "empty partition");
    orc_mt64 s;
    mt_seed(&s, seed);
    uint32_t* order = (uint32_t*)malloc(n * sizeof(uint32_t));
    for (size_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
    for (size_t i = n - 1; i > 0; --i) {
        size_t j = (size_t)uniform_index(&s, i + 1);
        uint32_t t = order[i];
        order[i] = order[j];
        order[j] = t;
    }
    for (size_t i = 0; i < n; ++i) assignment[order[i]] = (uint32_t)(i % n_sub);
    free(order);
    return ORC_OK;
}

/* inc/partition.hpp:59-74 */
int orc_contiguous_partition(size_t n, uint32_t n_sub, uint32_t* assignment) {
    if (n_sub < 1 || n < n_sub)
        return fail(ORC_VALIDATION, "cannot split %zu neurons into %u sub-experts", n, n_sub);
    size_t base = n / n_sub, extra = n % n_sub, pos = 0;
    for (uint32_t s = 0; s < n_sub; ++s) {
        size_t cap = base + (s < extra ? 1 : 0);
        for (size_t c = 0; c < cap; ++c) assignment[pos++] = s;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Counter-based synthetic generator for the large configs.
 * Element i of stream `seed` is a pure function of (seed, i), so the GPU
 * fill kernel (paper_2510_19366_b200/csrc/pack.cu synth_fill_kernel) and this CPU fill agree
 * bit for bit at any size without replaying a sequential stream.
 *   state = mix(seed + G); u_i = (mix(state + (i+1) G) >> 11) * 2^-53
 *   value = float((u_i * 2 - 1) * scale)
 * mix = SplitMix64 finaliser, G = 0x9E3779B97F4A7C15.                      */

static inline uint64_t sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline float synth_value(uint64_t state, uint64_t i, double scale) {
    const uint64_t G = 0x9E3779B97F4A7C15ULL;
    double u = (double)(sm_mix(state + (i + 1) * G) >> 11) * 0x1.0p-53;
    return (float)((u * 2.0 - 1.0) * scale);
}

uint64_t orc_synth_state(uint64_t seed) { return sm_mix(seed + 0x9E3779B97F4A7C15ULL); }

/* out[j] = value(first + j), j < n */
void orc_synth_fill(uint64_t seed, uint64_t first, size_t n, double scale, float* out) {
    uint64_t st = orc_synth_state(seed);
    for (size_t j = 0; j < n; ++j) out[j] = synth_value(st, first + j, scale);
}

/* Same stream laid out transposed: out[c * rows + r] = value(r * cols + c).
 * Lets the oracle receive w_gate / w_up neuron-major without a transpose.   */
void orc_synth_fill_t(uint64_t seed, size_t rows, size_t cols, double scale, float* out) {
    uint64_t st = orc_synth_state(seed);
    for (size_t r = 0; r < rows; ++r)
        for (size_t c = 0; c < cols; ++c) out[c * rows + r] = synth_value(st, (uint64_t)r * cols + c, scale);
}

/* ------------------------------------------------------------------------ */
/* Expert numerics: inc/expert.hpp                                          */

/* inc/expert.hpp:41 */
static double silu(double x) { return x / (1.0 + exp(-x)); }
double orc_silu(double x) { return silu(x); }

static int validate_weights(size_t d, size_t ff, const float* wg, const float* wu, const float* wd) {
    /* inc/expert.hpp:25-39 */
    if (d < 1 || ff < 1) return fail(ORC_VALIDATION, "toy expert needs d_model >= 1 and d_ff >= 1");
    if (!wg || !wu || !wd) return fail(ORC_VALIDATION, "toy expert weight shapes do not match");
    const float* ws[3] = {wg, wu, wd};
    for (int m = 0; m < 3; ++m)
        for (size_t i = 0; i < d * ff; ++i)
            if (!isfinite(ws[m][i])) return fail(ORC_VALIDATION, "toy expert weight is not finite");
    return ORC_OK;
}

static int check_input(size_t d, const float* x, size_t nx) {
    /* inc/expert.hpp:50-58 */
    if (nx != d) return fail(ORC_VALIDATION, "input length %zu does not match d_model %zu", nx, d);
    for (size_t i = 0; i < d; ++i)
        if (!isfinite(x[i])) return fail(ORC_VALIDATION, "input vector is not finite");
    return ORC_OK;
}

/* inc/expert.hpp:62-75.  Neuron j: a[j] = float(silu(g) * u) with
 * g = sum_i double(x_i) * double(wg[i][j]), i ascending.                    */
static float neuron_activation_mpex(size_t d, size_t ff, const float* wg, const float* wu,
                                    const float* x, size_t j) {
    double g = 0.0, u = 0.0;
    for (size_t i = 0; i < d; ++i) {
        const double xi = x[i];
        g += xi * (double)wg[i * ff + j];
        u += xi * (double)wu[i * ff + j];
    }
    return (float)(silu(g) * u);
}

/* Same arithmetic with the neuron's weights contiguous (wgT[j][i]).        */
static float neuron_activation_nm(size_t d, const float* wgT, const float* wuT, const float* x,
                                  size_t j) {
    const float* gr = wgT + j * d;
    const float* ur = wuT + j * d;
    double g = 0.0, u = 0.0;
    for (size_t i = 0; i < d; ++i) {
        const double xi = x[i];
        g += xi * (double)gr[i];
        u += xi * (double)ur[i];
    }
    return (float)(silu(g) * u);
}

int orc_intermediate(size_t d, size_t ff, const float* wg, const float* wu, const float* x, float* a) {
    for (size_t j = 0; j < ff; ++j) a[j] = neuron_activation_mpex(d, ff, wg, wu, x, j);
    return ORC_OK;
}

/* inc/expert.hpp:79-96 */
int orc_toy_ffn_forward(size_t d, size_t ff, const float* wg, const float* wu, const float* wd,
                        const float* x, size_t nx, float* y, float* a) {
    int rc = validate_weights(d, ff, wg, wu, wd);
    if (rc) return rc;
    if ((rc = check_input(d, x, nx))) return rc;
    orc_intermediate(d, ff, wg, wu, x, a);
    double* acc = (double*)calloc(d, sizeof(double));
    for (size_t j = 0; j < ff; ++j) {
        const double aj = a[j];
        if (aj == 0.0) continue;
        const float* down = wd + j * d;
        for (size_t i = 0; i < d; ++i) acc[i] += aj * (double)down[i];
    }
    for (size_t i = 0; i < d; ++i) y[i] = (float)acc[i];
    free(acc);
    return ORC_OK;
}

/* inc/partition.hpp:34-46 (validate(Partition)) */
int orc_validate_partition(uint32_t n_sub, size_t n, const uint32_t* assignment) {
    if (n_sub < 1) return fail(ORC_VALIDATION, "partition needs at least one sub-expert");
    if (n < n_sub) return fail(ORC_VALIDATION, "partition needs at least as many neurons as sub-experts");
    size_t* sizes = (size_t*)calloc(n_sub, sizeof(size_t));
    for (size_t c = 0; c < n; ++c) {
        if (assignment[c] >= n_sub) {
            free(sizes);
            return fail(ORC_VALIDATION, "partition label %u out of range for N=%u", assignment[c], n_sub);
        }
        ++sizes[assignment[c]];
    }
    size_t lo = sizes[0], hi = sizes[0];
    for (uint32_t s = 1; s < n_sub; ++s) {
        if (sizes[s] < lo) lo = sizes[s];
        if (sizes[s] > hi) hi = sizes[s];
    }
    free(sizes);
    if (lo == 0) return fail(ORC_VALIDATION, "every sub-expert must be non-empty");
    if (hi - lo > 1) return fail(ORC_VALIDATION, "partition is not balanced: sizes range from %zu to %zu", lo, hi);
    return ORC_OK;
}

/* inc/expert.hpp:101-135.  Unweighted output restricted to the active
 * sub-experts; neurons accumulated in ascending global index.              */
int orc_partitioned_forward(size_t d, size_t ff, const float* wg, const float* wu, const float* wd,
                            uint32_t n_sub, size_t n_assign, const uint32_t* assignment,
                            const float* x, size_t nx, const uint32_t* active, size_t n_active,
                            float* y) {
    int rc = validate_weights(d, ff, wg, wu, wd);
    if (rc) return rc;
    if ((rc = orc_validate_partition(n_sub, n_assign, assignment))) return rc;
    if ((rc = check_input(d, x, nx))) return rc;
    if (n_assign != ff)
        return fail(ORC_VALIDATION, "partition covers %zu neurons but the expert has d_ff %zu", n_assign, ff);
    uint8_t* is_active = (uint8_t*)calloc(n_sub, 1);
    for (size_t k = 0; k < n_active; ++k) {
        uint32_t n = active[k];
        if (n >= n_sub) {
            free(is_active);
            return fail(ORC_VALIDATION, "active sub-expert %u out of range for N=%u", n, n_sub);
        }
        if (is_active[n]) {
            free(is_active);
            return fail(ORC_VALIDATION, "active sub-expert list has duplicates");
        }
        is_active[n] = 1;
    }
    float* a = (float*)malloc(ff * sizeof(float));
    orc_intermediate(d, ff, wg, wu, x, a); /* all neurons, as :121 does */
    double* acc = (double*)calloc(d, sizeof(double));
    for (size_t j = 0; j < ff; ++j) {
        if (!is_active[assignment[j]]) continue;
        const double aj = a[j];
        if (aj == 0.0) continue;
        const float* down = wd + j * d;
        for (size_t i = 0; i < d; ++i) acc[i] += aj * (double)down[i];
    }
    for (size_t i = 0; i < d; ++i) y[i] = (float)acc[i];
    free(acc);
    free(a);
    free(is_active);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Routing: inc/gating.hpp                                                  */

/* inc/gating.hpp:107-125.  gate lists in CSR form: ids[off[n] .. off[n+1]).
 * Restates validate(GateSet) (:33-43) too.                                 */
int orc_proxy_scores(const float* act, size_t n_act, uint32_t n_sub, uint32_t r,
                     const uint32_t* off, const uint32_t* ids, double* scores) {
    if (n_sub < 1 || r < 1) return fail(ORC_VALIDATION, "gate set shape is inconsistent");
    for (uint32_t n = 0; n < n_sub; ++n) {
        if (off[n + 1] <= off[n]) return fail(ORC_VALIDATION, "every sub-expert needs at least one gate neuron");
        for (uint32_t q = off[n] + 1; q < off[n + 1]; ++q)
            if (ids[q] < ids[q - 1]) return fail(ORC_VALIDATION, "gate neuron lists must be ascending");
    }
    for (uint32_t n = 0; n < n_sub; ++n) {
        double sum = 0.0;
        for (uint32_t q = off[n]; q < off[n + 1]; ++q) {
            if (ids[q] >= n_act)
                return fail(ORC_VALIDATION, "gate neuron %u out of range for activation vector of length %zu", ids[q], n_act);
            sum += act[ids[q]];
        }
        scores[n] = sum / (double)(off[n + 1] - off[n]);
    }
    return ORC_OK;
}

/* Total order of inc/gating.hpp:138-141: score descending, index ascending. */
static const double* g_sort_scores;
static int by_score_desc(const void* pa, const void* pb) {
    uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
    double sa = g_sort_scores[a], sb = g_sort_scores[b];
    if (sa != sb) return sa > sb ? -1 : 1;
    return a < b ? -1 : (a > b);
}
static int by_u32(const void* pa, const void* pb) {
    uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
    return a < b ? -1 : (a > b);
}

/* Rank-order all n indices (insertion sort: thread safe, n <= a few hundred). */
static void rank_order(const double* scores, size_t n, uint32_t* order) {
    for (size_t i = 0; i < n; ++i) {
        uint32_t v = (uint32_t)i;
        size_t p = i;
        while (p > 0) {
            uint32_t u = order[p - 1];
            int before = scores[v] > scores[u] || (scores[v] == scores[u] && v < u);
            if (!before) break;
            order[p] = u;
            --p;
        }
        order[p] = v;
    }
}

/* inc/gating.hpp:129-145.  gap (optional): score(k-th) - score((k+1)-th) of
 * the total order, +inf when k == n; the near-tie measure of SURVEY 8(c).  */
int orc_select_topk(const double* scores, size_t n, uint32_t k, uint32_t* out, double* gap) {
    if (k < 1 || k > n) return fail(ORC_VALIDATION, "k_active = %u out of range [1, %zu]", k, n);
    uint32_t* order = (uint32_t*)malloc(n * sizeof(uint32_t));
    rank_order(scores, n, order);
    if (gap) *gap = (k < n) ? scores[order[k - 1]] - scores[order[k]] : INFINITY;
    memcpy(out, order, k * sizeof(uint32_t));
    qsort(out, k, sizeof(uint32_t), by_u32);
    free(order);
    return ORC_OK;
}
/* qsort-based variant kept for the single-threaded KAT path. */
int orc_select_topk_qsort(const double* scores, size_t n, uint32_t k, uint32_t* out) {
    if (k < 1 || k > n) return fail(ORC_VALIDATION, "k_active = %u out of range [1, %zu]", k, n);
    uint32_t* order = (uint32_t*)malloc(n * sizeof(uint32_t));
    for (size_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
    g_sort_scores = scores;
    qsort(order, n, sizeof(uint32_t), by_score_desc);
    memcpy(out, order, k * sizeof(uint32_t));
    qsort(out, k, sizeof(uint32_t), by_u32);
    free(order);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Layer composition (no reference code; SURVEY 8(c) restatement).          */

/* logits[t][g] = sum_i double(x[t][i]) * double(wr[i][g]), i ascending,
 * the accumulation rule of inc/expert.hpp:64-71 applied to the router.     */
int orc_router_logits(size_t T, size_t d, size_t G, const float* x, const float* wr, double* logits) {
    for (size_t t = 0; t < T; ++t) {
        double* l = logits + t * G;
        for (size_t g = 0; g < G; ++g) l[g] = 0.0;
        const float* xt = x + t * d;
        for (size_t i = 0; i < d; ++i) {
            const double xi = xt[i];
            const float* w = wr + i * G;
            for (size_t g = 0; g < G; ++g) l[g] += xi * (double)w[g];
        }
    }
    return ORC_OK;
}

/* Per token: sel = select_topk_subexperts(logits_t, k_t) (ascending ids);
 * mode 0 ("unit"):   w = 1 (the reference's unweighted sum);
 * mode 1 ("softmax_renorm"): p = softmax(logits_t) in double,
 *                            w_g = p_g / sum_{sel} p.
 * Unused slots j >= k_t hold sel = 0xFFFFFFFF, w = 0.                      */
int orc_route(size_t T, size_t G, const double* logits, const uint32_t* k_per_token, uint32_t k_scalar,
              uint32_t k_max, int mode, uint32_t* sel, float* w, double* gap) {
    uint32_t* tmp = (uint32_t*)malloc(G * sizeof(uint32_t));
    for (size_t t = 0; t < T; ++t) {
        const uint32_t k = k_per_token ? k_per_token[t] : k_scalar;
        if (k > k_max) {
            free(tmp);
            return fail(ORC_VALIDATION, "token %zu: k = %u exceeds k_max = %u", t, k, k_max);
        }
        const double* l = logits + t * G;
        int rc = orc_select_topk(l, G, k, tmp, gap ? gap + t : NULL);
        if (rc) {
            free(tmp);
            return rc;
        }
        double mx = l[0];
        for (size_t g = 1; g < G; ++g)
            if (l[g] > mx) mx = l[g];
        double z = 0.0;
        for (uint32_t j = 0; j < k; ++j) z += exp(l[tmp[j]] - mx);
        for (uint32_t j = 0; j < k_max; ++j) {
            sel[t * k_max + j] = j < k ? tmp[j] : 0xFFFFFFFFu;
            w[t * k_max + j] = j < k ? (mode == 1 ? (float)(exp(l[tmp[j]] - mx) / z) : 1.0f) : 0.0f;
        }
    }
    free(tmp);
    return ORC_OK;
}

/* Bucketing: counts[g] = #(t, j) with sel = g; offsets =
 * exclusive scan (G+1 entries); inside bucket g entries are ordered by
 * ascending token.  perm_tok[pos] = t, slot_row[t][j] = pos.               */
int orc_bucket(size_t T, size_t G, uint32_t k_max, const uint32_t* sel, uint32_t* counts,
               uint32_t* offsets, uint32_t* perm_tok, uint32_t* slot_row) {
    memset(counts, 0, G * sizeof(uint32_t));
    for (size_t t = 0; t < T; ++t)
        for (uint32_t j = 0; j < k_max; ++j) {
            uint32_t g = sel[t * k_max + j];
            if (g == 0xFFFFFFFFu) continue;
            if (g >= G) return fail(ORC_VALIDATION, "token %zu selects sub-expert %u >= %zu", t, g, G);
            ++counts[g];
        }
    offsets[0] = 0;
    for (size_t g = 0; g < G; ++g) offsets[g + 1] = offsets[g] + counts[g];
    uint32_t* cursor = (uint32_t*)malloc(G * sizeof(uint32_t));
    memcpy(cursor, offsets, G * sizeof(uint32_t));
    for (size_t t = 0; t < T; ++t)
        for (uint32_t j = 0; j < k_max; ++j) {
            uint32_t g = sel[t * k_max + j];
            if (slot_row) slot_row[t * k_max + j] = 0xFFFFFFFFu;
            if (g == 0xFFFFFFFFu) continue;
            uint32_t pos = cursor[g]++;
            if (perm_tok) perm_tok[pos] = (uint32_t)t;
            if (slot_row) slot_row[t * k_max + j] = pos;
        }
    free(cursor);
    return ORC_OK;
}

/* Layer forward given a routing (sel, w).  Sub-expert g = e * S + s.
 *   weight_mode 1: y_t = float( sum_{g in sel_t ascending} double(w) *
 *                              double(partitioned_forward(e, p_e, x_t, {s})) )
 *   weight_mode 0: y_t = float( sum_{e ascending} double(
 *                              partitioned_forward(e, p_e, x_t, active_e(t))) )
 *                  i.e. one reference call per parent expert with all of its
 *                  selected sub-experts active (the reference semantics).
 * partitioned_forward is evaluated through its definition: the activation of
 * neuron j depends only on column j, and the down accumulation visits the
 * active neurons in ascending j, so restricting the work to the members of
 * the active sub-experts is bit-identical to inc/expert.hpp:101-135.
 * layout 0: wg/wu per expert are MPEX row-major d x ff; layout 1: neuron-
 * major ff x d (same numbers, contiguous per neuron).                      */
typedef struct {
    size_t E, S, d, ff, T;
    uint32_t k_max;
    int weight_mode, layout;
    const float* const* wg;
    const float* const* wu;
    const float* const* wd;
    const uint32_t* const* assignment;
    const float* x;
    const uint32_t* sel;
    const float* w;
    float* y;
    size_t t0, t1;
} layer_job;

static void* layer_worker(void* arg) {
    layer_job* jb = (layer_job*)arg;
    const size_t d = jb->d, ff = jb->ff, S = jb->S, E = jb->E;
    double* yacc = (double*)malloc(d * sizeof(double));
    double* pacc = (double*)malloc(d * sizeof(double));
    uint8_t* act = (uint8_t*)malloc(S);
    for (size_t t = jb->t0; t < jb->t1; ++t) {
        const float* xt = jb->x + t * d;
        for (size_t i = 0; i < d; ++i) yacc[i] = 0.0;
        const uint32_t* st = jb->sel + t * jb->k_max;
        const float* wt = jb->w + t * jb->k_max;
        for (size_t e = 0; e < E; ++e) {
            /* collect the active sub-experts of expert e for this token */
            size_t n_act = 0;
            memset(act, 0, S);
            for (uint32_t j = 0; j < jb->k_max; ++j)
                if (st[j] != 0xFFFFFFFFu && st[j] / S == e) {
                    act[st[j] % S] = 1;
                    ++n_act;
                }
            if (!n_act) continue;
            const uint32_t* asg = jb->assignment[e];
            /* calls: unit mode -> one call with all active; weighted -> one per s */
            for (size_t s = 0; s < S; ++s) {
                if (jb->weight_mode == 1 && !act[s]) continue;
                if (jb->weight_mode == 0 && s > 0) break;
                for (size_t i = 0; i < d; ++i) pacc[i] = 0.0;
                for (size_t j = 0; j < ff; ++j) {
                    int on = jb->weight_mode == 1 ? (asg[j] == s) : act[asg[j]];
                    if (!on) continue;
                    const float aj_f = jb->layout == 1
                                           ? neuron_activation_nm(d, jb->wg[e], jb->wu[e], xt, j)
                                           : neuron_activation_mpex(d, ff, jb->wg[e], jb->wu[e], xt, j);
                    const double aj = aj_f;
                    if (aj == 0.0) continue;
                    const float* down = jb->wd[e] + j * d;
                    for (size_t i = 0; i < d; ++i) pacc[i] += aj * (double)down[i];
                }
                double wgt = 1.0;
                if (jb->weight_mode == 1) {
                    for (uint32_t j = 0; j < jb->k_max; ++j)
                        if (st[j] == e * S + s) wgt = (double)wt[j];
                }
                for (size_t i = 0; i < d; ++i) yacc[i] += wgt * (double)(float)pacc[i];
            }
        }
        for (size_t i = 0; i < d; ++i) jb->y[t * d + i] = (float)yacc[i];
    }
    free(yacc);
    free(pacc);
    free(act);
    return NULL;
}

int orc_layer_forward(size_t E, size_t S, size_t d, size_t ff, const float* const* wg,
                      const float* const* wu, const float* const* wd, const uint32_t* const* assignment,
                      int layout, size_t T, const float* x, uint32_t k_max, const uint32_t* sel,
                      const float* w, int weight_mode, float* y, int nthreads) {
    for (size_t e = 0; e < E; ++e) {
        int rc = orc_validate_partition((uint32_t)S, ff, assignment[e]);
        if (rc) return rc;
    }
    for (size_t q = 0; q < T * k_max; ++q)
        if (sel[q] != 0xFFFFFFFFu && sel[q] >= E * S)
            return fail(ORC_VALIDATION, "selection %u out of range for %zu sub-experts", sel[q], E * S);
    if (nthreads < 1) nthreads = 1;
    if ((size_t)nthreads > T) nthreads = T ? (int)T : 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
    layer_job* jobs = (layer_job*)malloc(sizeof(layer_job) * nthreads);
    for (int q = 0; q < nthreads; ++q) {
        layer_job jb = {E, S, d, ff, T, k_max, weight_mode, layout, wg, wu, wd, assignment, x, sel, w, y,
                        T * q / nthreads, T * (q + 1) / nthreads};
        jobs[q] = jb;
        pthread_create(&th[q], NULL, layer_worker, &jobs[q]);
    }
    for (int q = 0; q < nthreads; ++q) pthread_join(th[q], NULL);
    free(th);
    free(jobs);
    return ORC_OK;
}

/* Proxy-gate router (inc/gating.hpp:107-145): scores_t[g] =
 * proxy_scores(|a_t restricted to expert e's gate neurons|, gates_e)[s], i.e.
 * the mean |activation| over the gate neurons of sub-expert s, where the
 * activation of gate neuron j is inc/expert.hpp:62-75 for that neuron.
 * gates in CSR form over the global sub-expert id g = e*S + s; ids are
 * neuron indices within expert e.                                          */
int orc_proxy_router_scores(size_t E, size_t S, size_t d, size_t ff, const float* const* wg,
                            const float* const* wu, int layout, const uint32_t* off, const uint32_t* ids,
                            size_t T, const float* x, double* scores) {
    for (size_t t = 0; t < T; ++t) {
        const float* xt = x + t * d;
        for (size_t g = 0; g < E * S; ++g) {
            size_t e = g / S;
            if (off[g + 1] <= off[g]) return fail(ORC_VALIDATION, "every sub-expert needs at least one gate neuron");
            double sum = 0.0;
            for (uint32_t q = off[g]; q < off[g + 1]; ++q) {
                if (q > off[g] && ids[q] < ids[q - 1]) return fail(ORC_VALIDATION, "gate neuron lists must be ascending");
                if (ids[q] >= ff) return fail(ORC_VALIDATION, "gate neuron %u out of range", ids[q]);
                float a = layout == 1 ? neuron_activation_nm(d, wg[e], wu[e], xt, ids[q])
                                      : neuron_activation_mpex(d, ff, wg[e], wu[e], xt, ids[q]);
                sum += fabsf(a);
            }
            scores[t * E * S + g] = sum / (double)(off[g + 1] - off[g]);
        }
    }
    return ORC_OK;
}
