// proxy.cu -- the reference's training-free proxy-gate router ("CG"),
// per token, the activations of the E*S*r gate neurons
// (inc/expert.hpp:62-75 restricted to those neurons), then proxy_scores
// (inc/gating.hpp:107-125): score_g = sum_{n in gates_g} |a_n| / |gates_g| in
// double, and select_topk_subexperts (inc/gating.hpp:129-145) over them.
//
// Two paths, both certified:
//  * exact (fp32 layers, bf16 layers the tensor-core router cannot take):
//    proxy_exact_act_kernel accumulates every gate / up dot product in fp64,
//    one thread per (token, gate neuron), i ascending -- the reference's own
//    arithmetic (the fp32 x fp32 products are exact in fp64, so FMA == its
//    multiply-then-add) -- then the reference's float rounding of a_n, the
//    double mean, and the top-k;
//  * tensor core (bf16 layers, Mixtral / Qwen serving shapes): the gate and
//    up columns of the gate neurons are one [2 NR x d] matrix split into three
//    bf16 planes and run through the linear router's tcgen05 kernel
//    (router_tc.cu, fp32 partials per K split); proxy_topk_kernel forms the
//    scores with a per-neuron error bound propagated through SiLU, the
//    product and the float rounding, certifies each token's selection
//    (k-th/(k+1)-th gap > 2 guard + 1e-6) and queues the rest;
//    proxy_fixup_kernel recomputes the uncertain window's gate neurons in
//    fp64 and re-selects (+inf above the window, exact in it, -inf below).
#include <cfloat>

#include "mp_common.cuh"
#include "mp_kernels.h"
#include "mp_topk.cuh"

namespace mp {

namespace {

// ---------------------------------------------------------------- exact path
// CTA = 32 tokens (lanes) x 32 gate neurons (warps); K staged in smem chunks.
constexpr uint32_t XT = 32, XR = 32, XK = 32;
constexpr uint32_t kMaxItems = 1024;  // gate neurons per exact batch of the fixup

template <typename Tx>
__global__ void __launch_bounds__(1024) proxy_exact_act_kernel(const Tx* __restrict__ x, uint32_t T, uint32_t d,
                                                               const float* __restrict__ gate_rows,
                                                               const float* __restrict__ up_rows, uint32_t NR,
                                                               float* __restrict__ act) {
    __shared__ double xs[XK][XT + 1];
    __shared__ float gs[XR][XK + 1], us[XR][XK + 1];
    const uint32_t lane = threadIdx.x % 32, warp = threadIdx.x / 32;
    const uint32_t t0 = blockIdx.x * XT, r0 = blockIdx.y * XR;
    double g = 0.0, u = 0.0;
    for (uint32_t k0 = 0; k0 < d; k0 += XK) {
        __syncthreads();
        {
            const uint32_t tt = warp, kk = lane;  // 32 x 32 tiles, one element per thread
            xs[kk][tt] = (t0 + tt < T && k0 + kk < d) ? static_cast<double>(to_f32(x[(size_t)(t0 + tt) * d + k0 + kk]))
                                                      : 0.0;
            const bool ok = r0 + tt < NR && k0 + kk < d;
            gs[tt][kk] = ok ? gate_rows[(size_t)(r0 + tt) * d + k0 + kk] : 0.0f;
            us[tt][kk] = ok ? up_rows[(size_t)(r0 + tt) * d + k0 + kk] : 0.0f;
        }
        __syncthreads();
        const uint32_t kn = min(XK, d - k0);
        for (uint32_t kk = 0; kk < kn; ++kk) {  // i ascending: the reference's order
            const double xv = xs[kk][lane];
            g = fma(xv, static_cast<double>(gs[warp][kk]), g);
            u = fma(xv, static_cast<double>(us[warp][kk]), u);
        }
    }
    const uint32_t t = t0 + lane, r = r0 + warp;
    if (t < T && r < NR) act[(size_t)t * NR + r] = fabsf(static_cast<float>(g / (1.0 + exp(-g)) * u));
}

// score[t][g] = (sum_{r in gates_g, ascending} act[t][r]) / |gates_g| (double)
__global__ void __launch_bounds__(256) proxy_reduce_kernel(const float* __restrict__ act, uint32_t T, uint32_t NR,
                                                           const uint32_t* __restrict__ off, uint32_t G,
                                                           double* __restrict__ scores) {
    const size_t n = (size_t)T * G;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
        const uint32_t t = q / G, g = q % G;
        double sum = 0.0;
        for (uint32_t r = off[g]; r < off[g + 1]; ++r) sum += act[(size_t)t * NR + r];
        scores[q] = sum / static_cast<double>(off[g + 1] - off[g]);
    }
}

// ---------------------------------------------------------------- tensor-core path
// |SiLU(G) U - SiLU(G*) U*| with |G - G*|, |U - U*| <= e (|SiLU'| <= 1.0999),
// plus the float rounding of both values: an upper bound on the error of |a|.
__device__ __forceinline__ void proxy_neuron(double Gv, double Uv, double e, float& af, float& ea) {
    const double sg = Gv / (1.0 + exp(-Gv));
    const double a = sg * Uv;
    const double pre = 1.1 * e * (fabs(Uv) + e) + (fabs(sg) + 1.1 * e) * e;
    af = fabsf(static_cast<float>(a));
    // rn() is monotone: |rn(a) - rn(a*)| <= |a - a*| + ulp(max); 1 + 1e-6 covers the fp64
    // arithmetic here and the float rounding of the bound itself
    ea = static_cast<float>((pre + 0x1.0p-23 * (fabs(a) + pre)) * (1.0 + 1e-6) + 1e-30);
}

// Warp per token (8 per CTA).  partial: fp32 [ks][T][Npad] with the gate
// columns at [0, NR) and the up columns at [NR, 2 NR).  Scores of all G
// sub-experts to pscore [T][G]; certified tokens get their selection here,
// the others go to flagged[2 ..] with (a, b, guard) in pwin [T][3].
template <int NC>
__global__ void __launch_bounds__(256) proxy_topk_kernel(const float* __restrict__ partial, uint32_t ks, uint32_t T,
                                                         uint32_t NR, uint32_t Npad, const uint32_t* __restrict__ off,
                                                         uint32_t G, uint32_t k_max, const uint32_t* __restrict__ kpt,
                                                         uint32_t k_scalar, int weight_mode, uint32_t* __restrict__ sel,
                                                         float* __restrict__ wout, int* __restrict__ err,
                                                         RouterGuard rg, double* __restrict__ pscore,
                                                         double* __restrict__ pwin, uint32_t* __restrict__ flagged) {
    extern __shared__ __align__(16) unsigned char psm[];
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    float2* ae = reinterpret_cast<float2*>(psm) + (size_t)warp * NR;  // [NR] (|a|, error bound)
    double* sc = reinterpret_cast<double*>(psm + sizeof(float2) * 8 * NR) + (size_t)warp * G;
    const uint32_t t = blockIdx.x * 8 + warp;
    griddep_wait();
    griddep_launch();
    if (t >= T) return;
    double xn = 0.0;
    for (uint32_t s = lane; s < rg.ks; s += 32) xn += rg.xnorm[(size_t)s * T + t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xn += __shfl_xor_sync(0xffffffffu, xn, o);
    const double e = rg.coef * xn + rg.floor_abs;
    for (uint32_t n = lane; n < NR; n += 32) {
        double Gv = 0.0, Uv = 0.0;
        for (uint32_t s = 0; s < ks; ++s) {
            const float* row = partial + ((size_t)s * T + t) * Npad;
            Gv += static_cast<double>(__ldcg(row + n));
            Uv += static_cast<double>(__ldcg(row + NR + n));
        }
        float af, ea;
        proxy_neuron(Gv, Uv, e, af, ea);
        ae[n] = make_float2(af, ea);
    }
    __syncwarp();
    double guard = 0.0;
    for (uint32_t g = lane; g < G; g += 32) {
        double sum = 0.0, esum = 0.0;
        for (uint32_t r = off[g]; r < off[g + 1]; ++r) {
            sum += static_cast<double>(ae[r].x);
            esum += static_cast<double>(ae[r].y);
        }
        const double cnt = static_cast<double>(off[g + 1] - off[g]);
        sc[g] = sum / cnt;
        pscore[(size_t)t * G + g] = sum / cnt;
        guard = fmax(guard, esum / cnt * (1.0 + 1e-9));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) guard = fmax(guard, __shfl_xor_sync(0xffffffffu, guard, o));
    if (!isfinite(guard)) guard = 0.0;  // non-finite input: raised by the dispatch scan
    __syncwarp();
    const uint32_t kt = token_k(kpt, k_scalar, t, k_max, G, err);
    double vk[2];
    const double gap = warp_topk_token<NC>(sc, G, kt, k_max, weight_mode, sel + (size_t)t * k_max,
                                           wout + (size_t)t * k_max, nullptr, vk);
    const double a = __shfl_sync(0xffffffffu, vk[0], 0), b = __shfl_sync(0xffffffffu, vk[1], 0);
    if (gap < 2.0 * guard + kNearTie && lane == 0) {
        flagged[2 + atomicAdd(&flagged[0], 1u)] = t;
        pwin[(size_t)t * 3 + 0] = a;
        pwin[(size_t)t * 3 + 1] = b;
        pwin[(size_t)t * 3 + 2] = guard;
    }
}

// CTA per flagged token: the gate neurons of every sub-expert in the
// uncertainty window recomputed in fp64 (warp per neuron, x row staged in
// smem), the window's exact scores, and the re-selection.
template <typename Tx>
__global__ void __launch_bounds__(1024) proxy_fixup_kernel(const Tx* __restrict__ x, uint32_t d,
                                                           const float* __restrict__ gate_rows,
                                                           const float* __restrict__ up_rows,
                                                           const uint32_t* __restrict__ off, uint32_t G,
                                                           uint32_t k_max, const uint32_t* __restrict__ kpt,
                                                           uint32_t k_scalar, int weight_mode,
                                                           uint32_t* __restrict__ sel, float* __restrict__ wout,
                                                           int* __restrict__ err, const double* __restrict__ pscore,
                                                           const double* __restrict__ pwin,
                                                           uint32_t* __restrict__ flagged) {
    extern __shared__ double xs_d[];  // [d]
    __shared__ double sc[kMaxG], key[kMaxG];
    __shared__ uint32_t wlist[kMaxG], gstart[kMaxG];
    __shared__ uint32_t items[kMaxItems];
    __shared__ float iact[kMaxItems];
    __shared__ uint32_t n_w, b1_s, n_items;
    const uint32_t n = flagged[0];
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (uint32_t f = blockIdx.x; f < n; f += gridDim.x) {
        const uint32_t t = flagged[2 + f];
        const double a = pwin[(size_t)t * 3], b = pwin[(size_t)t * 3 + 1], gd = pwin[(size_t)t * 3 + 2];
        if (threadIdx.x == 0) n_w = 0;
        for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) xs_d[i] = static_cast<double>(to_f32(x[(size_t)t * d + i]));
        __syncthreads();
        for (uint32_t g = threadIdx.x; g < G; g += blockDim.x) {
            const double v = pscore[(size_t)t * G + g];
            sc[g] = v;
            const bool in_w = v >= b - 2.0 * gd && v <= a + 2.0 * gd;
            key[g] = v > a + 2.0 * gd ? DBL_MAX : (in_w ? v : -DBL_MAX);
            if (in_w) wlist[atomicAdd(&n_w, 1u)] = g;
        }
        __syncthreads();
        // the window's gate neurons in batches of <= kMaxItems (pack_gates caps a
        // sub-expert's gate list at kMaxItems for this path)
        for (uint32_t b0 = 0; b0 < n_w;) {
            if (threadIdx.x == 0) {
                uint32_t b1 = b0, m = 0;
                while (b1 < n_w && m + (off[wlist[b1] + 1] - off[wlist[b1]]) <= kMaxItems) {
                    gstart[b1] = m;
                    for (uint32_t r = off[wlist[b1]]; r < off[wlist[b1] + 1]; ++r) items[m++] = r;
                    ++b1;
                }
                b1_s = b1;
                n_items = m;
            }
            __syncthreads();
            const uint32_t b1 = b1_s, ni = n_items;
            for (uint32_t it = warp; it < ni; it += blockDim.x / 32) {
                const uint32_t r = items[it];
                const float* gw = gate_rows + (size_t)r * d;
                const float* uw = up_rows + (size_t)r * d;
                double ag[4] = {0, 0, 0, 0}, au[4] = {0, 0, 0, 0};
                uint32_t i = lane;
                for (; i + 96 < d; i += 128) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        ag[q] = fma(xs_d[i + 32 * q], static_cast<double>(__ldg(gw + i + 32 * q)), ag[q]);
                        au[q] = fma(xs_d[i + 32 * q], static_cast<double>(__ldg(uw + i + 32 * q)), au[q]);
                    }
                }
                for (; i < d; i += 32) {
                    ag[0] = fma(xs_d[i], static_cast<double>(__ldg(gw + i)), ag[0]);
                    au[0] = fma(xs_d[i], static_cast<double>(__ldg(uw + i)), au[0]);
                }
                double Gv = (ag[0] + ag[1]) + (ag[2] + ag[3]), Uv = (au[0] + au[1]) + (au[2] + au[3]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    Gv += __shfl_xor_sync(0xffffffffu, Gv, o);
                    Uv += __shfl_xor_sync(0xffffffffu, Uv, o);
                }
                if (lane == 0) iact[it] = fabsf(static_cast<float>(Gv / (1.0 + exp(-Gv)) * Uv));
            }
            __syncthreads();
            // exact scores of this batch: gate neurons in ascending order (inc/gating.hpp:114-123)
            for (uint32_t q = b0 + threadIdx.x; q < b1; q += blockDim.x) {
                const uint32_t g = wlist[q], cnt = off[g + 1] - off[g];
                double sum = 0.0;
                for (uint32_t r = 0; r < cnt; ++r) sum += static_cast<double>(iact[gstart[q] + r]);
                sc[g] = key[g] = sum / static_cast<double>(cnt);
            }
            __syncthreads();
            b0 = b1;
        }
        if (warp == 0) {
            const uint32_t kt = token_k(kpt, k_scalar, t, k_max, G, err);
            // the k-th / (k+1)-th keys both lie in the window: the gap is exact
            const double egap = warp_topk_token<kMaxG / 32>(sc, G, kt, k_max, weight_mode, sel + (size_t)t * k_max,
                                                            wout + (size_t)t * k_max, key);
            if (lane == 0 && egap < kNearTie) atomicAdd(&flagged[1], 1u);
        }
        __syncthreads();
    }
}

}  // namespace

// Top-k over exact double scores [T][G] with the near-tie count (stats[1]).
void launch_router_scores_topk(const float* scores, uint32_t T, uint32_t G, uint32_t k_max, const uint32_t* kpt,
                               uint32_t k, int weight_mode, uint32_t* sel, float* w, int* err, uint32_t* stats,
                               cudaStream_t s);

void launch_proxy_scores(int dtype, const void* x, uint32_t T, uint32_t d, const float* gate_w, const float* up_w,
                         const uint32_t* gate_off, uint32_t NR, uint32_t G, float* scores_buf, cudaStream_t s) {
    // scores_buf holds [T][G] doubles followed by the [T][NR] activation scratch
    double* scores = reinterpret_cast<double*>(scores_buf);
    float* act = reinterpret_cast<float*>(scores + (size_t)T * G);
    const dim3 grid((T + XT - 1) / XT, (NR + XR - 1) / XR);
    if (dtype == 1)
        proxy_exact_act_kernel<__nv_bfloat16><<<grid, 1024, 0, s>>>(static_cast<const __nv_bfloat16*>(x), T, d,
                                                                   gate_w, up_w, NR, act);
    else
        proxy_exact_act_kernel<float><<<grid, 1024, 0, s>>>(static_cast<const float*>(x), T, d, gate_w, up_w, NR, act);
    proxy_reduce_kernel<<<592, 256, 0, s>>>(act, T, NR, gate_off, G, scores);
}

void launch_proxy_tc_topk(const float* partial, uint32_t ks, uint32_t T, uint32_t NR, uint32_t Npad,
                          const uint32_t* gate_off, uint32_t G, uint32_t k_max, const uint32_t* kpt, uint32_t k,
                          int weight_mode, uint32_t* sel, float* w, int* err, const RouterGuard& rg, double* pscore,
                          double* pwin, uint32_t* flagged, cudaStream_t s) {
    const size_t smem = 8 * (sizeof(float2) * NR + sizeof(double) * G);
    auto go = [&](auto kern) {
        func_attr_once(reinterpret_cast<const void*>(kern), 200 * 1024);
        launch_k(kern, dim3((T + 7) / 8), dim3(256), smem, s, partial, ks, T, NR, Npad, gate_off, G, k_max, kpt, k,
                 weight_mode, sel, w, err, rg, pscore, pwin, flagged);
    };
    if (G <= 64)
        go(proxy_topk_kernel<2>);
    else if (G <= 128)
        go(proxy_topk_kernel<4>);
    else
        go(proxy_topk_kernel<8>);
}

void launch_proxy_fixup(const void* x, uint32_t d, const float* gate_w, const float* up_w, const uint32_t* gate_off,
                        uint32_t G, uint32_t k_max, const uint32_t* kpt, uint32_t k, int weight_mode, uint32_t* sel,
                        float* w, int* err, const double* pscore, const double* pwin, uint32_t* flagged, int num_sms,
                        cudaStream_t s) {
    const size_t smem = sizeof(double) * d;
    auto kern = proxy_fixup_kernel<__nv_bfloat16>;
    func_attr_once(reinterpret_cast<const void*>(kern), 200 * 1024);
    kern<<<num_sms, 1024, smem, s>>>(static_cast<const __nv_bfloat16*>(x), d, gate_w, up_w, gate_off, G, k_max, kpt,
                                     k, weight_mode, sel, w, err, pscore, pwin, flagged);
}

}  // namespace mp
