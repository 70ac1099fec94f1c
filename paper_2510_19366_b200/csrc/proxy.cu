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
//    product and the float rounding, certifies each token's selection with
//    per-sub-expert bounds (lowest lower bound inside the top-k above the
//    highest upper bound outside, by more than the 1e-6 near-tie width) and
//    queues the rest; proxy_fixup_kernel recomputes the uncertain
//    sub-experts' gate neurons in fp64 and re-selects (+inf certainly in,
//    exact uncertain, -inf certainly out).
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
constexpr uint32_t kFixThreads = 512;

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
// columns at [0, NR) and the up columns at [NR, 2 NR).  Every sub-expert g
// gets a score s_g and an error bound e_g; the top-k of the scores is
// certified when the smallest lower bound inside it (A) exceeds the largest
// upper bound outside it (B) by more than the near-tie width: then the exact
// top-k is the same and no exact gap is < 1e-6.  Otherwise the token goes to
// flagged[2 ..] with its scores in pscore [T][G] and a class per sub-expert in
// pclass [T][G]: +1 certainly selected (lower bound > B), -1 certainly not
// (upper bound < A), 0 uncertain -- recomputed exactly by proxy_fixup_kernel.
template <int NC>
__global__ void __launch_bounds__(256) proxy_topk_kernel(const float* __restrict__ partial, uint32_t ks, uint32_t T,
                                                         uint32_t NR, uint32_t Npad, const uint32_t* __restrict__ off,
                                                         uint32_t G, uint32_t k_max, const uint32_t* __restrict__ kpt,
                                                         uint32_t k_scalar, int weight_mode, uint32_t* __restrict__ sel,
                                                         float* __restrict__ wout, int* __restrict__ err,
                                                         RouterGuard rg, const __nv_bfloat16* __restrict__ x,
                                                         uint32_t d, double* __restrict__ pscore,
                                                         int8_t* __restrict__ pclass, uint32_t* __restrict__ flagged) {
    extern __shared__ __align__(16) unsigned char psm[];
    __shared__ uint32_t selm[8][kMaxG / 32];
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    float2* ae = reinterpret_cast<float2*>(psm) + (size_t)warp * NR;  // [NR] (|a|, error bound)
    double* sc = reinterpret_cast<double*>(psm + sizeof(float2) * 8 * NR) + (size_t)warp * 2 * G;
    double* ec = sc + G;  // per sub-expert score error bound
    const uint32_t t = blockIdx.x * 8 + warp;
    griddep_wait();
    griddep_launch();
    if (t >= T) return;
    const double xn = warp_row_abs_sum(x + (size_t)t * d, d);
    double e = rg.coef * xn + rg.floor_abs;
    if (!isfinite(e)) e = 0.0;  // non-finite input: raised by the dispatch scan
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
    if (lane < kMaxG / 32) selm[warp][lane] = 0;
    __syncwarp();
    for (uint32_t g = lane; g < G; g += 32) {
        double sum = 0.0, esum = 0.0;
        for (uint32_t r = off[g]; r < off[g + 1]; ++r) {
            sum += static_cast<double>(ae[r].x);
            esum += static_cast<double>(ae[r].y);
        }
        const double cnt = static_cast<double>(off[g + 1] - off[g]);
        sc[g] = sum / cnt;
        ec[g] = esum / cnt * (1.0 + 1e-9);
    }
    __syncwarp();
    const uint32_t kt = token_k(kpt, k_scalar, t, k_max, G, err);
    uint32_t* srow = sel + (size_t)t * k_max;
    warp_topk_token<NC>(sc, G, kt, k_max, weight_mode, srow, wout + (size_t)t * k_max);
    __syncwarp();
    for (uint32_t j = lane; j < kt; j += 32) {
        const uint32_t g = srow[j];
        atomicOr(&selm[warp][g >> 5], 1u << (g & 31));
    }
    __syncwarp();
    double A = DBL_MAX, B = -DBL_MAX;  // min lower bound inside, max upper bound outside
    for (uint32_t g = lane; g < G; g += 32) {
        if ((selm[warp][g >> 5] >> (g & 31)) & 1u)
            A = fmin(A, sc[g] - ec[g]);
        else
            B = fmax(B, sc[g] + ec[g]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        A = fmin(A, __shfl_xor_sync(0xffffffffu, A, o));
        B = fmax(B, __shfl_xor_sync(0xffffffffu, B, o));
    }
    if (A - B > kNearTie) return;  // certified (k == G: B = -DBL_MAX)
    for (uint32_t g = lane; g < G; g += 32) {
        const bool in = (selm[warp][g >> 5] >> (g & 31)) & 1u;
        pscore[(size_t)t * G + g] = sc[g];
        pclass[(size_t)t * G + g] = in ? (sc[g] - ec[g] > B ? 1 : 0) : (sc[g] + ec[g] < A ? -1 : 0);
    }
    if (lane == 0) flagged[2 + atomicAdd(&flagged[0], 1u)] = t;
}

// CTA per flagged token: the gate neurons of every uncertain sub-expert
// recomputed in fp64 (warp per neuron, x row staged in smem, 16-byte weight
// loads with 16 in flight per lane), the exact scores, and the re-selection
// on (+inf certainly selected, exact uncertain, -inf certainly not).
template <typename Tx>
__global__ void __launch_bounds__(kFixThreads) proxy_fixup_kernel(const Tx* __restrict__ x, uint32_t d,
                                                                  const float* __restrict__ gate_rows,
                                                                  const float* __restrict__ up_rows,
                                                                  const uint32_t* __restrict__ off, uint32_t G,
                                                                  uint32_t k_max, const uint32_t* __restrict__ kpt,
                                                                  uint32_t k_scalar, int weight_mode,
                                                                  uint32_t* __restrict__ sel, float* __restrict__ wout,
                                                                  int* __restrict__ err,
                                                                  const double* __restrict__ pscore,
                                                                  const int8_t* __restrict__ pclass,
                                                                  uint32_t* __restrict__ flagged) {
    extern __shared__ __align__(16) double xs_d[];  // [d]
    __shared__ double sc[kMaxG], key[kMaxG];
    __shared__ uint32_t wlist[kMaxG], gstart[kMaxG];
    __shared__ uint32_t items[kMaxItems];
    __shared__ float iact[kMaxItems];
    __shared__ uint32_t n_w, b1_s, n_items;
    const uint32_t n = flagged[0];
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32, nwarps = blockDim.x / 32;
    for (uint32_t f = blockIdx.x; f < n; f += gridDim.x) {
        const uint32_t t = flagged[2 + f];
        if (threadIdx.x == 0) n_w = 0;
        for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) xs_d[i] = static_cast<double>(to_f32(x[(size_t)t * d + i]));
        __syncthreads();
        for (uint32_t g = threadIdx.x; g < G; g += blockDim.x) {
            const double v = pscore[(size_t)t * G + g];
            const int8_t c = pclass[(size_t)t * G + g];
            sc[g] = v;
            key[g] = c > 0 ? DBL_MAX : (c < 0 ? -DBL_MAX : v);
            if (c == 0) wlist[atomicAdd(&n_w, 1u)] = g;
        }
        __syncthreads();
        // the uncertain sub-experts' gate neurons in batches of <= kMaxItems
        // (pack_gates caps a sub-expert's gate list at kMaxItems for this path)
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
            for (uint32_t it = warp; it < ni; it += nwarps) {
                const uint32_t r = items[it];
                const float* gw = gate_rows + (size_t)r * d;
                const float* uw = up_rows + (size_t)r * d;
                double ag = 0.0, au = 0.0;
                if ((d % 4) == 0) {
                    // lane owns 4 consecutive inputs per 128-wide step; 8 steps in flight
                    constexpr uint32_t U = 8;
                    for (uint32_t i0 = 4 * lane; i0 < d; i0 += U * 128) {
                        float4 gv[U], uv[U];
#pragma unroll
                        for (uint32_t u = 0; u < U; ++u) {
                            const uint32_t i = i0 + u * 128;
                            gv[u] = i < d ? __ldg(reinterpret_cast<const float4*>(gw + i)) : make_float4(0, 0, 0, 0);
                            uv[u] = i < d ? __ldg(reinterpret_cast<const float4*>(uw + i)) : make_float4(0, 0, 0, 0);
                        }
#pragma unroll
                        for (uint32_t u = 0; u < U; ++u) {
                            const uint32_t i = i0 + u * 128;
                            if (i >= d) break;
                            const double* xv = xs_d + i;
                            ag = fma(xv[0], (double)gv[u].x, ag);
                            ag = fma(xv[1], (double)gv[u].y, ag);
                            ag = fma(xv[2], (double)gv[u].z, ag);
                            ag = fma(xv[3], (double)gv[u].w, ag);
                            au = fma(xv[0], (double)uv[u].x, au);
                            au = fma(xv[1], (double)uv[u].y, au);
                            au = fma(xv[2], (double)uv[u].z, au);
                            au = fma(xv[3], (double)uv[u].w, au);
                        }
                    }
                } else {
                    for (uint32_t i = lane; i < d; i += 32) {
                        ag = fma(xs_d[i], static_cast<double>(__ldg(gw + i)), ag);
                        au = fma(xs_d[i], static_cast<double>(__ldg(uw + i)), au);
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    ag += __shfl_xor_sync(0xffffffffu, ag, o);
                    au += __shfl_xor_sync(0xffffffffu, au, o);
                }
                if (lane == 0) iact[it] = fabsf(static_cast<float>(ag / (1.0 + exp(-ag)) * au));
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
            // the k-th / (k+1)-th keys both lie among the uncertain: the gap is exact
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
                          int weight_mode, uint32_t* sel, float* w, int* err, const RouterGuard& rg, const void* x,
                          uint32_t d, double* pscore, int8_t* pclass, uint32_t* flagged, cudaStream_t s) {
    const size_t smem = 8 * (sizeof(float2) * NR + 2 * sizeof(double) * G);
    auto go = [&](auto kern) {
        func_attr_once(reinterpret_cast<const void*>(kern), 200 * 1024);
        launch_k(kern, dim3((T + 7) / 8), dim3(256), smem, s, partial, ks, T, NR, Npad, gate_off, G, k_max, kpt, k,
                 weight_mode, sel, w, err, rg, static_cast<const __nv_bfloat16*>(x), d, pscore, pclass, flagged);
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
                        float* w, int* err, const double* pscore, const int8_t* pclass, uint32_t* flagged,
                        int num_sms, cudaStream_t s) {
    const size_t smem = sizeof(double) * d;
    auto kern = proxy_fixup_kernel<__nv_bfloat16>;
    func_attr_once(reinterpret_cast<const void*>(kern), 200 * 1024);
    kern<<<3 * num_sms, kFixThreads, smem, s>>>(static_cast<const __nv_bfloat16*>(x), d, gate_w, up_w, gate_off, G,
                                                k_max, kpt, k, weight_mode, sel, w, err, pscore, pclass, flagged);
}

}  // namespace mp
