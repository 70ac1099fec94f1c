// proxy.cu -- the reference's training-free proxy-gate router ("CG"),
// per token, the activations of the E*S*r gate neurons
// (inc/expert.hpp:62-75 restricted to those neurons), then
// proxy_scores (inc/gating.hpp:107-125): score_g = sum_{n in gates_g} |a_n| /
// |gates_g| in double, and select_topk_subexperts (route.cu) over them.
// The two dot products per gate neuron use the router's accumulation scheme
// (fp32 FFMA partials over 16 inputs, fp64 across partials).
#include <cfloat>

#include "mp_common.cuh"
#include "mp_kernels.h"

namespace mp {

namespace {

constexpr uint32_t TB = 32, RB = 64, KC = 32;

template <typename Tx>
__global__ void __launch_bounds__(256) proxy_act_kernel(const Tx* __restrict__ x, uint32_t T, uint32_t d,
                                                        const float* __restrict__ gate_rows,
                                                        const float* __restrict__ up_rows, uint32_t NR,
                                                        float* __restrict__ act) {
    __shared__ float xs[KC][TB + 1];
    __shared__ __align__(16) float gs[KC][RB + 4];
    __shared__ __align__(16) float us[KC][RB + 4];
    const uint32_t tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    const uint32_t t0 = blockIdx.x * TB, r0 = blockIdx.y * RB;
    double ag[2][4] = {}, au[2][4] = {};
    float pg[2][4] = {}, pu[2][4] = {};
    for (uint32_t k0 = 0; k0 < d; k0 += KC) {
        __syncthreads();
        for (uint32_t q = tid; q < TB * KC; q += 256) {
            const uint32_t t = q / KC, kk = q % KC;
            xs[kk][t] = (t0 + t < T && k0 + kk < d) ? to_f32(x[(size_t)(t0 + t) * d + k0 + kk]) : 0.0f;
        }
        for (uint32_t q = tid; q < RB * KC; q += 256) {
            const uint32_t r = q / KC, kk = q % KC;
            const bool ok = r0 + r < NR && k0 + kk < d;
            gs[kk][r] = ok ? gate_rows[(size_t)(r0 + r) * d + k0 + kk] : 0.0f;
            us[kk][r] = ok ? up_rows[(size_t)(r0 + r) * d + k0 + kk] : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (uint32_t kk = 0; kk < KC; ++kk) {
            const float xa = xs[kk][2 * ty], xb = xs[kk][2 * ty + 1];
            const float4 g4 = *reinterpret_cast<const float4*>(&gs[kk][4 * tx]);
            const float4 u4 = *reinterpret_cast<const float4*>(&us[kk][4 * tx]);
            const float gv[4] = {g4.x, g4.y, g4.z, g4.w}, uv[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                pg[0][b] = fmaf(xa, gv[b], pg[0][b]);
                pg[1][b] = fmaf(xb, gv[b], pg[1][b]);
                pu[0][b] = fmaf(xa, uv[b], pu[0][b]);
                pu[1][b] = fmaf(xb, uv[b], pu[1][b]);
            }
            if ((kk & 15u) == 15u) {
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        ag[a][b] += (double)pg[a][b];
                        au[a][b] += (double)pu[a][b];
                        pg[a][b] = pu[a][b] = 0.0f;
                    }
            }
        }
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint32_t t = t0 + 2 * ty + a, r = r0 + 4 * tx + b;
            if (t < T && r < NR) {
                const double g = ag[a][b];
                const float av = static_cast<float>(g / (1.0 + exp(-g)) * au[a][b]);  // inc/expert.hpp:72
                act[(size_t)t * NR + r] = fabsf(av);
            }
        }
}

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

}  // namespace

void launch_proxy_scores(int dtype, const void* x, uint32_t T, uint32_t d, const float* gate_w, const float* up_w,
                         const uint32_t* gate_off, uint32_t NR, uint32_t G, float* scores_buf, cudaStream_t s) {
    // scores_buf holds [T][G] doubles followed by the [T][NR] activation scratch
    double* scores = reinterpret_cast<double*>(scores_buf);
    float* act = reinterpret_cast<float*>(scores + (size_t)T * G);
    const dim3 grid((T + TB - 1) / TB, (NR + RB - 1) / RB);
    if (dtype == 1)
        proxy_act_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x), T, d, gate_w, up_w,
                                                             NR, act);
    else
        proxy_act_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(x), T, d, gate_w, up_w, NR, act);
    proxy_reduce_kernel<<<592, 256, 0, s>>>(act, T, NR, gate_off, G, scores);
}

}  // namespace mp
