// mp_topk.cuh -- warp-level top-k selection shared by the routers (route.cu,
// proxy.cu): select_topk_subexperts (inc/gating.hpp:129-145) -- total order
// score desc / index asc, ascending output -- plus the softmax-renormalised
// weights of the selection and the k-th/(k+1)-th gap (the near-tie measure).
#pragma once

#include <cfloat>

#include "mp_common.cuh"
#include "mp_kernels.h"

namespace mp {
namespace {

constexpr double kNearTie = 1e-6;  // the routing contract's near-tie window (logit units)

// sum_i |x_i| of one bf16 row, to every lane of the warp (the input of the
// router certification bound).  16-byte loads, all of a lane's loads in
// flight when d % 8 == 0 and the row is 16-byte aligned.  fp32 partial sums
// per lane (relative error < 2^-16 at d <= 2^16, inside the bound's margin),
// fp64 across lanes.
__device__ __forceinline__ double warp_row_abs_sum(const __nv_bfloat16* __restrict__ xr, uint32_t d) {
    const uint32_t lane = lane_id();
    float s = 0.0f;
    if ((d % 8) == 0 && (reinterpret_cast<uintptr_t>(xr) & 15u) == 0) {
        for (uint32_t c = lane * 8; c < d; c += 256) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(xr + c));
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int h = 0; h < 4; ++h)
                s += fabsf(__uint_as_float(w[h] << 16)) + fabsf(__uint_as_float(w[h] & 0xFFFF0000u));
        }
    } else {
        for (uint32_t c = lane; c < d; c += 32) s += fabsf(__bfloat162float(xr[c]));
    }
    double r = static_cast<double>(s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    return r;
}

// ---------------------------------------------------------------- top-k
// One warp selects the k_t best of G scores for one token (score desc,
// index asc -- inc/gating.hpp:138-141), emits them in ascending index order
// (inc/gating.hpp:143) with their softmax-renormalised weights.
// Returns (to every lane) the gap between the k-th and (k+1)-th best score
// (+inf when k == G): the near-tie measure of the routing contract.
// keys (nullable): selection keys replacing sc for the ranking only (the
// exact re-selection of near-tie tokens); the weights always use sc.
// vk_out (nullable): the k-th and (k+1)-th best keys.
// msk_row / slot_row16 (nullable, shared memory): the selection as a bit mask
// over the G ids (ceil(G / 32) words, every word written) and, for each
// selected id, its slot in sel_row -- the bucketing ranks' input, without
// reading sel_row back from global memory.
// NC: 32-candidate chunks per lane held in registers (G <= 32 NC); smaller NC
// for small G trims the unrolled per-round work (Mixtral: G = 64 -> NC = 2)
template <int NC = kMaxG / 32>
__device__ double warp_topk_token(const double* __restrict__ sc, uint32_t G, uint32_t k, uint32_t k_max,
                                  int weight_mode, uint32_t* __restrict__ sel_row, float* __restrict__ w_row,
                                  const double* __restrict__ keys = nullptr, double* vk_out = nullptr,
                                  uint32_t* msk_row = nullptr, uint16_t* slot_row16 = nullptr) {
    const uint32_t lane = lane_id();
    const uint32_t nc = (G + 31) / 32;
    double v[NC];
    uint32_t taken = 0;  // bit c: value c of this lane selected
    const double* kv = keys ? keys : sc;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const uint32_t g = lane + 32u * c;
        v[c] = (c < (int)nc && g < G) ? kv[g] : -DBL_MAX;
    }
    double vmax = 0.0, vk = 0.0, vk1 = -INFINITY;
    const uint32_t rounds = k < G ? k + 1 : k;
    for (uint32_t r = 0; r < rounds; ++r) {
        double bv = -INFINITY;
        uint32_t bi = 0xFFFFFFFFu;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const uint32_t g = lane + 32u * c;
            if (c < (int)nc && g < G && !((taken >> c) & 1u) && v[c] > bv) {
                bv = v[c];
                bi = g;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (r == 0) vmax = bv;
        if (r == k) {  // the (k+1)-th best: measured, not taken
            vk1 = bv;
            break;
        }
        vk = bv;
        if (bi != 0xFFFFFFFFu && (bi & 31u) == lane) taken |= 1u << (bi >> 5);
    }
    if (vk_out && lane == 0) {
        vk_out[0] = vk;
        vk_out[1] = vk1;
    }
    if (keys) {  // weights from the logits, max over the selection (contains the top-1)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const uint32_t g = lane + 32u * c;
            v[c] = (c < (int)nc && g < G) ? sc[g] : -DBL_MAX;
        }
        double m = -DBL_MAX;
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if ((taken >> c) & 1u) m = fmax(m, v[c]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
        vmax = m;
    }
    // softmax over all G cancels in the renormalisation: w_g = e^(l_g - m) / sum_sel
    // (each exponential evaluated once)
    double z = 0.0;
    double ex[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        ex[c] = ((taken >> c) & 1u) ? exp(v[c] - vmax) : 0.0;
        z += ex[c];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
    // ascending-index emission: index order is (c, lane)
    uint32_t base = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if (c >= (int)nc) break;
        const bool mine = (taken >> c) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, mine);
        if (msk_row && lane == 0) msk_row[c] = bal;  // selection bit mask, word c = ids 32c .. 32c + 31
        if (mine) {
            const uint32_t pos = base + __popc(bal & ((1u << lane) - 1u));
            sel_row[pos] = lane + 32u * c;
            w_row[pos] = weight_mode == 1 ? static_cast<float>(ex[c] / z) : 1.0f;
            if (msk_row) slot_row16[lane + 32u * c] = static_cast<uint16_t>(pos);
        }
        base += __popc(bal);
    }
    for (uint32_t j = k + lane; j < k_max; j += 32) {
        sel_row[j] = kSelNone;
        w_row[j] = 0.0f;
    }
    return k < G ? vk - vk1 : INFINITY;
}

// Fast selection for the tensor-core router: keys are the fp32-rounded logits
// (rounding <= 2^-24 |logit|, inside the per-token certification guard), packed
// with the index into one order-preserving u64 (key bits high, ~index low:
// larger packed value = larger key, then lower index), so each argmax step is
// one 64-bit shuffle + max.  Weights use the fp64 logits `vals`.  Returns the
// key gap between the k-th and (k+1)-th best (+inf when k == G); vk_out gets
// both keys (as double).
__device__ __forceinline__ uint64_t pack_key(float v, uint32_t g) {
    uint32_t b = __float_as_uint(v);
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // order-preserving
    return (static_cast<uint64_t>(b) << 32) | static_cast<uint32_t>(~g);
}
__device__ __forceinline__ float unpack_key(uint64_t p) {
    uint32_t b = static_cast<uint32_t>(p >> 32);
    b = (b & 0x80000000u) ? (b & 0x7FFFFFFFu) : ~b;
    return __uint_as_float(b);
}

template <int NC = kMaxG / 32>
__device__ double warp_topk_fast(const double* __restrict__ vals, uint32_t G, uint32_t k, uint32_t k_max,
                                 int weight_mode, uint32_t* __restrict__ sel_row, float* __restrict__ w_row,
                                 double* vk_out, uint32_t* msk_row = nullptr, uint16_t* slot_row16 = nullptr) {
    const uint32_t lane = lane_id();
    const uint32_t nc = (G + 31) / 32;
    uint64_t v[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const uint32_t g = lane + 32u * c;
        v[c] = (c < (int)nc && g < G) ? pack_key(static_cast<float>(vals[g]), g) : 0ull;
    }
    uint32_t taken = 0;
    uint64_t pk = 0, pk1 = 0;
    const uint32_t rounds = k < G ? k + 1 : k;
    for (uint32_t r = 0; r < rounds; ++r) {
        uint64_t best = 0;
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if (!((taken >> c) & 1u) && v[c] > best) best = v[c];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const uint64_t o = __shfl_xor_sync(0xffffffffu, best, off);
            best = o > best ? o : best;
        }
        if (r == k) {
            pk1 = best;
            break;
        }
        pk = best;
        const uint32_t g = ~static_cast<uint32_t>(best);
        if ((g & 31u) == lane) taken |= 1u << (g >> 5);
    }
    const double vk = unpack_key(pk), vk1 = k < G ? (double)unpack_key(pk1) : -INFINITY;
    if (vk_out && lane == 0) {
        vk_out[0] = vk;
        vk_out[1] = vk1;
    }
    double m = -DBL_MAX;
#pragma unroll
    for (int c = 0; c < NC; ++c)
        if ((taken >> c) & 1u) m = fmax(m, vals[lane + 32u * c]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    double z = 0.0;
    double ex[NC];  // each exponential evaluated once
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        ex[c] = ((taken >> c) & 1u) ? exp(vals[lane + 32u * c] - m) : 0.0;
        z += ex[c];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
    uint32_t base = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if (c >= (int)nc) break;
        const bool mine = (taken >> c) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, mine);
        if (msk_row && lane == 0) msk_row[c] = bal;  // selection bit mask, word c = ids 32c .. 32c + 31
        if (mine) {
            const uint32_t pos = base + __popc(bal & ((1u << lane) - 1u));
            sel_row[pos] = lane + 32u * c;
            w_row[pos] = weight_mode == 1 ? static_cast<float>(ex[c] / z) : 1.0f;
            if (msk_row) slot_row16[lane + 32u * c] = static_cast<uint16_t>(pos);
        }
        base += __popc(bal);
    }
    for (uint32_t j = k + lane; j < k_max; j += 32) {
        sel_row[j] = kSelNone;
        w_row[j] = 0.0f;
    }
    return k < G ? vk - vk1 : INFINITY;
}

__device__ __forceinline__ uint32_t token_k(const uint32_t* kpt, uint32_t k, uint32_t t, uint32_t k_max, uint32_t G,
                                            int* err) {
    uint32_t kt = kpt ? kpt[t] : k;
    if (kt < 1 || kt > k_max || kt > G) {
        if (err) atomicOr(err, 1);
        kt = kt < 1 ? 1 : (kt > k_max ? k_max : kt);
        if (kt > G) kt = G;
    }
    return kt;
}

}  // namespace
}  // namespace mp
