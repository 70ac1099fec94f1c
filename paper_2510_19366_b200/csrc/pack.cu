// pack.cu -- load-time layout packer and data utilities.
//
// The offline refactoring engine hands over a Partition (inc/partition.hpp:
// 15-20) and MPEX weights (inc/io.hpp:210-251: w_gate/w_up d x ff row-major,
// w_down ff x d).  Neuron j owns column j of w_gate/w_up and row j of w_down
// (inc/expert.hpp:14-16), so a sub-expert is a set of neurons.  The packer
// gathers each sub-expert's members (ascending, subexpert_members
// inc/partition.hpp:49-55) into contiguous K-major blocks:
//   W1[g] : (2*w_pad) x d_pad, rows in blocks of 128 = 64 gate rows then the
//           64 up rows of the same neurons (kIlv; fused SwiGLU epilogue),
//   W2[g] : d_pad x w_pad (K = neurons contiguous),
// zero padded: a zero neuron contributes SiLU(0)*0*W_down = 0 exactly.
#include "mp_common.cuh"
#include "mp_kernels.h"

namespace mp {

namespace {

template <typename Tw>
__global__ void pack_w1_kernel(const float* __restrict__ wg, const float* __restrict__ wu, uint32_t d, uint32_t ff,
                               const int32_t* __restrict__ nmap, uint32_t w_pad, uint32_t d_pad,
                               Tw* __restrict__ W1) {
    // block: 32 rows (r) x 32 columns (i) of one sub-expert s
    __shared__ float tile[32][33];
    const uint32_t s = blockIdx.z;
    const uint32_t r0 = blockIdx.y * 32, i0 = blockIdx.x * 32;
    const uint32_t tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    const uint32_t rows = 2 * w_pad;
    // read: thread (ty -> i, tx -> r), row i of w_gate / w_up at column j(r)
    for (uint32_t q = ty; q < 32; q += 8) {
        const uint32_t i = i0 + q, r = r0 + tx;
        float v = 0.0f;
        if (i < d && r < rows) {
            const uint32_t blk = r / (2 * kIlv), within = r % (2 * kIlv);
            const uint32_t c = blk * kIlv + (within % kIlv);
            const int32_t j = nmap[(size_t)s * w_pad + c];
            if (j >= 0) v = (within < kIlv ? wg : wu)[(size_t)i * ff + j];
        }
        tile[tx][q] = v;
    }
    __syncthreads();
    // write: thread (ty -> r, tx -> i), coalesced along i
    for (uint32_t q = ty; q < 32; q += 8) {
        const uint32_t r = r0 + q, i = i0 + tx;
        if (r < rows && i < d_pad) W1[((size_t)s * rows + r) * d_pad + i] = from_f32<Tw>(tile[q][tx]);
    }
}

template <typename Tw>
__global__ void pack_w2_kernel(const float* __restrict__ wd, uint32_t d, const int32_t* __restrict__ nmap,
                               uint32_t w_pad, uint32_t d_pad, Tw* __restrict__ W2) {
    // block: 32 neurons (c) x 32 outputs (i) of one sub-expert s
    __shared__ float tile[32][33];
    const uint32_t s = blockIdx.z;
    const uint32_t c0 = blockIdx.y * 32, i0 = blockIdx.x * 32;
    const uint32_t tx = threadIdx.x, ty = threadIdx.y;
    for (uint32_t q = ty; q < 32; q += 8) {  // read rows j(c) of w_down, coalesced along i
        const uint32_t c = c0 + q, i = i0 + tx;
        float v = 0.0f;
        if (c < w_pad && i < d) {
            const int32_t j = nmap[(size_t)s * w_pad + c];
            if (j >= 0) v = wd[(size_t)j * d + i];
        }
        tile[q][tx] = v;
    }
    __syncthreads();
    for (uint32_t q = ty; q < 32; q += 8) {  // write W2[s][i][c], coalesced along c
        const uint32_t i = i0 + q, c = c0 + tx;
        if (i < d_pad && c < w_pad) W2[((size_t)s * d_pad + i) * w_pad + c] = from_f32<Tw>(tile[tx][q]);
    }
}

__global__ void transpose_router_kernel(const float* __restrict__ wr, uint32_t d, uint32_t G, uint32_t G_pad,
                                        float* __restrict__ wrT) {
    const size_t n = (size_t)G_pad * d;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
        const uint32_t g = q / d, i = q % d;
        wrT[q] = g < G ? wr[(size_t)i * G + g] : 0.0f;
    }
}

// Gate-neuron rows for the proxy router: gate_rows[n][i] = w_gate[i][j_n].
__global__ void pack_gate_rows_kernel(const float* __restrict__ wg, const float* __restrict__ wu, uint32_t d,
                                      uint32_t ff, const uint32_t* __restrict__ neurons, uint32_t n,
                                      float* __restrict__ gate_rows, float* __restrict__ up_rows) {
    const size_t tot = (size_t)n * d;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < tot; q += (size_t)gridDim.x * blockDim.x) {
        const uint32_t r = q / d, i = q % d;
        const uint32_t j = neurons[r];
        gate_rows[q] = wg[(size_t)i * ff + j];
        up_rows[q] = wu[(size_t)i * ff + j];
    }
}

__global__ void finite_check_kernel(const float* __restrict__ p, size_t n, int* __restrict__ flag) {
    bool bad = false;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x)
        bad |= !isfinite(p[q]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

__global__ void absmax_kernel(const float* __restrict__ p, size_t n, float* __restrict__ out) {
    float m = 0.0f;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x)
        m = fmaxf(m, fabsf(p[q]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    // non-negative floats order like their bit patterns
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned int*>(out), __float_as_uint(m));
}

// Counter-based generator, bit-identical to orc_synth_fill (oracle/moe_oracle.c).
__device__ __forceinline__ uint64_t sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

template <typename T>
__global__ void synth_fill_kernel(T* __restrict__ dst, size_t n, uint64_t state, uint64_t first, double scale) {
    const uint64_t G = 0x9E3779B97F4A7C15ULL;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x) {
        const uint64_t z = sm_mix(state + (first + j + 1) * G);
        const double u = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
        const double v = __dmul_rn(__dsub_rn(__dmul_rn(u, 2.0), 1.0), scale);
        dst[j] = from_f32<T>(__double2float_rn(v));
    }
}

// state = mix(seed + G): the stream origin of orc_synth_state.
uint64_t sm_mix_host(uint64_t seed) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

}  // namespace

void launch_pack_w1(int dtype, const float* wg, const float* wu, uint32_t d, uint32_t ff, const int32_t* nmap,
                    uint32_t S, uint32_t w_pad, uint32_t d_pad, void* W1_e, cudaStream_t s) {
    const dim3 grid((d_pad + 31) / 32, (2 * w_pad + 31) / 32, S), block(32, 8);
    if (dtype == 1)
        pack_w1_kernel<__nv_bfloat16><<<grid, block, 0, s>>>(wg, wu, d, ff, nmap, w_pad, d_pad,
                                                             static_cast<__nv_bfloat16*>(W1_e));
    else
        pack_w1_kernel<float><<<grid, block, 0, s>>>(wg, wu, d, ff, nmap, w_pad, d_pad, static_cast<float*>(W1_e));
}

void launch_pack_w2(int dtype, const float* wd, uint32_t d, uint32_t ff, const int32_t* nmap, uint32_t S,
                    uint32_t w_pad, uint32_t d_pad, void* W2_e, cudaStream_t s) {
    (void)ff;
    const dim3 grid((d_pad + 31) / 32, (w_pad + 31) / 32, S), block(32, 8);
    if (dtype == 1)
        pack_w2_kernel<__nv_bfloat16><<<grid, block, 0, s>>>(wd, d, nmap, w_pad, d_pad,
                                                             static_cast<__nv_bfloat16*>(W2_e));
    else
        pack_w2_kernel<float><<<grid, block, 0, s>>>(wd, d, nmap, w_pad, d_pad, static_cast<float*>(W2_e));
}

void launch_transpose_router(const float* wr, uint32_t d, uint32_t G, uint32_t G_pad, float* wrT, cudaStream_t s) {
    transpose_router_kernel<<<592, 256, 0, s>>>(wr, d, G, G_pad, wrT);
}

void launch_pack_gate_rows(const float* wg, const float* wu, uint32_t d, uint32_t ff, const uint32_t* neurons,
                           uint32_t n, float* gate_rows, float* up_rows, cudaStream_t s) {
    pack_gate_rows_kernel<<<592, 256, 0, s>>>(wg, wu, d, ff, neurons, n, gate_rows, up_rows);
}

void launch_finite_check(const float* p, size_t n, int* flag, cudaStream_t s) {
    finite_check_kernel<<<1184, 256, 0, s>>>(p, n, flag);
}

__global__ void l2_prefetch_kernel(const char* __restrict__ p, size_t bytes) {
    constexpr size_t kChunk = 32768;
    for (size_t off = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * kChunk; off < bytes;
         off += (size_t)gridDim.x * blockDim.x * kChunk) {
        const uint32_t n = static_cast<uint32_t>(bytes - off < kChunk ? bytes - off : kChunk) & ~15u;
        if (n)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(p + off)), "r"(n)
                         : "memory");
    }
}

void launch_l2_prefetch(const void* p, size_t bytes, cudaStream_t s) {
    l2_prefetch_kernel<<<16, 128, 0, s>>>(static_cast<const char*>(p), bytes);
}

void launch_absmax(const float* p, size_t n, float* out, cudaStream_t s) {
    absmax_kernel<<<592, 256, 0, s>>>(p, n, out);
}

void launch_synth_fill(void* dst, int dtype, size_t n, uint64_t seed, uint64_t first, double scale, cudaStream_t s) {
    const uint64_t state = sm_mix_host(seed);
    if (dtype == 1)
        synth_fill_kernel<__nv_bfloat16><<<1184, 256, 0, s>>>(static_cast<__nv_bfloat16*>(dst), n, state, first, scale);
    else
        synth_fill_kernel<float><<<1184, 256, 0, s>>>(static_cast<float*>(dst), n, state, first, scale);
}

}  // namespace mp
