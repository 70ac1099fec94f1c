// mma_cost.cu -- microbenchmark: cycles per tcgen05.mma.cta_group::1.kind::f16
// (M=128, K=16, both operands in shared memory, SW128 K-major) as a function
// of N, with one or two accumulators per k-step.  One CTA per SM, operands
// resident in smem (no TMA), throughput measured over many MMAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2510_19366_b200/csrc tests/probes/mma_cost.cu -o tests/probes/mma_cost -lcuda
#include <cstdio>
#include <vector>

#include "mp_common.cuh"

using namespace mp;

__global__ void __launch_bounds__(128, 1) mma_cost_kernel(uint32_t n, uint32_t two, uint32_t iters, uint64_t* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = base;              // 128 rows x 64 bf16 (16 KB)
    uint8_t* sB = base + 16384;      // 256 rows x 64 bf16 (32 KB)
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_slot;
    for (uint32_t i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(base)[i] = 0x3f803f80u;  // bf16 1.0
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc<512>(&tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = umma_idesc_bf16(128, n);
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        uint64_t t0 = clock64();
        for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) {
                umma_bf16(tmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc, 1);
                if (two) umma_bf16(tmem + 256, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + 16384 + k * 32),
                                   idesc, 1);
            }
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        uint64_t t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// CTA-pair variant: cta_group::2, M in {128, 256}, N = 256, one accumulator chain
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_cost_pair_kernel(uint32_t m, uint32_t two, uint32_t iters, uint64_t* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = base;
    uint8_t* sB = base + 16384;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_slot;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (uint32_t i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(base)[i] = 0x3f803f80u;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0 && rank == 0 && m == 0) {
        // mixed shapes: blocks of 112 MMAs alternating M=256 (acc 0) and M=128 (acc 256)
        const uint32_t i256 = umma_idesc_bf16(256, 256), i128 = umma_idesc_bf16(128, 256);
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        uint64_t t0 = clock64();
        for (uint32_t it = 0; it < iters / 28; ++it) {
            const uint32_t idesc = (it & 1u) ? i128 : i256;
            const uint32_t d = tmem + ((it & 1u) ? 256 : 0);
            for (uint32_t kb = 0; kb < 28; ++kb)
#pragma unroll
                for (uint32_t k = 0; k < 4; ++k)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                        "l"(umma_desc_sw128(a0 + k * 32)), "l"(umma_desc_sw128(b0 + k * 32)), "r"(idesc), "r"(1u)
                        : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"(static_cast<uint16_t>(1))
            : "memory");
        mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
    } else if (threadIdx.x == 0 && rank == 0) {
        const uint32_t idesc = umma_idesc_bf16(m, 256);
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        uint64_t t0 = clock64();
        for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) {
                const uint32_t d = tmem + ((two && (k & 1)) ? 256 : 0);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                    "l"(umma_desc_sw128(a0 + k * 32)), "l"(umma_desc_sw128(b0 + k * 32)), "r"(idesc), "r"(1u)
                    : "memory");
            }
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"(static_cast<uint16_t>(1))
            : "memory");
        mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x < 32) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// CTA-pair M=256 with N in {32..256} and 1/2/4 accumulator chains (swapped
// remainder tiles of gemm_tc2.cu): cycles per MMA, operands resident in smem
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_cost_pair_n_kernel(uint32_t n, uint32_t chains, uint32_t iters, uint64_t* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = base;
    uint8_t* sB = base + 16384;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_slot;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (uint32_t i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(base)[i] = 0x3f803f80u;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0 && rank == 0) {
        const uint32_t idesc = umma_idesc_bf16(256, n);
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        uint64_t t0 = clock64();
        uint32_t j = 0;
        for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k, ++j) {
                const uint32_t d = tmem + (j % chains) * n;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                    "l"(umma_desc_sw128(a0 + k * 32)), "l"(umma_desc_sw128(b0 + k * 32)), "r"(idesc), "r"(1u)
                    : "memory");
            }
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"(static_cast<uint16_t>(1))
            : "memory");
        mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x < 32) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint64_t* d_out;
    cudaMalloc(&d_out, sms * sizeof(uint64_t));
    const size_t smem = 1024 + 16384 + 32768;
    cudaFuncSetAttribute(mma_cost_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint32_t iters = 2000;
    printf("N,accumulators,cycles_per_mma,floor_N_over_2,flop_per_cycle_per_sm\n");
    for (uint32_t two = 0; two < 2; ++two)
        for (uint32_t n : {16u, 32u, 48u, 64u, 96u, 128u, 160u, 192u, 256u}) {
            if (two && n > 128) continue;  // second B operand at smem row 128 (256-row buffer)
            mma_cost_kernel<<<sms, 128, smem>>>(n, two, iters, d_out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            std::vector<uint64_t> h(sms);
            cudaMemcpy(h.data(), d_out, sms * 8, cudaMemcpyDeviceToHost);
            double mean = 0;
            for (auto v : h) mean += v;
            mean /= sms;
            const double n_mma = double(iters) * 4 * (two ? 2 : 1);
            const double cpm = mean / n_mma;
            printf("%u,%u,%.1f,%.1f,%.0f\n", n, two + 1, cpm, n / 2.0, 2.0 * 128 * n * 16 / cpm);
        }
    cudaFuncSetAttribute(mma_cost_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    printf("pair: M,accumulators,cycles_per_mma (N=256),floor\n");
    for (uint32_t two = 0; two < 2; ++two)
        for (uint32_t m : {128u, 256u, 0u}) {
            if (m == 0 && two) continue;
            cudaMemset(d_out, 0, sms * 8);
            mma_cost_pair_kernel<<<sms, 128, smem>>>(m, two, iters, d_out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            std::vector<uint64_t> h(sms);
            cudaMemcpy(h.data(), d_out, sms * 8, cudaMemcpyDeviceToHost);
            double mean = 0;
            int n = 0;
            for (auto v : h)
                if (v) mean += v, ++n;
            mean /= n;
            if (m == 0)  // alternating blocks: expected (128 + 64) / 2 = 96 cycles per MMA
                printf("alternating M=256/M=128 blocks,%.1f cycles per MMA (96 expected)\n",
                       mean / (double(iters / 28 * 28) * 4));
            else
                printf("%u,%u,%.1f,%.1f\n", m, two + 1, mean / (double(iters) * 4), m * 256.0 / 512);
        }
    cudaFuncSetAttribute(mma_cost_pair_n_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    printf("pair M=256: N,chains,cycles_per_mma,floor_N_over_2\n");
    for (uint32_t chains : {1u, 2u, 4u})
        for (uint32_t n : {32u, 64u, 128u, 256u}) {
            if (chains * n > 512) continue;
            cudaMemset(d_out, 0, sms * 8);
            mma_cost_pair_n_kernel<<<sms, 128, smem>>>(n, chains, iters, d_out);
            if (cudaDeviceSynchronize() != cudaSuccess) return 1;
            std::vector<uint64_t> h(sms);
            cudaMemcpy(h.data(), d_out, sms * 8, cudaMemcpyDeviceToHost);
            double mean = 0;
            int c = 0;
            for (auto v : h)
                if (v) mean += v, ++c;
            printf("%u,%u,%.1f,%.1f\n", n, chains, mean / c / (double(iters) * 4), n / 2.0);
        }
    return 0;
}
