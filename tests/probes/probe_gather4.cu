// probe_gather4.cu -- hardware probe (not product code): does
// cp.async.bulk.tensor.2d.tile::gather4 write four arbitrary rows into a
// 128B-swizzled smem tile exactly where a plain TMA tile load of those rows
// would put them?  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o probe probe_gather4.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tm_tile, const __grid_constant__ CUtensorMap tm_g4,
                      const int* rows, uint16_t* out_tile, uint16_t* out_g4) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* a = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
    uint8_t* b = a + 16384;
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(32768));
        // plain tile: rows 0..127 of the "gathered" source (see host)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su32(a)),
            "l"((uint64_t)&tm_tile), "r"(0), "r"(0), "r"(su32(&bar)));
        for (int q = 0; q < 32; ++q) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, "
                "{%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(b + q * 512)),
                "l"((uint64_t)&tm_g4), "r"(0), "r"(rows[4 * q]), "r"(rows[4 * q + 1]), "r"(rows[4 * q + 2]),
                "r"(rows[4 * q + 3]), "r"(su32(&bar)));
        }
    }
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(su32(&bar)));
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) {
        out_tile[i] = ((uint16_t*)a)[i];
        out_g4[i] = ((uint16_t*)b)[i];
    }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const int R = 512, C = 64;
    std::vector<uint16_t> src(R * C), gathered(128 * C);
    for (int r = 0; r < R; ++r)
        for (int c = 0; c < C; ++c) src[r * C + c] = (uint16_t)(r * 64 + c);
    std::vector<int> rows(128);
    for (int i = 0; i < 128; ++i) rows[i] = (i * 37 + 11) % R;
    for (int i = 0; i < 128; ++i)
        for (int c = 0; c < C; ++c) gathered[i * C + c] = src[rows[i] * C + c];
    uint16_t *d_src, *d_gat, *o1, *o2;
    int* d_rows;
    CK(cudaMalloc(&d_src, R * C * 2));
    CK(cudaMalloc(&d_gat, 128 * C * 2));
    CK(cudaMalloc(&o1, 16384));
    CK(cudaMalloc(&o2, 16384));
    CK(cudaMalloc(&d_rows, 128 * 4));
    CK(cudaMemcpy(d_src, src.data(), R * C * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_gat, gathered.data(), 128 * C * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_rows, rows.data(), 128 * 4, cudaMemcpyHostToDevice));
    void* fp;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
    EncFn enc = (EncFn)fp;
    CUtensorMap t1, t2;
    cuuint64_t g1[2] = {64, 128}, s1[1] = {128};
    cuuint32_t b1[2] = {64, 128}, es[2] = {1, 1};
    CUresult r1 = enc(&t1, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d_gat, g1, s1, b1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int box_rows = argc > 1 ? atoi(argv[1]) : 1;
    cuuint64_t g2[2] = {64, (cuuint64_t)R}, s2[1] = {128};
    cuuint32_t b2[2] = {64, (cuuint32_t)box_rows};
    CUresult r2 = enc(&t2, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d_src, g2, s2, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode tile=%d gather(box rows %d)=%d\n", (int)r1, box_rows, (int)r2);
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000));
    probe<<<1, 128, 40000>>>(t1, t2, d_rows, o1, o2);
    CK(cudaDeviceSynchronize());
    std::vector<uint16_t> h1(8192), h2(8192);
    CK(cudaMemcpy(h1.data(), o1, 16384, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2.data(), o2, 16384, cudaMemcpyDeviceToHost));
    int mism = 0;
    for (int i = 0; i < 8192; ++i) mism += h1[i] != h2[i];
    printf("gather4 vs tile layout mismatches: %d of 8192\n", mism);
    if (mism) {
        for (int i = 0; i < 16; ++i) printf("%d:%d/%d ", i, h1[i], h2[i]);
        printf("\n");
        for (int i = 512; i < 528; ++i) printf("%d:%d/%d ", i, h1[i], h2[i]);
        printf("\n");
    }
    return 0;
}
