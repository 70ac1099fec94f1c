// pdl_gap.cu -- per-boundary cost of dependent kernel launches on one stream:
// a chain of N short kernels (each touching a little global memory), plain
// stream order vs programmatic dependent launch (griddepcontrol.wait).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tests/probes/pdl_gap.cu -o tests/probes/pdl_gap
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step_kernel(float* buf, int n, int pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) buf[i] = buf[i] * 1.0001f + 1.0f;
}

int main() {
    const int n = 148 * 256, chain = 8, reps = 200;
    float* buf;
    cudaMalloc(&buf, n * sizeof(float));
    cudaMemset(buf, 0, n * sizeof(float));
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int pdl = 0; pdl < 2; ++pdl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl;
        for (int w = 0; w < 20; ++w) cudaLaunchKernelEx(&cfg, step_kernel, buf, n, pdl);
        cudaEventRecord(e0, s);
        for (int r = 0; r < reps; ++r)
            for (int c = 0; c < chain; ++c) cudaLaunchKernelEx(&cfg, step_kernel, buf, n, pdl);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%s: %.2f us per kernel (chain of %d x %d)\n", pdl ? "PDL" : "plain", ms * 1e3 / (reps * chain), chain,
               reps);
    }
    return 0;
}
