// FP64 RED throughput over a buffer (diagnostic for the H accumulate's placement sensitivity):
// every warp of a full grid adds into consecutive 8-byte entries of [p, p + n), 32 entries per
// instruction, so the L2 atomic units see the buffer's pages evenly.
// nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o libredprobe.so red_probe.cu
#include <cuda_runtime.h>
#include <cstdint>

__global__ void k_red(double* p, int64_t n, int iters) {
    const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    for (int it = 0; it < iters; ++it)
        for (int64_t i = t; i < n; i += nthreads)
            asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p + ((i * 2654435761ll + it) % n)), "d"(1.0)
                         : "memory");
}

extern "C" float red_probe(double* p, int64_t n, int iters) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_red<<<148 * 8, 256>>>(p, n, 1);
    cudaEventRecord(a);
    k_red<<<148 * 8, 256>>>(p, n, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
}
