// DMMA (mma.sync.m8n8k4.f64) issue/latency probe: throughput vs independent
// accumulator chains per warp and warps per SM. Prints one JSON line per case.
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int CH, int LDS_PER>
__global__ void k_probe(double* out, int iters) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1e-3 * i;
    __syncthreads();
    double c[CH][2];
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
    double a = threadIdx.x * 1e-3, b = 0.999;
    int idx = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (LDS_PER) {
                a = sm[(idx + 37 * i + it) & 1023];
            }
            dmma(c[i], a, b);
        }
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) r += c[i][0] + c[i][1];
    if (r == 1234.5) out[0] = r;
}

template <int CH, int LDS>
void run(int warps_per_block, int blocks_per_sm, int sms, double* out) {
    const int iters = 2048 / CH;
    dim3 grid(sms * blocks_per_sm), block(32 * warps_per_block);
    k_probe<CH, LDS><<<grid, block>>>(out, iters);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_probe<CH, LDS><<<grid, block>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double dmmas = (double)grid.x * warps_per_block * iters * CH;
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double cycles = ms * 1e-3 * clk * 1e3;
    std::printf("{\"chains\": %d, \"lds\": %d, \"warps_per_sm\": %d, \"tflops\": %.2f, \"dmma_per_sm_per_kcycle\": %.1f}\n",
                CH, LDS, warps_per_block * blocks_per_sm, dmmas * 512 / (ms * 1e-3) / 1e12,
                dmmas / sms / cycles * 1000);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 64);
    for (int w : {4, 8, 16, 32}) {
        run<1, 0>(w, 1, sms, out);
        run<2, 0>(w, 1, sms, out);
        run<4, 0>(w, 1, sms, out);
        run<8, 0>(w, 1, sms, out);
        run<2, 1>(w, 1, sms, out);
        run<4, 1>(w, 1, sms, out);
    }
    return 0;
}
