// FP64 roofline probes for B200 (sm_100a): DFMA pipe, DMMA (mma.sync m8n8k4 f64)
// pipe, and L2 FP64 atomic (RED.ADD.F64) throughput. MEASURED_PEAKS.json has
// no FP64 entry, so the grid pass's roofline denominator comes from here and
// from cuBLAS DGEMM (bench.py). Prints one JSON line.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));            \
            std::exit(1);                                                           \
        }                                                                           \
    } while (0)

constexpr int kIters = 4096;

__global__ void k_dfma(double* out, double s) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 1e-7);
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += a[i];
    if (r == 12345.678) out[0] = r;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void k_dmma(double* out, double s) {
    double c[CHAINS][2];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = 0.0;
    const double a = threadIdx.x * 1e-3, b = s;
    for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) dmma(c[i], a, b);
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) r += c[i][0] + c[i][1];
    if (r == 12345.678) out[0] = r;
}

// DMMA and DFMA at once: even warps run DMMA chains, odd warps DFMA chains (or every warp interleaves
// both when `both`), to see whether the two FP64 paths share one pipe.
__global__ void k_mixed(double* out, double s, int both) {
    const int warp = threadIdx.x >> 5;
    double c[8][2], a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        c[i][0] = c[i][1] = 0.0;
        a[i] = threadIdx.x * 1e-3 + i;
    }
    const double x = threadIdx.x * 1e-3;
    const bool do_mma = both || !(warp & 1), do_fma = both || (warp & 1);
    for (int it = 0; it < kIters / 4; ++it) {
        if (do_mma) {
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(c[i], x, s);
        }
        if (do_fma) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 1e-7);
        }
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += c[i][0] + c[i][1] + a[i];
    if (r == 12345.678) out[0] = r;
}

// RED.ADD.F64 into an L2-resident array of n doubles; each warp adds 32
// consecutive doubles (coalesced) or scattered lanes.
__global__ void k_red(double* arr, long long n, int per_thread, int scattered) {
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    for (int i = 0; i < per_thread; ++i) {
        long long base = ((tid >> 5) * 7919ll + i * 104729ll) * 32;
        long long idx = scattered ? (base + lane * 97) % n : (base + lane) % n;
        atomicAdd(arr + idx, 1.0);
    }
}

static float time_ms(void (*launch)(void*), void* arg, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    launch(arg);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(a));
        launch(arg);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    return best;
}

struct Cfg {
    double* out;
    int blocks, threads;
    long long n;
    int per_thread, scattered;
};

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double* out;
    CK(cudaMalloc(&out, 64 << 20));
    CK(cudaMemset(out, 0, 64 << 20));
    Cfg cfg{out, sms * 8, 256, 0, 0, 0};

    float t_dfma = time_ms([](void* p) {
        Cfg* c = (Cfg*)p;
        k_dfma<<<c->blocks, c->threads>>>(c->out, 0.999999);
    }, &cfg, 5);
    const double f_dfma = 2.0 * 8 * kIters * (double)cfg.blocks * cfg.threads;

    float t_dmma = time_ms([](void* p) {
        Cfg* c = (Cfg*)p;
        k_dmma<8><<<c->blocks, c->threads>>>(c->out, 0.999999);
    }, &cfg, 5);
    const double f_dmma = 512.0 * 8 * (kIters / 4) * (double)cfg.blocks * (cfg.threads / 32);

    float t_dmma4 = time_ms([](void* p) {
        Cfg* c = (Cfg*)p;
        k_dmma<2><<<c->blocks, c->threads>>>(c->out, 0.999999);
    }, &cfg, 5);
    const double f_dmma4 = 512.0 * 2 * (kIters / 4) * (double)cfg.blocks * (cfg.threads / 32);

    float t_mix = time_ms([](void* p) {
        Cfg* c = (Cfg*)p;
        k_mixed<<<c->blocks, c->threads>>>(c->out, 0.999999, 0);
    }, &cfg, 5);
    // half the warps: 8 DMMAs (512 FMA each) per iteration; the other half: 32 DFMAs per lane
    const double f_mix = (double)cfg.blocks * (cfg.threads / 64) * (kIters / 4) *
                         (8 * 512.0 * 2 + 32 * 32 * 2.0);
    float t_both = time_ms([](void* p) {
        Cfg* c = (Cfg*)p;
        k_mixed<<<c->blocks, c->threads>>>(c->out, 0.999999, 1);
    }, &cfg, 5);
    const double f_both = (double)cfg.blocks * (cfg.threads / 32) * (kIters / 4) * (8 * 512.0 * 2 + 32 * 32 * 2.0);

    Cfg rc{out, sms * 16, 256, (4ll << 20) / 8, 64, 0};
    float t_red = time_ms([](void* p) {
        Cfg* c = (Cfg*)p;
        k_red<<<c->blocks, c->threads>>>(c->out, c->n, c->per_thread, c->scattered);
    }, &rc, 5);
    const double n_red = (double)rc.blocks * rc.threads * rc.per_thread;
    rc.scattered = 1;
    float t_red_s = time_ms([](void* p) {
        Cfg* c = (Cfg*)p;
        k_red<<<c->blocks, c->threads>>>(c->out, c->n, c->per_thread, c->scattered);
    }, &rc, 5);

    std::printf(
        "{\"sms\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"dmma_2chain_tflops\": %.3f, "
        "\"red_f64_coalesced_gops\": %.2f, \"red_f64_scattered_gops\": %.2f, "
        "\"dmma_dfma_split_warps_tflops\": %.3f, \"dmma_dfma_same_warp_tflops\": %.3f}\n",
        sms, f_dfma / t_dfma * 1e-9, f_dmma / t_dmma * 1e-9, f_dmma4 / t_dmma4 * 1e-9, n_red / t_red * 1e-6,
        n_red / t_red_s * 1e-6, f_mix / t_mix * 1e-9, f_both / t_both * 1e-9);
    return 0;
}
