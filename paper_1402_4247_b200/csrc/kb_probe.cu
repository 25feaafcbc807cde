// HBM calibration probe: the paper's Table 2 experiment
// (/root/reference/PAPER.md:56, SPEC.md:463-471 microbench_normalize) --
// "normalized: divided every element of a vector by its norm -- n vectors
// which consist of n elements". On B200 this is a pure streaming kernel:
// read every element twice (the second read of a row hits L2, which holds the
// ~150 rows in flight) and write it once, so the compulsory HBM traffic is
// 2 * nvec * len * 8 bytes and the achieved fraction of the copy bandwidth
// calibrates the HBM roofline the grid pass is measured against.
//
// One CTA (256 threads) per vector; deterministic fixed-order reduction;
// zero vectors stay zero.
#include <algorithm>

#include "kb_internal.cuh"

namespace kbg {

namespace {

// CTA loops over rows blockIdx.x, blockIdx.x + gridDim.x, ... (one row per CTA
// unless nvec exceeds the grid limit).
__global__ void __launch_bounds__(256) k_normalize(double* __restrict__ x, int64_t nvec, int64_t len, bool vec2) {
    __shared__ double part[8];
    for (int64_t v = blockIdx.x; v < nvec; v += gridDim.x) {
        double* row = x + v * len;
        double ss = 0.0;
        if (vec2) {
            const double2* r2 = reinterpret_cast<const double2*>(row);
            const int64_t n2 = len / 2;
            int64_t i = threadIdx.x;
            for (; i + 3 * 256 < n2; i += 4 * 256) {  // 4 loads in flight per thread
                const double2 a = r2[i], b = r2[i + 256], c = r2[i + 512], d = r2[i + 768];
                ss += ((a.x * a.x + a.y * a.y) + (b.x * b.x + b.y * b.y)) + ((c.x * c.x + c.y * c.y) + (d.x * d.x + d.y * d.y));
            }
            for (; i < n2; i += 256) {
                const double2 a = r2[i];
                ss += a.x * a.x + a.y * a.y;
            }
        } else {
            for (int64_t i = threadIdx.x; i < len; i += 256) ss += row[i] * row[i];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
        __syncthreads();
        double tot = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) tot += part[w];
        __syncthreads();  // part is reused by the next row
        if (tot == 0.0) continue;
        const double nrm = sqrt(tot);
        if (vec2) {
            double2* r2 = reinterpret_cast<double2*>(row);
            for (int64_t i = threadIdx.x; i < len / 2; i += 256) {
                const double2 a = r2[i];
                r2[i] = make_double2(a.x / nrm, a.y / nrm);
            }
        } else {
            for (int64_t i = threadIdx.x; i < len; i += 256) row[i] = row[i] / nrm;
        }
    }
}

}  // namespace

int launch_normalize(double* d_x, int64_t nvec, int64_t len, cudaStream_t st) {
    if (nvec == 0 || len == 0) return 0;
    const bool vec2 = (len % 2 == 0) && (reinterpret_cast<uintptr_t>(d_x) % 16 == 0);
    // one CTA per row (all rows resident or queued): measured faster than
    // capping the rows in flight to fit L2 (n = 10000: 0.31 vs 0.39 ms)
    const int64_t grid = std::min<int64_t>(nvec, 0x7fffffff);
    k_normalize<<<static_cast<unsigned>(grid), 256, 0, st>>>(d_x, nvec, len, vec2);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

}  // namespace kbg
