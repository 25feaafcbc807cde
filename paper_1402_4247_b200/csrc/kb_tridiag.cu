// Symmetric tridiagonal eigensolver on the GPU: the step between
// tridiagonalize and back_transform of Eigen_HH, which the
// reference does with implicit-shift QL on the host (kband::solve_tridiag,
// /root/reference/proj/src/tridiag.cpp:14-110) and the paper with LAPACK on
// the CPUs. QL's rotation chain is sequential; here both halves
// are parallel over the spectrum instead:
//   eigenvalues  multisection on the Sturm count (kband::sturm_count,
//                tridiag.cpp:112-124, same pivot guard): one warp per
//                eigenvalue, 32 shifts per round (each lane one Sturm
//                sequence), the interval shrinks 33x per round;
//   eigenvectors inverse iteration (LU with partial pivoting of T - lambda I,
//                three solves from a deterministic start), one thread per
//                vector -- or per cluster of near-degenerate eigenvalues,
//                computed in order with modified Gram-Schmidt inside the
//                iteration (LAPACK dstein; repeated eigenvalues separated by
//                10 eps ||T|| first) -- then two windowed symmetric
//                re-orthogonalizations among close neighbours (k_tri_orth):
//                all parallel, no sequential chain across a dense spectrum.
// Scratch is interleaved [k][thread] so a warp's threads touch consecutive
// addresses at every step of their (sequential) recurrences.
#include <cfloat>
#include <cstdlib>

#include "kb_internal.cuh"

namespace kbg {

namespace {

__device__ __forceinline__ int sturm_count_dev(const double* d, const double* e2, int n, double x) {
    int c = 0;
    double q = 0.0;
    for (int i = 0; i < n; ++i) {
        q = (i == 0) ? d[0] - x : d[i] - x - e2[i - 1] / q;
        if (q == 0.0) q = -1e-300;  // pivot-underflow guard: a zero pivot counts as below (tridiag.cpp:121)
        if (q < 0.0) ++c;
    }
    return c;
}

// aux[0], aux[1]: Gershgorin interval, widened so count(lo) = 0 and count(hi) = n;
// aux[2]: ||T||_1 (max row sum). One CTA, fixed-order reductions.
__global__ void __launch_bounds__(256) k_tri_bounds(int n, const double* __restrict__ d, const double* __restrict__ e,
                                                    double* __restrict__ aux) {
    double lo = DBL_MAX, hi = -DBL_MAX, nrm = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < n ? fabs(e[i]) : 0.0);
        lo = fmin(lo, d[i] - r);
        hi = fmax(hi, d[i] + r);
        nrm = fmax(nrm, fabs(d[i]) + r);
    }
    __shared__ double s[3][256];
    s[0][threadIdx.x] = lo;
    s[1][threadIdx.x] = hi;
    s[2][threadIdx.x] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < static_cast<int>(blockDim.x); ++k) {
            lo = fmin(lo, s[0][k]);
            hi = fmax(hi, s[1][k]);
            nrm = fmax(nrm, s[2][k]);
        }
        const double pad = 4.0 * DBL_EPSILON * fmax(nrm, 1e-300) + 1e-300;
        aux[0] = lo - pad;
        aux[1] = hi + pad;
        aux[2] = nrm;
    }
}

// One warp per eigenvalue index; d and e^2 staged in shared memory per CTA.
__global__ void __launch_bounds__(128) k_tri_eigvals(int n, const double* __restrict__ d, const double* __restrict__ e,
                                                     const double* __restrict__ aux, double* __restrict__ w) {
    extern __shared__ double tsm[];
    double* sd = tsm;
    double* se2 = tsm + n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        sd[i] = d[i];
        se2[i] = i + 1 < n ? e[i] * e[i] : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int idx = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (idx >= n) return;
    double lo = aux[0], hi = aux[1];  // count(lo) <= idx < count(hi)
    for (int round = 0; round < 48; ++round) {
        const double wdt = hi - lo;
        if (wdt <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) || wdt <= 1e-300) break;
        const double x = lo + wdt * (static_cast<double>(lane + 1) / 33.0);
        const int c = sturm_count_dev(sd, se2, n, x);
        const unsigned m = __ballot_sync(0xffffffffu, c > idx);
        const int k = m ? __ffs(m) - 1 : 32;  // counts are monotone in x: the first shift above idx
        const double xk = __shfl_sync(0xffffffffu, x, k & 31);
        const double xk1 = __shfl_sync(0xffffffffu, x, (k + 31) & 31);
        const double nlo = k > 0 ? xk1 : lo, nhi = k < 32 ? xk : hi;
        if (nlo == lo && nhi == hi) break;  // shifts no longer distinct at this precision
        lo = nlo;
        hi = nhi;
    }
    if (lane == 0) w[idx] = 0.5 * (lo + hi);
}

__device__ __forceinline__ double start_value(int j, int k) {
    uint32_t h = static_cast<uint32_t>(j) * 0x9E3779B1u ^ (static_cast<uint32_t>(k) + 0x7F4A7C15u) * 0x85EBCA77u;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    return (static_cast<double>(h & 0xFFFFFF) + 0.5) / 16777216.0 - 0.5;
}

// Near-degenerate eigenvalues (gaps below kTightGap ||T||_1) are computed in
// order by one thread with re-orthogonalization inside the inverse iteration
// (LAPACK dstein); every other vector independently, in parallel. Inverse
// iteration leaves a vector's components along neighbours of order
// eps ||T|| / gap (<= 2e-7 above the tight threshold); k_tri_orth then removes
// them with two windowed symmetric (Loewdin, first-order) corrections over the
// neighbours closer than 1e-3 ||T||_1, each squaring the loss.
constexpr double kTightGap = 1e-9;
constexpr int kOrthWindow = 32;

// One thread per cluster (started by its first member). z: [n][n] row-major,
// column j = eigenvector j. Scratch (interleaved, stride n): lower multipliers,
// 1/pivots, super diagonals u1, u2, swap flags, right-hand side. Every array
// has its own restrict-qualified pointer and the recurrences carry their state
// in registers, so the (independent) loads of later steps can be issued ahead
// of the dependent chain.
__global__ void __launch_bounds__(128) k_tri_eigvecs(int n, const double* __restrict__ d, const double* __restrict__ e,
                                                     const double* __restrict__ w, const double* __restrict__ aux,
                                                     double* __restrict__ scr, double* __restrict__ z) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const double tnorm = fmax(aux[2], DBL_MIN);
    const double ctol = kTightGap * tnorm, pertol = 10.0 * DBL_EPSILON * tnorm;
    if (t > 0 && w[t] - w[t - 1] < ctol) return;  // not the first member of its (near-degenerate) cluster
    int end = t + 1;
    while (end < n && w[end] - w[end - 1] < ctol) ++end;
    const int64_t S = n;
    const int64_t nn = static_cast<int64_t>(n) * n;
    double* __restrict__ Lm = scr + t;  // element k at [k * S]
    double* __restrict__ Pi = scr + nn + t;
    double* __restrict__ U1 = scr + 2 * nn + t;
    double* __restrict__ U2 = scr + 3 * nn + t;
    double* __restrict__ Sw = scr + 4 * nn + t;
    double* __restrict__ B = scr + 5 * nn + t;
    const double tiny = DBL_EPSILON * tnorm;
    double lprev = 0.0;
    for (int j = t; j < end; ++j) {
        double* __restrict__ zj = z + j;  // element k at [k * n]
        double lam = w[j];
        if (j > t && lam - lprev < pertol) lam = lprev + pertol;
        lprev = lam;
        if (n == 1) {
            zj[0] = 1.0;
            continue;
        }
        // LU of T - lam I with partial pivoting (rows k, k+1), LAPACK dgttrf layout
        double dk = d[0] - lam, uk = e[0];
#pragma unroll 4
        for (int k = 0; k < n - 1; ++k) {
            const double lk = e[k];  // sub-diagonal entry below dk
            const double dn = d[k + 1] - lam, un = k + 1 < n - 1 ? e[k + 1] : 0.0;
            const int64_t o = k * S;
            if (fabs(dk) >= fabs(lk)) {
                const double piv = fabs(dk) < tiny ? copysign(tiny, dk) : dk;
                const double f = lk / piv;
                Lm[o] = f;
                Pi[o] = 1.0 / piv;
                U1[o] = uk;
                U2[o] = 0.0;
                Sw[o] = 0.0;
                dk = dn - f * uk;
                uk = un;
            } else {
                const double f = dk / lk;
                Lm[o] = f;
                Pi[o] = 1.0 / lk;
                U1[o] = dn;
                U2[o] = un;
                Sw[o] = 1.0;
                dk = uk - f * dn;
                uk = -f * un;
            }
        }
        Pi[(n - 1) * S] = 1.0 / (fabs(dk) < tiny ? copysign(tiny, dk) : dk);
        for (int k = 0; k < n; ++k) B[k * S] = start_value(j, k);
        for (int it = 0; it < 3; ++it) {
            // forward: apply the row interchanges and L (b_k carried in a register)
            double bk = B[0];
#pragma unroll 8
            for (int k = 0; k < n - 1; ++k) {
                const int64_t o = k * S;
                const double bn = B[o + S], f = Lm[o];
                const bool sw = Sw[o] != 0.0;
                B[o] = sw ? bn : bk;
                bk = sw ? bk - f * bn : bn - f * bk;
            }
            B[(n - 1) * S] = bk;
            // back substitution with U (diagonal, u1, u2) into column j of z
            double x2 = 0.0, x1 = bk * Pi[(n - 1) * S];
            zj[static_cast<int64_t>(n - 1) * n] = x1;
            double nrm = x1 * x1;
#pragma unroll 8
            for (int k = n - 2; k >= 0; --k) {
                const int64_t o = k * S;
                const double x = (B[o] - U1[o] * x1 - U2[o] * x2) * Pi[o];
                zj[static_cast<int64_t>(k) * n] = x;
                nrm += x * x;
                x2 = x1;
                x1 = x;
            }
            // re-orthogonalize against the earlier members of the cluster, normalize
            if (j > t) {
                for (int p = t; p < j; ++p) {
                    const double* __restrict__ zp = z + p;
                    double dot = 0.0;
                    for (int k = 0; k < n; ++k) dot += zp[static_cast<int64_t>(k) * n] * zj[static_cast<int64_t>(k) * n];
                    for (int k = 0; k < n; ++k) zj[static_cast<int64_t>(k) * n] -= dot * zp[static_cast<int64_t>(k) * n];
                }
                nrm = 0.0;
                for (int k = 0; k < n; ++k) nrm += zj[static_cast<int64_t>(k) * n] * zj[static_cast<int64_t>(k) * n];
            }
            const double sc = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
#pragma unroll 8
            for (int k = 0; k < n; ++k) {
                const double v = zj[static_cast<int64_t>(k) * n] * sc;
                zj[static_cast<int64_t>(k) * n] = v;
                B[k * S] = v;
            }
        }
    }
}

// Shared-memory variant (n <= kTriSmemMaxN): one warp per cluster, the LU factors and the
// right-hand side in the CTA's shared memory, so every step of lane 0's sequential recurrences is a
// shared-memory access instead of a DRAM round trip through the interleaved scratch (at n = 2048 the
// scratch of all vectors is 200 MB, past L2); normalization and re-orthogonalization use all lanes.
constexpr int kTriSmemMaxN = 5120;

__global__ void __launch_bounds__(32) k_tri_eigvecs_smem(int n, const double* __restrict__ d,
                                                         const double* __restrict__ e, const double* __restrict__ w,
                                                         const double* __restrict__ aux, double* __restrict__ z) {
    extern __shared__ double vsm[];
    const int t = blockIdx.x, lane = threadIdx.x;
    const double tnorm = fmax(aux[2], DBL_MIN);
    const double ctol = kTightGap * tnorm, pertol = 10.0 * DBL_EPSILON * tnorm;
    if (t > 0 && w[t] - w[t - 1] < ctol) return;  // not the first member of its (near-degenerate) cluster
    int end = t + 1;
    while (end < n && w[end] - w[end - 1] < ctol) ++end;
    double* __restrict__ Lm = vsm;
    double* __restrict__ Pi = vsm + n;
    double* __restrict__ U1 = vsm + 2 * n;
    double* __restrict__ U2 = vsm + 3 * n;
    double* __restrict__ B = vsm + 4 * n;  // right-hand side, then the solution in place
    unsigned char* __restrict__ Sw = reinterpret_cast<unsigned char*>(vsm + 5 * n);
    const double tiny = DBL_EPSILON * tnorm;
    double lprev = 0.0;
    for (int j = t; j < end; ++j) {
        double lam = w[j];
        if (j > t && lam - lprev < pertol) lam = lprev + pertol;
        lprev = lam;
        if (n == 1) {
            if (lane == 0) z[0] = 1.0;
            continue;
        }
        if (lane == 0) {
            double dk = d[0] - lam, uk = e[0];
            for (int k = 0; k < n - 1; ++k) {
                const double lk = e[k];
                const double dn = d[k + 1] - lam, un = k + 1 < n - 1 ? e[k + 1] : 0.0;
                if (fabs(dk) >= fabs(lk)) {
                    const double piv = fabs(dk) < tiny ? copysign(tiny, dk) : dk;
                    const double f = lk / piv;
                    Lm[k] = f;
                    Pi[k] = 1.0 / piv;
                    U1[k] = uk;
                    U2[k] = 0.0;
                    Sw[k] = 0;
                    dk = dn - f * uk;
                    uk = un;
                } else {
                    const double f = dk / lk;
                    Lm[k] = f;
                    Pi[k] = 1.0 / lk;
                    U1[k] = dn;
                    U2[k] = un;
                    Sw[k] = 1;
                    dk = uk - f * dn;
                    uk = -f * un;
                }
            }
            Pi[n - 1] = 1.0 / (fabs(dk) < tiny ? copysign(tiny, dk) : dk);
        }
        for (int k = lane; k < n; k += 32) B[k] = start_value(j, k);
        __syncwarp();
        for (int it = 0; it < 3; ++it) {
            if (lane == 0) {
                double bk = B[0];
                for (int k = 0; k < n - 1; ++k) {
                    const double bn = B[k + 1], f = Lm[k];
                    const bool sw = Sw[k] != 0;
                    B[k] = sw ? bn : bk;
                    bk = sw ? bk - f * bn : bn - f * bk;
                }
                double x2 = 0.0, x1 = bk * Pi[n - 1];
                B[n - 1] = x1;
                for (int k = n - 2; k >= 0; --k) {
                    const double x = (B[k] - U1[k] * x1 - U2[k] * x2) * Pi[k];
                    B[k] = x;
                    x2 = x1;
                    x1 = x;
                }
            }
            __syncwarp();
            // re-orthogonalize against the earlier members of the cluster (columns of z), normalize
            for (int p = t; p < j; ++p) {
                double dot = 0.0;
                for (int k = lane; k < n; k += 32) dot += z[static_cast<int64_t>(k) * n + p] * B[k];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
                for (int k = lane; k < n; k += 32) B[k] -= dot * z[static_cast<int64_t>(k) * n + p];
                __syncwarp();
            }
            double nrm = 0.0;
            for (int k = lane; k < n; k += 32) nrm += B[k] * B[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
            const double sc = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
            for (int k = lane; k < n; k += 32) B[k] *= sc;
            __syncwarp();
        }
        for (int k = lane; k < n; k += 32) z[static_cast<int64_t>(k) * n + j] = B[k];
        __syncwarp();
    }
}

// One windowed symmetric correction: zout_j = (z_j - 1/2 sum_k (z_k . z_j) z_k) / norm, k over the
// neighbours of j (|w_k - w_j| < 1e-3 ||T||_1, at most kOrthWindow each side). One warp per vector:
// lanes split the rows, and since the window's columns are a contiguous segment of each row, one pass
// gathers all (per-lane partial) dots, reduced with shuffles, and a second applies the correction.
__global__ void __launch_bounds__(128) k_tri_orth_warp(int n, const double* __restrict__ w,
                                                       const double* __restrict__ aux, const double* __restrict__ zin,
                                                       double* __restrict__ zout) {
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (j >= n) return;
    const double ortol = 1e-3 * fmax(aux[2], DBL_MIN);
    int lo = j, hi = j;
    while (lo > 0 && j - lo < kOrthWindow && w[j] - w[lo - 1] < ortol) --lo;
    while (hi + 1 < n && hi - j < kOrthWindow && w[hi + 1] - w[j] < ortol) ++hi;
    if (lo == hi) {
        for (int64_t i = lane; i < n; i += 32) zout[i * n + j] = zin[i * n + j];
        return;
    }
    const int nw = hi - lo + 1;
    double dots[2 * kOrthWindow + 1];
    for (int k = 0; k < nw; ++k) dots[k] = 0.0;
    for (int64_t i = lane; i < n; i += 32) {
        const double* __restrict__ row = zin + i * n + lo;
        const double zj = zin[i * n + j];
        for (int k = 0; k < nw; ++k) dots[k] += row[k] * zj;
    }
    for (int k = 0; k < nw; ++k) {
        double v = dots[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        dots[k] = k == j - lo ? 0.0 : 0.5 * v;
    }
    double nrm = 0.0;
    for (int64_t i = lane; i < n; i += 32) {
        const double* __restrict__ row = zin + i * n + lo;
        double v = zin[i * n + j];
        for (int k = 0; k < nw; ++k) v -= dots[k] * row[k];
        zout[i * n + j] = v;
        nrm += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    const double sc = 1.0 / sqrt(nrm);
    for (int64_t i = lane; i < n; i += 32) zout[i * n + j] *= sc;
}

}  // namespace

size_t tridiag_scratch_doubles(int n, bool vectors) {
    if (!vectors) return 4;
    const bool smem = n <= kTriSmemMaxN && !std::getenv("KBG_TRI_GLOBAL");
    return 4 + (smem ? 1 : 6) * static_cast<size_t>(n) * n;  // smem path: only the re-orthogonalization buffer
}

int launch_tridiag_solve(int n, const double* d_d, const double* d_e, bool vectors, double* d_w, double* d_z,
                         double* d_scr, cudaStream_t st) {
    double* aux = d_scr;  // [4]: interval, ||T||_1; inverse-iteration scratch after it
    d_scr += 4;
    k_tri_bounds<<<1, 256, 0, st>>>(n, d_d, d_e, aux);
    const size_t smem = 2 * static_cast<size_t>(n) * sizeof(double);
    KBG_CUDA(cudaFuncSetAttribute(k_tri_eigvals, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    const unsigned blocks = static_cast<unsigned>((static_cast<int64_t>(n) * 32 + 127) / 128);
    k_tri_eigvals<<<blocks, 128, smem, st>>>(n, d_d, d_e, aux, d_w);
    KBG_CUDA(cudaGetLastError());
    if (!vectors) return 2;
    const unsigned g = static_cast<unsigned>((n + 127) / 128);
    if (n <= kTriSmemMaxN && !std::getenv("KBG_TRI_GLOBAL")) {
        const size_t vs = 5 * static_cast<size_t>(n) * sizeof(double) + ((n + 15) & ~15);
        KBG_CUDA(cudaFuncSetAttribute(k_tri_eigvecs_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(vs)));
        k_tri_eigvecs_smem<<<static_cast<unsigned>(n), 32, vs, st>>>(n, d_d, d_e, d_w, aux, d_z);
    } else {
        k_tri_eigvecs<<<g, 128, 0, st>>>(n, d_d, d_e, d_w, aux, d_scr, d_z);
    }
    // two windowed corrections, ping-pong through the (now free) LU scratch
    const unsigned gw = static_cast<unsigned>((static_cast<int64_t>(n) * 32 + 127) / 128);
    k_tri_orth_warp<<<gw, 128, 0, st>>>(n, d_w, aux, d_z, d_scr);
    k_tri_orth_warp<<<gw, 128, 0, st>>>(n, d_w, aux, d_scr, d_z);
    KBG_CUDA(cudaGetLastError());
    return 5;
}

}  // namespace kbg
