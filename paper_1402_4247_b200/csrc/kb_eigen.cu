// Eigen_HH on the GPU: the paper's hot path downstream of
// the grid pass -- Householder tridiagonalization of the Hermitian H(k)
// (procedures 1-6 per stage), the eigenvector rearrangement (back transform)
// and the column normalization -- following the reference's kband
// conventions exactly (/root/reference/proj/src/householder.cpp):
//   tridiagonalize    householder.cpp:60-251 (records: reflector u, h, s, phase)
//   back_transform    householder.cpp:253-305
//   normalize_columns householder.cpp:307-331
// The tridiagonal QL solve between them stays with the caller, as in the
// paper (LAPACK dstevx/dstegr/dstedc on the CPUs).
//
// B200 design. The working matrix (n <= 6144: <= 604 MB, L2-resident up to
// n ~ 2800) stays on the device. tridiagonalize is one cooperative persistent
// kernel, one CTA per SM: per stage every CTA rebuilds the reflector from row
// i (redundantly, fixed-order reductions -> identical in every CTA), warps
// compute p = B u / h one row each (hemv, procedure 4), a grid barrier, every
// CTA forms K and q (procedures 4-5), warps apply the rank-2 update to their
// rows (her2, procedure 6), a second grid barrier. Both sweeps stream the
// trailing block from L2: BLAS-2, bound by L2 bandwidth and the two grid
// barriers per stage. back_transform gives each warp one eigenvector column,
// kept in shared memory through all n - 1 reflectors (read from L2), so no
// barrier is needed at all. All reductions have a fixed order: bitwise
// deterministic run to run.
#include <cooperative_groups.h>
#include <cublas_v2.h>

#include <algorithm>
#include <cstdlib>

#include "kb_internal.cuh"

namespace cg = cooperative_groups;

namespace kbg {

namespace {

constexpr double kSkipNorm = 1e-300;  // householder.cpp:46
// Unroll of the fused per-row sweep (her2 update + next hemv): keeps several L2 loads of a row in
// flight per lane; measured n = 1040 10.4 -> 8.2 ms (4), 8.5 (8).
#ifndef KBG_TRI_UNROLL
#define KBG_TRI_UNROLL 4
#endif
constexpr int kTriUnroll = KBG_TRI_UNROLL;
constexpr int kTriThreads = 512;      // 16 warps per CTA
constexpr int kTriWarps = kTriThreads / 32;

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// Fixed-order CTA sum of one double per thread (identical in every CTA).
__device__ double cta_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < kTriWarps; ++i) t += red[i];
    return t;
}

struct TriOut {
    double* d;      // [n]
    double* e;      // [n - 1]
    double2* u;     // [n - 1][n]
    double* h;      // [n - 1]
    double* s;      // [n - 1]
    double2* ph;    // [n - 1]
};

// Stage-j reflector from the (updated) row j, redundantly in every CTA
// (procedures 1-2): un[c] = conj(row j, c) for c > j, s, pivot phase, h.
// Returns (h, s) and the phase through bc; un[lo] is the shifted pivot.
template <class RowVal>
__device__ void build_reflector(int n, int j, RowVal&& rowval, double2* un, double* red, double2* bc) {
    const int lo = j + 1, tid = threadIdx.x;
    double s2 = 0.0;
    for (int c = lo + tid; c < n; c += kTriThreads) {
        const double2 x = rowval(c);
        un[c] = make_double2(x.x, -x.y);
        s2 += x.x * x.x + x.y * x.y;
    }
    s2 = cta_sum(s2, red);
    if (tid == 0) {
        const double s = sqrt(s2);
        const double2 u0 = un[lo];
        const double piv = hypot(u0.x, u0.y);
        const double2 phs = piv > 0.0 ? make_double2(u0.x / piv, u0.y / piv) : make_double2(1.0, 0.0);
        const double h = s >= kSkipNorm ? s * (s + piv) : 0.0;
        if (h != 0.0) un[lo] = make_double2(u0.x + phs.x * s, u0.y + phs.y * s);
        bc[0] = phs;
        bc[1] = make_double2(h, s);
    }
    __syncthreads();
}

// Record of stage j (procedure 3), CTA 0.
__device__ void write_record(int n, int j, double dj, const double2* un, const double2* bc, const TriOut& out) {
    if (blockIdx.x != 0) return;
    const double h = bc[1].x, s = bc[1].y;
    const double2 phs = bc[0];
    if (threadIdx.x == 0) {
        out.d[j] = dj;
        out.e[j] = h == 0.0 ? 0.0 : s;
        out.h[j] = h;
        out.s[j] = s;
        out.ph[j] = h == 0.0 ? make_double2(1.0, 0.0) : make_double2(-phs.x, -phs.y);
    }
    double2* uj = out.u + static_cast<int64_t>(j) * n;
    for (int r = threadIdx.x; r < n; r += kTriThreads)
        uj[r] = (h == 0.0 || r <= j) ? make_double2(0.0, 0.0) : un[r];
}

// Procedure-6 term u_r conj(q_c) + q_r conj(u_c) (householder.cpp:211-224).
__device__ __forceinline__ double2 her2_term(double2 ur, double2 qr, double2 uc, double2 qc) {
    return make_double2(ur.x * qc.x + ur.y * qc.y + qr.x * uc.x + qr.y * uc.y,
                        ur.y * qc.x - ur.x * qc.y + qr.y * uc.x - qr.x * uc.y);
}

// One grid barrier and one pass over the trailing block per stage: the
// rank-2 update of stage i (procedure 6) and the hemv of stage i + 1
// (procedure 4) are fused -- every CTA first rebuilds row i + 1 as updated by
// stage i (it needs u, q of stage i only), forms reflector i + 1 from it, then
// each warp updates its rows r >= i + 2 in registers and immediately
// accumulates p_{i+1}[r] from the updated values. Row/column i + 1 are never
// read again, so they are not stored. p is double-buffered across stages.
__global__ void __launch_bounds__(kTriThreads, 1) k_tridiag(int n, double2* __restrict__ B, double2* __restrict__ p2,
                                                            TriOut out, double sign) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double2 tri_smem[];
    double2* ucur = tri_smem;           // [n] reflector of stage i
    double2* unxt = tri_smem + n;       // [n] reflector of stage i + 1
    double2* q = tri_smem + 2 * n;      // [n] p then q of stage i
    __shared__ double red[kTriWarps];
    __shared__ double2 bc[2];
    const int tid = threadIdx.x, lane = tid & 31;
    const int gwarp = blockIdx.x * kTriWarps + (tid >> 5), nwarp = gridDim.x * kTriWarps;
    // prologue: reflector 0 from row 0 and its hemv
    build_reflector(n, 0, [&](int c) { return B[c]; }, ucur, red, bc);
    write_record(n, 0, B[0].x, ucur, bc, out);
    double hcur = bc[1].x;
    if (hcur != 0.0) {
        for (int r = 1 + gwarp; r < n; r += nwarp) {
            const double2* br = B + static_cast<int64_t>(r) * n;
            double ar = 0.0, ai = 0.0;
            for (int c = 1 + lane; c < n; c += 32) {
                const double2 x = br[c], y = ucur[c];
                ar += x.x * y.x - x.y * y.y;
                ai += x.x * y.y + x.y * y.x;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                ar += __shfl_xor_sync(0xffffffffu, ar, o);
                ai += __shfl_xor_sync(0xffffffffu, ai, o);
            }
            if (lane == 0) p2[r] = make_double2(ar / hcur, ai / hcur);
        }
    }
    grid.sync();
    for (int i = 0; i + 1 < n; ++i) {
        const int lo = i + 1, lo2 = i + 2;
        const double2* pin = p2 + (i & 1) * n;
        double2* pout = p2 + ((i + 1) & 1) * n;
        // procedures 4 (dot) and 5 of stage i: K = Re(p . u) / 2h, q = p - K u
        if (hcur != 0.0) {
            double dr = 0.0;
            for (int r = lo + tid; r < n; r += kTriThreads) {
                const double2 pr = pin[r];
                q[r] = pr;
                dr += pr.x * ucur[r].x + pr.y * ucur[r].y;
            }
            const double K = cta_sum(dr, red) / (2.0 * hcur);
            for (int r = lo + tid; r < n; r += kTriThreads) {
                const double2 pr = q[r], ur = ucur[r];
                q[r] = make_double2(pr.x - K * ur.x, pr.y - K * ur.y);
            }
            __syncthreads();
        }
        // row lo as updated by stage i -> reflector of stage lo (d[lo] from its diagonal)
        const bool upd = hcur != 0.0;
        const double2 ul = upd ? ucur[lo] : make_double2(0.0, 0.0), ql = upd ? q[lo] : make_double2(0.0, 0.0);
        auto rowval = [&](int c) {
            double2 b = B[static_cast<int64_t>(lo) * n + c];
            if (upd) {
                const double2 x = her2_term(ul, ql, ucur[c], q[c]);
                b.x += sign * x.x;
                b.y += sign * x.y;
            }
            return b;
        };
        double hnxt = 0.0;
        if (lo2 < n) {
            build_reflector(n, lo, rowval, unxt, red, bc);
            write_record(n, lo, rowval(lo).x, unxt, bc, out);
            hnxt = bc[1].x;
        } else if (blockIdx.x == 0 && tid == 0) {
            out.d[lo] = rowval(lo).x;
        }
        // fused pass over rows/columns >= lo2: stage-i update + stage-(i+1) hemv
        if (upd || hnxt != 0.0) {
            for (int r = lo2 + gwarp; r < n; r += nwarp) {
                double2* br = B + static_cast<int64_t>(r) * n;
                const double2 ur = upd ? ucur[r] : make_double2(0.0, 0.0), qr = upd ? q[r] : make_double2(0.0, 0.0);
                double ar = 0.0, ai = 0.0;
#if KBG_TRI_UNROLL > 1
#pragma unroll kTriUnroll
#endif
                for (int c = lo2 + lane; c < n; c += 32) {
                    double2 b = br[c];
                    if (upd) {
                        const double2 x = her2_term(ur, qr, ucur[c], q[c]);
                        b.x += sign * x.x;
                        b.y += sign * x.y;
                        br[c] = b;
                    }
                    const double2 y = unxt[c];
                    ar += b.x * y.x - b.y * y.y;
                    ai += b.x * y.y + b.y * y.x;
                }
                if (hnxt != 0.0) {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        ar += __shfl_xor_sync(0xffffffffu, ar, o);
                        ai += __shfl_xor_sync(0xffffffffu, ai, o);
                    }
                    if (lane == 0) pout[r] = make_double2(ar / hnxt, ai / hnxt);
                }
            }
            grid.sync();
        }
        double2* t = ucur;
        ucur = unxt;
        unxt = t;
        hcur = hnxt;
        __syncthreads();  // the swapped buffers are rewritten next stage
    }
}

// Cumulative chased-out phases (householder.cpp:264-273), sequential like the
// reference: dph[row] for rows 1..n-1, dph[0] = 1.
__global__ void k_phase_prefix(int n, const double* __restrict__ h, const double2* __restrict__ ph,
                               double2* __restrict__ dph) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double2 acc = make_double2(1.0, 0.0);
    dph[0] = acc;
    for (int k = 0; k + 1 < n; ++k) {
        if (h[k] > 0.0) acc = cmul(acc, ph[k]);
        dph[k + 1] = acc;
    }
}

// W = Q Y: one warp per eigenvector column j, the column in shared memory;
// reflectors applied in reverse stage order (householder.cpp:275-296).
constexpr int kBtWarps = 4;  // max warps (columns) per CTA; fewer when n is large
__global__ void __launch_bounds__(kBtWarps * 32) k_back_transform(int n, int m, const double* __restrict__ Y,
                                                                  const double2* __restrict__ U,
                                                                  const double* __restrict__ h,
                                                                  const double2* __restrict__ dph,
                                                                  double2* __restrict__ W) {
    extern __shared__ double2 bt_smem[];
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.x * (blockDim.x >> 5) + wi;
    if (j >= m) return;
    double2* w = bt_smem + static_cast<int64_t>(wi) * n;
    for (int r = lane; r < n; r += 32) {
        const double y = Y[static_cast<int64_t>(r) * m + j];
        const double2 f = dph[r];
        w[r] = r == 0 ? make_double2(y, 0.0) : make_double2(y * f.x, y * f.y);
    }
    __syncwarp();
    for (int k = n - 2; k >= 0; --k) {
        const double hk = h[k];
        if (hk == 0.0) continue;
        const int lo = k + 1;
        const double2* uk = U + static_cast<int64_t>(k) * n;
        double ar = 0.0, ai = 0.0;  // u^H w
#pragma unroll 4
        for (int r = lo + lane; r < n; r += 32) {
            const double2 x = uk[r], y = w[r];
            ar += x.x * y.x + x.y * y.y;
            ai += x.x * y.y - x.y * y.x;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ar += __shfl_xor_sync(0xffffffffu, ar, o);
            ai += __shfl_xor_sync(0xffffffffu, ai, o);
        }
        ar /= hk;
        ai /= hk;
#pragma unroll 4
        for (int r = lo + lane; r < n; r += 32) {
            const double2 x = uk[r];
            double2 y = w[r];
            y.x -= x.x * ar - x.y * ai;
            y.y -= x.x * ai + x.y * ar;
            w[r] = y;
        }
        __syncwarp();
    }
    for (int r = lane; r < n; r += 32) W[static_cast<int64_t>(r) * m + j] = w[r];
}

// Columns to unit 2-norm in row order (linalg.cpp:214-218, householder.cpp:307-331):
// one thread per column; exact products/sums so the norms match the reference bitwise.
__global__ void k_normalize_columns(int64_t n, int64_t m, double2* __restrict__ C, int* __restrict__ zero_col) {
    const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (j >= m) return;
    double s = 0.0;
    for (int64_t r = 0; r < n; ++r) {
        const double2 v = C[r * m + j];
        s = __dadd_rn(s, __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y)));
    }
    const double nrm = sqrt(s);
    if (nrm < kSkipNorm) {
        atomicMin(zero_col, static_cast<int>(j));
        return;
    }
    const double inv = 1.0 / nrm;
    for (int64_t r = 0; r < n; ++r) {
        double2 v = C[r * m + j];
        v.x = __dmul_rn(v.x, inv);
        v.y = __dmul_rn(v.y, inv);
        C[r * m + j] = v;
    }
}

// HermitianMatrix::from (linalg.cpp:44-63): defect max |A_ij - conj(A_ji)|
// (bit pattern, atomicMax), then A_ij = avg, A_ji = conj(avg), diagonal real.
__global__ void k_hermitian_repair(int n, double2* __restrict__ A, unsigned long long* defect) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t nn = static_cast<int64_t>(n) * n;
    double d = 0.0;
    if (t < nn) {
        const int i = static_cast<int>(t / n), j = static_cast<int>(t - static_cast<int64_t>(i) * n);
        if (j >= i) {
            const double2 a = A[t], b = A[static_cast<int64_t>(j) * n + i];
            d = hypot(a.x - b.x, a.y + b.y);
            if (!isfinite(a.x) || !isfinite(a.y) || !isfinite(b.x) || !isfinite(b.y)) d = __longlong_as_double(0x7ff0000000000000ll);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    if ((threadIdx.x & 31) == 0) atomicMax(defect, static_cast<unsigned long long>(__double_as_longlong(d)));
}

__global__ void k_hermitian_apply(int n, double2* __restrict__ A) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<int64_t>(n) * n) return;
    const int i = static_cast<int>(t / n), j = static_cast<int>(t - static_cast<int64_t>(i) * n);
    if (j < i) return;
    if (j == i) {
        A[t].y = 0.0;
        return;
    }
    const double2 a = A[t], b = A[static_cast<int64_t>(j) * n + i];
    const double2 avg = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
    A[t] = avg;
    A[static_cast<int64_t>(j) * n + i] = make_double2(avg.x, -avg.y);
}

}  // namespace

int launch_hermitian_repair(int n, double* d_A, unsigned long long* d_defect, bool apply, cudaStream_t st) {
    const int64_t nn = static_cast<int64_t>(n) * n;
    if (nn == 0) return 0;
    const unsigned grid = static_cast<unsigned>((nn + 255) / 256);
    if (!apply)
        k_hermitian_repair<<<grid, 256, 0, st>>>(n, reinterpret_cast<double2*>(d_A), d_defect);
    else
        k_hermitian_apply<<<grid, 256, 0, st>>>(n, reinterpret_cast<double2*>(d_A));
    KBG_CUDA(cudaGetLastError());
    return 1;
}

size_t hh_tridiag_smem(int n) { return 3 * static_cast<size_t>(n) * sizeof(double2); }

int launch_hh_tridiagonalize(int n, double* d_B, double* d_p, double* d, double* e, double* u, double* h, double* s,
                             double* ph, double sign, cudaStream_t st) {
    if (n <= 0) return 0;
    if (n == 1) {
        KBG_CUDA(cudaMemcpyAsync(d, d_B, sizeof(double), cudaMemcpyDeviceToDevice, st));
        return 0;
    }
    int dev = 0, sms = 0, per_sm = 0;
    KBG_CUDA(cudaGetDevice(&dev));
    KBG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t smem = hh_tridiag_smem(n);
    KBG_CUDA(cudaFuncSetAttribute(k_tridiag, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    KBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tridiag, kTriThreads, smem));
    if (per_sm < 1) throw Error(KBG_ERR_DIMENSION, "tridiagonalize: n too large for the cooperative kernel");
    // rows per warp: no more CTAs than rows of work keep busy
    int grid = std::max(1, std::min(sms, (n + kTriWarps - 1) / kTriWarps));
    if (const char* g = std::getenv("KBG_TRI_GRID")) grid = std::max(1, std::min(sms * per_sm, std::atoi(g)));  // tuning
    TriOut o{d, e, reinterpret_cast<double2*>(u), h, s, reinterpret_cast<double2*>(ph)};
    int nn = n;
    double2* B = reinterpret_cast<double2*>(d_B);
    double2* P = reinterpret_cast<double2*>(d_p);
    void* args[] = {&nn, &B, &P, &o, &sign};  // P: 2 n complex (double-buffered p)
    KBG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_tridiag), dim3(grid), dim3(kTriThreads), args,
                                         smem, st));
    KBG_CUDA(cudaGetLastError());
    return 1;
}

int launch_hh_back_transform(int n, int m, const double* d_Y, const double* d_U, const double* d_h,
                             const double* d_ph, double* d_dph, double* d_W, cudaStream_t st) {
    if (n <= 0 || m <= 0) return 0;
    k_phase_prefix<<<1, 32, 0, st>>>(n, d_h, reinterpret_cast<const double2*>(d_ph), reinterpret_cast<double2*>(d_dph));
    const int nw = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kBtWarps, (227 * 1024) / (n * 16))));
    const size_t smem = static_cast<size_t>(nw) * n * sizeof(double2);
    KBG_CUDA(cudaFuncSetAttribute(k_back_transform, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    k_back_transform<<<static_cast<unsigned>((m + nw - 1) / nw), nw * 32, smem, st>>>(
        n, m, d_Y, reinterpret_cast<const double2*>(d_U), d_h, reinterpret_cast<const double2*>(d_dph),
        reinterpret_cast<double2*>(d_W));
    KBG_CUDA(cudaGetLastError());
    return 2;
}

// ---- blocked (compact WY) back transform ------------------------------------------
// W = P_0 P_1 ... P_{n-2} D Y with P_k = I - u_k u_k^H / h_k (householder.cpp:275-296; D the chased
// phases). Reflectors are grouped in blocks of kWyBlock: P_k0 ... P_k0+K-1 = I - V T V^H (LAPACK
// zlarft, forward, columnwise: T upper triangular, T_ii = tau_i = 1/h_i, T(0:i, i) = -tau_i T(0:i,0:i)
// V(:,0:i)^H v_i), and each block is applied with ZGEMMs, last block first: W -= V (T (V^H W)). W is
// kept column-major (n x m, ld n) during the sweep; V is the block's rows of U read as a column-major
// n x K matrix, restricted to its nonzero rows k0+1..n-1.
constexpr int kWyBlock = 64;
constexpr int kWySplit = 16;

namespace {

// W_cm[j][r] = D_r Y[r][j]
__global__ void k_bt_wy_init(int n, int m, const double* __restrict__ Y, const double2* __restrict__ dph,
                             double2* __restrict__ Wc) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < static_cast<int64_t>(n) * m;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = t / n, r = t % n;
        const double y = Y[r * m + j];
        const double2 f = dph[r];
        Wc[t] = r == 0 ? make_double2(y, 0.0) : make_double2(y * f.x, y * f.y);
    }
}

__global__ void k_bt_wy_out(int n, int m, const double2* __restrict__ Wc, double2* __restrict__ W) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < static_cast<int64_t>(n) * m;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = t / m, j = t % m;
        W[t] = Wc[j * n + r];
    }
}

// T (K x K, column-major, upper) of one block from G = V^H V (K x K, column-major) and h.
// One CTA of K threads; column i needs the finished columns 0..i-1.
__global__ void k_bt_wy_larft(int K, const double2* __restrict__ G, const double* __restrict__ h,
                              double2* __restrict__ T) {
    const int r = threadIdx.x;
    for (int i = 0; i < K; ++i) {
        const double tau = h[i] != 0.0 ? 1.0 / h[i] : 0.0;
        double2 acc = make_double2(0.0, 0.0);
        if (r < i) {  // (T(0:i,0:i) G(0:i, i))_r, T upper: columns c >= r
            for (int c = r; c < i; ++c) acc = cadd(acc, cmul(T[c * K + r], G[i * K + c]));
            T[i * K + r] = make_double2(-tau * acc.x, -tau * acc.y);
        } else if (r == i) {
            T[i * K + i] = make_double2(tau, 0.0);
        } else if (r < K) {
            T[i * K + r] = make_double2(0.0, 0.0);
        }
        __syncthreads();
    }
}

// out = sum over chunks of P[c] (fixed order: deterministic)
__global__ void k_bt_wy_sum(int64_t len, int chunks, const double2* __restrict__ P, double2* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= len) return;
    double2 a = P[i];
    for (int c = 1; c < chunks; ++c) a = cadd(a, P[c * len + i]);
    out[i] = a;
}

cublasHandle_t wy_handle() {
    static thread_local cublasHandle_t hnd = nullptr;
    static thread_local int dev = -1;
    int cur = 0;
    KBG_CUDA(cudaGetDevice(&cur));
    if (!hnd || dev != cur) {
        if (cublasCreate(&hnd) != CUBLAS_STATUS_SUCCESS) throw Error(KBG_ERR_CUDA, "cublasCreate failed");
        dev = cur;
    }
    return hnd;
}

void cublas_ok(cublasStatus_t s, const char* what) {
    if (s != CUBLAS_STATUS_SUCCESS) throw Error(KBG_ERR_CUDA, std::string("back_transform: ") + what + " failed");
}

}  // namespace

int launch_hh_back_transform_wy(int n, int m, const double* d_Y, const double* d_U, const double* d_h,
                                const double* d_ph, double* d_dph, double* d_W, double* d_scr, cudaStream_t st) {
    if (n <= 0 || m <= 0) return 0;
    const int K = kWyBlock;
    double2* Wc = reinterpret_cast<double2*>(d_scr);                     // n x m
    double2* G = Wc + static_cast<int64_t>(n) * m;                       // K x K
    double2* T = G + K * K;                                              // K x K
    double2* X = T + K * K;                                              // K x m
    double2* X2 = X + static_cast<int64_t>(K) * m;                       // K x m
    double2* P = X2 + static_cast<int64_t>(K) * m;                       // kWySplit partials of K x max(K, m)
    const double2* U = reinterpret_cast<const double2*>(d_U);
    k_phase_prefix<<<1, 32, 0, st>>>(n, d_h, reinterpret_cast<const double2*>(d_ph), reinterpret_cast<double2*>(d_dph));
    k_bt_wy_init<<<148 * 4, 256, 0, st>>>(n, m, d_Y, reinterpret_cast<const double2*>(d_dph), Wc);
    cublasHandle_t hb = wy_handle();
    cublas_ok(cublasSetStream(hb, st), "cublasSetStream");
    const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0),
                          mone = make_cuDoubleComplex(-1.0, 0.0);
    auto z = [](const double2* p) { return reinterpret_cast<const cuDoubleComplex*>(p); };
    auto zm = [](double2* p) { return reinterpret_cast<cuDoubleComplex*>(p); };
    int launches = 2;
    const int nref = n - 1;
    for (int k0 = ((nref - 1) / K) * K; k0 >= 0; k0 -= K) {
        const int kb = std::min(K, nref - k0);
        const int r0 = k0 + 1, rows = n - r0;  // nonzero rows of the block's reflectors
        const cuDoubleComplex* V = z(U + static_cast<int64_t>(k0) * n + r0);  // column i = u_{k0+i}, ld n
        // G = V^H V, T = larft(G, h); X = V^H W. Both reduce over the long row dimension into a small
        // output, so they are split over row chunks (strided-batched ZGEMMs into partials + a
        // fixed-order sum): a plain ZGEMM of that shape runs on a handful of CTAs.
        cuDoubleComplex* Wr = zm(Wc + r0);
        const int chunks = std::max(1, std::min(kWySplit, rows / 128));
        const int clen = (rows + chunks - 1) / chunks, last = rows - (chunks - 1) * clen;
        auto splitk = [&](const cuDoubleComplex* B, int ncol, double2* out, const char* what) {
            // full chunks batched; the (shorter) last chunk separately; then sum in chunk order
            if (chunks > 1)
                cublas_ok(cublasZgemmStridedBatched(hb, CUBLAS_OP_C, CUBLAS_OP_N, kb, ncol, clen, &one, V, n, clen, B,
                                                    n, clen, &zero, zm(P), kb, static_cast<long long>(kb) * ncol,
                                                    chunks - 1),
                          what);
            cublas_ok(cublasZgemm(hb, CUBLAS_OP_C, CUBLAS_OP_N, kb, ncol, last, &one, V + (chunks - 1) * clen, n,
                                  B + (chunks - 1) * clen, n, &zero, zm(P + static_cast<int64_t>(chunks - 1) * kb * ncol),
                                  kb),
                      what);
            k_bt_wy_sum<<<(kb * ncol + 255) / 256, 256, 0, st>>>(static_cast<int64_t>(kb) * ncol, chunks, P, out);
        };
        splitk(V, kb, G, "ZGEMM V^H V");
        k_bt_wy_larft<<<1, ((kb + 31) / 32) * 32, 0, st>>>(kb, G, d_h + k0, T);
        // X = V^H W, X2 = T X, W -= V X2 (rows r0..n-1 of W)
        splitk(Wr, m, X, "ZGEMM V^H W");
        cublas_ok(cublasZgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, kb, m, kb, &one, z(T), kb, z(X), kb, &zero, zm(X2), kb),
                  "ZGEMM T X");
        cublas_ok(cublasZgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, rows, m, kb, &mone, V, n, z(X2), kb, &one, Wr, n),
                  "ZGEMM W -= V X");
        launches += 5;
    }
    k_bt_wy_out<<<148 * 4, 256, 0, st>>>(n, m, Wc, reinterpret_cast<double2*>(d_W));
    KBG_CUDA(cudaGetLastError());
    return launches + 1;
}

size_t hh_back_transform_wy_scratch(int n, int m) {
    const size_t wide = std::max<size_t>(kWyBlock, m);
    return 2 * (static_cast<size_t>(n) * m + 2 * kWyBlock * kWyBlock + 2 * static_cast<size_t>(kWyBlock) * m +
                static_cast<size_t>(kWySplit) * kWyBlock * wide);
}

int launch_hh_normalize_columns(int64_t n, int64_t m, double* d_C, int* d_zero, cudaStream_t st) {
    if (n <= 0 || m <= 0) return 0;
    k_normalize_columns<<<static_cast<unsigned>((m + 127) / 128), 128, 0, st>>>(n, m, reinterpret_cast<double2*>(d_C),
                                                                               d_zero);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

}  // namespace kbg
