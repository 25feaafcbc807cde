// Formats either side of the grid pass: the pair-sparse
// real-space blocks the grid kernels read (DM) and write (H) <-> the
// reference's RealSpaceOperator (dense n x n block per lattice offset R,
// /root/reference/SPEC.md:213-216), its Bloch image M(k) = sum_R
// exp(+2 pi i k.R) M_R (Part 1 bloch_transform) and the
// real-space folding of k-resolved density matrices DM(R) = sum_k w_k
// exp(-2 pi i k.R) rho_k (Part 6 density_matrices).
//
// All of these are HBM-bound gathers/scatters (a few flops per byte). The
// dense side is the large one (nk n^2 complex values vs nnz pair values), so
// the Bloch kernel maps consecutive threads to consecutive columns of one
// dense row (coalesced 16-byte stores); the pair-side kernels give each pair
// block to one warp. Every output element is produced by exactly one thread
// summing its terms in a fixed order (pair order over R, k order over k) --
// no atomics, bitwise deterministic.
#include "kb_internal.cuh"

namespace kbg {

namespace {

// (cos, sin)(2 pi sign k.R) per (k, pair): sincospi keeps the reduction exact.
__global__ void k_phase(int nk, int64_t npair, const double* __restrict__ kpts, const int32_t* __restrict__ pair_R,
                        double sign, double2* __restrict__ out) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= nk * npair) return;
    const int k = static_cast<int>(t / npair);
    const int64_t p = t - k * npair;
    const double* kk = kpts + 3 * k;
    const int32_t* R = pair_R + 3 * p;
    const double kr = (kk[0] * R[0] + kk[1] * R[1]) + kk[2] * R[2];
    double s, c;
    sincospi(2.0 * kr, &s, &c);
    out[t] = make_double2(c, sign * s);
}

// M(k)[row][col] = sum over the (a, b, R) pairs of the atom pair (a, b), in
// pair order, of phase(k, p) * M_p[i][j], for every k. blockIdx.x = row,
// threads over 256 consecutive columns; each thread reads its M entries once
// (L1 serves the re-reads) and writes its element of all nk images.
__global__ void __launch_bounds__(256) k_bloch(int nk, int n, int natom, const int32_t* __restrict__ orb_atom,
                                               const int32_t* __restrict__ orb_off, const int32_t* __restrict__ run,
                                               const int64_t* __restrict__ pair_off, int64_t npair,
                                               const double* __restrict__ M, const double2* __restrict__ phase,
                                               double2* __restrict__ out) {
    const int row = blockIdx.x;
    const int col = blockIdx.y * 256 + threadIdx.x;
    if (col >= n) return;
    const int a = orb_atom[row], b = orb_atom[col];
    const int i = row - orb_off[a], j = col - orb_off[b];
    const int nb = orb_off[b + 1] - orb_off[b];
    const int64_t ab = static_cast<int64_t>(a) * natom + b;
    const int p0 = run[2 * ab], p1 = run[2 * ab + 1];
    const int64_t nn = static_cast<int64_t>(n) * n, rc = static_cast<int64_t>(row) * n + col;
    for (int k = 0; k < nk; ++k) {
        double re = 0.0, im = 0.0;
        const double2* ph = phase + static_cast<int64_t>(k) * npair;
        for (int p = p0; p < p1; ++p) {
            const double v = M[pair_off[p] + i * nb + j];
            const double2 e = ph[p];
            re += e.x * v;
            im += e.y * v;
        }
        out[k * nn + rc] = make_double2(re, im);
    }
}

// One warp per atom pair (a, b) (8 per CTA): the pairs of its run share the
// rho_k block (same rows and columns, different R), so each element is read
// from HBM once per k and the run's other offsets hit L1.
// DM_p[i][j] = Re sum_k w_k exp(-2 pi i k.R_p) rho_k[row][col]; the largest
// |imaginary part| goes to *max_imag (bit pattern, atomicMax on >= 0 doubles).
__global__ void __launch_bounds__(256) k_fold(int nk, int n, int nrun, const int32_t* __restrict__ runs,
                                              const int32_t* __restrict__ pair_a, const int32_t* __restrict__ pair_b,
                                              const int64_t* __restrict__ pair_off, int64_t npair,
                                              const int32_t* __restrict__ orb_off, const double* __restrict__ w,
                                              const double2* __restrict__ phase, const double2* __restrict__ rho_k,
                                              double* __restrict__ out, unsigned long long* max_imag) {
    const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    double im_abs = 0.0;
    if (r < nrun) {
        const int p0 = runs[r], p1 = runs[r + 1];
        const int a = pair_a[p0], b = pair_b[p0];
        const int nb = orb_off[b + 1] - orb_off[b], ne = (orb_off[a + 1] - orb_off[a]) * nb;
        const int64_t nn = static_cast<int64_t>(n) * n;
        for (int q = lane; q < ne; q += 32) {
            const int64_t rc = static_cast<int64_t>(orb_off[a] + q / nb) * n + orb_off[b] + q % nb;
            for (int p = p0; p < p1; ++p) {
                double re = 0.0, im = 0.0;
#pragma unroll 4
                for (int k = 0; k < nk; ++k) {
                    const double2 x = rho_k[k * nn + rc];
                    const double2 c = phase[static_cast<int64_t>(k) * npair + p];  // (cos, -sin)
                    re += w[k] * (c.x * x.x - c.y * x.y);
                    im += w[k] * (c.x * x.y + c.y * x.x);
                }
                out[pair_off[p] + q] = re;
                im_abs = fmax(im_abs, fabs(im));
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) im_abs = fmax(im_abs, __shfl_xor_sync(0xffffffffu, im_abs, o));
    if (lane == 0 && max_imag) atomicMax(max_imag, static_cast<unsigned long long>(__double_as_longlong(im_abs)));
}

// pair-sparse <-> dense blocks [nR][n][n], one warp per pair; to_dense:
// dense[rid][row][col] = x[e], else x[e] = dense[...].
__global__ void __launch_bounds__(256) k_realspace(int n, int64_t npair, const int32_t* __restrict__ pair_a,
                                                   const int32_t* __restrict__ pair_b,
                                                   const int64_t* __restrict__ pair_off,
                                                   const int32_t* __restrict__ rid,
                                                   const int32_t* __restrict__ orb_off, bool to_dense,
                                                   double* __restrict__ sparse, double* __restrict__ dense) {
    const int64_t p = blockIdx.x * 8ll + (threadIdx.x >> 5);
    if (p >= npair) return;
    const int a = pair_a[p], b = pair_b[p];
    const int nb = orb_off[b + 1] - orb_off[b], ne = (orb_off[a + 1] - orb_off[a]) * nb;
    const int64_t base = (static_cast<int64_t>(rid[p]) * n + orb_off[a]) * n + orb_off[b];
    for (int q = threadIdx.x & 31; q < ne; q += 32) {
        const int64_t d = base + static_cast<int64_t>(q / nb) * n + q % nb;
        if (to_dense)
            dense[d] = sparse[pair_off[p] + q];
        else
            sparse[pair_off[p] + q] = dense[d];
    }
}

// D[r][i] = w[i] * C[r][i] (complex C, real weights), row-major n x m.
__global__ void k_scale_states(int64_t total, int m, const double2* __restrict__ C, const double* __restrict__ w,
                               double2* __restrict__ D) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= total) return;
    const double f = w[t % m];
    const double2 c = C[t];
    D[t] = make_double2(f * c.x, f * c.y);
}

unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

int launch_phase(int nk, int64_t npair, const double* d_kpts, const int32_t* pair_R, double sign, double2* d_phase,
                 cudaStream_t st) {
    if (nk * npair == 0) return 0;
    k_phase<<<blocks_for(nk * npair, 256), 256, 0, st>>>(nk, npair, d_kpts, pair_R, sign, d_phase);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

int launch_bloch(const FormatIndex& f, const DevIndex& ix, int nk, const double* d_M, const double2* d_phase,
                 double* d_out, cudaStream_t st) {
    if (f.n == 0) return 0;
    const dim3 grid(static_cast<unsigned>(f.n), blocks_for(f.n, 256));
    k_bloch<<<grid, 256, 0, st>>>(nk, f.n, f.natom, f.orb_atom, f.orb_off, f.run, ix.pair_off, ix.npair, d_M, d_phase,
                                  reinterpret_cast<double2*>(d_out));
    KBG_CUDA(cudaGetLastError());
    return 1;
}

int launch_fold(const FormatIndex& f, const DevIndex& ix, int nk, const double* d_w, const double2* d_phase,
                const double* d_rho_k, double* d_out, unsigned long long* d_max_imag, cudaStream_t st) {
    if (f.nrun == 0) return 0;
    k_fold<<<blocks_for(f.nrun, 8), 256, 0, st>>>(nk, f.n, f.nrun, f.runs, ix.pair_a, ix.pair_b, ix.pair_off,
                                                  ix.npair, f.orb_off, d_w, d_phase,
                                                  reinterpret_cast<const double2*>(d_rho_k), d_out, d_max_imag);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

int launch_realspace(const FormatIndex& f, const DevIndex& ix, bool to_dense, double* d_sparse, double* d_dense,
                     cudaStream_t st) {
    if (ix.npair == 0) return 0;
    k_realspace<<<blocks_for(ix.npair, 8), 256, 0, st>>>(f.n, ix.npair, ix.pair_a, ix.pair_b, ix.pair_off, f.rid,
                                                         f.orb_off, to_dense, d_sparse, d_dense);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

int launch_scale_states(int n, int m, const double* d_C, const double* d_w, double* d_D, cudaStream_t st) {
    const int64_t total = static_cast<int64_t>(n) * m;
    if (total == 0) return 0;
    k_scale_states<<<blocks_for(total, 256), 256, 0, st>>>(total, m, reinterpret_cast<const double2*>(d_C), d_w,
                                                           reinterpret_cast<double2*>(d_D));
    KBG_CUDA(cudaGetLastError());
    return 1;
}

void free_formats(FormatIndex& f) {
    for (void* p : {static_cast<void*>(f.orb_atom), static_cast<void*>(f.orb_off), static_cast<void*>(f.run),
                    static_cast<void*>(f.rid), static_cast<void*>(f.runs)})
        if (p) cudaFree(p);
    f = FormatIndex();
}

}  // namespace kbg
