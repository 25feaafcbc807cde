// V_eff from rho on the grid: the step between the density
// pass (G3) and the Hamiltonian pass (G4) of one SCF iteration.
//   V_H:  Poisson in G space, V_H(G) = 4 pi rho(G) / |G|^2, V_H(G = 0) = 0
//         (neutralizing background); cuFFT D2Z / Z2D (library FFTs).
//   V_x:  exchange-only local spin density (Slater), V_x,s = -(6 rho_s / pi)^(1/3)
//         (nspin = 1: rho_s = rho / 2, i.e. -(3 rho / pi)^(1/3)).
//   V_eff,s = V_H + V_x,s + V_loc (V_loc optional).
// Energies: E_H = 1/2 sum V_H rho dV, E_x = -3/4 (6/pi)^(1/3) sum_s sum rho_s^(4/3) dV,
// reduced in a fixed order (two passes) -> deterministic.
// Hartree atomic units; rho in e/bohr^3, C-order grid (k fastest), like the
// density pass writes it. Elementwise work is HBM-bound: one read of rho and
// V_loc, one write of V_eff per spin, plus the FFT round trip.
#include <cufft.h>

#include <cmath>

#include "kb_internal.cuh"

namespace kbg {

namespace {

constexpr double kPi = 3.14159265358979323846;

// rho_tot = sum_s rho_s -> real FFT input
__global__ void k_rho_total(int64_t n, int nspin, const double* __restrict__ rho, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = nspin == 2 ? rho[i] + rho[n + i] : rho[i];
}

// rho(G) -> V_H(G) (with the 1/N of the inverse transform folded in).
// G = 2 pi (m1 b1 + m2 b2 + m3 b3), b_i rows of A^-T; m wrapped to (-N/2, N/2].
__global__ void k_poisson(int N0, int N1, int N2, const double* __restrict__ B, cufftDoubleComplex* __restrict__ f) {
    const int H2 = N2 / 2 + 1;
    const int64_t total = static_cast<int64_t>(N0) * N1 * H2;
    const double scale = 4.0 * kPi / (static_cast<double>(N0) * N1 * N2);
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int k = static_cast<int>(t % H2);
        const int64_t r = t / H2;
        const int j = static_cast<int>(r % N1), i = static_cast<int>(r / N1);
        const int m0 = i <= N0 / 2 ? i : i - N0, m1 = j <= N1 / 2 ? j : j - N1, m2 = k;
        double g[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) g[c] = 2.0 * kPi * (m0 * B[c] + m1 * B[3 + c] + m2 * B[6 + c]);
        const double g2 = g[0] * g[0] + g[1] * g[1] + g[2] * g[2];
        const double s = (m0 == 0 && m1 == 0 && m2 == 0) ? 0.0 : scale / g2;
        f[t].x *= s;
        f[t].y *= s;
    }
}

// V_eff,s = V_H + V_x,s (+ V_loc); per-block partial energies (fixed order).
__global__ void __launch_bounds__(256) k_veff(int64_t n, int nspin, const double* __restrict__ rho,
                                              const double* __restrict__ vh, const double* __restrict__ vloc,
                                              double* __restrict__ veff, double* __restrict__ part) {
    const double cx = -cbrt(6.0 / kPi);  // V_x,s = cx rho_s^(1/3)
    double eh = 0.0, ex = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double h = vh[i];
        const double vl = vloc ? vloc[i] : 0.0;
        double rt = 0.0;
        for (int s = 0; s < nspin; ++s) {
            const double rs = nspin == 2 ? fmax(rho[s * n + i], 0.0) : 0.5 * fmax(rho[i], 0.0);
            const double c = cbrt(rs);
            veff[s * n + i] = h + cx * c + vl;
            ex += (nspin == 2 ? 1.0 : 2.0) * rs * c;
            rt += nspin == 2 ? rho[s * n + i] : rho[i];
        }
        eh += h * rt;
    }
    __shared__ double sh[2][8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        eh += __shfl_xor_sync(0xffffffffu, eh, o);
        ex += __shfl_xor_sync(0xffffffffu, ex, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sh[0][threadIdx.x >> 5] = eh;
        sh[1][threadIdx.x >> 5] = ex;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < 8; ++w) {
            a += sh[0][w];
            b += sh[1][w];
        }
        part[2 * blockIdx.x] = a;
        part[2 * blockIdx.x + 1] = b;
    }
}

__global__ void k_energy_final(int nblk, const double* __restrict__ part, double dV, double* __restrict__ e) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double a = 0.0, b = 0.0;
    for (int i = 0; i < nblk; ++i) {
        a += part[2 * i];
        b += part[2 * i + 1];
    }
    e[0] = 0.5 * a * dV;
    e[1] = -0.75 * cbrt(6.0 / kPi) * b * dV;
}

void cufft_check(cufftResult r, const char* what) {
    if (r != CUFFT_SUCCESS) throw Error(KBG_ERR_CUDA, std::string(what) + ": cuFFT error " + std::to_string(r));
}

}  // namespace

void VeffPlan::release() {
    if (planned) {
        cufftDestroy(static_cast<cufftHandle>(fwd));
        cufftDestroy(static_cast<cufftHandle>(inv));
    }
    if (work) cudaFree(work);
    if (B) cudaFree(B);
    *this = VeffPlan();
}

int run_veff(VeffPlan& vp, const int N[3], const double Ainv[9], int nspin, const double* d_rho, const double* d_vloc,
             double dV, double* d_veff, double* d_energy, cudaStream_t st) {
    const int64_t n = static_cast<int64_t>(N[0]) * N[1] * N[2];
    const int64_t nc = static_cast<int64_t>(N[0]) * N[1] * (N[2] / 2 + 1);
    const int64_t nr = (n + 1) & ~int64_t(1);  // complex spectrum 16-byte aligned
    const int sms_grid = 148 * 4;
    if (!vp.planned) {
        cufftHandle f, i;
        cufft_check(cufftPlan3d(&f, N[0], N[1], N[2], CUFFT_D2Z), "cufftPlan3d D2Z");
        cufft_check(cufftPlan3d(&i, N[0], N[1], N[2], CUFFT_Z2D), "cufftPlan3d Z2D");
        vp.fwd = static_cast<int>(f);
        vp.inv = static_cast<int>(i);
        // work: real grid (rho_tot, then V_H) | complex half spectrum | energy partials
        KBG_CUDA(cudaMalloc(&vp.work, (nr + 2 * nc + 2 * sms_grid) * sizeof(double)));
        // reciprocal basis b_i = rows of A^-T: (A^-1)^T rows = columns of A^-1
        double Bh[9];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) Bh[3 * r + c] = Ainv[3 * c + r];
        KBG_CUDA(cudaMalloc(&vp.B, 9 * sizeof(double)));
        KBG_CUDA(cudaMemcpy(vp.B, Bh, sizeof(Bh), cudaMemcpyHostToDevice));
        vp.planned = true;
    }
    double* real = vp.work;
    cufftDoubleComplex* spec = reinterpret_cast<cufftDoubleComplex*>(vp.work + nr);
    double* part = vp.work + nr + 2 * nc;
    cufft_check(cufftSetStream(static_cast<cufftHandle>(vp.fwd), st), "cufftSetStream");
    cufft_check(cufftSetStream(static_cast<cufftHandle>(vp.inv), st), "cufftSetStream");
    k_rho_total<<<sms_grid, 256, 0, st>>>(n, nspin, d_rho, real);
    cufft_check(cufftExecD2Z(static_cast<cufftHandle>(vp.fwd), real, spec), "cufftExecD2Z");
    k_poisson<<<sms_grid, 256, 0, st>>>(N[0], N[1], N[2], vp.B, spec);
    cufft_check(cufftExecZ2D(static_cast<cufftHandle>(vp.inv), spec, real), "cufftExecZ2D");
    k_veff<<<sms_grid, 256, 0, st>>>(n, nspin, d_rho, real, d_vloc, d_veff, part);
    if (d_energy) k_energy_final<<<1, 32, 0, st>>>(sms_grid, part, dV, d_energy);
    KBG_CUDA(cudaGetLastError());
    return 4 + (d_energy ? 1 : 0);
}

}  // namespace kbg
