// V_eff from rho on the grid: the step between the density
// pass (G3) and the Hamiltonian pass (G4) of one SCF iteration.
//   V_H:  Poisson in G space, V_H(G) = 4 pi rho(G) / |G|^2, V_H(G = 0) = 0
//         (neutralizing background); cuFFT D2Z / Z2D (library FFTs).
//   V_x:  local spin density exchange (Slater), V_x,s = -(6 rho_s / pi)^(1/3)
//         (nspin = 1: rho_s = rho / 2, i.e. -(3 rho / pi)^(1/3)).
//   V_c:  with KBG_OPT_XC = 1, the Perdew-Wang 1992 LSDA correlation (full LDA).
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

// rho_tot = sum_s rho_s -> real FFT input; a non-finite rho anywhere raises *bad
// (the host API turns it into KBG_ERR_NONFINITE before returning V_eff).
__global__ void k_rho_total(int64_t n, int nspin, const double* __restrict__ rho, double* __restrict__ out,
                            unsigned int* bad) {
    bool fin = true;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double r0 = rho[i], r1 = nspin == 2 ? rho[n + i] : 0.0;
        fin = fin && isfinite(r0) && isfinite(r1);
        out[i] = nspin == 2 ? r0 + r1 : r0;
    }
    if (bad && !__all_sync(0xffffffffu, fin) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
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

// Perdew-Wang 1992 LSDA correlation (Phys. Rev. B 45, 13244; Table I, p = 1,
// Hartree): G(rs) and dG/drs for eps_c(rs, 0), eps_c(rs, 1) and -alpha_c(rs).
__device__ __forceinline__ void pw92_g(double rs, double sr, double A, double a1, double b1, double b2, double b3,
                                       double b4, double& g, double& dg) {
    const double q0 = -2.0 * A * (1.0 + a1 * rs);
    const double q1 = 2.0 * A * (b1 * sr + b2 * rs + b3 * rs * sr + b4 * rs * rs);
    const double q1p = A * (b1 / sr + 2.0 * b2 + 3.0 * b3 * sr + 4.0 * b4 * rs);
    const double lg = log1p(1.0 / q1);
    g = q0 * lg;
    dg = -2.0 * A * a1 * lg - q0 * q1p / (q1 * q1 + q1);
}

// eps_c and v_c,up / v_c,down at total density n > 0, polarization zeta.
__device__ void pw92(double n, double zeta, double& eps, double& vu, double& vd) {
    zeta = fmin(1.0, fmax(-1.0, zeta));
    const double rs = cbrt(3.0 / (4.0 * kPi * n)), sr = sqrt(rs);
    double e0, d0, e1, d1, ma, dma;
    pw92_g(rs, sr, 0.031091, 0.21370, 7.5957, 3.5876, 1.6382, 0.49294, e0, d0);
    if (zeta == 0.0) {  // unpolarized: f(0) = f'(0) = 0, the other two fits drop out (same bits)
        eps = e0;
        vu = vd = e0 - rs / 3.0 * d0;
        return;
    }
    pw92_g(rs, sr, 0.015545, 0.20548, 14.1189, 6.1977, 3.3662, 0.62517, e1, d1);
    pw92_g(rs, sr, 0.016887, 0.11125, 10.357, 3.6231, 0.88026, 0.49671, ma, dma);
    const double ac = -ma, dac = -dma, fz0 = 1.709921;
    const double c43 = 0.5198420997897464;  // 2^(4/3) - 2
    const double cp = cbrt(1.0 + zeta), cm = cbrt(1.0 - zeta);
    const double f = ((1.0 + zeta) * cp + (1.0 - zeta) * cm - 2.0) / c43;
    const double fp = (4.0 / 3.0) * (cp - cm) / c43;
    const double z3 = zeta * zeta * zeta, z4 = z3 * zeta;
    eps = e0 + ac * f / fz0 * (1.0 - z4) + (e1 - e0) * f * z4;
    const double de_rs = d0 + dac * f / fz0 * (1.0 - z4) + (d1 - d0) * f * z4;
    const double de_z = ac / fz0 * (fp * (1.0 - z4) - 4.0 * z3 * f) + (e1 - e0) * (fp * z4 + 4.0 * z3 * f);
    const double common = eps - rs / 3.0 * de_rs - zeta * de_z;
    vu = common + de_z;
    vd = common - de_z;
}

// V_eff,s = V_H + V_x,s [+ V_c,s (xc = 1)] (+ V_loc); per-block partial energies (fixed order):
// part[0] sum V_H rho, part[1] sum_s rho_s^(4/3) (exchange), part[2] sum n eps_c.
template <int XC>
__global__ void __launch_bounds__(256) k_veff(int64_t n, int nspin, const double* __restrict__ rho,
                                              const double* __restrict__ vh, const double* __restrict__ vloc,
                                              double* __restrict__ veff, double* __restrict__ part) {
    const double cx = -cbrt(6.0 / kPi);  // V_x,s = cx rho_s^(1/3)
    double eh = 0.0, ex = 0.0, ec = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double h = vh[i];
        const double vl = vloc ? vloc[i] : 0.0;
        double rt = 0.0, sp[2] = {0.0, 0.0};
        for (int s = 0; s < nspin; ++s) {
            const double rs = nspin == 2 ? fmax(rho[s * n + i], 0.0) : 0.5 * fmax(rho[i], 0.0);
            const double c = cbrt(rs);
            sp[s] = rs;
            veff[s * n + i] = h + cx * c + vl;
            ex += (nspin == 2 ? 1.0 : 2.0) * rs * c;
            rt += nspin == 2 ? rho[s * n + i] : rho[i];
        }
        if (XC == 1) {
            const double up = sp[0], dn = nspin == 2 ? sp[1] : sp[0], nt = up + dn;
            if (nt > 1e-30) {
                double eps, vu, vd;
                pw92(nt, (up - dn) / nt, eps, vu, vd);
                veff[i] += vu;
                if (nspin == 2) veff[n + i] += vd;
                ec += nt * eps;
            }
        }
        eh += h * rt;
    }
    __shared__ double sh[3][8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        eh += __shfl_xor_sync(0xffffffffu, eh, o);
        ex += __shfl_xor_sync(0xffffffffu, ex, o);
        ec += __shfl_xor_sync(0xffffffffu, ec, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sh[0][threadIdx.x >> 5] = eh;
        sh[1][threadIdx.x >> 5] = ex;
        sh[2][threadIdx.x >> 5] = ec;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0, c = 0.0;
        for (int w = 0; w < 8; ++w) {
            a += sh[0][w];
            b += sh[1][w];
            c += sh[2][w];
        }
        part[3 * blockIdx.x] = a;
        part[3 * blockIdx.x + 1] = b;
        part[3 * blockIdx.x + 2] = c;
    }
}

// e[0] = E_H, e[1] = E_xc (exchange, plus PW92 correlation when xc = 1)
__global__ void k_energy_final(int nblk, const double* __restrict__ part, double dV, double* __restrict__ e) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double a = 0.0, b = 0.0, c = 0.0;
    for (int i = 0; i < nblk; ++i) {
        a += part[3 * i];
        b += part[3 * i + 1];
        c += part[3 * i + 2];
    }
    e[0] = 0.5 * a * dV;
    e[1] = -0.75 * cbrt(6.0 / kPi) * b * dV + c * dV;
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

int run_veff(VeffPlan& vp, const int N[3], const double Ainv[9], int nspin, int xc, const double* d_rho,
             const double* d_vloc, double dV, double* d_veff, double* d_energy, cudaStream_t st, unsigned int* d_bad) {
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
        KBG_CUDA(cudaMalloc(&vp.work, (nr + 2 * nc + 3 * sms_grid) * sizeof(double)));
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
    k_rho_total<<<sms_grid, 256, 0, st>>>(n, nspin, d_rho, real, d_bad);
    cufft_check(cufftExecD2Z(static_cast<cufftHandle>(vp.fwd), real, spec), "cufftExecD2Z");
    k_poisson<<<sms_grid, 256, 0, st>>>(N[0], N[1], N[2], vp.B, spec);
    cufft_check(cufftExecZ2D(static_cast<cufftHandle>(vp.inv), spec, real), "cufftExecZ2D");
    if (xc == 1)
        k_veff<1><<<sms_grid, 256, 0, st>>>(n, nspin, d_rho, real, d_vloc, d_veff, part);
    else
        k_veff<0><<<sms_grid, 256, 0, st>>>(n, nspin, d_rho, real, d_vloc, d_veff, part);
    if (d_energy) k_energy_final<<<1, 32, 0, st>>>(sms_grid, part, dV, d_energy);
    KBG_CUDA(cudaGetLastError());
    return 4 + (d_energy ? 1 : 0);
}

}  // namespace kbg
