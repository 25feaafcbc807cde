// C++ host over the kbgrid C-ABI (include/kbgrid.hpp), as kband's pipeline
// would use it: synthetic Fe3O4 primitive cell -> index -> rho and H on the
// GPU -> electron-count identity sum_r rho dV = sum_ab Tr(DM_ab S_ba) and the
// kband-style error taxonomy. Exit code 0 on success. Run by
// tests/test_gpu_cpp_host.py.
#include <cmath>
#include <cstdio>
#include <vector>

#include "kbgrid.hpp"
#include "kbgsynth.h"

int main() {
    kbg_synth* s = nullptr;
    if (kbg_synth_create(KBG_CELL_PRIMITIVE, 1, 100.0, 1402, 1024, &s) != KBG_OK) return 2;
    const kbg_system* sys = kbg_synth_system(s);
    const double dV = kbg_synth_dV(s);
    try {
        kbg::GridPass gp(*sys, 0);
        gp.build_index();
        const kbg_index ix = gp.view();
        std::vector<double> dm(ix.nnz), veff(ix.npts), ones(ix.npts, 1.0);
        kbg_synth_dm(s, &ix, 1, 1402, dm.data());
        kbg_synth_veff(s, 1, 1402, veff.data());
        const std::vector<double> rho = gp.density(dm);
        const std::vector<double> S = gp.hamiltonian(ones, dV);
        const std::vector<double> H = gp.hamiltonian(veff, dV);
        const kbg::PairList pl = gp.pairs();
        std::vector<int> norb(sys->natom);
        for (int a = 0; a < sys->natom; ++a) {
            const kbg_species& sp = sys->spec[sys->species[a]];
            norb[a] = 0;
            for (int r = 0; r < sp.nrad; ++r) norb[a] += 2 * sp.l[r] + 1;
        }
        double ne = 0.0, tr = 0.0, e = 0.0, trh = 0.0;
        for (int64_t p = 0; p < ix.npts; ++p) {
            ne += rho[p] * dV;
            e += rho[p] * veff[p] * dV;
        }
        for (size_t p = 0; p + 1 < pl.off.size(); ++p) {
            const int na = norb[pl.a[p]], nb = norb[pl.b[p]];
            const int64_t q = pl.mirror[p];
            for (int i = 0; i < na; ++i)
                for (int j = 0; j < nb; ++j) {
                    tr += dm[pl.off[p] + i * nb + j] * S[pl.off[q] + j * na + i];
                    trh += dm[pl.off[p] + i * nb + j] * H[pl.off[q] + j * na + i];
                }
        }
        std::printf("electrons: grid %.15f  Tr(DM S) %.15f\nenergy:    grid %.15f  Tr(DM H) %.15f\n", ne, tr, e, trh);
        if (std::fabs(ne - tr) > 1e-10 * std::fmax(1.0, std::fabs(ne))) return 3;
        if (std::fabs(e - trh) > 1e-10 * std::fmax(1.0, std::fabs(e))) return 4;
        // the one-call SCF drop-in gives the same rho bitwise and H within atomics' rounding
        const auto [rho2, H2] = gp.grid_pass(dm, veff, dV);
        for (int64_t p = 0; p < ix.npts; ++p)
            if (rho2[p] != rho[p]) return 7;
        double hmax = 0.0, hdiff = 0.0;
        for (int64_t p = 0; p < ix.nnz; ++p) {
            hmax = std::fmax(hmax, std::fabs(H[p]));
            hdiff = std::fmax(hdiff, std::fabs(H2[p] - H[p]));
        }
        if (hdiff > 1e-13 * hmax) return 8;
        // Eigen_HH end to end on a small Hermitian matrix: residual || A c - eps c ||
        {
            const int64_t n = 40;
            std::vector<double> a(2 * n * n);
            for (int64_t i = 0; i < n; ++i)
                for (int64_t j = 0; j <= i; ++j) {
                    const double re = std::cos(0.37 * (i + 1) * (j + 2)), im = i == j ? 0.0 : std::sin(0.11 * (i + 3) * j);
                    a[2 * (i * n + j)] = re;
                    a[2 * (i * n + j) + 1] = im;
                    a[2 * (j * n + i)] = re;
                    a[2 * (j * n + i) + 1] = -im;
                }
            const kbg::EigenResult er = kbg::eigen_hh(n, a);
            double res = 0.0;
            for (int64_t k = 0; k < n; ++k)
                for (int64_t i = 0; i < n; ++i) {
                    double sr = -er.eigenvalues[k] * er.eigenvectors[2 * (i * n + k)];
                    double si = -er.eigenvalues[k] * er.eigenvectors[2 * (i * n + k) + 1];
                    for (int64_t j = 0; j < n; ++j) {
                        const double ar = a[2 * (i * n + j)], ai = a[2 * (i * n + j) + 1];
                        const double cr = er.eigenvectors[2 * (j * n + k)], ci = er.eigenvectors[2 * (j * n + k) + 1];
                        sr += ar * cr - ai * ci;
                        si += ar * ci + ai * cr;
                    }
                    res = std::fmax(res, std::hypot(sr, si));
                }
            std::printf("eigen_hh n=%lld: max residual %.3e\n", static_cast<long long>(n), res);
            if (res > 1e-10 * n) return 9;
        }
        bool threw = false;
        try {
            gp.density(std::vector<double>(3));
        } catch (const kbg::DimensionError& err) {
            threw = true;
            std::printf("DimensionError as expected: %s\n", err.what());
        }
        if (!threw) return 5;
        threw = false;
        std::vector<double> bad = dm;
        bad[0] += 1.0;
        try {
            gp.density(bad);
        } catch (const kbg::ConsistencyError& err) {
            threw = true;
            std::printf("ConsistencyError as expected: %s\n", err.what());
        }
        if (!threw) return 6;
    } catch (const kbg::Error& err) {
        std::fprintf(stderr, "kbg error: %s\n", err.what());
        kbg_synth_free(s);
        return 1;
    }
    kbg_synth_free(s);
    std::printf("grid_pass_demo ok\n");
    return 0;
}
