// kbgrid.hpp -- C++ host interface over the kbgrid C-ABI, in the reference's
// conventions (header-only).
//
// This is what kband's band pipeline would call between Part 6
// (density_matrices) and Part 1
// (bloch_transform): free-function style, inputs by const&,
// results returned by value (/root/reference/proj/include/kband/linalg.hpp:75-80),
// failures thrown as the kband error taxonomy (common.hpp:21-38) with the
// library's message naming the failing field or index.
//
// Define KBG_USE_KBAND_ERRORS before including this header inside the kband
// tree to throw kband::ConfigError etc. directly; otherwise kbg::ConfigError
// etc. (same names, same hierarchy) are used.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "kbgrid.h"

#ifdef KBG_USE_KBAND_ERRORS
#include "kband/common.hpp"
#endif

namespace kbg {

#ifdef KBG_USE_KBAND_ERRORS
using Error = kband::Error;
using ConfigError = kband::ConfigError;
using DimensionError = kband::DimensionError;
using ConsistencyError = kband::ConsistencyError;
using ConvergenceError = kband::ConvergenceError;
#else
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct DimensionError : Error {
    using Error::Error;
};
struct ConsistencyError : Error {
    using Error::Error;
};
struct ConvergenceError : Error {
    using Error::Error;
};
#endif
struct DeviceError : Error {
    using Error::Error;
};

inline void throw_status(int st, const std::string& what) {
    switch (st) {
        case KBG_OK: return;
        case KBG_ERR_CONFIG: throw ConfigError(what);
        case KBG_ERR_DIMENSION: throw DimensionError(what);
        case KBG_ERR_CONSISTENCY: throw ConsistencyError(what);
        case KBG_ERR_NONFINITE: throw ConvergenceError(what);
        default: throw DeviceError(what);
    }
}

// Pair-sparse real-space blocks (DM in, H out): the layout of kbg_index.
struct PairList {
    std::vector<int32_t> a, b, R;     // R: 3 per pair
    std::vector<int64_t> off;         // npair + 1
    std::vector<int32_t> mirror;      // index of (b, a, -R)
    int64_t nnz = 0;
};

// One grid pass context (one GPU, or one shard of a multi-GPU grid).
class GridPass {
public:
    GridPass(const kbg_system& sys, int device = 0, int rank = 0, int nranks = 1) {
        const int st = kbg_create_sharded(&sys, device, rank, nranks, &ctx_);
        if (st != KBG_OK) throw_status(st, std::string("kbg_create: ") + kbg_status_string(st));
    }
    ~GridPass() { kbg_destroy(ctx_); }
    GridPass(const GridPass&) = delete;
    GridPass& operator=(const GridPass&) = delete;
    GridPass(GridPass&& o) noexcept : ctx_(std::exchange(o.ctx_, nullptr)) {}

    // Index build (once per geometry): bit-exact lists, task lists and the
    // orbital cache.
    void build_index() { check(kbg_build_index(ctx_), "kbg_build_index"); }

    kbg_index view() const {
        kbg_index ix;
        check(kbg_index_view(ctx_, &ix), "kbg_index_view");
        return ix;
    }

    PairList pairs() const {
        const kbg_index ix = view();
        PairList p;
        p.a.assign(ix.pair_a, ix.pair_a + ix.npair);
        p.b.assign(ix.pair_b, ix.pair_b + ix.npair);
        p.R.assign(ix.pair_R, ix.pair_R + 3 * ix.npair);
        p.off.assign(ix.pair_off, ix.pair_off + ix.npair + 1);
        p.mirror.assign(ix.pair_mirror, ix.pair_mirror + ix.npair);
        p.nnz = ix.nnz;
        return p;
    }

    // rho[nspin][npts] = sum_ab phi_a DM_ab phi_b   (dm: [nspin][nnz])
    std::vector<double> density(const std::vector<double>& dm, int nspin = 1) const {
        const kbg_index ix = view();
        if (static_cast<int64_t>(dm.size()) != nspin * ix.nnz)
            throw DimensionError("density: dm has " + std::to_string(dm.size()) + " values, expected nspin*nnz = " +
                                 std::to_string(nspin * ix.nnz));
        std::vector<double> rho(static_cast<size_t>(nspin) * ix.npts);
        check(kbg_density(ctx_, nspin, dm.data(), rho.data()), "kbg_density");
        return rho;
    }

    // h[nspin][nnz] = sum_r phi_a V dV phi_b   (veff: [nspin][npts])
    std::vector<double> hamiltonian(const std::vector<double>& veff, double dV, int nspin = 1) const {
        const kbg_index ix = view();
        if (static_cast<int64_t>(veff.size()) != nspin * ix.npts)
            throw DimensionError("hamiltonian: veff has " + std::to_string(veff.size()) +
                                 " values, expected nspin*npts = " + std::to_string(nspin * ix.npts));
        std::vector<double> h(static_cast<size_t>(nspin) * ix.nnz);
        check(kbg_hamiltonian(ctx_, nspin, veff.data(), dV, h.data()), "kbg_hamiltonian");
        return h;
    }

    // One SCF grid pass (kbg_grid_pass): rho from dm and h from veff, the two halves overlapped on two
    // streams; pinned host buffers are read / written in place by the kernels.
    std::pair<std::vector<double>, std::vector<double>> grid_pass(const std::vector<double>& dm,
                                                                  const std::vector<double>& veff, double dV,
                                                                  int nspin = 1) const {
        const kbg_index ix = view();
        if (static_cast<int64_t>(dm.size()) != nspin * ix.nnz || static_cast<int64_t>(veff.size()) != nspin * ix.npts)
            throw DimensionError("grid_pass: dm must hold nspin*nnz and veff nspin*npts values");
        std::vector<double> rho(static_cast<size_t>(nspin) * ix.npts), h(static_cast<size_t>(nspin) * ix.nnz);
        check(kbg_grid_pass(ctx_, nspin, dm.data(), veff.data(), dV, rho.data(), h.data()), "kbg_grid_pass");
        return {std::move(rho), std::move(h)};
    }

    // Device-pointer variants (stream = cudaStream_t).
    void density_dev(int nspin, const double* d_dm, double* d_rho, void* stream = nullptr) const {
        check(kbg_density_dev(ctx_, nspin, d_dm, d_rho, stream), "kbg_density_dev");
    }
    void hamiltonian_dev(int nspin, const double* d_veff, double dV, double* d_h, void* stream = nullptr) const {
        check(kbg_hamiltonian_dev(ctx_, nspin, d_veff, dV, d_h, stream), "kbg_hamiltonian_dev");
    }

    kbg_tally tally() const {
        kbg_tally t;
        check(kbg_last_tally(ctx_, &t), "kbg_last_tally");
        return t;
    }

    kbg_ctx* handle() const { return ctx_; }

private:
    void check(int st, const char* what) const {
        if (st != KBG_OK) throw_status(st, std::string(what) + ": " + kbg_last_error(ctx_));
    }
    kbg_ctx* ctx_ = nullptr;
};

// ---- Eigen_HH (kband::eigen_hh / solve_tridiag, householder.hpp:78-80, tridiag.hpp:18-21) ----
struct EigenResult {
    std::vector<double> eigenvalues;   // ascending
    std::vector<double> eigenvectors;  // [n][n] complex interleaved (re, im), columns; empty if not wanted
};

// a: [n][n] Hermitian, complex interleaved row-major; the whole pipeline device-resident.
inline EigenResult eigen_hh(int64_t n, const std::vector<double>& a, bool want_vectors = true) {
    if (static_cast<int64_t>(a.size()) != 2 * n * n) throw DimensionError("eigen_hh: a must hold 2*n*n doubles");
    EigenResult r;
    r.eigenvalues.resize(n);
    if (want_vectors) r.eigenvectors.resize(2 * n * n);
    const int st = kbg_hh_eigen(n, a.data(), want_vectors ? 1 : 0, r.eigenvalues.data(),
                                want_vectors ? r.eigenvectors.data() : nullptr);
    if (st != KBG_OK) throw_status(st, std::string("kbg_hh_eigen: ") + kbg_hh_last_error());
    return r;
}

// Real symmetric tridiagonal (d [n], e [n-1]); eigenvectors as the columns of a real [n][n].
inline std::pair<std::vector<double>, std::vector<double>> solve_tridiag(const std::vector<double>& d,
                                                                         const std::vector<double>& e,
                                                                         bool want_vectors = true) {
    const int64_t n = static_cast<int64_t>(d.size());
    if (n < 1 || static_cast<int64_t>(e.size()) + 1 != n)
        throw DimensionError("solve_tridiag: off-diagonal length must be n-1");
    std::vector<double> w(n), z(want_vectors ? n * n : 0), ee = e;
    if (ee.empty()) ee.push_back(0.0);
    const int st = kbg_tridiag_solve(n, d.data(), ee.data(), want_vectors ? 1 : 0, w.data(),
                                     want_vectors ? z.data() : nullptr);
    if (st != KBG_OK) throw_status(st, std::string("kbg_tridiag_solve: ") + kbg_hh_last_error());
    return {std::move(w), std::move(z)};
}

}  // namespace kbg
