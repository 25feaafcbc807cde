// C shim over the reference's own kband library -- TEST INFRASTRUCTURE.
//
// oracle/Makefile (target `ref`) compiles this file together with the
// reference's sources where they lie (/root/reference/proj/src/{common,
// householder,linalg,tridiag}.cpp; no copies) into oracle/_ref/libkband_ref.so.
// It pins the GPU Eigen_HH pieces to the reference itself:
//   tridiagonalize   /root/reference/proj/src/householder.cpp:60-251
//   back_transform   householder.cpp:253-305
//   normalize_columns householder.cpp:307-331
//   solve_tridiag    tridiag.cpp:14-110 (the host step the paper keeps on CPUs)
//   eigen_hh         householder.cpp:333-351
// Only tests/ and bench.py's reference leg load it. Complex arrays are
// interleaved (re, im) doubles, row-major.
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>

#include "kband/householder.hpp"
#include "kband/linalg.hpp"
#include "kband/tridiag.hpp"

using kband::Complex;

namespace {

thread_local char g_err[512];

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_err[0] = 0;
        return 0;
    } catch (const kband::DimensionError& e) {
        std::strncpy(g_err, e.what(), sizeof(g_err) - 1);
        return 2;
    } catch (const kband::ConsistencyError& e) {
        std::strncpy(g_err, e.what(), sizeof(g_err) - 1);
        return 3;
    } catch (const kband::ConvergenceError& e) {
        std::strncpy(g_err, e.what(), sizeof(g_err) - 1);
        return 4;
    } catch (const std::exception& e) {
        std::strncpy(g_err, e.what(), sizeof(g_err) - 1);
        return 1;
    }
}

kband::HermitianMatrix hermitian(int64_t n, const double* a) {
    kband::DenseMatrix m(n, n);
    std::memcpy(static_cast<void*>(m.data()), a, sizeof(Complex) * n * n);
    return kband::HermitianMatrix::from(std::move(m));
}

kband::ThreadTeam* team_of(int threads, kband::ThreadTeam& storage) { return threads > 1 ? &storage : nullptr; }

}  // namespace

extern "C" {

const char* kbr_last_error() { return g_err; }

// Records: u [(n-1) x n] complex (row i = reflector of stage i, zeros when
// skipped), h, s [n-1], phase [n-1] complex.
int kbr_tridiagonalize(int64_t n, const double* a, int fault_sign, double* d, double* e, double* u, double* h,
                       double* s, double* phase) {
    return guarded([&] {
        kband::ProcedurePlan plan = kband::ProcedurePlan::host_serial();
        plan.fault_proc6_sign = fault_sign != 0;
        const kband::TridiagReal t = kband::tridiagonalize(hermitian(n, a), plan);
        std::memcpy(d, t.d.data(), sizeof(double) * n);
        if (n > 1) std::memcpy(e, t.e.data(), sizeof(double) * (n - 1));
        for (int64_t i = 0; i + 1 < n; ++i) {
            const auto& r = t.records[i];
            h[i] = r.h;
            s[i] = r.s;
            phase[2 * i] = r.phase.real();
            phase[2 * i + 1] = r.phase.imag();
            double* ui = u + 2 * i * n;
            if (r.u.empty())
                std::memset(ui, 0, sizeof(double) * 2 * n);
            else
                std::memcpy(ui, r.u.data(), sizeof(Complex) * n);
        }
    });
}

// W = back_transform(records, Y): Y real [n x m] (tridiagonal eigenvectors), W complex [n x m].
int kbr_back_transform(int64_t n, int64_t m, const double* u, const double* h, const double* s,
                       const double* phase, const double* y, double* w, int threads) {
    return guarded([&] {
        std::vector<kband::HouseholderRecord> recs(n > 0 ? n - 1 : 0);
        for (int64_t i = 0; i + 1 < n; ++i) {
            auto& r = recs[i];
            r.stage = static_cast<std::size_t>(i);
            r.h = h[i];
            r.s = s[i];
            r.phase = Complex(phase[2 * i], phase[2 * i + 1]);
            if (r.h != 0.0) {
                r.u.resize(n);
                std::memcpy(static_cast<void*>(r.u.data()), u + 2 * i * n, sizeof(Complex) * n);
            }
        }
        kband::DenseMatrix Y(n, m);
        for (int64_t i = 0; i < n * m; ++i) Y.data()[i] = Complex(y[i], 0.0);
        kband::ThreadTeam team(threads > 1 ? threads : 1);
        const kband::DenseMatrix W = kband::back_transform(recs, Y, team_of(threads, team));
        std::memcpy(w, static_cast<const void*>(W.data()), sizeof(Complex) * n * m);
    });
}

int kbr_normalize_columns(int64_t n, int64_t m, double* c) {
    return guarded([&] {
        kband::DenseMatrix C(n, m);
        std::memcpy(static_cast<void*>(C.data()), c, sizeof(Complex) * n * m);
        const kband::DenseMatrix O = kband::normalize_columns(C);
        std::memcpy(c, static_cast<const void*>(O.data()), sizeof(Complex) * n * m);
    });
}

// Eigenvalues ascending [n]; z real [n x n] (column j = eigenvector j) if want_vectors.
int kbr_solve_tridiag(int64_t n, const double* d, const double* e, int want_vectors, double* evals, double* z) {
    return guarded([&] {
        kband::TridiagProblem p;
        p.d.assign(d, d + n);
        p.e.assign(e, e + (n > 0 ? n - 1 : 0));
        const kband::TridiagEigenResult r = kband::solve_tridiag(p, want_vectors != 0);
        std::memcpy(evals, r.eigenvalues.data(), sizeof(double) * n);
        if (want_vectors)
            for (int64_t i = 0; i < n * n; ++i) z[i] = r.eigenvectors->data()[i].real();
    });
}

// T^H H T (linalg.cpp triple_product): t [n x m], h [n x n] Hermitian, c [m x m].
int kbr_triple_product(int64_t n, int64_t m, const double* t, const double* h, double* c) {
    return guarded([&] {
        kband::DenseMatrix T(n, m);
        std::memcpy(static_cast<void*>(T.data()), t, sizeof(Complex) * n * m);
        const kband::HermitianMatrix C = kband::triple_product(T, hermitian(n, h));
        std::memcpy(c, static_cast<const void*>(C.dense().data()), sizeof(Complex) * m * m);
    });
}

// Full reference eigensolver; vectors complex [n x n] (columns) if want_vectors.
int kbr_eigen_hh(int64_t n, const double* a, int want_vectors, int threads, double* evals, double* vecs) {
    return guarded([&] {
        kband::ThreadTeam team(threads > 1 ? threads : 1);
        const kband::ProcedurePlan plan =
            threads > 1 ? kband::ProcedurePlan::host_threaded() : kband::ProcedurePlan::host_serial();
        const kband::EigenResult r = kband::eigen_hh(hermitian(n, a), want_vectors != 0, plan, team_of(threads, team));
        std::memcpy(evals, r.eigenvalues.data(), sizeof(double) * n);
        if (want_vectors) std::memcpy(vecs, static_cast<const void*>(r.eigenvectors->data()), sizeof(Complex) * n * n);
    });
}

}  // extern "C"
