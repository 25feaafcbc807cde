/*
 * oracle.h -- CPU oracle for the NAO grid pass (liboracle.so).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker / the timed CPU baseline. The product (libkbgrid.so)
 * never links or calls it.
 *
 * PARITY UNPINNED: arxiv/paper_1402_4247 ships no implementation, test,
 * golden vector or fixture for this path (SURVEY.md sections 0 and 8(c); the
 * arithmetic lives in OpenMX 3.6, which is not vendored). This oracle is a
 * first-principles restatement of the definitions in include/kbgrid.h written
 * in the reference's conventions:
 *   - error taxonomy -> status codes (kband common.hpp:21-38),
 *   - deterministic fixed-chunk threading, results bitwise independent of the
 *     thread count (common.hpp:58-64, common.cpp:41-47),
 *   - plain loops as the independent brute-force check (test_support.hpp:35-44).
 * It is cross-checked against an independent numpy restatement
 * (tests/golden/make_golden.py) and against analytic identities (tests/).
 */
#ifndef KBG_ORACLE_H
#define KBG_ORACLE_H

#include "../include/kbgrid.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kbo_ctx kbo_ctx;

int kbo_create(const kbg_system* sys, kbo_ctx** out);
int kbo_build_index(kbo_ctx* ctx);
int kbo_index_view(kbo_ctx* ctx, kbg_index* out);
/* threads <= 0: hardware concurrency. */
int kbo_density(kbo_ctx* ctx, int nspin, const double* dm, double* rho, int threads);
int kbo_hamiltonian(kbo_ctx* ctx, int nspin, const double* veff, double dV, double* h, int threads);
/* Block-range variants [b0, b1): rho is zeroed and filled on the range's
 * points; h is zeroed and receives the range's contributions (rank emulation
 * and bounded CPU-baseline samples). */
int kbo_density_range(kbo_ctx* ctx, int nspin, const double* dm, double* rho, int threads, int64_t b0, int64_t b1);
int kbo_hamiltonian_range(kbo_ctx* ctx, int nspin, const double* veff, double dV, double* h, int threads, int64_t b0,
                          int64_t b1);
/* Orbitals of cover `c` of block `block` on its 64 slots: out[M][64]. */
int kbo_block_orbitals(kbo_ctx* ctx, int64_t block, double* out, int64_t cap, int* m_out);
/* Orbitals of one species centred at the origin evaluated at displacement d
 * (d2 computed by the library): out[norb]; zero if outside rc. */
int kbo_orbitals_at(kbo_ctx* ctx, int species, const double* d, double* out);
const char* kbo_last_error(const kbo_ctx* ctx);
/* HBM probe host backend (Table 2 normalization). */
int kbo_normalize_rows(double* x, int64_t nvec, int64_t len, int threads);
void kbo_destroy(kbo_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif
