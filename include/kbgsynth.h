/*
 * kbgsynth.h -- synthetic Fe3O4 inputs for the grid pass (libkbgsynth.so).
 *
 * Input generator (component G0). It is neither the
 * product nor the checker: it produces the byte-identical inputs that both
 * libkbgrid.so (GPU) and the CPU oracle consume. Seeded std::mt19937_64 as in
 * the reference's fixtures (/root/reference/proj/tests/test_support.hpp:9);
 * doubles are drawn as (x >> 11) * 2^-53 so the stream is bit-reproducible.
 *
 * Structure: magnetite Fd-3m, a = 8.396 A, Fe 8a, Fe 16d, O 32e (x = 0.2549)
 * with the four FCC translations; canonical atom order = site list order,
 * then translation, supercell index outermost. Primitive cell = the 14 site
 * representatives in the FCC primitive lattice a/2 (0,1,1),(1,0,1),(1,1,0).
 * Grid rule: N_i = smallest 2^a 3^b 5^c >= ceil(|a_i| sqrt(Ecut[Ry]) / pi).
 * Basis: Fe s2p2d1 (rc 6.0 bohr), O s2p2 (rc 5.0 bohr);
 * R(r) = N r^l exp(-alpha r^2) (1 - (r/rc)^2)^3, int R^2 r^2 dr = 1.
 */
#ifndef KBGSYNTH_H
#define KBGSYNTH_H

#include <stdint.h>

#include "kbgrid.h"

#ifdef __cplusplus
extern "C" {
#endif

#define KBG_CELL_PRIMITIVE 0
#define KBG_CELL_CUBIC 1

typedef struct kbg_synth kbg_synth;

/* kind: KBG_CELL_PRIMITIVE (rep must be 1) or KBG_CELL_CUBIC (rep x rep x rep
 * supercell of the 56-atom cell). ntab: radial table points (1024 default). */
int kbg_synth_create(int kind, int rep, double ecut_ry, uint64_t seed, int ntab, kbg_synth** out);
const kbg_system* kbg_synth_system(const kbg_synth* s);
double kbg_synth_dV(const kbg_synth* s);
/* veff: [nspin][npts]. Gaussian wells on atoms + 0.1 * low-G cosine field. */
int kbg_synth_veff(const kbg_synth* s, int nspin, uint64_t seed, double* veff);
/* dm: [nspin][nnz] in the pair order of `idx` (from kbg_index_view or the
 * oracle). U(-1,1) * exp(-|tau_a - t_b(R)| / 2 bohr), DM_ba(-R) = DM_ab(R)^T. */
int kbg_synth_dm(const kbg_synth* s, const kbg_index* idx, int nspin, uint64_t seed, double* dm);
void kbg_synth_free(kbg_synth* s);

/* Tabulate u(r) = R(r)/r^l = N exp(-alpha r^2) (1-(r/rc)^2)^3 and du/dr on
 * ntab uniform points of [0, rc], normalised so that int_0^rc R^2 r^2 dr = 1.
 * out: [ntab][2]. Returns the normalisation constant N. */
double kbg_synth_radial_table(int l, double alpha, double rc, int ntab, double* out);

/* Smallest 2^a 3^b 5^c >= n. */
int kbg_synth_good_size(int n);

#ifdef __cplusplus
}
#endif

#endif /* KBGSYNTH_H */
