// CPU oracle of the NAO grid pass -- TEST INFRASTRUCTURE (see oracle.h).
//
// Parity unpinned (no reference implementation exists).
// Definitions follow include/kbgrid.h; conventions follow the reference:
//   errors           /root/reference/proj/include/kband/common.hpp:21-38
//   fixed chunking   /root/reference/proj/src/common.cpp:41-47 (chunk_of)
//   serial reductions /root/reference/proj/include/kband/common.hpp:58-64
// Compile with -ffp-contract=off: the sphere-membership and pair-distance
// expressions must round exactly as the GPU's __dmul_rn/__dadd_rn sequence.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

namespace kbo {

// kband::Error taxonomy (common.hpp:21-38) mapped onto kbgrid.h status codes.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct Species {
    std::vector<int> l;
    double rc = 0;
    int ntab = 0;
    std::vector<double> table;
    int norb = 0;
};

struct Cover {
    int32_t atom;
    int32_t R[3];
    uint64_t mask;
};

struct Index {
    int nblk[3] = {0, 0, 0};
    int64_t nblock = 0;
    std::vector<int32_t> blk_ptr, cov_atom, cov_R, pair_a, pair_b, pair_R, pair_mirror;
    std::vector<uint64_t> cov_mask;
    std::vector<int64_t> pair_off;
    std::map<std::tuple<int, int, int, int, int>, int64_t> pair_id;
    int64_t nbpair = 0, natompt = 0;
    double sum_m = 0, sum_m2 = 0;
    bool built = false;
};

constexpr double C00 = 0.28209479177387814;  // 1/(2 sqrt(pi))
constexpr double C1 = 0.4886025119029199;    // sqrt(3/(4 pi))
constexpr double C20 = 0.31539156525252005;  // sqrt(5/(16 pi))
constexpr double C22 = 0.5462742152960396;   // sqrt(15/(16 pi))
constexpr double C2 = 1.0925484305920792;    // sqrt(15/(4 pi))

inline int slot_of(int li, int lj, int lk) {
    return ((((li >> 1) * 2 + (lj >> 1)) * 2 + (lk >> 1)) * 8) + ((li & 1) * 2 + (lj & 1)) * 2 + (lk & 1);
}

// Fixed contiguous chunking (kband chunk_of, common.cpp:41-47): chunk t of
// [0,n) over T threads.
inline void chunk_of(int64_t n, int T, int t, int64_t& b, int64_t& e) {
    int64_t base = n / T, rem = n % T;
    b = t * base + std::min<int64_t>(t, rem);
    e = b + base + (t < rem ? 1 : 0);
}

template <class F>
void parallel_for(int64_t n, int threads, F&& fn) {
    if (threads <= 1 || n < 2) {
        fn(int64_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t) {
        int64_t b, e;
        chunk_of(n, threads, t, b, e);
        if (b < e) th.emplace_back([&fn, b, e] { fn(b, e); });
    }
    for (auto& x : th) x.join();
}

struct Oracle {
    double A[9];
    double Ainv[9];
    int N[3];
    int natom = 0;
    std::vector<int> species;
    std::vector<double> tau;
    std::vector<Species> spec;
    std::vector<int64_t> basis_off;
    Index idx;
    std::string last_error;

    // ---- system -----------------------------------------------------------
    void load(const kbg_system& s) {
        if (s.natom < 1) throw Error(KBG_ERR_CONFIG, "system: natom must be >= 1");
        if (s.nspecies < 1 || !s.spec) throw Error(KBG_ERR_CONFIG, "system: no species");
        if (!s.species || !s.tau) throw Error(KBG_ERR_CONFIG, "system: null species/tau");
        for (int c = 0; c < 3; ++c)
            if (s.grid[c] < 1) throw Error(KBG_ERR_DIMENSION, "system: grid[" + std::to_string(c) + "] < 1");
        std::memcpy(A, s.lattice, sizeof(A));
        double det = A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
                     A[2] * (A[3] * A[7] - A[4] * A[6]);
        if (!(std::fabs(det) > 1e-12)) throw Error(KBG_ERR_CONFIG, "system: singular lattice");
        Ainv[0] = (A[4] * A[8] - A[5] * A[7]) / det;
        Ainv[1] = (A[2] * A[7] - A[1] * A[8]) / det;
        Ainv[2] = (A[1] * A[5] - A[2] * A[4]) / det;
        Ainv[3] = (A[5] * A[6] - A[3] * A[8]) / det;
        Ainv[4] = (A[0] * A[8] - A[2] * A[6]) / det;
        Ainv[5] = (A[2] * A[3] - A[0] * A[5]) / det;
        Ainv[6] = (A[3] * A[7] - A[4] * A[6]) / det;
        Ainv[7] = (A[1] * A[6] - A[0] * A[7]) / det;
        Ainv[8] = (A[0] * A[4] - A[1] * A[3]) / det;
        std::memcpy(N, s.grid, sizeof(N));
        natom = s.natom;
        spec.resize(s.nspecies);
        for (int t = 0; t < s.nspecies; ++t) {
            const kbg_species& in = s.spec[t];
            Species& sp = spec[t];
            if (in.nrad < 1 || !in.l || !in.table)
                throw Error(KBG_ERR_CONFIG, "species " + std::to_string(t) + ": empty radial list");
            if (!(in.rc > 0)) throw Error(KBG_ERR_CONFIG, "species " + std::to_string(t) + ": rc <= 0");
            if (in.ntab < 4) throw Error(KBG_ERR_CONFIG, "species " + std::to_string(t) + ": ntab < 4");
            sp.l.assign(in.l, in.l + in.nrad);
            sp.rc = in.rc;
            sp.ntab = in.ntab;
            sp.table.assign(in.table, in.table + static_cast<size_t>(in.nrad) * in.ntab * 2);
            sp.norb = 0;
            for (int l : sp.l) {
                if (l < 0 || l > KBG_MAX_L)
                    throw Error(KBG_ERR_CONFIG, "species " + std::to_string(t) + ": l out of range");
                sp.norb += 2 * l + 1;
            }
            if (sp.norb > KBG_MAX_ORB_PER_ATOM)
                throw Error(KBG_ERR_CONFIG, "species " + std::to_string(t) + ": too many orbitals");
        }
        species.assign(s.species, s.species + natom);
        tau.assign(s.tau, s.tau + 3 * natom);
        basis_off.assign(natom + 1, 0);
        for (int a = 0; a < natom; ++a) {
            if (species[a] < 0 || species[a] >= s.nspecies)
                throw Error(KBG_ERR_CONFIG, "atom " + std::to_string(a) + ": bad species id");
            for (int c = 0; c < 3; ++c)
                if (!std::isfinite(tau[3 * a + c]))
                    throw Error(KBG_ERR_NONFINITE, "atom " + std::to_string(a) + ": non-finite position");
            basis_off[a + 1] = basis_off[a] + spec[species[a]].norb;
        }
    }

    void frac(const double* r, double f[3]) const {
        for (int c = 0; c < 3; ++c) f[c] = r[0] * Ainv[0 * 3 + c] + r[1] * Ainv[1 * 3 + c] + r[2] * Ainv[2 * 3 + c];
    }
    void extent(double rho, double e[3]) const {
        for (int c = 0; c < 3; ++c)
            e[c] = rho * std::sqrt(Ainv[c] * Ainv[c] + Ainv[3 + c] * Ainv[3 + c] + Ainv[6 + c] * Ainv[6 + c]) *
                       (1.0 + 1e-9) + 1e-12;
    }
    // Exact expressions shared with the GPU (kbgrid.h conventions).
    void point_pos(int i, int j, int k, double r[3]) const {
        double fi = static_cast<double>(i) / N[0], fj = static_cast<double>(j) / N[1],
               fk = static_cast<double>(k) / N[2];
        for (int c = 0; c < 3; ++c) r[c] = (fi * A[c] + fj * A[3 + c]) + fk * A[6 + c];
    }
    void image_pos(int a, const int R[3], double t[3]) const {
        for (int c = 0; c < 3; ++c)
            t[c] = tau[3 * a + c] + ((R[0] * A[c] + R[1] * A[3 + c]) + R[2] * A[6 + c]);
    }
    static double dist2(const double d[3]) { return (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]; }

    static bool canonical(int a, int b, const int R[3]) {
        if (a != b) return a < b;
        if (R[0] != 0) return R[0] > 0;
        if (R[1] != 0) return R[1] > 0;
        return R[2] >= 0;
    }
    // Pair existence, evaluated in the canonical orientation so that the list
    // is closed under (a,b,R) -> (b,a,-R) bit-for-bit.
    bool pair_test(int a, int b, const int R[3]) const {
        int aa = a, bb = b, RR[3] = {R[0], R[1], R[2]};
        if (!canonical(a, b, R)) {
            aa = b;
            bb = a;
            RR[0] = -R[0];
            RR[1] = -R[1];
            RR[2] = -R[2];
        }
        double t[3], d[3];
        image_pos(bb, RR, t);
        for (int c = 0; c < 3; ++c) d[c] = t[c] - tau[3 * aa + c];
        double s = spec[species[aa]].rc + spec[species[bb]].rc;
        return dist2(d) < s * s;
    }

    // ---- G1 index ---------------------------------------------------------
    void build_index() {
        Index& X = idx;
        X = Index();
        for (int c = 0; c < 3; ++c) X.nblk[c] = (N[c] + KBG_BLOCK_EDGE - 1) / KBG_BLOCK_EDGE;
        X.nblock = static_cast<int64_t>(X.nblk[0]) * X.nblk[1] * X.nblk[2];
        std::vector<std::vector<Cover>> per_block(X.nblock);
        for (int a = 0; a < natom; ++a) {
            const Species& sp = spec[species[a]];
            const double rc2 = sp.rc * sp.rc;
            double f[3], e[3];
            frac(&tau[3 * a], f);
            extent(sp.rc, e);
            int Rlo[3], Rhi[3];
            for (int c = 0; c < 3; ++c) {
                Rlo[c] = static_cast<int>(std::floor(-f[c] - e[c])) - 1;
                Rhi[c] = static_cast<int>(std::ceil(1.0 - f[c] + e[c])) + 1;
            }
            int R[3];
            for (R[0] = Rlo[0]; R[0] <= Rhi[0]; ++R[0])
                for (R[1] = Rlo[1]; R[1] <= Rhi[1]; ++R[1])
                    for (R[2] = Rlo[2]; R[2] <= Rhi[2]; ++R[2]) {
                        int lo[3], hi[3];
                        bool empty = false;
                        for (int c = 0; c < 3; ++c) {
                            lo[c] = std::max(0, static_cast<int>(std::floor((f[c] + R[c] - e[c]) * N[c])) - 1);
                            hi[c] = std::min(N[c] - 1, static_cast<int>(std::ceil((f[c] + R[c] + e[c]) * N[c])) + 1);
                            if (lo[c] > hi[c]) empty = true;
                        }
                        if (empty) continue;
                        double t[3];
                        image_pos(a, R, t);
                        std::map<int64_t, uint64_t> masks;
                        for (int i = lo[0]; i <= hi[0]; ++i)
                            for (int j = lo[1]; j <= hi[1]; ++j)
                                for (int k = lo[2]; k <= hi[2]; ++k) {
                                    double r[3], d[3];
                                    point_pos(i, j, k, r);
                                    for (int c = 0; c < 3; ++c) d[c] = r[c] - t[c];
                                    if (dist2(d) < rc2) {
                                        int64_t b = (static_cast<int64_t>(i / 4) * X.nblk[1] + j / 4) * X.nblk[2] + k / 4;
                                        masks[b] |= uint64_t(1) << slot_of(i & 3, j & 3, k & 3);
                                    }
                                }
                        for (auto& kv : masks) per_block[kv.first].push_back({a, {R[0], R[1], R[2]}, kv.second});
                    }
        }
        X.blk_ptr.assign(X.nblock + 1, 0);
        for (int64_t b = 0; b < X.nblock; ++b) {
            X.blk_ptr[b + 1] = X.blk_ptr[b] + static_cast<int32_t>(per_block[b].size());
            for (auto& cv : per_block[b]) {
                X.cov_atom.push_back(cv.atom);
                for (int c = 0; c < 3; ++c) X.cov_R.push_back(cv.R[c]);
                X.cov_mask.push_back(cv.mask);
            }
        }
        // Pairs (a, b, R) sorted lexicographically.
        X.pair_off.push_back(0);
        for (int a = 0; a < natom; ++a) {
            double fa[3];
            frac(&tau[3 * a], fa);
            for (int b = 0; b < natom; ++b) {
                double fb[3], e[3];
                frac(&tau[3 * b], fb);
                extent(spec[species[a]].rc + spec[species[b]].rc, e);
                int Rlo[3], Rhi[3];
                for (int c = 0; c < 3; ++c) {
                    double df = fb[c] - fa[c];
                    Rlo[c] = static_cast<int>(std::floor(-df - e[c])) - 1;
                    Rhi[c] = static_cast<int>(std::ceil(-df + e[c])) + 1;
                }
                int R[3];
                for (R[0] = Rlo[0]; R[0] <= Rhi[0]; ++R[0])
                    for (R[1] = Rlo[1]; R[1] <= Rhi[1]; ++R[1])
                        for (R[2] = Rlo[2]; R[2] <= Rhi[2]; ++R[2]) {
                            if (!pair_test(a, b, R)) continue;
                            X.pair_id[std::make_tuple(a, b, R[0], R[1], R[2])] = static_cast<int64_t>(X.pair_a.size());
                            X.pair_a.push_back(a);
                            X.pair_b.push_back(b);
                            for (int c = 0; c < 3; ++c) X.pair_R.push_back(R[c]);
                            X.pair_off.push_back(X.pair_off.back() +
                                                 spec[species[a]].norb * spec[species[b]].norb);
                        }
            }
        }
        const int64_t npair = static_cast<int64_t>(X.pair_a.size());
        X.pair_mirror.assign(npair, -1);
        for (int64_t p = 0; p < npair; ++p) {
            auto it = X.pair_id.find(std::make_tuple(X.pair_b[p], X.pair_a[p], -X.pair_R[3 * p], -X.pair_R[3 * p + 1],
                                                     -X.pair_R[3 * p + 2]));
            if (it == X.pair_id.end())
                throw Error(KBG_ERR_CONSISTENCY, "build_index: pair " + std::to_string(p) + " has no mirror");
            X.pair_mirror[p] = static_cast<int32_t>(it->second);
        }
        // Block-pair consistency + statistics.
        for (int64_t b = 0; b < X.nblock; ++b) {
            const int c0 = X.blk_ptr[b], c1 = X.blk_ptr[b + 1];
            for (int ci = c0; ci < c1; ++ci)
                for (int cj = ci; cj < c1; ++cj) {
                    if ((X.cov_mask[ci] & X.cov_mask[cj]) == 0) continue;
                    lookup_pair(ci, cj, b);
                    ++X.nbpair;
                }
            for (int s = 0; s < 64; ++s) {
                int64_t m = 0;
                for (int ci = c0; ci < c1; ++ci)
                    if ((X.cov_mask[ci] >> s) & 1) m += spec[species[X.cov_atom[ci]]].norb;
                X.sum_m += static_cast<double>(m);
                X.sum_m2 += static_cast<double>(m) * static_cast<double>(m);
            }
            for (int ci = c0; ci < c1; ++ci) X.natompt += __builtin_popcountll(X.cov_mask[ci]);
        }
        X.built = true;
    }

    // Pair id of covers (ci, cj): binary search of (a, b, R) in the lexicographically sorted pair list.
    int64_t lookup_pair(int ci, int cj, int64_t blk) const {
        const Index& X = idx;
        const int key[5] = {X.cov_atom[ci], X.cov_atom[cj], X.cov_R[3 * cj] - X.cov_R[3 * ci],
                            X.cov_R[3 * cj + 1] - X.cov_R[3 * ci + 1], X.cov_R[3 * cj + 2] - X.cov_R[3 * ci + 2]};
        auto less = [&](int64_t p) {  // pair p < key
            const int v[5] = {X.pair_a[p], X.pair_b[p], X.pair_R[3 * p], X.pair_R[3 * p + 1], X.pair_R[3 * p + 2]};
            for (int c = 0; c < 5; ++c)
                if (v[c] != key[c]) return v[c] < key[c];
            return false;
        };
        int64_t lo = 0, hi = static_cast<int64_t>(X.pair_a.size());
        while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if (less(mid))
                lo = mid + 1;
            else
                hi = mid;
        }
        const bool hit = lo < static_cast<int64_t>(X.pair_a.size()) && X.pair_a[lo] == key[0] &&
                         X.pair_b[lo] == key[1] && X.pair_R[3 * lo] == key[2] && X.pair_R[3 * lo + 1] == key[3] &&
                         X.pair_R[3 * lo + 2] == key[4];
        if (!hit)
            throw Error(KBG_ERR_CONSISTENCY, "block " + std::to_string(blk) + ": covers " + std::to_string(ci) +
                                                 "," + std::to_string(cj) + " share points but form no pair");
        return lo;
    }

    // ---- G2 orbitals ------------------------------------------------------
    void orbitals(const Species& sp, const double d[3], double d2, double* out) const {
        const double r = std::sqrt(d2);
        const double h = sp.rc / (sp.ntab - 1);
        const double x = r / h;
        int k = static_cast<int>(x);
        if (k > sp.ntab - 2) k = sp.ntab - 2;
        const double t = x - k;
        const double omt = 1.0 - t;
        const double h00 = (1.0 + 2.0 * t) * omt * omt;
        const double h10 = t * omt * omt;
        const double h01 = t * t * (3.0 - 2.0 * t);
        const double h11 = t * t * (t - 1.0);
        int o = 0;
        for (size_t rad = 0; rad < sp.l.size(); ++rad) {
            const double* T = &sp.table[(rad * sp.ntab + k) * 2];
            const double u = h00 * T[0] + h10 * h * T[1] + h01 * T[2] + h11 * h * T[3];
            switch (sp.l[rad]) {
                case 0: out[o++] = C00 * u; break;
                case 1:
                    out[o++] = C1 * d[0] * u;
                    out[o++] = C1 * d[1] * u;
                    out[o++] = C1 * d[2] * u;
                    break;
                default:
                    out[o++] = C20 * (2.0 * d[2] * d[2] - d[0] * d[0] - d[1] * d[1]) * u;
                    out[o++] = C22 * (d[0] * d[0] - d[1] * d[1]) * u;
                    out[o++] = C2 * d[0] * d[1] * u;
                    out[o++] = C2 * d[0] * d[2] * u;
                    out[o++] = C2 * d[1] * d[2] * u;
                    break;
            }
        }
    }

    // Phi for all covers of block b: phi[(row)*64 + slot], rows = concatenated orbitals.
    int block_phi(int64_t b, std::vector<double>& phi, std::vector<int>& row0) const {
        const Index& X = idx;
        const int c0 = X.blk_ptr[b], c1 = X.blk_ptr[b + 1];
        row0.assign(c1 - c0 + 1, 0);
        for (int c = c0; c < c1; ++c) row0[c - c0 + 1] = row0[c - c0] + spec[species[X.cov_atom[c]]].norb;
        const int M = row0.back();
        phi.assign(static_cast<size_t>(M) * 64, 0.0);
        const int bi = static_cast<int>(b / (static_cast<int64_t>(X.nblk[1]) * X.nblk[2]));
        const int bj = static_cast<int>((b / X.nblk[2]) % X.nblk[1]);
        const int bk = static_cast<int>(b % X.nblk[2]);
        double out[KBG_MAX_ORB_PER_ATOM];
        for (int c = c0; c < c1; ++c) {
            const int a = X.cov_atom[c];
            const Species& sp = spec[species[a]];
            double t[3];
            image_pos(a, &X.cov_R[3 * c], t);
            for (int li = 0; li < 4; ++li)
                for (int lj = 0; lj < 4; ++lj)
                    for (int lk = 0; lk < 4; ++lk) {
                        const int s = slot_of(li, lj, lk);
                        if (!((X.cov_mask[c] >> s) & 1)) continue;
                        double r[3], d[3];
                        point_pos(bi * 4 + li, bj * 4 + lj, bk * 4 + lk, r);
                        for (int q = 0; q < 3; ++q) d[q] = r[q] - t[q];
                        orbitals(sp, d, dist2(d), out);
                        for (int o = 0; o < sp.norb; ++o) phi[static_cast<size_t>(row0[c - c0] + o) * 64 + s] = out[o];
                    }
        }
        return M;
    }

    int64_t point_of(int64_t b, int s, bool* valid) const {
        const Index& X = idx;
        const int bi = static_cast<int>(b / (static_cast<int64_t>(X.nblk[1]) * X.nblk[2]));
        const int bj = static_cast<int>((b / X.nblk[2]) % X.nblk[1]);
        const int bk = static_cast<int>(b % X.nblk[2]);
        const int o = s >> 3, w = s & 7;
        const int li = ((o >> 2) & 1) * 2 + ((w >> 2) & 1);
        const int lj = ((o >> 1) & 1) * 2 + ((w >> 1) & 1);
        const int lk = (o & 1) * 2 + (w & 1);
        const int i = bi * 4 + li, j = bj * 4 + lj, k = bk * 4 + lk;
        *valid = (i < N[0] && j < N[1] && k < N[2]);
        return (static_cast<int64_t>(i) * N[1] + j) * N[2] + k;
    }

    // ---- G3 density: rho(s) = sum_{ci,cj ∋ s} phi_ci(s)^T DM(ci,cj) phi_cj(s) ---
    // Per block and row cover ci: Y_ci(s) = sum_cj DM(ci,cj) phi_cj(s) over the
    // covers cj sharing points with ci (all 64 slots at once: phi is exactly 0
    // outside a cover's mask, so the extra terms are exact zeros), then
    // rho(s) += sum_i phi_ci,i(s) Y_ci,i(s). Full (ci, cj) range, no symmetry
    // used. Blocks write disjoint points: bitwise independent of the thread count.
    void density(int nspin, const double* dm, double* rho, int threads, int64_t blo, int64_t bhi) const {
        const Index& X = idx;
        const int64_t npts = static_cast<int64_t>(N[0]) * N[1] * N[2];
        const int64_t nnz = X.pair_off.back();
        for (int64_t p = 0; p < nspin * npts; ++p) rho[p] = 0.0;
        parallel_for(bhi - blo, threads, [&](int64_t b0, int64_t b1) {
            std::vector<double> phi;
            std::vector<int> row0;
            std::vector<int64_t> off;
            double y[KBG_MAX_ORB_PER_ATOM][64];
            double acc[64];
            for (int64_t b = blo + b0; b < blo + b1; ++b) {
                const int c0 = X.blk_ptr[b], c1 = X.blk_ptr[b + 1];
                if (c0 == c1) continue;
                block_phi(b, phi, row0);
                const int nc = c1 - c0;
                off.assign(static_cast<size_t>(nc) * nc, -1);
                for (int i = 0; i < nc; ++i)
                    for (int j = 0; j < nc; ++j)
                        if (X.cov_mask[c0 + i] & X.cov_mask[c0 + j]) off[i * nc + j] = X.pair_off[lookup_pair(c0 + i, c0 + j, b)];
                for (int sp = 0; sp < nspin; ++sp) {
                    const double* D = dm + sp * nnz;
                    for (int s = 0; s < 64; ++s) acc[s] = 0.0;
                    for (int i = 0; i < nc; ++i) {
                        const int na = spec[species[X.cov_atom[c0 + i]]].norb;
                        for (int ii = 0; ii < na; ++ii)
                            for (int s = 0; s < 64; ++s) y[ii][s] = 0.0;
                        for (int j = 0; j < nc; ++j) {
                            if (off[i * nc + j] < 0) continue;
                            const int nb = spec[species[X.cov_atom[c0 + j]]].norb;
                            const double* blk = D + off[i * nc + j];
                            for (int ii = 0; ii < na; ++ii)
                                for (int jj = 0; jj < nb; ++jj) {
                                    const double d = blk[ii * nb + jj];
                                    const double* pj = &phi[static_cast<size_t>(row0[j] + jj) * 64];
                                    for (int s = 0; s < 64; ++s) y[ii][s] += d * pj[s];
                                }
                        }
                        for (int ii = 0; ii < na; ++ii) {
                            const double* pi = &phi[static_cast<size_t>(row0[i] + ii) * 64];
                            for (int s = 0; s < 64; ++s) acc[s] += pi[s] * y[ii][s];
                        }
                    }
                    for (int s = 0; s < 64; ++s) {
                        bool valid;
                        const int64_t pt = point_of(b, s, &valid);
                        if (valid) rho[sp * npts + pt] = acc[s];
                    }
                }
            }
        });
    }

    // ---- G4 hamiltonian: all ordered cover pairs --------------------------
    // Blocks are processed in windows of kWindow (fixed, independent of the
    // thread count). Phase 1, parallel over the window's blocks: each block's
    // tiles T(ci, cj) = sum_s phi_ci(s) w(s) phi_cj(s)^T for every ordered cover
    // pair with common points (full na x nb, no symmetry used). Phase 2,
    // parallel over contiguous pair ranges: each thread adds the window's tiles
    // of its pairs into H in block order, then (ci, cj) order. Every entry is
    // therefore summed in one fixed order: results are bitwise independent of
    // the thread count (kband common.hpp:58-64).
    static constexpr int64_t kWindow = 512;
    struct Tile {
        int64_t pair;
        int64_t off;  // into the block's tile values
        int na, nb;
    };
    void hamiltonian(int nspin, const double* veff, double dV, double* h, int threads, int64_t blo,
                     int64_t bhi) const {
        const Index& X = idx;
        const int64_t npts = static_cast<int64_t>(N[0]) * N[1] * N[2];
        const int64_t nnz = X.pair_off.back();
        const int64_t npair = static_cast<int64_t>(X.pair_a.size());
        for (int64_t p = 0; p < nspin * nnz; ++p) h[p] = 0.0;
        std::vector<std::vector<Tile>> tiles(kWindow);
        std::vector<std::vector<double>> vals(kWindow);
        for (int64_t w0 = blo; w0 < bhi; w0 += kWindow) {
            const int64_t w1 = std::min(bhi, w0 + kWindow);
            parallel_for(w1 - w0, threads, [&](int64_t i0, int64_t i1) {
                std::vector<double> phi;
                std::vector<int> row0;
                double w[64];
                for (int64_t i = i0; i < i1; ++i) {
                    const int64_t b = w0 + i;
                    std::vector<Tile>& T = tiles[i];
                    std::vector<double>& V = vals[i];
                    T.clear();
                    V.clear();
                    const int c0 = X.blk_ptr[b], c1 = X.blk_ptr[b + 1];
                    if (c0 == c1) continue;
                    block_phi(b, phi, row0);
                    for (int sp = 0; sp < nspin; ++sp) {
                        for (int s = 0; s < 64; ++s) {
                            bool valid;
                            const int64_t pt = point_of(b, s, &valid);
                            w[s] = valid ? veff[sp * npts + pt] * dV : 0.0;
                        }
                        for (int ci = c0; ci < c1; ++ci) {
                            const int na = spec[species[X.cov_atom[ci]]].norb;
                            for (int cj = c0; cj < c1; ++cj) {
                                const uint64_t both = X.cov_mask[ci] & X.cov_mask[cj];
                                if (!both) continue;
                                const int nb = spec[species[X.cov_atom[cj]]].norb;
                                const int64_t pair = lookup_pair(ci, cj, b);
                                T.push_back({pair + sp * npair, static_cast<int64_t>(V.size()), na, nb});
                                V.resize(V.size() + static_cast<size_t>(na) * nb, 0.0);
                                double* blk = V.data() + T.back().off;
                                // sum over the octets (8 consecutive slots) holding common points, in
                                // 8 slot-lanes combined in a fixed tree: exact zeros outside the masks
                                for (int ii = 0; ii < na; ++ii) {
                                    const double* pa = &phi[static_cast<size_t>(row0[ci - c0] + ii) * 64];
                                    double aw[64];
                                    for (int s = 0; s < 64; ++s) aw[s] = pa[s] * w[s];
                                    for (int jj = 0; jj < nb; ++jj) {
                                        const double* pb = &phi[static_cast<size_t>(row0[cj - c0] + jj) * 64];
                                        double l[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                                        for (int o = 0; o < 8; ++o) {
                                            if (!((both >> (8 * o)) & 0xFFu)) continue;
                                            for (int k = 0; k < 8; ++k) l[k] += aw[8 * o + k] * pb[8 * o + k];
                                        }
                                        blk[ii * nb + jj] = ((l[0] + l[1]) + (l[2] + l[3])) + ((l[4] + l[5]) + (l[6] + l[7]));
                                    }
                                }
                            }
                        }
                    }
                }
            });
            parallel_for(nspin * npair, threads, [&](int64_t p0, int64_t p1) {
                for (int64_t i = 0; i < w1 - w0; ++i)
                    for (const Tile& t : tiles[i]) {
                        if (t.pair < p0 || t.pair >= p1) continue;
                        const int64_t sp = t.pair / npair, p = t.pair - sp * npair;
                        double* dst = h + sp * nnz + X.pair_off[p];
                        const double* src = vals[i].data() + t.off;
                        for (int e = 0; e < t.na * t.nb; ++e) dst[e] += src[e];
                    }
            });
        }
    }
};

}  // namespace kbo

struct kbo_ctx {
    kbo::Oracle o;
};

namespace {
template <class F>
int guard(kbo_ctx* ctx, F&& fn) {
    try {
        fn();
        if (ctx) ctx->o.last_error.clear();
        return KBG_OK;
    } catch (const kbo::Error& e) {
        if (ctx) ctx->o.last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        if (ctx) ctx->o.last_error = e.what();
        return KBG_ERR_CONSISTENCY;
    }
}
int nthreads(int t) {
    if (t > 0) return t;
    unsigned h = std::thread::hardware_concurrency();
    return h ? static_cast<int>(h) : 1;
}
}  // namespace

extern "C" int kbo_create(const kbg_system* sys, kbo_ctx** out) {
    if (!sys || !out) return KBG_ERR_CONFIG;
    auto* c = new kbo_ctx();
    int st = guard(c, [&] { c->o.load(*sys); });
    if (st != KBG_OK) {
        std::fprintf(stderr, "kbo_create: %s\n", c->o.last_error.c_str());
        delete c;
        *out = nullptr;
        return st;
    }
    *out = c;
    return KBG_OK;
}

extern "C" int kbo_build_index(kbo_ctx* ctx) {
    if (!ctx) return KBG_ERR_CONFIG;
    return guard(ctx, [&] { ctx->o.build_index(); });
}

extern "C" int kbo_index_view(kbo_ctx* ctx, kbg_index* out) {
    if (!ctx || !out) return KBG_ERR_CONFIG;
    const kbo::Index& X = ctx->o.idx;
    if (!X.built) {
        ctx->o.last_error = "index_view: index not built";
        return KBG_ERR_CONFIG;
    }
    std::memset(out, 0, sizeof(*out));
    out->npts = static_cast<int64_t>(ctx->o.N[0]) * ctx->o.N[1] * ctx->o.N[2];
    for (int c = 0; c < 3; ++c) out->nblk[c] = X.nblk[c];
    out->nblock = X.nblock;
    out->ncover = static_cast<int64_t>(X.cov_atom.size());
    out->blk_ptr = X.blk_ptr.data();
    out->cov_atom = X.cov_atom.data();
    out->cov_R = X.cov_R.data();
    out->cov_mask = X.cov_mask.data();
    out->npair = static_cast<int64_t>(X.pair_a.size());
    out->pair_a = X.pair_a.data();
    out->pair_b = X.pair_b.data();
    out->pair_R = X.pair_R.data();
    out->pair_off = X.pair_off.data();
    out->pair_mirror = X.pair_mirror.data();
    out->nnz = X.pair_off.back();
    out->nbpair = X.nbpair;
    out->natompt = X.natompt;
    out->sum_m = X.sum_m;
    out->sum_m2 = X.sum_m2;
    return KBG_OK;
}

extern "C" int kbo_density_range(kbo_ctx* ctx, int nspin, const double* dm, double* rho, int threads, int64_t b0,
                                 int64_t b1) {
    if (!ctx || !dm || !rho) return KBG_ERR_CONFIG;
    if (nspin < 1 || nspin > 2) {
        ctx->o.last_error = "density: nspin must be 1 or 2";
        return KBG_ERR_CONFIG;
    }
    if (!ctx->o.idx.built) {
        ctx->o.last_error = "density: index not built";
        return KBG_ERR_CONFIG;
    }
    if (b0 < 0 || b1 > ctx->o.idx.nblock || b0 > b1) {
        ctx->o.last_error = "density: bad block range";
        return KBG_ERR_DIMENSION;
    }
    return guard(ctx, [&] { ctx->o.density(nspin, dm, rho, nthreads(threads), b0, b1); });
}

extern "C" int kbo_density(kbo_ctx* ctx, int nspin, const double* dm, double* rho, int threads) {
    if (!ctx) return KBG_ERR_CONFIG;
    return kbo_density_range(ctx, nspin, dm, rho, threads, 0, ctx->o.idx.nblock);
}

extern "C" int kbo_hamiltonian_range(kbo_ctx* ctx, int nspin, const double* veff, double dV, double* h, int threads,
                                     int64_t b0, int64_t b1) {
    if (!ctx || !veff || !h) return KBG_ERR_CONFIG;
    if (nspin < 1 || nspin > 2) {
        ctx->o.last_error = "hamiltonian: nspin must be 1 or 2";
        return KBG_ERR_CONFIG;
    }
    if (!ctx->o.idx.built) {
        ctx->o.last_error = "hamiltonian: index not built";
        return KBG_ERR_CONFIG;
    }
    if (b0 < 0 || b1 > ctx->o.idx.nblock || b0 > b1) {
        ctx->o.last_error = "hamiltonian: bad block range";
        return KBG_ERR_DIMENSION;
    }
    return guard(ctx, [&] { ctx->o.hamiltonian(nspin, veff, dV, h, nthreads(threads), b0, b1); });
}

extern "C" int kbo_hamiltonian(kbo_ctx* ctx, int nspin, const double* veff, double dV, double* h, int threads) {
    if (!ctx) return KBG_ERR_CONFIG;
    return kbo_hamiltonian_range(ctx, nspin, veff, dV, h, threads, 0, ctx->o.idx.nblock);
}

extern "C" int kbo_block_orbitals(kbo_ctx* ctx, int64_t block, double* out, int64_t cap, int* m_out) {
    if (!ctx || !out || !m_out) return KBG_ERR_CONFIG;
    if (!ctx->o.idx.built || block < 0 || block >= ctx->o.idx.nblock) {
        ctx->o.last_error = "block_orbitals: bad block";
        return KBG_ERR_DIMENSION;
    }
    return guard(ctx, [&] {
        std::vector<double> phi;
        std::vector<int> row0;
        int M = ctx->o.block_phi(block, phi, row0);
        *m_out = M;
        if (static_cast<int64_t>(M) * 64 > cap) throw kbo::Error(KBG_ERR_DIMENSION, "block_orbitals: cap too small");
        std::memcpy(out, phi.data(), sizeof(double) * phi.size());
    });
}

extern "C" int kbo_orbitals_at(kbo_ctx* ctx, int species, const double* d, double* out) {
    if (!ctx || !d || !out) return KBG_ERR_CONFIG;
    if (species < 0 || species >= static_cast<int>(ctx->o.spec.size())) return KBG_ERR_CONFIG;
    const kbo::Species& sp = ctx->o.spec[species];
    double d2 = kbo::Oracle::dist2(d);
    if (!(d2 < sp.rc * sp.rc)) {
        for (int o = 0; o < sp.norb; ++o) out[o] = 0.0;
        return KBG_OK;
    }
    ctx->o.orbitals(sp, d, d2, out);
    return KBG_OK;
}

// Table 2 normalization: the host backend of
// the HBM probe, x[v][:] /= ||x[v]||, rows split over `threads` in fixed
// contiguous chunks; zero rows stay zero.
extern "C" int kbo_normalize_rows(double* x, int64_t nvec, int64_t len, int threads) {
    if (!x || nvec < 0 || len < 0) return KBG_ERR_CONFIG;
    kbo::parallel_for(nvec, threads, [&](int64_t v0, int64_t v1) {
        for (int64_t v = v0; v < v1; ++v) {
            double* r = x + v * len;
            double ss = 0.0;
            for (int64_t i = 0; i < len; ++i) ss += r[i] * r[i];
            if (ss == 0.0) continue;
            const double nrm = std::sqrt(ss);
            for (int64_t i = 0; i < len; ++i) r[i] /= nrm;
        }
    });
    return KBG_OK;
}

extern "C" const char* kbo_last_error(const kbo_ctx* ctx) { return ctx ? ctx->o.last_error.c_str() : "null ctx"; }
extern "C" void kbo_destroy(kbo_ctx* ctx) { delete ctx; }
