// Device helpers shared by the index build and the grid kernels.
#pragma once

#include "kb_internal.cuh"

namespace kbg {

// Real-solid-harmonic constants (same literals as the oracle).
constexpr double kC00 = 0.28209479177387814;  // 1/(2 sqrt(pi))
constexpr double kC1 = 0.4886025119029199;    // sqrt(3/(4 pi))
constexpr double kC20 = 0.31539156525252005;  // sqrt(5/(16 pi))
constexpr double kC22 = 0.5462742152960396;   // sqrt(15/(16 pi))
constexpr double kC2 = 1.0925484305920792;    // sqrt(15/(4 pi))

// Slot (0..63) -> block-local (li, lj, lk). Octet o = slot>>3 is a 2x2x2 cube,
// quad q = slot>>2 a 1x2x2 square (include/kbgrid.h).
__device__ __forceinline__ void slot_decode(int s, int& li, int& lj, int& lk) {
    const int o = s >> 3, w = s & 7;
    li = ((o >> 2) & 1) * 2 + ((w >> 2) & 1);
    lj = ((o >> 1) & 1) * 2 + ((w >> 1) & 1);
    lk = (o & 1) * 2 + (w & 1);
}

// Exact-rounding expressions of include/kbgrid.h (no contraction).
__device__ __forceinline__ void point_pos_exact(const SysParams& P, int i, int j, int k, double r[3]) {
    const double fi = __ddiv_rn(static_cast<double>(i), static_cast<double>(P.N[0]));
    const double fj = __ddiv_rn(static_cast<double>(j), static_cast<double>(P.N[1]));
    const double fk = __ddiv_rn(static_cast<double>(k), static_cast<double>(P.N[2]));
#pragma unroll
    for (int c = 0; c < 3; ++c)
        r[c] = __dadd_rn(__dadd_rn(__dmul_rn(fi, P.A[c]), __dmul_rn(fj, P.A[3 + c])), __dmul_rn(fk, P.A[6 + c]));
}

__device__ __forceinline__ void image_pos_exact(const SysParams& P, const double* tau, int R0, int R1, int R2,
                                                double t[3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
        t[c] = __dadd_rn(tau[c], __dadd_rn(__dadd_rn(__dmul_rn(static_cast<double>(R0), P.A[c]),
                                                     __dmul_rn(static_cast<double>(R1), P.A[3 + c])),
                                           __dmul_rn(static_cast<double>(R2), P.A[6 + c])));
}

__device__ __forceinline__ double dist2_exact(const double d[3]) {
    return __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2]));
}

// Orbitals of one atom at two points (displacements d[h], squared lengths d2[h],
// h = 0, 1): cubic Hermite on the uniform radial table (u = R / r^l and du/dr)
// times real solid harmonics in the fixed order of include/kbgrid.h; one sink
// call per orbital with both values (the geometry cache's 16-byte stores).
// `tables` may point to shared memory (staged copy of the table array) or
// global memory.
template <class Sink>
__device__ __forceinline__ void eval_orbitals_pair(const DevSpecies& sp, const double* __restrict__ tables,
                                                   const double (&d)[2][3], const double (&d2)[2], Sink&& sink) {
    // Explicit round-to-nearest operations in the oracle's exact expression order
    // (oracle/kbg_oracle.cpp orbitals(), compiled with -ffp-contract=off): no compiler-chosen FMA
    // contraction, so every kernel that inlines this produces the same Phi bits -- the oracle's.
    auto m = [](double x, double y) { return __dmul_rn(x, y); };
    auto p = [](double x, double y) { return __dadd_rn(x, y); };
    auto s = [](double x, double y) { return __dsub_rn(x, y); };
    double h00[2], h10h[2], h01[2], h11h[2];
    const double* tab[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const double x = __ddiv_rn(__dsqrt_rn(d2[h]), sp.h);
        int k = static_cast<int>(x);
        if (k > sp.ntab - 2) k = sp.ntab - 2;
        const double t = s(x, static_cast<double>(k));
        const double omt = s(1.0, t);
        h00[h] = m(m(p(1.0, m(2.0, t)), omt), omt);
        h10h[h] = m(m(m(t, omt), omt), sp.h);
        h01[h] = m(m(t, t), s(3.0, m(2.0, t)));
        h11h[h] = m(m(m(t, t), s(t, 1.0)), sp.h);
        tab[h] = tables + sp.tab_off + 2 * k;
    }
    int o = 0;
    for (int rad = 0; rad < sp.nrad; ++rad) {
        double u[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double2 a = *reinterpret_cast<const double2*>(tab[h] + static_cast<long long>(rad) * sp.ntab * 2);
            const double2 b = *reinterpret_cast<const double2*>(tab[h] + static_cast<long long>(rad) * sp.ntab * 2 + 2);
            u[h] = p(p(p(m(h00[h], a.x), m(h10h[h], a.y)), m(h01[h], b.x)), m(h11h[h], b.y));
        }
        const int l = sp.l[rad];
        if (l == 0) {
            sink(o++, m(kC00, u[0]), m(kC00, u[1]));
        } else if (l == 1) {
#pragma unroll
            for (int c = 0; c < 3; ++c) sink(o++, m(m(kC1, d[0][c]), u[0]), m(m(kC1, d[1][c]), u[1]));
        } else {
            double v[5][2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double x = d[h][0], y = d[h][1], z = d[h][2];
                v[0][h] = m(m(kC20, s(s(m(m(2.0, z), z), m(x, x)), m(y, y))), u[h]);
                v[1][h] = m(m(kC22, s(m(x, x), m(y, y))), u[h]);
                v[2][h] = m(m(m(kC2, x), y), u[h]);
                v[3][h] = m(m(m(kC2, x), z), u[h]);
                v[4][h] = m(m(m(kC2, y), z), u[h]);
            }
#pragma unroll
            for (int q = 0; q < 5; ++q) sink(o++, v[q][0], v[q][1]);
        }
    }
}

__device__ __forceinline__ int64_t block_id(const SysParams& P, int bi, int bj, int bk) {
    return (static_cast<int64_t>(bi) * P.nblk[1] + bj) * P.nblk[2] + bk;
}

__device__ __forceinline__ void block_decode(const SysParams& P, int64_t b, int& bi, int& bj, int& bk) {
    bk = static_cast<int>(b % P.nblk[2]);
    const int64_t t = b / P.nblk[2];
    bj = static_cast<int>(t % P.nblk[1]);
    bi = static_cast<int>(t / P.nblk[1]);
}

// Lexicographic pair key (a, b, R0, R1, R2); |R_c| < 512, natom^2 < 2^33.
__host__ __device__ __forceinline__ int64_t pair_key(int a, int b, int R0, int R1, int R2, int natom) {
    return ((static_cast<int64_t>(a) * natom + b) << 30) | (static_cast<int64_t>(R0 + 512) << 20) |
           (static_cast<int64_t>(R1 + 512) << 10) | static_cast<int64_t>(R2 + 512);
}

__device__ __forceinline__ int64_t find_pair(const int64_t* __restrict__ keys, int64_t n, int64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < n && keys[lo] == key) ? lo : -1;
}

}  // namespace kbg

namespace kbg {

// Row groups of a block (shared by the task builder and the grid kernels):
// consecutive covers are packed into groups of <= kGroupRows orbitals; a cover
// with more orbitals forms a group of its own. Rows are not padded: a group's
// 8-row DMMA tiles may run into the next group's rows, which the kernels mask
// out. norb(c) gives the orbital count of local cover c; g_rows = actual rows.
// Returns the group count. (Padding every cover to a multiple of 4 rows would
// give all fragment rows the same shared-memory swizzle, but the extra rows do
// not fit two rho buffers into shared memory at the coarse end of the sweep.)

template <class NorbF>
__host__ __device__ inline int make_groups(int ncov, NorbF norb, int* g_first, int* g_end, int* g_row0,
                                           int* g_rows, int* c_row0, int* c_group) {
    int ng = 0, next_row = 0, cur = 0;  // cur = rows used by the open group (0: none open)
    for (int c = 0; c < ncov; ++c) {
        const int n = norb(c);
        if (cur == 0 || cur + n > kGroupRows) {
            if (cur > 0) {
                g_rows[ng - 1] = cur;
                next_row = g_row0[ng - 1] + g_rows[ng - 1];
            }
            g_first[ng] = c;
            g_row0[ng] = next_row;
            ++ng;
            cur = 0;
        }
        c_row0[c] = g_row0[ng - 1] + cur;
        c_group[c] = ng - 1;
        cur += n;
        g_end[ng - 1] = c + 1;
        if (cur >= kGroupRows) {
            g_rows[ng - 1] = cur;
            next_row = g_row0[ng - 1] + g_rows[ng - 1];
            cur = 0;
        }
    }
    if (cur > 0) g_rows[ng - 1] = cur;
    return ng;
}

__host__ __device__ __forceinline__ uint32_t quads_of(uint64_t m) {
    uint32_t q = 0;
    for (int i = 0; i < 16; ++i) q |= static_cast<uint32_t>(((m >> (4 * i)) & 0xFull) != 0) << i;
    return q;
}

__host__ __device__ __forceinline__ uint32_t octets_of(uint64_t m) {
    uint32_t q = 0;
    for (int i = 0; i < 8; ++i) q |= static_cast<uint32_t>(((m >> (8 * i)) & 0xFFull) != 0) << i;
    return q;
}

}  // namespace kbg
