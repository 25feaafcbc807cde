// Device core of the grid kernels, shared by the one-CTA-per-block kernels
// (kb_grid.cu) and the persistent warp-specialized kernels (kb_persist.cu).
//
// Per grid block (4x4x4 points = 64 slots) a shared-memory buffer holds
//   Phi      FP64, rows x 64 slots: the covers' (atom images') orbitals, rows
//            packed into row groups of <= 16 orbitals (two 8-row DMMA tiles);
//            Phi[row][slot] at row*64 + (slot ^ 4*(row & 3)), so any 4
//            consecutive rows x 4 slots (a half-warp DMMA fragment) hit 32 banks;
//   tables   covers, groups, pair offsets off2d[ci][cj], row -> (cover,
//            orbital), partner octets, this block's warp task list.
// H task (group g, partner cj >= first(g)): C(16 x 8*TN) += Phi_g diag(V dV)
//   Phi_cj^T over the common 1x2x2 quads with mma.sync.m8n8k4.f64 (SASS
//   DMMA); canonical rows (cover ci <= cj) are scattered with FP64 atomics.
// rho task (group g, octet part h of kRhoOct octets, partner range): Y(16 x 8 slots) +=
//   D'(16 x n_cj) Phi_cj(n_cj x 8) over the partners cj in the range in registers, D' =
//   repacked DM (x2 off the (a,a,0) blocks: the symmetric half), then
//   rho(slot) += sum_rows Phi_g * Y once per task.
#pragma once

#include <type_traits>

#include "kb_device.cuh"


// L2 policy of the persistent kernels: 1 streams the geometry cache with
// evict_first; 2 also loads the repacked DM with evict_last.
#ifndef KBG_L2_HINT
#define KBG_L2_HINT 1
#endif

// H tiles: 1 = permuted B-fragment column order (hcol_of_n): the scatter's RED instructions touch half
// the L2 sectors, which removes the H pass's dependence on where the output buffer lies in memory
// (56 atoms: 0.321-0.382 ms over 21 buffer placements -> 0.3185-0.3205; deterministic 0.539 -> 0.429)
#ifndef KBG_H_PERMCOL
#define KBG_H_PERMCOL 1
#endif
// rho D' gather: 1 = predicated loads (no per-lane branch around rows without a pair to the partner;
// the density pass 0.352 -> 0.343 ms at 56 atoms and no register spills), 0 = branch + zero fill.
// H pair tiles (h_tile2): 1 = quad addresses as byte offsets, one XOR + one add per operand (56 atoms H
// 0.3185 -> 0.3164 ms, 448 atoms 2.376 -> 2.353 ms; the same in the single-partner h_tile adds spills
// and measured slower); 0 = element indices scaled per access
#ifndef KBG_H_BYTEADDR
#define KBG_H_BYTEADDR 1
#endif
#ifndef KBG_RHO_PGATHER
#define KBG_RHO_PGATHER 1
#endif

namespace kbg {
namespace core {

struct CoverS {
    double t[3];
    uint64_t mask;
    int row0;
    int norb;
    int sp;
    int grp;
};

struct GroupS {
    int first, end, row0, rows, tm;  // covers [first, end), Phi rows [row0, row0 + rows), tm = ceil(rows / 8)
};

struct Meta {
    int64_t block;  // grid block staged in this buffer (-1: end of work)
    int ncov, ngrp, rows, done;
    int next;  // task queue head (dynamic schedule)
};

constexpr uint8_t kNoCover = 0xFF;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// Predicated DMMA: issued in straight-line code, executed only when `on`
// (uniform across the warp) -- no branch between independent accumulators.
__device__ __forceinline__ void dmma_if(double (&c)[2], double a, double b, uint32_t on) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        " setp.ne.u32 p, %4, 0;\n"
        " @p mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        "}\n"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b), "r"(on));
}

// Octets (2x2x2 cubes, 8 consecutive slots) with any bit set: OR-fold each
// byte into its low bit, then gather the 8 low bits with one multiply.
__device__ __forceinline__ uint32_t octet_bits(uint64_t m) {
    m |= m >> 4;
    m |= m >> 2;
    m |= m >> 1;
    return static_cast<uint32_t>(((m & 0x0101010101010101ull) * 0x0102040810204080ull) >> 56);
}

__device__ __forceinline__ int swz(int row) { return (row & 3) << 2; }
__device__ __forceinline__ int phi_idx(int row, int slot) { return row * 64 + (slot ^ swz(row)); }

// Dynamic shared memory of every grid kernel. Buffers are addressed by byte
// offsets from this symbol (not by pointers kept in structs) so the compiler
// always emits shared-memory loads/stores (LDS/STS), never generic LD/ST.
extern __shared__ __align__(16) unsigned char kbg_smem[];

struct Smem {
    uint32_t base;  // byte offset of this buffer in kbg_smem; o_* are relative to it
    uint32_t o_meta, o_cov, o_grp, o_off2d, o_rcov, o_rorb, o_pom, o_pbits, o_task, o_wptr, o_acc, o_phi;
    __device__ __forceinline__ Meta* meta() const { return reinterpret_cast<Meta*>(kbg_smem + base + o_meta); }
    __device__ __forceinline__ CoverS* cov() const { return reinterpret_cast<CoverS*>(kbg_smem + base + o_cov); }
    __device__ __forceinline__ GroupS* grp() const { return reinterpret_cast<GroupS*>(kbg_smem + base + o_grp); }
    // [ncov][ncov] offset of canonical pair (ci <= cj) with common points (H: value, rho: repacked)
    __device__ __forceinline__ int32_t* off2d() const { return reinterpret_cast<int32_t*>(kbg_smem + base + o_off2d); }
    __device__ __forceinline__ uint8_t* rcov() const { return kbg_smem + base + o_rcov; }  // row -> cover (kNoCover: tail)
    __device__ __forceinline__ uint8_t* rorb() const { return kbg_smem + base + o_rorb; }  // row -> orbital in cover
    // [ngrp][ncov] octets shared by group g (rows ci <= cj) and cover cj
    __device__ __forceinline__ uint8_t* pom() const { return kbg_smem + base + o_pom; }
    // [ngrp][8 / kRhoOct] covers cj with a shared octet in part h
    __device__ __forceinline__ uint64_t* pbits() const { return reinterpret_cast<uint64_t*>(kbg_smem + base + o_pbits); }
    __device__ __forceinline__ Task* task() const { return reinterpret_cast<Task*>(kbg_smem + base + o_task); }
    __device__ __forceinline__ int32_t* wptr() const { return reinterpret_cast<int32_t*>(kbg_smem + base + o_wptr); }
    // H: w[nspin][64];  rho: racc[nspin][acc_warps][64]
    __device__ __forceinline__ double* acc() const { return reinterpret_cast<double*>(kbg_smem + base + o_acc); }
    __device__ __forceinline__ double* phi() const { return reinterpret_cast<double*>(kbg_smem + base + o_phi); }
};

__host__ __device__ __forceinline__ size_t align16(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }

// Buffer layout: [tables | acc | Phi]. The tables section has a fixed size
// (table_bytes) and is exactly what the geometry cache stores per block and
// the persistent kernels' producer bulk-copies back (kb_cache.cu).
__host__ __device__ inline size_t tables_layout(const GridArgs& g, size_t* off) {
    size_t o = 0;
    const size_t mc = static_cast<size_t>(g.max_cover);
    off[0] = o;  // meta
    o += align16(sizeof(Meta));
    off[1] = o;  // covers
    o += align16(mc * sizeof(CoverS));
    off[2] = o;  // groups
    o += align16(mc * sizeof(GroupS));
    off[3] = o;  // off2d
    o += align16(mc * mc * sizeof(int32_t));
    off[4] = o;  // rcov
    o += align16(static_cast<size_t>(g.max_rows));
    off[5] = o;  // rorb
    o += align16(static_cast<size_t>(g.max_rows));
    off[6] = o;  // pom
    o += align16(mc * mc);
    off[7] = o;  // pbits
    o += align16(mc * (8 / kRhoOct) * sizeof(uint64_t));
    off[8] = o;  // tasks
    o += align16(static_cast<size_t>(g.max_tasks) * sizeof(Task));
    off[9] = o;  // wptr
    o += align16((kMaxTaskWarps + 1) * sizeof(int32_t));
    return o;
}

__host__ __device__ inline size_t table_bytes(const GridArgs& g) {
    size_t off[10];
    return tables_layout(g, off);
}

// Byte size of one buffer; off[] receives the section offsets (off[10] = acc,
// off[11] = Phi).
__host__ __device__ inline size_t buffer_layout(const GridArgs& g, size_t acc_doubles, size_t* off) {
    size_t o = tables_layout(g, off);
    off[10] = o;
    o += align16(acc_doubles * sizeof(double));
    off[11] = o;
    o += align16(static_cast<size_t>(g.max_rows) * 64 * sizeof(double));
    return o;
}

// Host: the layout of a buffer with `acc_doubles` accumulator doubles into
// g.lay (every launcher calls this before launching).
inline void set_layout(GridArgs& g, size_t acc_doubles) {
    size_t off[12];
    const size_t bytes = buffer_layout(g, acc_doubles, off);
    for (int i = 0; i < 12; ++i) g.lay[i] = static_cast<uint32_t>(off[i]);
    g.lay[12] = static_cast<uint32_t>(bytes);
}

// Buffer at byte offset `base` of kbg_smem, laid out as g.lay.
__device__ __forceinline__ Smem carve(uint32_t base, const GridArgs& g) {
    Smem s;
    s.base = base;
    s.o_meta = g.lay[0];
    s.o_cov = g.lay[1];
    s.o_grp = g.lay[2];
    s.o_off2d = g.lay[3];
    s.o_rcov = g.lay[4];
    s.o_rorb = g.lay[5];
    s.o_pom = g.lay[6];
    s.o_pbits = g.lay[7];
    s.o_task = g.lay[8];
    s.o_wptr = g.lay[9];
    s.o_acc = g.lay[10];
    s.o_phi = g.lay[11];
    return s;
}

__device__ __forceinline__ int64_t slot_point(const SysParams& P, int bi, int bj, int bk, int s, bool& valid) {
    int li, lj, lk;
    slot_decode(s, li, lj, lk);
    const int i = bi * 4 + li, j = bj * 4 + lj, k = bk * 4 + lk;
    valid = i < P.N[0] && j < P.N[1] && k < P.N[2];
    return (static_cast<int64_t>(i) * P.N[1] + j) * P.N[2] + k;
}

// Positions of slots 2l and 2l + 1 of block (bi, bj, bk). The geometry cache and stage_block share
// these expressions, written with explicit round-to-nearest operations (no FMA contraction left to
// the compiler, like the oracle's -ffp-contract=off), so both produce the same Phi bits in any kernel.
__device__ __forceinline__ void slot_pair_pos(const SysParams& P, int bi, int bj, int bk, int l, double (&r)[2][3]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        int li, lj, lk;
        slot_decode(2 * l + h, li, lj, lk);
        point_pos_exact(P, bi * 4 + li, bj * 4 + lj, bk * 4 + lk, r[h]);
    }
}

// Orbitals of one cover (image position t, slot mask, species) at slots 2l, 2l + 1 (positions r):
// sink(o, {value at 2l, value at 2l + 1}), exact zeros outside the mask.
template <class Sink>
__device__ __forceinline__ void phi_slot_pair(const SysParams& P, const double* __restrict__ tables,
                                              const double (&t)[3], uint64_t mask, int sp, const double (&r)[2][3],
                                              int l, Sink&& sink) {
    double d[2][3], d2[2];
    bool in[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        in[h] = (mask >> (2 * l + h)) & 1;
#pragma unroll
        for (int q = 0; q < 3; ++q) d[h][q] = __dsub_rn(r[h][q], t[q]);
        d2[h] = dist2_exact(d[h]);
        if (!in[h]) d2[h] = 0.0;  // unused value, keeps the table index in range
    }
    eval_orbitals_pair(P.sp[sp], tables, d, d2, [&](int o, double v0, double v1) {
        sink(o, make_double2(in[0] ? v0 : 0.0, in[1] ? v1 : 0.0));
    });
}

// Stages block b into buffer sm using threads [0, nt) (tid = this thread's
// index among them); sync() is a barrier over exactly those threads. For H
// (density = false) also stages w = V dV for every spin; for rho zeroes the
// per-warp accumulators. Returns ncov (0: nothing to compute).
template <class Sync>
__device__ int stage_block(const GridArgs& g, int64_t b, const Smem& sm, int tid, int nt, Sync&& sync, bool density,
                           int acc_warps, bool eval_phi = true) {
    const int c0 = g.blk_ptr[b];
    const int ncov = g.blk_ptr[b + 1] - c0;
    if (tid == 0) {
        sm.meta()->block = b;
        sm.meta()->ncov = ncov;
        sm.meta()->done = 0;
        sm.meta()->next = 0;
    }
    if (ncov == 0) {
        sync();
        return 0;
    }
    const SysParams& P = g.sys;
    if (tid < ncov) {
        CoverS& cv = sm.cov()[tid];
        const int a = g.cov_atom[c0 + tid];
        cv.sp = P.spc[a];
        cv.norb = P.sp[cv.sp].norb;
        cv.mask = g.cov_mask[c0 + tid];
        const int R0 = g.cov_R[3 * (c0 + tid)], R1 = g.cov_R[3 * (c0 + tid) + 1], R2 = g.cov_R[3 * (c0 + tid) + 2];
        image_pos_exact(P, P.tau + 3 * a, R0, R1, R2, cv.t);  // the oracle's expression, no contraction
    }
    const int64_t tp0 = g.t_ptr[b];
    const int ntask = static_cast<int>(g.t_ptr[b + 1] - tp0);
    for (int i = tid; i < ntask; i += nt) sm.task()[i] = g.tasks[tp0 + i];
    if (tid <= kMaxTaskWarps) sm.wptr()[tid] = g.t_wptr[b * (kMaxTaskWarps + 1) + tid];
    for (int i = tid; i < ncov * ncov; i += nt) sm.off2d()[i] = -1;
    for (int i = tid; i < g.max_rows; i += nt) sm.rcov()[i] = kNoCover;
    int bi, bj, bk;
    block_decode(P, b, bi, bj, bk);
    if (density) {
        for (int i = tid; i < g.nspin * acc_warps * 64; i += nt) sm.acc()[i] = 0.0;
    } else if (g.in) {
        for (int i = tid; i < g.nspin * 64; i += nt) {
            bool valid;
            const int64_t pt = slot_point(P, bi, bj, bk, i & 63, valid);
            const double v = valid ? g.in[(i >> 6) * g.npts + pt] : 0.0;
            sm.acc()[i] = v * (g.dV * g.sign);  // fault hook (sign -1) folded into w
            if (!isfinite(v) && g.vbits)  // non-finite V: flag for the host API (KBG_ERR_NONFINITE)
                atomicMax(const_cast<unsigned long long*>(g.vbits), 0x7ff8000000000000ull);
        }
    }
    sync();
    if (tid == 0) {
        int gf[kMaxCoverPerBlock], ge[kMaxCoverPerBlock], gr0[kMaxCoverPerBlock], grs[kMaxCoverPerBlock],
            cr0[kMaxCoverPerBlock], cg[kMaxCoverPerBlock];
        const int ng = make_groups(ncov, [&](int c) { return sm.cov()[c].norb; }, gf, ge, gr0, grs, cr0, cg);
        for (int q = 0; q < ng; ++q) sm.grp()[q] = GroupS{gf[q], ge[q], gr0[q], grs[q], (grs[q] + 7) >> 3};
        for (int c = 0; c < ncov; ++c) {
            sm.cov()[c].row0 = cr0[c];
            sm.cov()[c].grp = cg[c];
        }
        sm.meta()->ngrp = ng;
        sm.meta()->rows = gr0[ng - 1] + grs[ng - 1];
    }
    {
        const int64_t p0 = g.bp_ptr[b], p1 = g.bp_ptr[b + 1];
        for (int64_t e = p0 + tid; e < p1; e += nt) {
            const BPair bp = g.bp[e];
            sm.off2d()[(bp.cicj & 0xffff) * ncov + (bp.cicj >> 16)] = density ? bp.roff : static_cast<int32_t>(bp.off);
        }
    }
    sync();
    const int ngrp = sm.meta()->ngrp, rows = sm.meta()->rows;
    for (int i = tid; i < ngrp * ncov; i += nt) {
        const int q = i / ncov, cj = i % ncov;
        const GroupS& G = sm.grp()[q];
        uint64_t m = 0;
        if (cj >= G.first)
            for (int ci = G.first; ci < G.end && ci <= cj; ++ci) m |= sm.cov()[ci].mask & sm.cov()[cj].mask;
        sm.pom()[i] = static_cast<uint8_t>(octet_bits(m));
    }
    if (tid < ncov) {
        const CoverS& cv = sm.cov()[tid];
        for (int o = 0; o < cv.norb; ++o) {
            sm.rcov()[cv.row0 + o] = static_cast<uint8_t>(tid);
            sm.rorb()[cv.row0 + o] = static_cast<uint8_t>(o);
        }
    }
    if (eval_phi)
        for (int i = tid; i < 8 * 64; i += nt) sm.phi()[rows * 64 + i] = 0.0;  // tail rows (tile overrun)
    // two slots per thread, the same expressions as the geometry cache (kb_cache.cu k_phi_cache):
    // both Phi paths give the same bits, so H/rho do not depend on the kernel choice
    for (int task = tid; eval_phi && task < ncov * 32; task += nt) {
        const int c = task >> 5, l = task & 31;
        const CoverS& cv = sm.cov()[c];
        double r[2][3];
        slot_pair_pos(P, bi, bj, bk, l, r);
        phi_slot_pair(P, P.tables, cv.t, cv.mask, cv.sp, r, l, [&](int o, double2 v) {
            *reinterpret_cast<double2*>(sm.phi() + (cv.row0 + o) * 64 + ((2 * l) ^ swz(cv.row0 + o))) = v;
        });
    }
    sync();
    constexpr int kParts = 8 / kRhoOct;
    if (tid < ngrp * kParts) {
        const int q = tid / kParts, h = tid % kParts;
        uint64_t bits = 0;
        for (int cj = 0; cj < ncov; ++cj)
            if ((sm.pom()[q * ncov + cj] >> (kRhoOct * h)) & ((1u << kRhoOct) - 1u)) bits |= 1ull << cj;
        sm.pbits()[tid] = bits;
    }
    sync();
    return ncov;
}

// ---- H --------------------------------------------------------------------------
// Deterministic accumulation (KBG_OPT_DETERMINISTIC; scatter bit value 16).
// FP64 atomics add in arrival order, so plain RED.ADD.F64 makes H's last bits
// depend on the schedule. Instead every contribution v (one task's sum over
// the block points it covers) is split into two parts that lie on FIXED grids,
//   hi = round(v, g1), g1 = 2^(E-50);   lo = round(v - hi, g2), g2 = 2^(E-84),
// with 2^E >= max|w| * hbound >= sum of |contributions| of any H entry (kb_api.cu:
// h_bound). Every partial sum of the hi parts is then a multiple of g1 below
// 2^53 g1 and every partial sum of the lo parts a multiple of g2 below 2^53 g2:
// all additions are exact, so the two accumulators (interleaved [entry][2])
// hold the same bits whatever the order of the atomics -- across runs, kernels,
// and rank counts (the multi-GPU reduction adds the limbs the same way,
// kb_comm.cu). H = hi + lo is rounded once at the end (k_finalize). Rounding
// to a grid is two exact additions of C = 1.5 * 2^(k+52) (|x| < 2^(k+51)):
// (x + C) - C is x rounded to a multiple of 2^k.
struct HScale {
    double c1, c2;   // rounding constants of the hi and lo grids
    long long lo;    // offset (doubles) of an entry's lo limb from its hi limb (KBG_DET_SPLIT: nnz, else 1)
};
__shared__ HScale s_hscale;  // per CTA, set by thread 0 at kernel start

// FP64 reduction into global memory as a fire-and-forget RED (the compiler
// otherwise emits ATOMG with a discarded return value here).
__device__ __forceinline__ void red_add(double* p, double v) {
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// (C1, C2) from the bit pattern of max|V| (sign cleared; NaN/inf give NaN H)
// and wfac = |dV| * hbound.
__device__ __forceinline__ HScale hscale_of(unsigned long long vbits, double wfac, int64_t nnz) {
    HScale h;
    h.lo = KBG_DET_SPLIT ? nnz : 1;
    const double m = __longlong_as_double(static_cast<long long>(vbits & 0x7fffffffffffffffull)) * wfac;
    if (!(m <= 1.79e308)) {
        h.c1 = __longlong_as_double(0x7ff8000000000000ll);
        h.c2 = 0.0;
        return h;
    }
    int E = -900;
    if (m > 0.0) {
        int e;
        frexp(m, &e);  // m < 2^e
        E = e > -900 ? e : -900;
    }
    h.c1 = ldexp(1.5, E + 2);
    h.c2 = ldexp(1.5, E - 32);
    return h;
}

// Column of cj (within an 8-column tile) behind DMMA column n of the H tiles. With KBG_H_PERMCOL the
// B fragments load orbital rows in the order 0 6 1 7 2 4 3 5, so a RED instruction (fixed e of the C
// fragment's column pair 2q + e) covers 4 contiguous columns of every row -- half the L2 sectors of the
// identity order's alternate columns -- and the 4 rows of a half-warp's B loads keep distinct row & 3
// (conflict-free under the Phi swizzle).
__device__ __forceinline__ int hcol_of_n(int n) {
    return KBG_H_PERMCOL ? ((n & 1) ? 4 + ((n >> 1) ^ 2) : (n >> 1)) : n;
}

// Scatter of one accumulated tile: rows ra0 + [0, 8*TM) (group rows < rend),
// columns cb0 + [0, 8*TN) of cover cj; canonical rows (cover ci <= cj) only.
template <bool DET, int TM, int TN>
__device__ __forceinline__ void h_scatter(const Smem& sm, const double (&c)[TM][TN][2], int ncov, int cj, int ra0,
                                          int rend, int cb0, double* __restrict__ H, int scatter,
                                          int lane) {
    const int nb = sm.cov()[cj].norb;
    const double c1 = DET ? s_hscale.c1 : 0.0, c2 = DET ? s_hscale.c2 : 0.0;
    const long long lo_off = DET ? s_hscale.lo : 0;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int r = ra0 + 8 * i + (lane >> 2);
        const int ci = r < rend ? sm.rcov()[r] : kNoCover;
        const int off = ci <= cj ? sm.off2d()[ci * ncov + cj] : -1;  // kNoCover (255) fails ci <= cj
        const int ri = sm.rorb()[r];
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = cb0 + 8 * j + hcol_of_n((lane & 3) * 2 + e);
                if (off >= 0 && col < nb && !(KBG_EXPERIMENTS && (scatter & 2))) {
                    const double v = c[i][j][e];  // the fault hook's sign is folded into w
                    if (DET) {
                        const double hi = __dsub_rn(__dadd_rn(v, c1), c1);
                        const double lo = __dsub_rn(__dadd_rn(__dsub_rn(v, hi), c2), c2);
                        double* p = H + (KBG_DET_SPLIT ? 1 : 2) * (off + ri * nb + col);
                        if (!(KBG_EXPERIMENTS && (scatter & 8))) red_add(p, hi);  // bits 8, 4: timing
                        if (!(KBG_EXPERIMENTS && (scatter & 4))) red_add(p + lo_off, lo);  // experiments only
                    } else if (!(KBG_EXPERIMENTS && (scatter & 1))) {
                        red_add(H + off + ri * nb + col, v);
                    } else {
                        H[off + ri * nb + col] = v;
                    }
                }
            }
    }
}

// One partner: C(8*TM x 8*TN) += Phi_rows diag(w) Phi_cj^T over the quads in
// qm. Tiles with <= 2 DMMAs per quad alternate two accumulator sets.
template <bool DET, int TM, int TN>
__device__ __forceinline__ void h_tile(const Smem& sm, const double* __restrict__ w, int ncov, int cj, int ra0,
                                       int rend, int cb0, uint32_t qm, double* __restrict__ H, int scatter,
                                       int lane) {
    constexpr int NACC = (TM * TN <= 2) ? 2 : 1;
    double c[NACC][TM][TN][2];
#pragma unroll
    for (int u = 0; u < NACC; ++u)
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) c[u][i][j][0] = c[u][i][j][1] = 0.0;
    const CoverS& B = sm.cov()[cj];
    const int ra = ra0 + (lane >> 2), rb = B.row0 + cb0 + hcol_of_n(lane >> 2);
    const double* pa = sm.phi() + ra * 64 + (lane & 3);
    const double* pb = sm.phi() + rb * 64 + (lane & 3);
    const int sa = swz(ra), sb = swz(rb);  // 8-row steps keep row & 3
    const double* pw = w + (lane & 3);
    auto step = [&](int u, int q) {
        const int col = 4 * q;
        const double wv = pw[col];
        double a[TM], bb[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = pa[i * 512 + (col ^ sa)] * wv;
#pragma unroll
        for (int j = 0; j < TN; ++j) bb[j] = pb[j * 512 + (col ^ sb)];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) dmma(c[u][i][j], a[i], bb[j]);
    };
    while (qm) {
        const int q0 = __ffs(qm) - 1;
        qm &= qm - 1;
        if (NACC == 2 && qm) {
            const int q1 = __ffs(qm) - 1;
            qm &= qm - 1;
            step(0, q0);
            step(NACC - 1, q1);
        } else {
            step(0, q0);
        }
    }
    if (NACC == 2)
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                c[0][i][j][0] += c[NACC - 1][i][j][0];
                c[0][i][j][1] += c[NACC - 1][i][j][1];
            }
    h_scatter<DET, TM, TN>(sm, c[0], ncov, cj, ra0, rend, cb0, H, scatter, lane);
}

// Two partners sharing the group's (w-scaled) A fragments: per quad of
// q1 | q2 the A fragments are loaded and scaled once.
template <bool DET, int TM, int TN1, int TN2>
__device__ __forceinline__ void h_tile2(const Smem& sm, const double* __restrict__ w, int ncov, int cj1, int cj2,
                                        int ra0, int rend, uint32_t q1, uint32_t q2, double* __restrict__ H,
                                        int scatter, int lane) {
    double c1[TM][TN1][2], c2[TM][TN2][2];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
#pragma unroll
        for (int j = 0; j < TN1; ++j) c1[i][j][0] = c1[i][j][1] = 0.0;
#pragma unroll
        for (int j = 0; j < TN2; ++j) c2[i][j][0] = c2[i][j][1] = 0.0;
    }
    const int ra = ra0 + (lane >> 2);
    const int rb1 = sm.cov()[cj1].row0 + hcol_of_n(lane >> 2), rb2 = sm.cov()[cj2].row0 + hcol_of_n(lane >> 2);
    const double* pa = sm.phi() + ra * 64 + (lane & 3);
    const double* pb1 = sm.phi() + rb1 * 64 + (lane & 3);
    const double* pb2 = sm.phi() + rb2 * 64 + (lane & 3);
    const int sa = swz(ra), sb1 = swz(rb1), sb2 = swz(rb2);
    const double* pw = w + (lane & 3);
    // Three loops -- quads of both partners, of cj1 only, of cj2 only -- so every DMMA is
    // unconditional: a DMMA under a per-quad predicate the compiler cannot prove warp-uniform
    // costs a WARPSYNC + NOP pair each (SASS of the single merged loop, profiles/ncu_h_r2.txt).
#if KBG_H_BYTEADDR
    // byte offsets: the swizzled quad offset is one XOR of the quad's byte offset with the row's swizzle
    // bytes, added to a per-lane byte pointer (two instructions per operand address)
    const char* ca = reinterpret_cast<const char*>(pa);
    const char* cb1 = reinterpret_cast<const char*>(pb1);
    const char* cb2 = reinterpret_cast<const char*>(pb2);
    const char* cw = reinterpret_cast<const char*>(pw);
    const uint32_t sa8 = 8u * sa, sb18 = 8u * sb1, sb28 = 8u * sb2;
#endif
    auto run = [&](uint32_t qm, auto with1, auto with2) {
        constexpr bool W1 = decltype(with1)::value, W2 = decltype(with2)::value;
        while (qm) {
            const int q = __ffs(qm) - 1;
            qm &= qm - 1;
#if KBG_H_BYTEADDR
            const uint32_t qo = static_cast<uint32_t>(q) << 5;
            const double wv = *reinterpret_cast<const double*>(cw + qo);
            double a[TM];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = *reinterpret_cast<const double*>(ca + i * 4096 + (qo ^ sa8)) * wv;
#else
            const int col = 4 * q;
            const double wv = pw[col];
            double a[TM];
#pragma unroll
            for (int i = 0; i < TM; ++i)
                a[i] = pa[i * 512 + (col ^ sa)] * wv;
#endif
            if (W1) {
                double bb[TN1];
#pragma unroll
                for (int j = 0; j < TN1; ++j)
#if KBG_H_BYTEADDR
                    bb[j] = *reinterpret_cast<const double*>(cb1 + j * 4096 + (qo ^ sb18));
#else
                    bb[j] = pb1[j * 512 + (col ^ sb1)];
#endif
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN1; ++j) dmma(c1[i][j], a[i], bb[j]);
            }
            if (W2) {
                double bb[TN2];
#pragma unroll
                for (int j = 0; j < TN2; ++j)
#if KBG_H_BYTEADDR
                    bb[j] = *reinterpret_cast<const double*>(cb2 + j * 4096 + (qo ^ sb28));
#else
                    bb[j] = pb2[j * 512 + (col ^ sb2)];
#endif
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN2; ++j) dmma(c2[i][j], a[i], bb[j]);
            }
        }
    };
    run(q1 & q2, std::true_type{}, std::true_type{});
    run(q1 & ~q2, std::true_type{}, std::false_type{});
    run(q2 & ~q1, std::false_type{}, std::true_type{});
    h_scatter<DET, TM, TN1>(sm, c1, ncov, cj1, ra0, rend, 0, H, scatter, lane);
    h_scatter<DET, TM, TN2>(sm, c2, ncov, cj2, ra0, rend, 0, H, scatter, lane);
}

template <bool DET, int TM, int TN1>
__device__ __forceinline__ void h_tile2_tn2(int tn2, const Smem& sm, const double* w, int ncov, int cj1, int cj2,
                                            int ra0, int rend, uint32_t q1, uint32_t q2, double* H,
                                            int scatter, int lane) {
    if (tn2 == 2)
        h_tile2<DET, TM, TN1, 2>(sm, w, ncov, cj1, cj2, ra0, rend, q1, q2, H, scatter, lane);
    else
        h_tile2<DET, TM, TN1, 1>(sm, w, ncov, cj1, cj2, ra0, rend, q1, q2, H, scatter, lane);
}

// One H element into the accumulator (FP64 RED, or the deterministic two-limb split).
template <bool DET>
__device__ __forceinline__ void h_add(double* __restrict__ H, int64_t idx, double v) {
    if (DET) {
        const double hi = __dsub_rn(__dadd_rn(v, s_hscale.c1), s_hscale.c1);
        const double lo = __dsub_rn(__dadd_rn(__dsub_rn(v, hi), s_hscale.c2), s_hscale.c2);
        double* p = H + (KBG_DET_SPLIT ? 1 : 2) * idx;
        red_add(p, hi);
        red_add(p + s_hscale.lo, lo);
    } else {
        red_add(H + idx, v);
    }
}

// A5's sparse alternative (north star: DMMA "only where the atom-pair orbital block is dense enough,
// otherwise warp-shuffle reductions"): the same task as point-exact FP64 FMAs over the common points
// only (no quad padding). Lane l owns row (l & 15) of the group and 8 columns (half l >> 4) of the
// partner; per common point one A value (scaled by w) and 8 B values, which all 16 lanes of a half
// warp read at the same address (shared-memory broadcast). Selected per task by its point density
// (Task.pad2_, kb_tasks.cu) below the KBG_OPT_SPARSE_DFMA threshold (scatter bits 8..15).
template <bool DET>
__device__ __forceinline__ void h_task_dfma(const Smem& sm, const double* __restrict__ w, int ncov, const Task& t,
                                         double* __restrict__ H, int lane) {
    const GroupS& G = sm.grp()[t.g];
    const int r = G.row0 + (lane & 15);
    const bool row_ok = (lane & 15) < G.rows;
    const int ci = row_ok ? sm.rcov()[r] : kNoCover;
    const int ri = sm.rorb()[r];
    const double* phi = sm.phi();
    for (int k = 0; k < 2; ++k) {
        const int cj = k ? t.cj2 : t.cj;
        if (cj == kNoCover) break;
        const CoverS& B = sm.cov()[cj];
        uint64_t m = 0;  // exact common points of the group's canonical rows and cj
        for (int c = G.first; c < G.end && c <= cj; ++c) m |= sm.cov()[c].mask & B.mask;
        const int nb = B.norb, c0 = 8 * (lane >> 4);
        double acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.0;
        while (m) {
            const int p = __ffsll(m) - 1;
            m &= m - 1;
            const double a = phi[phi_idx(r, p)] * w[p];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int rb = B.row0 + min(c0 + j, nb - 1);
                acc[j] = fma(a, phi[phi_idx(rb, p)], acc[j]);
            }
        }
        const int off = ci <= cj ? sm.off2d()[ci * ncov + cj] : -1;
        if (off >= 0)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (c0 + j < nb) h_add<DET>(H, off + ri * nb + c0 + j, acc[j]);
    }
}

template <bool DET, bool SPARSE = false>
__device__ __forceinline__ void h_task(const Smem& sm, const double* w, int ncov, const Task& t, double* H,
                                       int scatter, int lane, bool dfma_warp = false) {
    if (SPARSE && (dfma_warp || t.pad2_ < ((scatter >> 8) & 0xFF))) {
        h_task_dfma<DET>(sm, w, ncov, t, H, lane);
        return;
    }
    const GroupS& G = sm.grp()[t.g];
    const int rend = G.row0 + G.rows;
    // quad masks made provably warp-uniform (a shuffle from lane 0): the DMMA loops over them then
    // need no WARPSYNC (mma.sync requires the converged warp)
    const uint32_t q1 = __shfl_sync(0xffffffffu, static_cast<uint32_t>(t.qmask), 0);
    if (t.cj2 != 0xFF) {  // paired partners: group <= 16 rows, partners <= 16 orbitals
        const uint32_t q2 = __shfl_sync(0xffffffffu, static_cast<uint32_t>(t.qmask2), 0);
        const int tn1 = (sm.cov()[t.cj].norb + 7) >> 3, tn2 = (sm.cov()[t.cj2].norb + 7) >> 3;
        if (G.tm == 2) {
            if (tn1 == 2)
                h_tile2_tn2<DET, 2, 2>(tn2, sm, w, ncov, t.cj, t.cj2, G.row0, rend, q1, q2, H, scatter,
                                  lane);
            else
                h_tile2_tn2<DET, 2, 1>(tn2, sm, w, ncov, t.cj, t.cj2, G.row0, rend, q1, q2, H, scatter,
                                  lane);
        } else {
            if (tn1 == 2)
                h_tile2_tn2<DET, 1, 2>(tn2, sm, w, ncov, t.cj, t.cj2, G.row0, rend, q1, q2, H, scatter,
                                  lane);
            else
                h_tile2_tn2<DET, 1, 1>(tn2, sm, w, ncov, t.cj, t.cj2, G.row0, rend, q1, q2, H, scatter,
                                  lane);
        }
        return;
    }
    const int nb = sm.cov()[t.cj].norb;
    const uint32_t qm = q1;
    for (int i0 = 0; i0 < G.tm; i0 += 2) {
        const int tm = min(2, G.tm - i0);
        for (int j0 = 0; j0 < (nb + 7) >> 3; j0 += 2) {
            const int tn = min(2, ((nb + 7) >> 3) - j0);
            const int ra0 = G.row0 + 8 * i0, cb0 = 8 * j0;
            if (tm == 2 && tn == 2)
                h_tile<DET, 2, 2>(sm, w, ncov, t.cj, ra0, rend, cb0, qm, H, scatter, lane);
            else if (tm == 2)
                h_tile<DET, 2, 1>(sm, w, ncov, t.cj, ra0, rend, cb0, qm, H, scatter, lane);
            else if (tn == 2)
                h_tile<DET, 1, 2>(sm, w, ncov, t.cj, ra0, rend, cb0, qm, H, scatter, lane);
            else
                h_tile<DET, 1, 1>(sm, w, ncov, t.cj, ra0, rend, cb0, qm, H, scatter, lane);
        }
    }
}

// ---- rho ------------------------------------------------------------------------
// Repacked DM (k_dm_repack): canonical pair blocks, rows padded to 16-column
// chunks, column j = 16c + 4s + k stored at 16c + 4k + s and pre-scaled (x2
// except the (a,a,0) blocks). Lane k of a DMMA A fragment then reads its four
// K-step values as two 16-byte loads.
template <int TM>
__device__ __forceinline__ void gather_a(const Smem& sm, int ncov, const int (&rci)[TM], const int (&rri)[TM], int cj,
                                         int kc, const double* __restrict__ Dr, int lane, double (&a)[TM][4]) {
    const int stride = 16 * ((sm.cov()[cj].norb + 15) >> 4);
#if KBG_L2_HINT >= 2
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
#pragma unroll
    for (int t = 0; t < TM; ++t) {
        const int ci = rci[t];
        const int off = ci <= cj ? sm.off2d()[ci * ncov + cj] : -1;  // ci = kNoCover (255) fails ci <= cj
#if KBG_RHO_PGATHER
        // predicated loads (no divergent branch: rows without a pair to cj differ per lane)
        const uint32_t e = static_cast<uint32_t>(off) + static_cast<uint32_t>(rri[t] * stride + 16 * kc) +
                           4u * static_cast<uint32_t>(lane & 3);
        const double* p = Dr + e;
        asm("{\n\t.reg .pred q;\n\tsetp.ge.s32 q, %4, 0;\n\t"
            "mov.b64 %0, 0;\n\tmov.b64 %1, 0;\n\tmov.b64 %2, 0;\n\tmov.b64 %3, 0;\n\t"
            "@q ld.global.nc.v2.f64 {%0, %1}, [%5];\n\t@q ld.global.nc.v2.f64 {%2, %3}, [%5+16];\n\t}"
            : "=d"(a[t][0]), "=d"(a[t][1]), "=d"(a[t][2]), "=d"(a[t][3])
            : "r"(off), "l"(p));
#else
        if (off >= 0) {
            // 32-bit element offset (one IMAD.WIDE for the address instead of a 64-bit add chain)
            const uint32_t e = static_cast<uint32_t>(off) + static_cast<uint32_t>(rri[t] * stride + 16 * kc) +
                               4u * static_cast<uint32_t>(lane & 3);
            const double2* p = reinterpret_cast<const double2*>(Dr + e);
#if KBG_L2_HINT >= 2
            double2 v0, v1;
            asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v0.x), "=d"(v0.y) : "l"(p), "l"(pol));
            asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v1.x), "=d"(v1.y) : "l"(p + 1), "l"(pol));
#else
            const double2 v0 = __ldg(p), v1 = __ldg(p + 1);
#endif
            a[t][0] = v0.x;
            a[t][1] = v0.y;
            a[t][2] = v1.x;
            a[t][3] = v1.y;
        } else {
            a[t][0] = a[t][1] = a[t][2] = a[t][3] = 0.0;
        }
#endif
    }
}

// Order of one partner's DMMAs: 0 (default) octet-major, branching over octets
// outside the partner's overlap; 1 k-step-major, branching; 2 k-step-major over
// all octets of the part (Phi is exactly 0 outside a cover's support, so the
// extra products add exact zeros); 3 k-step-major with the DMMAs of octets
// outside the overlap predicated off; 4 octet pairs, both-active pairs with
// their DMMAs interleaved (4 accumulator chains in flight). With the octet mask
// made provably warp-uniform (KBG_RHO_UNIFORM: a shuffle from lane 0), order 0
// measures 0.359 ms for the 56-atom density pass vs 0.370 (3), 0.372 (3
// uniform), 0.373 (0 without the shuffle) and 0.402 (2); on the final tree
// 0.340 vs 0.379 (1) and 0.340 (4; 448 atoms 2.501 vs 2.510): the accumulator
// chains are not what limits rho.
#ifndef KBG_RHO_ORDER
#define KBG_RHO_ORDER 0
#endif
#ifndef KBG_RHO_UNIFORM
#define KBG_RHO_UNIFORM 1
#endif
template <int TM, int KS>
__device__ __forceinline__ void rho_partner(const double* __restrict__ pb, int swb, uint32_t om4,
                                            const double (&a)[TM][4], double (&y)[TM][kRhoOct][2], int colbase) {
#if KBG_RHO_ORDER == 0
#pragma unroll
    for (int o = 0; o < kRhoOct; ++o) {
        if (!((om4 >> o) & 1u)) continue;
        const int col = colbase + 8 * o;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const double bv = pb[s * 256 + (col ^ swb)];
#pragma unroll
            for (int t = 0; t < TM; ++t) dmma(y[t][o], a[t][s], bv);
        }
    }
#elif KBG_RHO_ORDER == 4
    // octet pairs: both active -> their DMMAs interleaved (4 accumulator chains in flight)
#pragma unroll
    for (int o = 0; o < kRhoOct; o += 2) {
        const uint32_t pm = (om4 >> o) & 3u;
        if (pm == 3u) {
#pragma unroll
            for (int s = 0; s < KS; ++s) {
                const double b0 = pb[s * 256 + ((colbase + 8 * o) ^ swb)];
                const double b1 = pb[s * 256 + ((colbase + 8 * o + 8) ^ swb)];
#pragma unroll
                for (int t = 0; t < TM; ++t) {
                    dmma(y[t][o], a[t][s], b0);
                    dmma(y[t][o + 1], a[t][s], b1);
                }
            }
        } else {
#pragma unroll
            for (int e = 0; e < 2; ++e) {  // compile-time accumulator index (no local memory)
                if (pm != (1u << e)) continue;
                const int col = colbase + 8 * (o + e);
#pragma unroll
                for (int s = 0; s < KS; ++s) {
                    const double bv = pb[s * 256 + (col ^ swb)];
#pragma unroll
                    for (int t = 0; t < TM; ++t) dmma(y[t][o + e], a[t][s], bv);
                }
            }
        }
    }
#elif KBG_RHO_ORDER == 3
#pragma unroll
    for (int s = 0; s < KS; ++s)
#pragma unroll
        for (int o = 0; o < kRhoOct; ++o) {
            const uint32_t on = (om4 >> o) & 1u;
            const double bv = pb[s * 256 + ((colbase + 8 * o) ^ swb)];
#pragma unroll
            for (int t = 0; t < TM; ++t) dmma_if(y[t][o], a[t][s], bv, on);
        }
#else
#pragma unroll
    for (int s = 0; s < KS; ++s)
#pragma unroll
        for (int o = 0; o < kRhoOct; ++o) {
            if (KBG_RHO_ORDER == 1 && !((om4 >> o) & 1u)) continue;
            const double bv = pb[s * 256 + ((colbase + 8 * o) ^ swb)];
#pragma unroll
            for (int t = 0; t < TM; ++t) dmma(y[t][o], a[t][s], bv);
        }
#endif
}

template <int TM>
__device__ void rho_task_rows(const Smem& sm, int ncov, int gi, int ra0, int h, int cbeg, int cend,
                              const double* __restrict__ Dr, double* __restrict__ racc, int lane) {
    const GroupS& G = sm.grp()[gi];
    const int rend = G.row0 + G.rows;
    int rci[TM], rri[TM];
#pragma unroll
    for (int t = 0; t < TM; ++t) {
        const int r = ra0 + 8 * t + (lane >> 2);
        rci[t] = r < rend ? sm.rcov()[r] : kNoCover;
        rri[t] = sm.rorb()[r];
    }
    double y[TM][kRhoOct][2];
#pragma unroll
    for (int t = 0; t < TM; ++t)
#pragma unroll
        for (int o = 0; o < kRhoOct; ++o) y[t][o][0] = y[t][o][1] = 0.0;
    const uint8_t* pom = sm.pom() + gi * ncov;
    uint64_t bits = sm.pbits()[(8 / kRhoOct) * gi + h] & (~0ull << cbeg) &
                    (cend >= 64 ? ~0ull : ((1ull << cend) - 1ull));
    const int colbase = 8 * kRhoOct * h + (lane >> 2);
    // one K chunk (<= 16 orbitals of cj from orbital 16 kc) of one partner, D' fragments in `a`
    auto chunk = [&](const CoverS& B, int kc, uint32_t om4, const double (&a)[TM][4]) {
        const int ks = min(4, (B.norb - 16 * kc + 3) >> 2);
        const int rb = B.row0 + 16 * kc + (lane & 3);
        const double* pb = sm.phi() + rb * 64;
        const int swb = swz(rb);
        switch (ks) {
            case 1: rho_partner<TM, 1>(pb, swb, om4, a, y, colbase); break;
            case 2: rho_partner<TM, 2>(pb, swb, om4, a, y, colbase); break;
            case 3: rho_partner<TM, 3>(pb, swb, om4, a, y, colbase); break;
            default: rho_partner<TM, 4>(pb, swb, om4, a, y, colbase); break;
        }
    };
    // Partners in two 32-bit passes (blocks rarely have more than 32 covers: the common pass costs
    // 32-bit find-first-set and clear instead of 64-bit ones). One fragment set: more warps per SM hide
    // the gather latency (a ping-pong prefetch spills at 96 and 128 registers).
    for (int w32 = 0; w32 < 2; ++w32) {
        uint32_t bits32 = static_cast<uint32_t>(bits >> (32 * w32));
        while (bits32) {
            const int cj = 32 * w32 + __ffs(bits32) - 1;
            bits32 &= bits32 - 1;
            double a[TM][4];
            gather_a<TM>(sm, ncov, rci, rri, cj, 0, Dr, lane, a);
#if KBG_RHO_UNIFORM
            // provably warp-uniform (shuffle from lane 0): the octet branches need no WARPSYNC
            const uint32_t om4 = __shfl_sync(0xffffffffu, (pom[cj] >> (kRhoOct * h)) & ((1u << kRhoOct) - 1u), 0);
#else
            const uint32_t om4 = (pom[cj] >> (kRhoOct * h)) & ((1u << kRhoOct) - 1u);
#endif
            const CoverS& B = sm.cov()[cj];
            for (int kc = 0;;) {  // K chunks of 16 orbitals (one for every Fe3O4 cover)
                chunk(B, kc, om4, a);
                if (16 * ++kc >= B.norb) break;
                gather_a<TM>(sm, ncov, rci, rri, cj, kc, Dr, lane, a);
            }
        }
    }
    // rho(slot) += sum over rows of Phi_row(slot) * Y(row, slot): per-lane
    // partial products v[j] (j = 2*octet + e), then a reduce-scatter over the
    // 8 row lanes (xor 16, 8, 4).
    constexpr int NV = 2 * kRhoOct;
    double v[NV];
#pragma unroll
    for (int o = 0; o < kRhoOct; ++o) {
        const int p = 8 * (kRhoOct * h + o) + 2 * (lane & 3);
        v[2 * o] = v[2 * o + 1] = 0.0;
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            const int r = ra0 + 8 * t + (lane >> 2);
            const double2 f2 = *reinterpret_cast<const double2*>(sm.phi() + phi_idx(r, p));
            v[2 * o] += f2.x * y[t][o][0];
            v[2 * o + 1] += f2.y * y[t][o][1];
        }
    }
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
    double w4[NV / 2];
#pragma unroll
    for (int i = 0; i < NV / 2; ++i) {
        const double send = b4 ? v[i] : v[i + NV / 2];
        const double keep = b4 ? v[i + NV / 2] : v[i];
        w4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    if (NV == 8) {  // 4 octets: lane l ends with j = l >> 2
        double w2[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double send = b3 ? w4[i] : w4[i + 2];
            const double keep = b3 ? w4[i + 2] : w4[i];
            w2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
        const double send = b2 ? w2[0] : w2[1];
        const double keep = b2 ? w2[1] : w2[0];
        const double tot = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        const int j = lane >> 2;
        racc[8 * (kRhoOct * h + (j >> 1)) + 2 * (lane & 3) + (j & 1)] += tot;
    } else {  // 2 octets: lane l (bit 2 clear) ends with j = (l >> 3) & 3
        const double send = b3 ? w4[0] : w4[1];
        const double keep = b3 ? w4[1] : w4[0];
        double tot = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        tot += __shfl_xor_sync(0xffffffffu, tot, 4);
        const int j = (lane >> 3) & 3;
        if (!b2) racc[8 * (kRhoOct * h + (j >> 1)) + 2 * (lane & 3) + (j & 1)] += tot;
    }
}

__device__ __forceinline__ void rho_task(const Smem& sm, int ncov, const Task& t, const double* Dr, double* racc,
                                         int lane) {
    const GroupS& G = sm.grp()[t.g];
    for (int i0 = 0; i0 < G.tm; i0 += 2) {
        if (G.tm - i0 >= 2)
            rho_task_rows<2>(sm, ncov, t.g, G.row0 + 8 * i0, t.half, t.cj, t.qmask, Dr, racc, lane);
        else
            rho_task_rows<1>(sm, ncov, t.g, G.row0 + 8 * i0, t.half, t.cj, t.qmask, Dr, racc, lane);
    }
}

}  // namespace core
}  // namespace kbg
