// G2+G3 / G2+G4: fused orbital evaluation + density / Hamiltonian contraction.
//
// One CTA per 4x4x4 grid block (64 slots). Phi (FP64, M rows x 64 slots) is
// evaluated once into shared memory; rows are the block's covers (atom
// images) packed into row groups of <= 16 orbitals (two 8-row DMMA tiles).
// Work is split into per-block task lists built at index time and
// LPT-balanced over the CTA's warps (kb_tasks.cu):
//   H  task (group g, partner cover cj >= first(g)):
//        C(16 x 8*TN) += Phi_g^T diag(V dV) Phi_cj over the common 1x2x2 quads,
//        mma.sync.m8n8k4.f64 (SASS DMMA), K = 4 slots of a quad; canonical rows
//        (cover ci <= cj) are scattered with FP64 atomics, mirrored afterwards.
//   rho task (group g, octet half h):
//        Y(16 x 8 slots) += D'(16 x n_cj) Phi_cj(n_cj x 8) summed over all
//        partners cj >= first(g) in registers (D' = 2 DM for ci < cj, DM for
//        ci == cj: the symmetric half), then once per task
//        rho(slot) += sum_rows Phi_g * Y. Per-warp shared accumulators are
//        summed in a fixed order, so rho is bitwise deterministic.
#include "kb_device.cuh"

namespace kbg {

namespace {

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

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// Octets (2x2x2 cubes, 8 consecutive slots) with any bit set: OR-fold each
// byte into its low bit, then gather the 8 low bits with one multiply.
__device__ __forceinline__ uint32_t octet_bits(uint64_t m) {
    m |= m >> 4;
    m |= m >> 2;
    m |= m >> 1;
    return static_cast<uint32_t>(((m & 0x0101010101010101ull) * 0x0102040810204080ull) >> 56);
}

// Phi[row][slot] lives at row*64 + (slot ^ 4*(row & 3)): any 4 consecutive
// rows x 4 consecutive slots (a half-warp DMMA fragment) hit 32 banks.
__device__ __forceinline__ int swz(int row) { return (row & 3) << 2; }
__device__ __forceinline__ int phi_idx(int row, int slot) { return row * 64 + (slot ^ swz(row)); }

constexpr uint8_t kNoCover = 0xFF;

struct Smem {
    double* phi;
    double* acc;  // w[64] (H) or racc[NW][64] (rho)
    CoverS* cov;
    GroupS* grp;
    int32_t* off2d;  // [ncov][ncov] value offset of canonical pair (ci <= cj) with common points, else -1
    uint8_t* rcov;   // [rows] cover of each Phi row (kNoCover for pad rows)
    uint8_t* rorb;   // [rows] orbital index inside that cover
    uint8_t* pom;    // [ngrp][ncov] octets shared by group g (rows ci <= cj) and cover cj
    uint64_t* pbits; // [ngrp][2] covers cj with a shared octet in half h
    Task* task;
    int32_t* wptr;   // [kTaskWarps + 1]
};

__host__ __device__ __forceinline__ size_t align16(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }

__host__ __device__ inline size_t smem_layout(const GridArgs& g, int acc_doubles, size_t* off) {
    size_t o = 0;
    off[0] = o;
    o += align16(static_cast<size_t>(g.max_rows) * 64 * sizeof(double));
    off[1] = o;
    o += align16(static_cast<size_t>(acc_doubles) * sizeof(double));
    off[2] = o;
    o += align16(static_cast<size_t>(g.max_cover) * sizeof(CoverS));
    off[3] = o;
    o += align16(static_cast<size_t>(g.max_cover) * sizeof(GroupS));
    off[4] = o;
    o += align16(static_cast<size_t>(g.max_cover) * g.max_cover * sizeof(int32_t));
    off[5] = o;
    o += align16(static_cast<size_t>(g.max_rows));
    off[6] = o;
    o += align16(static_cast<size_t>(g.max_rows));
    off[7] = o;
    o += align16(static_cast<size_t>(g.max_tasks) * sizeof(Task));
    off[8] = o;
    o += align16((kTaskWarps + 1) * sizeof(int32_t));
    off[9] = o;
    o += align16(static_cast<size_t>(g.max_cover) * g.max_cover);
    off[10] = o;
    o += align16(static_cast<size_t>(g.max_cover) * 2 * sizeof(uint64_t));
    return o;
}

__device__ __forceinline__ Smem carve(unsigned char* base, const GridArgs& g, int acc_doubles) {
    size_t off[11];
    smem_layout(g, acc_doubles, off);
    Smem s;
    s.phi = reinterpret_cast<double*>(base + off[0]);
    s.acc = reinterpret_cast<double*>(base + off[1]);
    s.cov = reinterpret_cast<CoverS*>(base + off[2]);
    s.grp = reinterpret_cast<GroupS*>(base + off[3]);
    s.off2d = reinterpret_cast<int32_t*>(base + off[4]);
    s.rcov = base + off[5];
    s.rorb = base + off[6];
    s.task = reinterpret_cast<Task*>(base + off[7]);
    s.wptr = reinterpret_cast<int32_t*>(base + off[8]);
    s.pom = base + off[9];
    s.pbits = reinterpret_cast<uint64_t*>(base + off[10]);
    return s;
}

struct Block {
    int ncov, ngrp, rows;  // rows: padded Phi rows in use (without the 8 tail rows)
};

// Stages block b: covers, row groups, row tables, pair-offset table, this
// kernel's task list, and Phi (zeros outside spheres and in pad rows).
__device__ Block stage_block(const GridArgs& g, int64_t b, const Smem& sm) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int c0 = g.blk_ptr[b];
    Block blk;
    blk.ncov = g.blk_ptr[b + 1] - c0;
    blk.ngrp = 0;
    blk.rows = 0;
    if (blk.ncov == 0) return blk;
    const int ncov = blk.ncov;
    const SysParams& P = g.sys;
    if (tid < ncov) {
        CoverS& cv = sm.cov[tid];
        const int a = g.cov_atom[c0 + tid];
        cv.sp = P.spc[a];
        cv.norb = P.sp[cv.sp].norb;
        cv.mask = g.cov_mask[c0 + tid];
        const int R0 = g.cov_R[3 * (c0 + tid)], R1 = g.cov_R[3 * (c0 + tid) + 1], R2 = g.cov_R[3 * (c0 + tid) + 2];
#pragma unroll
        for (int c = 0; c < 3; ++c) cv.t[c] = P.tau[3 * a + c] + ((R0 * P.A[c] + R1 * P.A[3 + c]) + R2 * P.A[6 + c]);
    }
    const int64_t tp0 = g.t_ptr[b];
    const int ntask = static_cast<int>(g.t_ptr[b + 1] - tp0);
    for (int i = tid; i < ntask; i += nt) sm.task[i] = g.tasks[tp0 + i];
    if (tid <= kTaskWarps) sm.wptr[tid] = g.t_wptr[b * (kTaskWarps + 1) + tid];
    for (int i = tid; i < ncov * ncov; i += nt) sm.off2d[i] = -1;
    for (int i = tid; i < g.max_rows; i += nt) sm.rcov[i] = kNoCover;
    __syncthreads();
    if (tid == 0) {
        int gf[kMaxCoverPerBlock], ge[kMaxCoverPerBlock], gr0[kMaxCoverPerBlock], grs[kMaxCoverPerBlock],
            cr0[kMaxCoverPerBlock], cg[kMaxCoverPerBlock];
        const int ng = make_groups(ncov, [&](int c) { return sm.cov[c].norb; }, gf, ge, gr0, grs, cr0, cg);
        for (int q = 0; q < ng; ++q) sm.grp[q] = GroupS{gf[q], ge[q], gr0[q], grs[q], (grs[q] + 7) >> 3};
        for (int c = 0; c < ncov; ++c) {
            sm.cov[c].row0 = cr0[c];
            sm.cov[c].grp = cg[c];
        }
        sm.cov[0].grp |= ng << 16;  // broadcast the group count
    }
    {
        const int64_t p0 = g.bp_ptr[b], p1 = g.bp_ptr[b + 1];
        for (int64_t e = p0 + tid; e < p1; e += nt) {
            const BPair bp = g.bp[e];
            sm.off2d[(bp.cicj & 0xffff) * ncov + (bp.cicj >> 16)] = static_cast<int32_t>(bp.off);
        }
    }
    __syncthreads();
    blk.ngrp = sm.cov[0].grp >> 16;
    const GroupS& lg = sm.grp[blk.ngrp - 1];
    blk.rows = lg.row0 + lg.rows;
    // partner octet table: pom[g][cj] = octets shared by cover cj and the rows
    // ci <= cj of group g; pbits[g][h] = the covers cj with a shared octet in half h
    for (int i = tid; i < blk.ngrp * 2; i += nt) sm.pbits[i] = 0;
    for (int i = tid; i < blk.ngrp * ncov; i += nt) {
        const int q = i / ncov, cj = i % ncov;
        const GroupS& G = sm.grp[q];
        uint64_t m = 0;
        if (cj >= G.first)
            for (int ci = G.first; ci < G.end && ci <= cj; ++ci) m |= sm.cov[ci].mask & sm.cov[cj].mask;
        sm.pom[i] = static_cast<uint8_t>(octet_bits(m));
    }
    __syncthreads();
    if (tid < blk.ngrp * 2) {
        const int q = tid >> 1, h = tid & 1;
        uint64_t bits = 0;
        for (int cj = 0; cj < ncov; ++cj)
            if ((sm.pom[q * ncov + cj] >> (4 * h)) & 0xF) bits |= 1ull << cj;
        sm.pbits[tid] = bits;
    }
    if (tid < ncov) {
        const CoverS& cv = sm.cov[tid];
        for (int o = 0; o < cv.norb; ++o) {
            sm.rcov[cv.row0 + o] = static_cast<uint8_t>(tid);
            sm.rorb[cv.row0 + o] = static_cast<uint8_t>(o);
        }
    }
    __syncthreads();
    // zero the pad rows (group padding + 8 tail rows for tile overrun)
    for (int i = tid; i < (blk.rows + 8) * 64; i += nt)
        if (sm.rcov[i >> 6] == kNoCover) sm.phi[i] = 0.0;
    int bi, bj, bk;
    block_decode(P, b, bi, bj, bk);
    for (int task = tid; task < ncov * 64; task += nt) {
        const int c = task >> 6, s = task & 63;
        const CoverS& cv = sm.cov[c];
        double* dst = sm.phi;
        const int row0 = cv.row0;
        if ((cv.mask >> s) & 1) {
            int li, lj, lk;
            slot_decode(s, li, lj, lk);
            const double fi = static_cast<double>(bi * 4 + li) / P.N[0];
            const double fj = static_cast<double>(bj * 4 + lj) / P.N[1];
            const double fk = static_cast<double>(bk * 4 + lk) / P.N[2];
            const double dx = (fi * P.A[0] + fj * P.A[3] + fk * P.A[6]) - cv.t[0];
            const double dy = (fi * P.A[1] + fj * P.A[4] + fk * P.A[7]) - cv.t[1];
            const double dz = (fi * P.A[2] + fj * P.A[5] + fk * P.A[8]) - cv.t[2];
            const double d2 = dx * dx + dy * dy + dz * dz;
            eval_orbitals(P.sp[cv.sp], P.tables, dx, dy, dz, d2,
                          [&](int o, double v) { dst[phi_idx(row0 + o, s)] = v; });
        } else {
            for (int o = 0; o < cv.norb; ++o) dst[phi_idx(row0 + o, s)] = 0.0;
        }
    }
    __syncthreads();
    return blk;
}

__device__ __forceinline__ int64_t slot_point(const SysParams& P, int bi, int bj, int bk, int s, bool& valid) {
    int li, lj, lk;
    slot_decode(s, li, lj, lk);
    const int i = bi * 4 + li, j = bj * 4 + lj, k = bk * 4 + lk;
    valid = i < P.N[0] && j < P.N[1] && k < P.N[2];
    return (static_cast<int64_t>(i) * P.N[1] + j) * P.N[2] + k;
}

// ---- H task ---------------------------------------------------------------------
// Output tile rows ra0 + [0, 8*TM) (inside group g) x columns cb0 + [0, 8*TN)
// of cover cj. Tiles with <= 2 DMMAs per quad alternate two accumulator sets.
template <int TM, int TN>
__device__ __forceinline__ void h_tile(const Smem& sm, int ncov, int cj, int ra0, int rend, int cb0, uint32_t qm,
                                       double* __restrict__ H, double sign, int scatter, int lane) {
    constexpr int NACC = (TM * TN <= 2) ? 2 : 1;
    double c[NACC][TM][TN][2];
#pragma unroll
    for (int u = 0; u < NACC; ++u)
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) c[u][i][j][0] = c[u][i][j][1] = 0.0;
    const CoverS& B = sm.cov[cj];
    const int ra = ra0 + (lane >> 2), rb = B.row0 + cb0 + (lane >> 2);
    const double* pa = sm.phi + ra * 64 + (lane & 3);
    const double* pb = sm.phi + rb * 64 + (lane & 3);
    const int sa = swz(ra), sb = swz(rb);  // 8-row steps keep row & 3
    const double* pw = sm.acc + (lane & 3);
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
    const int nb = B.norb;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int r = ra0 + 8 * i + (lane >> 2);
        const int ci = r < rend ? sm.rcov[r] : kNoCover;
        const int off = (ci != kNoCover && ci <= cj) ? sm.off2d[ci * ncov + cj] : -1;
        const int ri = sm.rorb[r];
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = cb0 + 8 * j + (lane & 3) * 2 + e;
                double v = c[0][i][j][e];
                if (NACC == 2) v += c[NACC - 1][i][j][e];
                if (off >= 0 && col < nb) {
                    if (scatter == 0)
                        atomicAdd(H + off + ri * nb + col, sign * v);
                    else
                        H[off + ri * nb + col] = sign * v;
                }
            }
    }
}

__device__ __forceinline__ void h_task(const Smem& sm, int ncov, const Task& t, double* H, double sign, int scatter,
                                       int lane) {
    const GroupS& G = sm.grp[t.g];
    const int nb = sm.cov[t.cj].norb;
    const uint32_t qm = t.qmask;
    for (int i0 = 0; i0 < G.tm; i0 += 2) {
        const int tm = min(2, G.tm - i0);
        for (int j0 = 0; j0 < (nb + 7) >> 3; j0 += 2) {
            const int tn = min(2, ((nb + 7) >> 3) - j0);
            const int ra0 = G.row0 + 8 * i0, cb0 = 8 * j0, rend = G.row0 + G.rows;
            if (tm == 2 && tn == 2)
                h_tile<2, 2>(sm, ncov, t.cj, ra0, rend, cb0, qm, H, sign, scatter, lane);
            else if (tm == 2)
                h_tile<2, 1>(sm, ncov, t.cj, ra0, rend, cb0, qm, H, sign, scatter, lane);
            else if (tn == 2)
                h_tile<1, 2>(sm, ncov, t.cj, ra0, rend, cb0, qm, H, sign, scatter, lane);
            else
                h_tile<1, 1>(sm, ncov, t.cj, ra0, rend, cb0, qm, H, sign, scatter, lane);
        }
    }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 2) k_hamiltonian(GridArgs g) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Smem sm = carve(smem_raw, g, 64);
    const int64_t b = g.blk_begin + blockIdx.x;
    const Block blk = stage_block(g, b, sm);
    if (blk.ncov == 0) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int bi, bj, bk;
    block_decode(g.sys, b, bi, bj, bk);
    for (int spin = 0; spin < g.nspin; ++spin) {
        if (tid < 64) {
            bool valid;
            const int64_t pt = slot_point(g.sys, bi, bj, bk, tid, valid);
            sm.acc[tid] = valid ? g.in[spin * g.npts + pt] * g.dV : 0.0;
        }
        __syncthreads();
        double* Hs = g.out + spin * g.nnz;
        for (int w = warp; w < kTaskWarps; w += NW)
            for (int e = sm.wptr[w]; e < sm.wptr[w + 1]; ++e) h_task(sm, blk.ncov, sm.task[e], Hs, g.sign, g.scatter, lane);
        __syncthreads();
    }
}

// ---- rho task -------------------------------------------------------------------
// Rows ra0 + [0, 8*TM) of group g; octets 4h..4h+3; partners cj >= first(g).
// A = D'(rows x 4 cols of cj) gathered from the pair blocks (prefetched one
// partner ahead), B = Phi_cj(4 cols x 8 slots), C = Y(rows x 8 slots).
template <int TM>
struct RowInfo {
    int ci[TM];
    int ri[TM];
};

template <int TM>
__device__ __forceinline__ void gather_a(const Smem& sm, int ncov, const RowInfo<TM>& ri, int cj, int kc,
                                         const double* __restrict__ Ds, int lane, double (&a)[TM][4]) {
    const int nb = sm.cov[cj].norb;
#pragma unroll
    for (int t = 0; t < TM; ++t) {
        const int ci = ri.ci[t];
        const int off = (ci <= cj) ? sm.off2d[ci * ncov + cj] : -1;  // ci = kNoCover (255) fails ci <= cj
        const double fac = ci < cj ? 2.0 : 1.0;
        const double* row = Ds + off + ri.ri[t] * nb + 16 * kc + (lane & 3);
        const int jmax = nb - 16 * kc - (lane & 3);
#pragma unroll
        for (int s = 0; s < 4; ++s) a[t][s] = (off >= 0 && 4 * s < jmax) ? fac * __ldg(row + 4 * s) : 0.0;
    }
}

template <int TM, int KS>
__device__ __forceinline__ void rho_partner(const double* __restrict__ pb, int swb, uint32_t om4,
                                            const double (&a)[TM][4], double (&y)[TM][4][2], int colbase) {
#pragma unroll
    for (int o = 0; o < 4; ++o) {
        if (!((om4 >> o) & 1u)) continue;
        const int col = colbase + 8 * o;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const double bv = pb[s * 256 + (col ^ swb)];
#pragma unroll
            for (int t = 0; t < TM; ++t) dmma(y[t][o], a[t][s], bv);
        }
    }
}

template <int TM>
__device__ void rho_task_rows(const Smem& sm, int ncov, int gi, int ra0, int h, const double* __restrict__ Ds,
                              double* __restrict__ racc, int lane) {
    const GroupS& G = sm.grp[gi];
    const int rend = G.row0 + G.rows;
    RowInfo<TM> ri;
#pragma unroll
    for (int t = 0; t < TM; ++t) {
        const int r = ra0 + 8 * t + (lane >> 2);
        ri.ci[t] = r < rend ? sm.rcov[r] : kNoCover;
        ri.ri[t] = sm.rorb[r];
    }
    double y[TM][4][2];
#pragma unroll
    for (int t = 0; t < TM; ++t)
#pragma unroll
        for (int o = 0; o < 4; ++o) y[t][o][0] = y[t][o][1] = 0.0;
    const uint8_t* pom = sm.pom + gi * ncov;
    uint64_t bits = sm.pbits[2 * gi + h];
    const int colbase = 32 * h + (lane >> 2);
    double nxt[TM][4];
    if (bits) gather_a<TM>(sm, ncov, ri, __ffsll(bits) - 1, 0, Ds, lane, nxt);
    while (bits) {
        const int cj = __ffsll(bits) - 1;
        bits &= bits - 1;
        const uint32_t om4 = (pom[cj] >> (4 * h)) & 0xFu;
        const CoverS& B = sm.cov[cj];
        double a[TM][4];
#pragma unroll
        for (int t = 0; t < TM; ++t)
#pragma unroll
            for (int s = 0; s < 4; ++s) a[t][s] = nxt[t][s];
        const int nkc = (B.norb + 15) >> 4;
        if (nkc == 1 && bits) gather_a<TM>(sm, ncov, ri, __ffsll(bits) - 1, 0, Ds, lane, nxt);
        for (int kc = 0; kc < nkc; ++kc) {
            if (kc > 0) gather_a<TM>(sm, ncov, ri, cj, kc, Ds, lane, a);
            const int ks = min(4, (B.norb - 16 * kc + 3) >> 2);
            const int rb = B.row0 + 16 * kc + (lane & 3);
            const double* pb = sm.phi + rb * 64;
            const int swb = swz(rb);
            switch (ks) {
                case 1: rho_partner<TM, 1>(pb, swb, om4, a, y, colbase); break;
                case 2: rho_partner<TM, 2>(pb, swb, om4, a, y, colbase); break;
                case 3: rho_partner<TM, 3>(pb, swb, om4, a, y, colbase); break;
                default: rho_partner<TM, 4>(pb, swb, om4, a, y, colbase); break;
            }
        }
        if (nkc > 1 && bits) gather_a<TM>(sm, ncov, ri, __ffsll(bits) - 1, 0, Ds, lane, nxt);
    }
    // rho(slot) += sum over rows of Phi_row(slot) * Y(row, slot)
#pragma unroll
    for (int o = 0; o < 4; ++o) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int p = 8 * (4 * h + o) + 2 * (lane & 3) + e;
            double v = 0.0;
#pragma unroll
            for (int t = 0; t < TM; ++t) {
                const int r = ra0 + 8 * t + (lane >> 2);
                v += sm.phi[phi_idx(r, p)] * y[t][o][e];
            }
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            if (lane < 4) racc[p] += v;
        }
    }
}

__device__ __forceinline__ void rho_task(const Smem& sm, int ncov, const Task& t, const double* Ds, double* racc,
                                         int lane) {
    const GroupS& G = sm.grp[t.g];
    for (int i0 = 0; i0 < G.tm; i0 += 2) {
        if (G.tm - i0 >= 2)
            rho_task_rows<2>(sm, ncov, t.g, G.row0 + 8 * i0, t.half, Ds, racc, lane);
        else
            rho_task_rows<1>(sm, ncov, t.g, G.row0 + 8 * i0, t.half, Ds, racc, lane);
    }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 2) k_density(GridArgs g) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Smem sm = carve(smem_raw, g, NW * 64);
    const int64_t b = g.blk_begin + blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int bi, bj, bk;
    block_decode(g.sys, b, bi, bj, bk);
    const Block blk = stage_block(g, b, sm);
    if (blk.ncov == 0) {
        if (tid < 64) {
            bool valid;
            const int64_t pt = slot_point(g.sys, bi, bj, bk, tid, valid);
            if (valid)
                for (int spin = 0; spin < g.nspin; ++spin) g.out[spin * g.npts + pt] = 0.0;
        }
        return;
    }
    double* racc = sm.acc + warp * 64;
    for (int spin = 0; spin < g.nspin; ++spin) {
        for (int i = lane; i < 64; i += 32) racc[i] = 0.0;
        __syncwarp();
        const double* Ds = g.in + spin * g.nnz;
        for (int w = warp; w < kTaskWarps; w += NW)
            for (int e = sm.wptr[w]; e < sm.wptr[w + 1]; ++e) rho_task(sm, blk.ncov, sm.task[e], Ds, racc, lane);
        __syncthreads();
        if (tid < 64) {
            double r = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) r += sm.acc[w * 64 + tid];
            bool valid;
            const int64_t pt = slot_point(g.sys, bi, bj, bk, tid, valid);
            if (valid) g.out[spin * g.npts + pt] = r;
        }
        __syncthreads();
    }
}

// ---- mirror: H_ba(-R) = H_ab(R)^T ------------------------------------------------
__global__ void k_mirror(SysParams P, int64_t npair, int nspin, int64_t nnz, const int32_t* __restrict__ pa,
                         const int32_t* __restrict__ pb, const int32_t* __restrict__ pR,
                         const int64_t* __restrict__ poff, const int32_t* __restrict__ mirror, double* h) {
    const int lane = threadIdx.x & 31;
    const int64_t p = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (p >= npair) return;
    const int a = pa[p], b = pb[p];
    const int R0 = pR[3 * p], R1 = pR[3 * p + 1], R2 = pR[3 * p + 2];
    const bool canon = (a != b) ? a < b : (R0 != 0 ? R0 > 0 : (R1 != 0 ? R1 > 0 : R2 >= 0));
    const int na = P.sp[P.spc[a]].norb, nb = P.sp[P.spc[b]].norb;
    const int64_t q = mirror[p];
    if (q == p) {
        // (a, a, 0): re-symmetrise (H + H^T)/2, like kband triple_product (linalg.cpp:120-128)
        for (int s = 0; s < nspin; ++s) {
            double* x = h + s * nnz + poff[p];
            for (int e = lane; e < na * na; e += 32) {
                const int i = e / na, j = e % na;
                if (i < j) {
                    const double v = 0.5 * (x[i * na + j] + x[j * na + i]);
                    x[i * na + j] = v;
                    x[j * na + i] = v;
                }
            }
        }
        return;
    }
    if (canon) return;
    for (int s = 0; s < nspin; ++s) {
        const double* src = h + s * nnz + poff[q];  // nb x na
        double* dst = h + s * nnz + poff[p];        // na x nb
        for (int e = lane; e < na * nb; e += 32) {
            const int i = e / nb, j = e % nb;
            dst[e] = src[j * na + i];
        }
    }
}

// ---- DM symmetry validation (host API only) ---------------------------------------
__global__ void k_dm_check(SysParams P, int64_t npair, int nspin, int64_t nnz, const int32_t* __restrict__ pa,
                           const int32_t* __restrict__ pb, const int64_t* __restrict__ poff,
                           const int32_t* __restrict__ mirror, const double* __restrict__ dm,
                           unsigned long long* out) {
    const int lane = threadIdx.x & 31;
    const int64_t p = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (p >= npair) return;
    const int na = P.sp[P.spc[pa[p]]].norb, nb = P.sp[P.spc[pb[p]]].norb;
    const int64_t q = mirror[p];
    double dmax = 0.0, amax = 0.0;
    bool finite = true;
    for (int s = 0; s < nspin; ++s) {
        const double* x = dm + s * nnz + poff[p];
        const double* y = dm + s * nnz + poff[q];
        for (int e = lane; e < na * nb; e += 32) {
            const int i = e / nb, j = e % nb;
            const double v = x[e];
            finite &= isfinite(v);
            dmax = fmax(dmax, fabs(v - y[j * na + i]));
            amax = fmax(amax, fabs(v));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    finite = __all_sync(0xffffffffu, finite);
    if (lane == 0) {
        atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(dmax)));
        atomicMax(out + 1, static_cast<unsigned long long>(__double_as_longlong(amax)));
        if (!finite) atomicMax(out + 2, 1ull);
    }
}

__global__ void k_block_orbitals(GridArgs g, int64_t b, double* out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Smem sm = carve(smem_raw, g, 64);
    const Block blk = stage_block(g, b, sm);
    // rows in cover order, without group padding
    int r0 = 0;
    for (int c = 0; c < blk.ncov; ++c) {
        const CoverS& cv = sm.cov[c];
        for (int i = threadIdx.x; i < cv.norb * 64; i += blockDim.x)
            out[static_cast<size_t>(r0) * 64 + i] = sm.phi[phi_idx(cv.row0 + (i >> 6), i & 63)];
        r0 += cv.norb;
    }
}

template <class K>
void set_smem(K kernel, size_t bytes) {
    KBG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
}

}  // namespace

size_t grid_smem_bytes(const GridArgs& g, int nwarps, bool density) {
    size_t off[11];
    return smem_layout(g, density ? nwarps * 64 : 64, off);
}

int launch_density(const GridArgs& g, int64_t nblk, int nwarps, cudaStream_t st) {
    if (nblk <= 0) return 0;
    const size_t smem = grid_smem_bytes(g, nwarps, true);
    if (nwarps == 4) {
        set_smem(k_density<4>, smem);
        k_density<4><<<static_cast<unsigned>(nblk), 128, smem, st>>>(g);
    } else {
        set_smem(k_density<8>, smem);
        k_density<8><<<static_cast<unsigned>(nblk), 256, smem, st>>>(g);
    }
    KBG_CUDA(cudaGetLastError());
    return 1;
}

int launch_hamiltonian(const GridArgs& g, int64_t nblk, int nwarps, cudaStream_t st) {
    if (nblk <= 0) return 0;
    const size_t smem = grid_smem_bytes(g, nwarps, false);
    if (nwarps == 4) {
        set_smem(k_hamiltonian<4>, smem);
        k_hamiltonian<4><<<static_cast<unsigned>(nblk), 128, smem, st>>>(g);
    } else {
        set_smem(k_hamiltonian<8>, smem);
        k_hamiltonian<8><<<static_cast<unsigned>(nblk), 256, smem, st>>>(g);
    }
    KBG_CUDA(cudaGetLastError());
    return 1;
}

int launch_mirror(const DevIndex& ix, const SysParams& sys, int nspin, double* h, cudaStream_t st) {
    if (ix.npair == 0) return 0;
    const unsigned grid = static_cast<unsigned>((ix.npair * 32 + 255) / 256);
    k_mirror<<<grid, 256, 0, st>>>(sys, ix.npair, nspin, ix.nnz, ix.pair_a, ix.pair_b, ix.pair_R, ix.pair_off,
                                   ix.pair_mirror, h);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

int launch_dm_check(const DevIndex& ix, const SysParams& sys, int nspin, const double* dm,
                    unsigned long long* d_out, cudaStream_t st) {
    if (ix.npair == 0) return 0;
    const unsigned grid = static_cast<unsigned>((ix.npair * 32 + 255) / 256);
    k_dm_check<<<grid, 256, 0, st>>>(sys, ix.npair, nspin, ix.nnz, ix.pair_a, ix.pair_b, ix.pair_off, ix.pair_mirror,
                                     dm, d_out);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

int launch_block_orbitals(const GridArgs& g, int64_t block, double* d_out, cudaStream_t st) {
    const size_t smem = grid_smem_bytes(g, 1, false);
    set_smem(k_block_orbitals, smem);
    k_block_orbitals<<<1, 256, smem, st>>>(g, block, d_out);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

}  // namespace kbg
