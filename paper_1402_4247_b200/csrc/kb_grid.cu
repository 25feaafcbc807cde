// G2+G3 / G2+G4: fused orbital evaluation + density / Hamiltonian contraction.
//
// One CTA per 4x4x4 grid block (64 slots). The block's orbitals Phi (FP64,
// one norb x 4 tile per cover and active quad) are evaluated once into shared
// memory; every
// canonical cover pair (ci <= cj) sharing points is then one warp task:
//   H : C(na x nb) += Phi_ci^T diag(V dV) Phi_cj  over active 1x2x2 quads
//       -> mma.sync.m8n8k4.f64 (SASS DMMA), M = orbitals of ci, N = orbitals
//       of cj, K = 4 slots of a quad; FP64 atomics into the canonical pair
//       block, mirrored afterwards.
//   rho: X(8 slots x nb) = Phi_ci^T(8 x na) DM(na x nb) per active 2x2x2 octet
//       -> DMMA with M = 8 slots, K = 4 orbitals of ci, N = 8 orbitals of cj;
//       rho(slot) += f * sum_j X Phi_cj (f = 2 off-diagonal, DM symmetric),
//       per-warp shared accumulators summed in fixed order (deterministic).
#include "kb_device.cuh"

namespace kbg {

namespace {

struct CoverS {
    double t[3];
    uint64_t mask;
    uint32_t qmask;  // active 1x2x2 quads
    int tbase;       // offset (doubles) of this cover's first quad tile
    int norb;
    int sp;
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t quad_mask(uint64_t m) {
    uint32_t q = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) q |= static_cast<uint32_t>(((m >> (4 * i)) & 0xFull) != 0) << i;
    return q;
}

__device__ __forceinline__ uint32_t octet_of_quads(uint32_t qm) {
    uint32_t o = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) o |= static_cast<uint32_t>(((qm >> (2 * i)) & 3u) != 0) << i;
    return o;
}

// Offset of the norb x 4 tile of quad q of cover cv (q must be active).
__device__ __forceinline__ int tile_of(const CoverS& cv, int q) {
    return cv.tbase + __popc(cv.qmask & ((1u << q) - 1u)) * cv.norb * 4;
}
// As tile_of, or the zero tile (offset 0) when q is inactive.
__device__ __forceinline__ int tile_or_zero(const CoverS& cv, int q) {
    return ((cv.qmask >> q) & 1u) ? tile_of(cv, q) : 0;
}

struct Smem {
    double* phi;  // [kZero zeros][tiles...][kTilePad zeros]
    double* acc;  // w[64] (H) or racc[NW][64] (rho)
    BPair* bp;    // this block's work items
    CoverS* cov;
};

__device__ __forceinline__ Smem carve(unsigned char* base, int max_phi, int acc_doubles, int max_bpairs) {
    Smem s;
    s.phi = reinterpret_cast<double*>(base);
    s.acc = s.phi + max_phi;
    s.bp = reinterpret_cast<BPair*>(s.acc + acc_doubles);
    s.cov = reinterpret_cast<CoverS*>(s.bp + max_bpairs);
    return s;
}

// Loads the covers and work items of block b into shared memory and evaluates
// Phi on the active quads. Returns the number of covers (uniform per CTA).
__device__ int stage_block(const GridArgs& g, int64_t b, const Smem& sm, int& nbp) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int c0 = g.blk_ptr[b], c1 = g.blk_ptr[b + 1];
    const int ncov = c1 - c0;
    const int64_t p0 = g.bp_ptr[b];
    nbp = static_cast<int>(g.bp_ptr[b + 1] - p0);
    if (ncov == 0) return 0;
    const SysParams& P = g.sys;
    if (tid < ncov) {
        CoverS& cv = sm.cov[tid];
        const int a = g.cov_atom[c0 + tid];
        cv.sp = P.spc[a];
        cv.norb = P.sp[cv.sp].norb;
        cv.mask = g.cov_mask[c0 + tid];
        cv.qmask = quad_mask(cv.mask);
        const int R0 = g.cov_R[3 * (c0 + tid)], R1 = g.cov_R[3 * (c0 + tid) + 1], R2 = g.cov_R[3 * (c0 + tid) + 2];
#pragma unroll
        for (int c = 0; c < 3; ++c) cv.t[c] = P.tau[3 * a + c] + ((R0 * P.A[c] + R1 * P.A[3 + c]) + R2 * P.A[6 + c]);
    }
    for (int i = tid; i < nbp; i += nt) sm.bp[i] = g.bp[p0 + i];
    for (int i = tid; i < kZero; i += nt) sm.phi[i] = 0.0;
    __syncthreads();
    if (tid < ncov) {
        int base = kZero;
        for (int c = 0; c < tid; ++c) base += __popc(sm.cov[c].qmask) * sm.cov[c].norb * 4;
        sm.cov[tid].tbase = base;
    }
    __syncthreads();
    const CoverS& last = sm.cov[ncov - 1];
    const int end = last.tbase + __popc(last.qmask) * last.norb * 4;
    for (int i = tid; i < kTilePad; i += nt) sm.phi[end + i] = 0.0;
    int bi, bj, bk;
    block_decode(P, b, bi, bj, bk);
    for (int task = tid; task < ncov * 64; task += nt) {
        const int c = task >> 6, s = task & 63;
        const CoverS& cv = sm.cov[c];
        if (!((cv.qmask >> (s >> 2)) & 1u)) continue;  // no tile for an inactive quad
        double* dst = sm.phi + tile_of(cv, s >> 2) + (s & 3);
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
            eval_orbitals(P.sp[cv.sp], P.tables, dx, dy, dz, d2, [&](int o, double v) { dst[4 * o] = v; });
        } else {
            for (int o = 0; o < cv.norb; ++o) dst[4 * o] = 0.0;
        }
    }
    __syncthreads();
    return ncov;
}

__device__ __forceinline__ int64_t slot_point(const SysParams& P, int bi, int bj, int bk, int s, bool& valid) {
    int li, lj, lk;
    slot_decode(s, li, lj, lk);
    const int i = bi * 4 + li, j = bj * 4 + lj, k = bk * 4 + lk;
    valid = i < P.N[0] && j < P.N[1] && k < P.N[2];
    return (static_cast<int64_t>(i) * P.N[1] + j) * P.N[2] + k;
}

// ---- H pair task ---------------------------------------------------------------
// C(na x nb) = sum over common quads q of A(na x 4) B(4 x nb), A = Phi_ci w,
// B = Phi_cj^T. The DMMA A/B fragments of a quad are 32 consecutive doubles of
// the quad tile (lane = 4*row + point). Pairs with <= 2 output tiles alternate
// two accumulator sets so that two independent DMMA chains are in flight.
template <int TM, int TN>
__device__ __forceinline__ void h_pair(const double* __restrict__ phi, const double* __restrict__ w, const CoverS& A,
                                       const CoverS& B, uint32_t qm, double* __restrict__ H, double sign, int scatter,
                                       int lane) {
    constexpr int NACC = (TM * TN <= 2) ? 2 : 1;
    double c[NACC][TM][TN][2];
#pragma unroll
    for (int u = 0; u < NACC; ++u)
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) c[u][i][j][0] = c[u][i][j][1] = 0.0;
    const double* pw = w + (lane & 3);
    auto step = [&](int u, int q) {
        const double wv = pw[4 * q];
        const double* ta = phi + tile_of(A, q) + lane;
        const double* tb = phi + tile_of(B, q) + lane;
        double a[TM], b[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = ta[32 * i] * wv;
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = tb[32 * j];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) dmma(c[u][i][j], a[i], b[j]);
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
    const int na = A.norb, nb = B.norb;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = i * 8 + (lane >> 2), col = j * 8 + (lane & 3) * 2 + e;
                double v = c[0][i][j][e];
                if (NACC == 2) v += c[NACC - 1][i][j][e];
                if (r < na && col < nb) {
                    if (scatter == 0)
                        atomicAdd(H + r * nb + col, sign * v);
                    else
                        H[r * nb + col] = sign * v;
                }
            }
}

template <int TM>
__device__ __forceinline__ void h_pair_tn(int tn, const double* phi, const double* w, const CoverS& A,
                                          const CoverS& B, uint32_t qm, double* H, double sign, int scatter,
                                          int lane) {
    switch (tn) {
        case 1: h_pair<TM, 1>(phi, w, A, B, qm, H, sign, scatter, lane); break;
        case 2: h_pair<TM, 2>(phi, w, A, B, qm, H, sign, scatter, lane); break;
        case 3: h_pair<TM, 3>(phi, w, A, B, qm, H, sign, scatter, lane); break;
        default: h_pair<TM, 4>(phi, w, A, B, qm, H, sign, scatter, lane); break;
    }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 2) k_hamiltonian(GridArgs g) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Smem sm = carve(smem_raw, g.max_phi, 64, g.max_bpairs);
    const int64_t b = g.blk_begin + blockIdx.x;
    int nbp;
    const int ncov = stage_block(g, b, sm, nbp);
    if (ncov == 0) return;
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
        for (int e = warp; e < nbp; e += NW) {
            const BPair bp = sm.bp[e];
            const CoverS& A = sm.cov[bp.cicj & 0xffff];
            const CoverS& B = sm.cov[bp.cicj >> 16];
            const uint32_t qm = quad_mask(A.mask & B.mask);
            const int tm = (A.norb + 7) >> 3, tn = (B.norb + 7) >> 3;
            double* H = Hs + bp.off;
            switch (tm) {
                case 1: h_pair_tn<1>(tn, sm.phi, sm.acc, A, B, qm, H, g.sign, g.scatter, lane); break;
                case 2: h_pair_tn<2>(tn, sm.phi, sm.acc, A, B, qm, H, g.sign, g.scatter, lane); break;
                case 3: h_pair_tn<3>(tn, sm.phi, sm.acc, A, B, qm, H, g.sign, g.scatter, lane); break;
                default: h_pair_tn<4>(tn, sm.phi, sm.acc, A, B, qm, H, g.sign, g.scatter, lane); break;
            }
        }
        __syncthreads();
    }
}

// ---- rho pair task -------------------------------------------------------------
// Per active octet o (quads 2o, 2o+1): X(8 slots x nb) = Phi_ci^T DM, the A
// fragment of lane l is Phi_ci[4s + (l&3)][slot] read from the tile of quad
// 2o + (l>>4) (zero tile when inactive). Fast path (na, nb <= 16): DM
// fragments in registers, prefetched one pair ahead; two octets per
// iteration for DMMA ILP.
constexpr int kFrag = 8;  // B fragments per lane for na, nb <= 16: (4 K-steps) x (2 N-tiles)

__device__ __forceinline__ void load_dfrag(const double* __restrict__ D, int na, int nb, int lane,
                                           double (&out)[kFrag]) {
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int k = 4 * s + (lane & 3), n = 8 * t + (lane >> 2);
            out[s * 2 + t] = (k < na && n < nb) ? __ldg(D + k * nb + n) : 0.0;
        }
}

template <int KS, int TN, int NO>
__device__ __forceinline__ void rho_octets(const double* __restrict__ phi, const CoverS& A, const CoverS& B,
                                           const int (&oct)[2], const double (&bf)[kFrag], double f,
                                           double* __restrict__ racc, int lane) {
    const int half = lane >> 4, pt = (lane >> 2) & 3;
    const double* ta[NO];
    const double* tb[NO];
#pragma unroll
    for (int o = 0; o < NO; ++o) {
        const int q = 2 * oct[o] + half;
        ta[o] = phi + tile_or_zero(A, q) + 4 * (lane & 3) + pt;
        tb[o] = phi + tile_or_zero(B, q) + 8 * (lane & 3) + pt;
    }
    double x[NO][TN][2];
#pragma unroll
    for (int o = 0; o < NO; ++o)
#pragma unroll
        for (int t = 0; t < TN; ++t) x[o][t][0] = x[o][t][1] = 0.0;
#pragma unroll
    for (int s = 0; s < KS; ++s) {
        double a[NO];
#pragma unroll
        for (int o = 0; o < NO; ++o) a[o] = ta[o][16 * s];
#pragma unroll
        for (int o = 0; o < NO; ++o)
#pragma unroll
            for (int t = 0; t < TN; ++t) dmma(x[o][t], a[o], bf[s * 2 + t]);
    }
#pragma unroll
    for (int o = 0; o < NO; ++o) {
        double part = 0.0;
#pragma unroll
        for (int t = 0; t < TN; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e) part += x[o][t][e] * tb[o][32 * t + 4 * e];
        part += __shfl_xor_sync(0xffffffffu, part, 1);
        part += __shfl_xor_sync(0xffffffffu, part, 2);
        if ((lane & 3) == 0) racc[8 * oct[o] + (lane >> 2)] += f * part;
    }
}

template <int KS, int TN>
__device__ __forceinline__ void rho_pair(const double* __restrict__ phi, const CoverS& A, const CoverS& B,
                                         uint32_t om, const double (&bf)[kFrag], double f, double* __restrict__ racc,
                                         int lane) {
    while (om) {
        int oct[2];
        oct[0] = __ffs(om) - 1;
        om &= om - 1;
        if (om) {
            oct[1] = __ffs(om) - 1;
            om &= om - 1;
            rho_octets<KS, TN, 2>(phi, A, B, oct, bf, f, racc, lane);
        } else {
            oct[1] = oct[0];
            rho_octets<KS, TN, 1>(phi, A, B, oct, bf, f, racc, lane);
        }
    }
}

// General path for atoms with more than 16 orbitals (not used by Fe3O4).
__device__ __noinline__ void rho_pair_big(const double* __restrict__ phi, const CoverS& A, const CoverS& B, uint32_t om,
                             const double* __restrict__ D, double f, double* __restrict__ racc, int lane) {
    const int na = A.norb, nb = B.norb;
    const int ks = (na + 3) >> 2, tn = (nb + 7) >> 3;
    const int half = lane >> 4, pt = (lane >> 2) & 3;
    while (om) {
        const int o = __ffs(om) - 1;
        om &= om - 1;
        const int q = 2 * o + half;
        const double* ta = phi + tile_or_zero(A, q) + 4 * (lane & 3) + pt;
        const double* tb = phi + tile_or_zero(B, q) + 8 * (lane & 3) + pt;
        double part = 0.0;
        for (int t = 0; t < tn; ++t) {
            double x[2] = {0.0, 0.0};
            for (int s = 0; s < ks; ++s) {
                const int k = 4 * s + (lane & 3), n = 8 * t + (lane >> 2);
                const double bv = (k < na && n < nb) ? __ldg(D + k * nb + n) : 0.0;
                dmma(x, ta[16 * s], bv);
            }
            part += x[0] * tb[32 * t] + x[1] * tb[32 * t + 4];
        }
        part += __shfl_xor_sync(0xffffffffu, part, 1);
        part += __shfl_xor_sync(0xffffffffu, part, 2);
        if ((lane & 3) == 0) racc[8 * o + (lane >> 2)] += f * part;
    }
}

template <int KS>
__device__ __forceinline__ void rho_pair_tn(int tn, const double* phi, const CoverS& A, const CoverS& B, uint32_t om,
                                            const double (&bf)[kFrag], double f, double* racc, int lane) {
    if (tn == 1)
        rho_pair<KS, 1>(phi, A, B, om, bf, f, racc, lane);
    else
        rho_pair<KS, 2>(phi, A, B, om, bf, f, racc, lane);
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 2) k_density(GridArgs g) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Smem sm = carve(smem_raw, g.max_phi, NW * 64, g.max_bpairs);
    const int64_t b = g.blk_begin + blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int bi, bj, bk;
    block_decode(g.sys, b, bi, bj, bk);
    int nbp;
    const int ncov = stage_block(g, b, sm, nbp);
    if (ncov == 0) {
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
        double nxt[kFrag];
        auto prefetch = [&](int e) {
            const BPair bp = sm.bp[e];
            const int na = sm.cov[bp.cicj & 0xffff].norb, nb = sm.cov[bp.cicj >> 16].norb;
            if (na <= 16 && nb <= 16) load_dfrag(Ds + bp.off, na, nb, lane, nxt);
        };
        if (warp < nbp) prefetch(warp);
        for (int e = warp; e < nbp; e += NW) {
            double cur[kFrag];
#pragma unroll
            for (int i = 0; i < kFrag; ++i) cur[i] = nxt[i];
            if (e + NW < nbp) prefetch(e + NW);
            const BPair bp = sm.bp[e];
            const int ci = bp.cicj & 0xffff, cj = bp.cicj >> 16;
            const CoverS& A = sm.cov[ci];
            const CoverS& B = sm.cov[cj];
            const uint32_t om = octet_of_quads(quad_mask(A.mask & B.mask));
            const double f = ci == cj ? 1.0 : 2.0;
            if (A.norb > 16 || B.norb > 16) {
                rho_pair_big(sm.phi, A, B, om, Ds + bp.off, f, racc, lane);
                continue;
            }
            const int ks = (A.norb + 3) >> 2, tn = (B.norb + 7) >> 3;
            switch (ks) {
                case 1: rho_pair_tn<1>(tn, sm.phi, A, B, om, cur, f, racc, lane); break;
                case 2: rho_pair_tn<2>(tn, sm.phi, A, B, om, cur, f, racc, lane); break;
                case 3: rho_pair_tn<3>(tn, sm.phi, A, B, om, cur, f, racc, lane); break;
                default: rho_pair_tn<4>(tn, sm.phi, A, B, om, cur, f, racc, lane); break;
            }
        }
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
    const Smem sm = carve(smem_raw, g.max_phi, 64, g.max_bpairs);
    int nbp;
    const int ncov = stage_block(g, b, sm, nbp);
    if (ncov == 0) return;
    // unpack the quad tiles to [orbital][slot] rows in cover order
    int r0 = 0;
    for (int c = 0; c < ncov; ++c) {
        const CoverS& cv = sm.cov[c];
        for (int i = threadIdx.x; i < cv.norb * 64; i += blockDim.x) {
            const int o = i >> 6, s = i & 63;
            out[static_cast<size_t>(r0) * 64 + i] = sm.phi[tile_or_zero(cv, s >> 2) + 4 * o + (s & 3)];
        }
        r0 += cv.norb;
    }
}

template <class K>
void set_smem(K kernel, size_t bytes) {
    KBG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
}

}  // namespace

size_t grid_smem_bytes(int max_phi, int max_cover, int max_bpairs, int nwarps, bool density) {
    return static_cast<size_t>(max_phi) * sizeof(double) +
           static_cast<size_t>(density ? nwarps * 64 : 64) * sizeof(double) +
           static_cast<size_t>(max_bpairs) * sizeof(BPair) + static_cast<size_t>(max_cover) * sizeof(CoverS);
}

int launch_density(const GridArgs& g, int64_t nblk, int nwarps, cudaStream_t st) {
    if (nblk <= 0) return 0;
    const size_t smem = grid_smem_bytes(g.max_phi, g.max_cover, g.max_bpairs, nwarps, true);
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
    const size_t smem = grid_smem_bytes(g.max_phi, g.max_cover, g.max_bpairs, nwarps, false);
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
    const size_t smem = grid_smem_bytes(g.max_phi, g.max_cover, g.max_bpairs, 1, false);
    set_smem(k_block_orbitals, smem);
    k_block_orbitals<<<1, 256, smem, st>>>(g, block, d_out);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

}  // namespace kbg
