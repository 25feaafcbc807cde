// G1: device index build (bit-exact with the oracle's lists).
//
// Candidate (atom, image) boxes are supersets; membership is decided only by
// the exact-rounding expression of include/kbgrid.h, so the resulting lists do
// not depend on how the boxes were computed.
#include <cub/cub.cuh>

#include "kb_device.cuh"

namespace kbg {

namespace {

template <class T>
T* dalloc(size_t n) {
    T* p = nullptr;
    if (n == 0) n = 1;
    KBG_CUDA(pool_malloc(&p, n * sizeof(T)));
    return p;
}

template <class T>
void dfree(T*& p) {
    if (p) pool_free(p);
    p = nullptr;
}

// Exclusive scan of n values into out[0..n] (out[n] = total).
template <class T>
T exclusive_scan(T* d_in_np1, T* d_out_np1, int64_t n, cudaStream_t st) {
    // d_in_np1[n] must be 0 so that out[n] is the total.
    size_t bytes = 0;
    KBG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, d_in_np1, d_out_np1, static_cast<int>(n + 1), st));
    void* tmp = dalloc<char>(bytes);
    KBG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, d_in_np1, d_out_np1, static_cast<int>(n + 1), st));
    T total;
    KBG_CUDA(cudaMemcpyAsync(&total, d_out_np1 + n, sizeof(T), cudaMemcpyDeviceToHost, st));
    KBG_CUDA(cudaStreamSynchronize(st));
    pool_free(tmp);
    return total;
}

__device__ __forceinline__ void frac_dev(const SysParams& P, const double* r, double f[3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) f[c] = r[0] * P.Ainv[c] + r[1] * P.Ainv[3 + c] + r[2] * P.Ainv[6 + c];
}

__device__ __forceinline__ void extent_dev(const SysParams& P, double rho, double e[3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
        e[c] = rho * sqrt(P.Ainv[c] * P.Ainv[c] + P.Ainv[3 + c] * P.Ainv[3 + c] + P.Ainv[6 + c] * P.Ainv[6 + c]) *
                   (1.0 + 1e-9) + 1e-12;
}

// ---- candidates -------------------------------------------------------------
__global__ void k_candidates(SysParams P, int64_t* count, const int64_t* off, Candidate* out) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= P.natom) return;
    const DevSpecies& sp = P.sp[P.spc[a]];
    double f[3], e[3];
    frac_dev(P, P.tau + 3 * a, f);
    extent_dev(P, sp.rc, e);
    int Rlo[3], Rhi[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        Rlo[c] = static_cast<int>(floor(-f[c] - e[c])) - 1;
        Rhi[c] = static_cast<int>(ceil(1.0 - f[c] + e[c])) + 1;
    }
    int64_t n = 0;
    for (int R0 = Rlo[0]; R0 <= Rhi[0]; ++R0)
        for (int R1 = Rlo[1]; R1 <= Rhi[1]; ++R1)
            for (int R2 = Rlo[2]; R2 <= Rhi[2]; ++R2) {
                const int R[3] = {R0, R1, R2};
                int lo[3], hi[3];
                bool empty = false;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    lo[c] = max(0, static_cast<int>(floor((f[c] + R[c] - e[c]) * P.N[c])) - 1);
                    hi[c] = min(P.N[c] - 1, static_cast<int>(ceil((f[c] + R[c] + e[c]) * P.N[c])) + 1);
                    empty |= lo[c] > hi[c];
                }
                if (empty) continue;
                if (out) {
                    Candidate& cd = out[off[a] + n];
                    cd.atom = a;
                    for (int c = 0; c < 3; ++c) {
                        cd.R[c] = R[c];
                        cd.lo[c] = lo[c];
                        cd.hi[c] = hi[c];
                    }
                }
                ++n;
            }
    if (count) count[a] = n;
}

__global__ void k_cand_tasks(const Candidate* cand, int64_t ncand, int64_t* ntask) {
    const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (c >= ncand) return;
    int64_t n = 1;
    for (int d = 0; d < 3; ++d) n *= (cand[c].hi[d] >> 2) - (cand[c].lo[d] >> 2) + 1;
    ntask[c] = n;
}

// One CTA per candidate; one warp per (candidate, block) task; lanes test
// slots lane and lane+32 with the exact expression and ballot the mask.
__global__ void k_cover_masks(SysParams P, const Candidate* __restrict__ cand, const int64_t* __restrict__ task_off,
                              int64_t ncand, int64_t* __restrict__ tkey, uint64_t* __restrict__ tmask,
                              unsigned long long* ncover) {
    const int64_t c = blockIdx.x;
    const Candidate cd = cand[c];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const DevSpecies& sp = P.sp[P.spc[cd.atom]];
    double t[3];
    image_pos_exact(P, P.tau + 3 * cd.atom, cd.R[0], cd.R[1], cd.R[2], t);
    const int b0[3] = {cd.lo[0] >> 2, cd.lo[1] >> 2, cd.lo[2] >> 2};
    const int nb[3] = {(cd.hi[0] >> 2) - b0[0] + 1, (cd.hi[1] >> 2) - b0[1] + 1, (cd.hi[2] >> 2) - b0[2] + 1};
    const int64_t n = static_cast<int64_t>(nb[0]) * nb[1] * nb[2];
    unsigned cnt = 0;
    for (int64_t tk = warp; tk < n; tk += nw) {
        const int bk = b0[2] + static_cast<int>(tk % nb[2]);
        const int bj = b0[1] + static_cast<int>((tk / nb[2]) % nb[1]);
        const int bi = b0[0] + static_cast<int>(tk / (static_cast<int64_t>(nb[2]) * nb[1]));
        uint64_t mask = 0;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int s = lane + 32 * half;
            int li, lj, lk;
            slot_decode(s, li, lj, lk);
            const int i = bi * 4 + li, j = bj * 4 + lj, k = bk * 4 + lk;
            bool in = false;
            if (i < P.N[0] && j < P.N[1] && k < P.N[2]) {
                double r[3], d[3];
                point_pos_exact(P, i, j, k, r);
#pragma unroll
                for (int q = 0; q < 3; ++q) d[q] = __dsub_rn(r[q], t[q]);
                in = dist2_exact(d) < sp.rc2;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, in);
            mask |= static_cast<uint64_t>(bal) << (32 * half);
        }
        if (lane == 0) {
            const int64_t slot = task_off[c] + tk;
            const int64_t blk = block_id(P, bi, bj, bk);
            tkey[slot] = mask ? blk * ncand + c : INT64_MAX;
            tmask[slot] = mask;
            cnt += mask != 0;
        }
    }
    if (lane == 0 && cnt) atomicAdd(ncover, static_cast<unsigned long long>(cnt));
}

__global__ void k_cover_finish(const int64_t* __restrict__ key, const uint64_t* __restrict__ mask, int64_t ncover,
                               int64_t ncand, const Candidate* __restrict__ cand, int32_t* cov_atom, int32_t* cov_R,
                               uint64_t* cov_mask, int32_t* blk_count) {
    const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= ncover) return;
    const int64_t blk = key[e] / ncand, c = key[e] % ncand;
    cov_atom[e] = cand[c].atom;
    for (int q = 0; q < 3; ++q) cov_R[3 * e + q] = cand[c].R[q];
    cov_mask[e] = mask[e];
    atomicAdd(&blk_count[blk], 1);
}

// ---- pairs ----------------------------------------------------------------
__device__ __forceinline__ bool canonical_dev(int a, int b, int R0, int R1, int R2) {
    if (a != b) return a < b;
    if (R0 != 0) return R0 > 0;
    if (R1 != 0) return R1 > 0;
    return R2 >= 0;
}

__device__ __forceinline__ bool pair_test_dev(const SysParams& P, int a, int b, int R0, int R1, int R2) {
    if (!canonical_dev(a, b, R0, R1, R2)) {
        const int t = a;
        a = b;
        b = t;
        R0 = -R0;
        R1 = -R1;
        R2 = -R2;
    }
    double tb[3], d[3];
    image_pos_exact(P, P.tau + 3 * b, R0, R1, R2, tb);
#pragma unroll
    for (int c = 0; c < 3; ++c) d[c] = __dsub_rn(tb[c], P.tau[3 * a + c]);
    const double s = __dadd_rn(P.sp[P.spc[a]].rc, P.sp[P.spc[b]].rc);
    return dist2_exact(d) < __dmul_rn(s, s);
}

__global__ void k_pairs(SysParams P, int64_t* count, const int64_t* off, int32_t* pa, int32_t* pb, int32_t* pR) {
    const int64_t ab = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (ab >= static_cast<int64_t>(P.natom) * P.natom) return;
    const int a = static_cast<int>(ab / P.natom), b = static_cast<int>(ab % P.natom);
    double fa[3], fb[3], e[3];
    frac_dev(P, P.tau + 3 * a, fa);
    frac_dev(P, P.tau + 3 * b, fb);
    extent_dev(P, P.sp[P.spc[a]].rc + P.sp[P.spc[b]].rc, e);
    int Rlo[3], Rhi[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double df = fb[c] - fa[c];
        Rlo[c] = static_cast<int>(floor(-df - e[c])) - 1;
        Rhi[c] = static_cast<int>(ceil(-df + e[c])) + 1;
    }
    int64_t n = 0;
    for (int R0 = Rlo[0]; R0 <= Rhi[0]; ++R0)
        for (int R1 = Rlo[1]; R1 <= Rhi[1]; ++R1)
            for (int R2 = Rlo[2]; R2 <= Rhi[2]; ++R2) {
                if (!pair_test_dev(P, a, b, R0, R1, R2)) continue;
                if (pa) {
                    const int64_t p = off[ab] + n;
                    pa[p] = a;
                    pb[p] = b;
                    pR[3 * p] = R0;
                    pR[3 * p + 1] = R1;
                    pR[3 * p + 2] = R2;
                }
                ++n;
            }
    if (count) count[ab] = n;
}

__global__ void k_pair_meta(SysParams P, int64_t npair, const int32_t* pa, const int32_t* pb, const int32_t* pR,
                            int64_t* size, int64_t* key) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p >= npair) return;
    size[p] = static_cast<int64_t>(P.sp[P.spc[pa[p]]].norb) * P.sp[P.spc[pb[p]]].norb;
    key[p] = pair_key(pa[p], pb[p], pR[3 * p], pR[3 * p + 1], pR[3 * p + 2], P.natom);
}

__global__ void k_pair_rsize(SysParams P, int64_t npair, const int32_t* pa, const int32_t* pb, const int32_t* pR,
                             int64_t* size) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p >= npair) return;
    const int a = pa[p], b = pb[p];
    if (!canonical_dev(a, b, pR[3 * p], pR[3 * p + 1], pR[3 * p + 2])) return;
    const int nb = P.sp[P.spc[b]].norb;
    size[p] = static_cast<int64_t>(P.sp[P.spc[a]].norb) * 16 * ((nb + 15) >> 4);
}

__global__ void k_pair_mirror(SysParams P, int64_t npair, const int32_t* pa, const int32_t* pb, const int32_t* pR,
                              const int64_t* key, int32_t* mirror, int* err) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p >= npair) return;
    const int64_t q = find_pair(key, npair, pair_key(pb[p], pa[p], -pR[3 * p], -pR[3 * p + 1], -pR[3 * p + 2], P.natom));
    mirror[p] = static_cast<int32_t>(q);
    if (q < 0) atomicCAS(err, 0, 1);
}

// Mirror work list: non-canonical pairs (dst) with their canonical mirror (src), and the (a, a, 0) pairs.
__global__ void k_mirror_items(SysParams P, int64_t npair, const int32_t* pa, const int32_t* pb, const int32_t* pR,
                               const int64_t* poff, const int32_t* mirror, MirrorItem* items, int* count) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p >= npair) return;
    const int64_t q = mirror[p];
    const int a = pa[p], b = pb[p];
    if (q != p && canonical_dev(a, b, pR[3 * p], pR[3 * p + 1], pR[3 * p + 2])) return;
    MirrorItem it;
    it.dst = poff[p];
    it.src = poff[q];
    it.na = P.sp[P.spc[a]].norb;
    it.nb = P.sp[P.spc[b]].norb;
    items[atomicAdd(count, 1)] = it;  // item order is free: every item writes its own block
}

// DM repack work list: one item per canonical pair (order free: every item writes its own block).
__global__ void k_repack_items(SysParams P, int64_t npair, const int32_t* pa, const int32_t* pb, const int32_t* pR,
                               const int64_t* poff, const int64_t* proff, const int32_t* mirror, RepackItem* items,
                               int* count) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p >= npair) return;
    const int a = pa[p], b = pb[p];
    const int R0 = pR[3 * p], R1 = pR[3 * p + 1], R2 = pR[3 * p + 2];
    if (!canonical_dev(a, b, R0, R1, R2)) return;
    RepackItem it;
    it.p = static_cast<int32_t>(p);
    it.src = poff[p];
    it.dst = proff[p];
    it.srq = poff[mirror[p]];
    it.na = P.sp[P.spc[a]].norb;
    it.nb = P.sp[P.spc[b]].norb;
    it.fac2 = !(a == b && R0 == 0 && R1 == 0 && R2 == 0);
    items[atomicAdd(count, 1)] = it;
}

// ---- block work items -------------------------------------------------------
struct Stats {
    unsigned long long sum_m, sum_m2, natompt;
    int max_phi, max_cover, max_bpairs;
};

__global__ void k_bp_count(SysParams P, int64_t nblock, const int32_t* __restrict__ blk_ptr,
                           const int32_t* __restrict__ cov_atom, const uint64_t* __restrict__ cov_mask,
                           int64_t* bp_count, int64_t* blk_cost, Stats* stats) {
    const int lane = threadIdx.x & 31;
    const int64_t b = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (b >= nblock) return;
    const int c0 = blk_ptr[b], c1 = blk_ptr[b + 1];
    long long cnt = 0, cost = 0;
    for (int ci = c0; ci < c1; ++ci) {
        const uint64_t mi = cov_mask[ci];
        const int na = P.sp[P.spc[cov_atom[ci]]].norb;
        for (int cj = ci + lane; cj < c1; cj += 32) {
            const uint64_t both = mi & cov_mask[cj];
            if (both) {
                ++cnt;
                // padded tile work, as the DMMA kernels execute it: rows and columns in 8-orbital tiles,
                // points in 1x2x2 quads (weights the shard split and the heaviest-first order)
                uint32_t nq = 0;
#pragma unroll
                for (int q = 0; q < 16; ++q) nq += ((both >> (4 * q)) & 0xFull) != 0;
                const int nb = P.sp[P.spc[cov_atom[cj]]].norb;
                cost += static_cast<long long>((na + 7) & ~7) * ((nb + 7) & ~7) * 4 * nq;
            }
        }
    }
    unsigned long long sm = 0, sm2 = 0, nap = 0;
    int rows = 0;
    for (int half = 0; half < 2; ++half) {
        const int s = lane + 32 * half;
        long long m = 0;
        for (int c = c0; c < c1; ++c)
            if ((cov_mask[c] >> s) & 1) m += P.sp[P.spc[cov_atom[c]]].norb;
        sm += m;
        sm2 += m * m;
    }
    for (int c = c0 + lane; c < c1; c += 32) {
        nap += __popcll(cov_mask[c]);
        uint32_t qm = 0;  // active 1x2x2 quads -> one norb x 4 tile each
        for (int q = 0; q < 16; ++q) qm |= static_cast<uint32_t>(((cov_mask[c] >> (4 * q)) & 0xFull) != 0) << q;
        rows += __popc(qm) * P.sp[P.spc[cov_atom[c]]].norb * 4;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        cost += __shfl_xor_sync(0xffffffffu, cost, o);
        sm += __shfl_xor_sync(0xffffffffu, sm, o);
        sm2 += __shfl_xor_sync(0xffffffffu, sm2, o);
        nap += __shfl_xor_sync(0xffffffffu, nap, o);
        rows += __shfl_xor_sync(0xffffffffu, rows, o);
    }
    if (lane == 0) {
        bp_count[b] = cnt;
        blk_cost[b] = cost;
        atomicAdd(&stats->sum_m, sm);
        atomicAdd(&stats->sum_m2, sm2);
        atomicAdd(&stats->natompt, nap);
        atomicMax(&stats->max_phi, rows);
        atomicMax(&stats->max_cover, c1 - c0);
        atomicMax(&stats->max_bpairs, static_cast<int>(cnt));
    }
}

__global__ void k_bp_fill(SysParams P, int64_t nblock, const int32_t* __restrict__ blk_ptr,
                          const int32_t* __restrict__ cov_atom, const int32_t* __restrict__ cov_R,
                          const uint64_t* __restrict__ cov_mask, const int64_t* __restrict__ bp_ptr,
                          const int64_t* __restrict__ pkey, const int64_t* __restrict__ poff,
                          const int64_t* __restrict__ proff, int64_t npair, BPair* bp,
                          int* err) {
    const int lane = threadIdx.x & 31;
    const int64_t b = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (b >= nblock) return;
    const int c0 = blk_ptr[b], c1 = blk_ptr[b + 1];
    int64_t pos = bp_ptr[b];
    for (int ci = c0; ci < c1; ++ci) {
        const uint64_t mi = cov_mask[ci];
        const int ai = cov_atom[ci];
        for (int cj0 = ci; cj0 < c1; cj0 += 32) {
            const int cj = cj0 + lane;
            uint64_t both = 0;
            if (cj < c1) both = mi & cov_mask[cj];
            const unsigned bal = __ballot_sync(0xffffffffu, both != 0);
            if (both) {
                const int aj = cov_atom[cj];
                const int64_t key = pair_key(ai, aj, cov_R[3 * cj] - cov_R[3 * ci], cov_R[3 * cj + 1] - cov_R[3 * ci + 1],
                                             cov_R[3 * cj + 2] - cov_R[3 * ci + 2], P.natom);
                const int64_t p = find_pair(pkey, npair, key);
                BPair e;
                e.cicj = (ci - c0) | ((cj - c0) << 16);
                e.roff = p >= 0 ? static_cast<int32_t>(proff[p]) : 0;
                e.off = p >= 0 ? poff[p] : 0;
                if (p < 0) atomicCAS(err, 0, static_cast<int>(b) + 1);
                bp[pos + __popc(bal & ((1u << lane) - 1u))] = e;
            }
            pos += __popc(bal);
        }
    }
}

}  // namespace

namespace {
__global__ void k_iota(int64_t b0, int64_t n, int64_t* out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = b0 + i;
}
}  // namespace

void block_order_device(DevIndex& ix, int64_t b0, int64_t b1, bool heaviest_first, cudaStream_t st) {
    const int64_t n = b1 - b0;
    ix.order = dalloc<int64_t>(std::max<int64_t>(1, n));
    ix.norder = n;
    if (n <= 0) return;
    int64_t* ids = heaviest_first ? dalloc<int64_t>(n) : ix.order;
    k_iota<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(b0, n, ids);
    KBG_CUDA(cudaGetLastError());
    if (!heaviest_first) return;
    int64_t* keys_out = dalloc<int64_t>(n);
    size_t bytes = 0;
    KBG_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, ix.blk_cost + b0, keys_out, ids, ix.order,
                                                       static_cast<int>(n), 0, 64, st));
    void* tmp = dalloc<char>(bytes);
    KBG_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, bytes, ix.blk_cost + b0, keys_out, ids, ix.order,
                                                       static_cast<int>(n), 0, 64, st));
    pool_free(tmp);
    pool_free(keys_out);
    pool_free(ids);
}

void free_index(DevIndex& ix) {
    free_cache(ix);
    free_tasks(ix);
    dfree(ix.blk_ptr);
    dfree(ix.cov_atom);
    dfree(ix.cov_R);
    dfree(ix.cov_mask);
    dfree(ix.pair_a);
    dfree(ix.pair_b);
    dfree(ix.pair_R);
    dfree(ix.pair_off);
    dfree(ix.pair_key);
    dfree(ix.pair_roff);
    dfree(ix.order);
    dfree(ix.pair_mirror);
    dfree(ix.mir);
    dfree(ix.rep);
    dfree(ix.mir_count);
    dfree(ix.bp_ptr);
    dfree(ix.bp);
    dfree(ix.blk_cost);
    ix = DevIndex();
}

void build_index_device(const SysParams& P, DevIndex& ix, cudaStream_t st) {
    free_index(ix);
    const int natom = P.natom;
    const int64_t nblock = static_cast<int64_t>(P.nblk[0]) * P.nblk[1] * P.nblk[2];
    ix.nblock = nblock;
    const int T = 256;
    auto grid_of = [](int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); };

    // 1. candidate images per atom
    int64_t* cnt = dalloc<int64_t>(natom + 1);
    int64_t* coff = dalloc<int64_t>(natom + 1);
    KBG_CUDA(cudaMemsetAsync(cnt, 0, (natom + 1) * sizeof(int64_t), st));
    k_candidates<<<grid_of(natom, 64), 64, 0, st>>>(P, cnt, nullptr, nullptr);
    KBG_CUDA(cudaGetLastError());
    const int64_t ncand = exclusive_scan(cnt, coff, natom, st);
    Candidate* cand = dalloc<Candidate>(ncand);
    k_candidates<<<grid_of(natom, 64), 64, 0, st>>>(P, nullptr, coff, cand);
    KBG_CUDA(cudaGetLastError());

    // 2. (candidate, block) tasks
    int64_t* tcnt = dalloc<int64_t>(ncand + 1);
    int64_t* toff = dalloc<int64_t>(ncand + 1);
    KBG_CUDA(cudaMemsetAsync(tcnt, 0, (ncand + 1) * sizeof(int64_t), st));
    k_cand_tasks<<<grid_of(ncand, T), T, 0, st>>>(cand, ncand, tcnt);
    const int64_t ntask = exclusive_scan(tcnt, toff, ncand, st);
    int64_t* tkey = dalloc<int64_t>(ntask);
    uint64_t* tmask = dalloc<uint64_t>(ntask);
    unsigned long long* d_ncover = dalloc<unsigned long long>(1);
    KBG_CUDA(cudaMemsetAsync(d_ncover, 0, sizeof(unsigned long long), st));
    k_cover_masks<<<static_cast<unsigned>(ncand), 256, 0, st>>>(P, cand, toff, ncand, tkey, tmask, d_ncover);
    KBG_CUDA(cudaGetLastError());

    // 3. sort by (block, candidate) -> cover lists
    int64_t* skey = dalloc<int64_t>(ntask);
    uint64_t* smask = dalloc<uint64_t>(ntask);
    {
        size_t bytes = 0;
        KBG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, tkey, skey, tmask, smask, static_cast<int>(ntask), 0,
                                                 64, st));
        void* tmp = dalloc<char>(bytes);
        KBG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, tkey, skey, tmask, smask, static_cast<int>(ntask), 0, 64,
                                                 st));
        KBG_CUDA(cudaStreamSynchronize(st));
        pool_free(tmp);
    }
    unsigned long long ncover_h = 0;
    KBG_CUDA(cudaMemcpy(&ncover_h, d_ncover, sizeof(ncover_h), cudaMemcpyDeviceToHost));
    ix.ncover = static_cast<int64_t>(ncover_h);
    ix.cov_atom = dalloc<int32_t>(ix.ncover);
    ix.cov_R = dalloc<int32_t>(3 * ix.ncover);
    ix.cov_mask = dalloc<uint64_t>(ix.ncover);
    int32_t* bcnt = dalloc<int32_t>(nblock + 1);
    ix.blk_ptr = dalloc<int32_t>(nblock + 1);
    KBG_CUDA(cudaMemsetAsync(bcnt, 0, (nblock + 1) * sizeof(int32_t), st));
    if (ix.ncover)
        k_cover_finish<<<grid_of(ix.ncover, T), T, 0, st>>>(skey, smask, ix.ncover, ncand, cand, ix.cov_atom, ix.cov_R,
                                                             ix.cov_mask, bcnt);
    KBG_CUDA(cudaGetLastError());
    exclusive_scan(bcnt, ix.blk_ptr, nblock, st);
    pool_free(bcnt);
    pool_free(tkey);
    pool_free(tmask);
    pool_free(skey);
    pool_free(smask);
    pool_free(tcnt);
    pool_free(toff);
    pool_free(d_ncover);
    pool_free(cand);
    pool_free(cnt);
    pool_free(coff);

    // 4. pairs (a, b, R), lexicographic
    const int64_t nab = static_cast<int64_t>(natom) * natom;
    int64_t* pcnt = dalloc<int64_t>(nab + 1);
    int64_t* poff = dalloc<int64_t>(nab + 1);
    KBG_CUDA(cudaMemsetAsync(pcnt, 0, (nab + 1) * sizeof(int64_t), st));
    k_pairs<<<grid_of(nab, 128), 128, 0, st>>>(P, pcnt, nullptr, nullptr, nullptr, nullptr);
    KBG_CUDA(cudaGetLastError());
    ix.npair = exclusive_scan(pcnt, poff, nab, st);
    ix.pair_a = dalloc<int32_t>(ix.npair);
    ix.pair_b = dalloc<int32_t>(ix.npair);
    ix.pair_R = dalloc<int32_t>(3 * ix.npair);
    k_pairs<<<grid_of(nab, 128), 128, 0, st>>>(P, nullptr, poff, ix.pair_a, ix.pair_b, ix.pair_R);
    KBG_CUDA(cudaGetLastError());
    pool_free(pcnt);
    pool_free(poff);
    int64_t* psize = dalloc<int64_t>(ix.npair + 1);
    ix.pair_off = dalloc<int64_t>(ix.npair + 1);
    ix.pair_key = dalloc<int64_t>(ix.npair);
    ix.pair_mirror = dalloc<int32_t>(ix.npair);
    KBG_CUDA(cudaMemsetAsync(psize, 0, (ix.npair + 1) * sizeof(int64_t), st));
    int* d_err = dalloc<int>(1);
    KBG_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), st));
    if (ix.npair) {
        k_pair_meta<<<grid_of(ix.npair, T), T, 0, st>>>(P, ix.npair, ix.pair_a, ix.pair_b, ix.pair_R, psize,
                                                        ix.pair_key);
        k_pair_mirror<<<grid_of(ix.npair, T), T, 0, st>>>(P, ix.npair, ix.pair_a, ix.pair_b, ix.pair_R, ix.pair_key,
                                                          ix.pair_mirror, d_err);
    }
    KBG_CUDA(cudaGetLastError());
    ix.nnz = exclusive_scan(psize, ix.pair_off, ix.npair, st);
    // repacked-DM sizes: canonical pairs only, rows padded to 16-column chunks
    KBG_CUDA(cudaMemsetAsync(psize, 0, (ix.npair + 1) * sizeof(int64_t), st));
    if (ix.npair) k_pair_rsize<<<grid_of(ix.npair, T), T, 0, st>>>(P, ix.npair, ix.pair_a, ix.pair_b, ix.pair_R, psize);
    KBG_CUDA(cudaGetLastError());
    ix.mir = dalloc<MirrorItem>(std::max<int64_t>(1, ix.npair));
    ix.mir_count = dalloc<int>(2);  // [0] mirror items, [1] repack items
    KBG_CUDA(cudaMemsetAsync(ix.mir_count, 0, 2 * sizeof(int), st));
    if (ix.npair)
        k_mirror_items<<<grid_of(ix.npair, T), T, 0, st>>>(P, ix.npair, ix.pair_a, ix.pair_b, ix.pair_R, ix.pair_off,
                                                           ix.pair_mirror, ix.mir, ix.mir_count);
    KBG_CUDA(cudaGetLastError());
    ix.pair_roff = dalloc<int64_t>(ix.npair + 1);
    ix.nrep = exclusive_scan(psize, ix.pair_roff, ix.npair, st);
    if (ix.nrep >= (int64_t(1) << 31)) throw Error(KBG_ERR_DIMENSION, "build_index: repacked density matrix too large");
    ix.rep = dalloc<RepackItem>(std::max<int64_t>(1, ix.npair));
    if (ix.npair)
        k_repack_items<<<grid_of(ix.npair, T), T, 0, st>>>(P, ix.npair, ix.pair_a, ix.pair_b, ix.pair_R, ix.pair_off,
                                                           ix.pair_roff, ix.pair_mirror, ix.rep, ix.mir_count + 1);
    KBG_CUDA(cudaGetLastError());
    pool_free(psize);
    int herr = 0;
    KBG_CUDA(cudaMemcpy(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (herr) {
        pool_free(d_err);
        throw Error(KBG_ERR_CONSISTENCY, "build_index: pair list not closed under (a,b,R) -> (b,a,-R)");
    }

    // 5. block work items (canonical cover pairs with shared points)
    int64_t* bpc = dalloc<int64_t>(nblock + 1);
    ix.bp_ptr = dalloc<int64_t>(nblock + 1);
    ix.blk_cost = dalloc<int64_t>(nblock);
    Stats* d_stats = dalloc<Stats>(1);
    KBG_CUDA(cudaMemsetAsync(bpc, 0, (nblock + 1) * sizeof(int64_t), st));
    KBG_CUDA(cudaMemsetAsync(d_stats, 0, sizeof(Stats), st));
    const unsigned wgrid = static_cast<unsigned>((nblock * 32 + T - 1) / T);
    k_bp_count<<<wgrid, T, 0, st>>>(P, nblock, ix.blk_ptr, ix.cov_atom, ix.cov_mask, bpc, ix.blk_cost, d_stats);
    KBG_CUDA(cudaGetLastError());
    ix.nbpair = exclusive_scan(bpc, ix.bp_ptr, nblock, st);
    pool_free(bpc);
    ix.bp = dalloc<BPair>(ix.nbpair);
    k_bp_fill<<<wgrid, T, 0, st>>>(P, nblock, ix.blk_ptr, ix.cov_atom, ix.cov_R, ix.cov_mask, ix.bp_ptr, ix.pair_key,
                                   ix.pair_off, ix.pair_roff, ix.npair, ix.bp, d_err);
    KBG_CUDA(cudaGetLastError());
    Stats hs;
    int hmir[2] = {0, 0};
    KBG_CUDA(cudaMemcpyAsync(&hs, d_stats, sizeof(Stats), cudaMemcpyDeviceToHost, st));
    KBG_CUDA(cudaMemcpyAsync(hmir, ix.mir_count, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    KBG_CUDA(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
    KBG_CUDA(cudaStreamSynchronize(st));
    pool_free(d_stats);
    pool_free(d_err);
    if (herr)
        throw Error(KBG_ERR_CONSISTENCY, "build_index: block " + std::to_string(herr - 1) +
                                             " has covers that share points but form no pair");
    ix.nmir = hmir[0];
    ix.nrep_items = hmir[1];
    ix.sum_m = static_cast<double>(hs.sum_m);
    ix.sum_m2 = static_cast<double>(hs.sum_m2);
    ix.natompt = static_cast<int64_t>(hs.natompt);
    ix.max_phi = hs.max_phi;
    ix.max_cover = hs.max_cover;
    ix.max_bpairs = hs.max_bpairs;
}

void copy_index_to_host(const DevIndex& ix, HostIndex& h, cudaStream_t st) {
    auto get = [&](auto& vec, const auto* src, int64_t n) {
        vec.resize(static_cast<size_t>(n));
        if (n) KBG_CUDA(cudaMemcpyAsync(vec.data(), src, n * sizeof(vec[0]), cudaMemcpyDeviceToHost, st));
    };
    get(h.blk_ptr, ix.blk_ptr, ix.nblock + 1);
    get(h.cov_atom, ix.cov_atom, ix.ncover);
    get(h.cov_R, ix.cov_R, 3 * ix.ncover);
    get(h.cov_mask, ix.cov_mask, ix.ncover);
    get(h.pair_a, ix.pair_a, ix.npair);
    get(h.pair_b, ix.pair_b, ix.npair);
    get(h.pair_R, ix.pair_R, 3 * ix.npair);
    get(h.pair_off, ix.pair_off, ix.npair + 1);
    get(h.pair_mirror, ix.pair_mirror, ix.npair);
    KBG_CUDA(cudaStreamSynchronize(st));
    h.valid = true;
}

}  // namespace kbg
