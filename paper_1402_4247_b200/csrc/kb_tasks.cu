// Per-block warp task lists for the grid kernels (built once per geometry,
// after the index). One thread per block: row groups (make_groups), the H
// tasks (group x partner cover, common quads) and the rho tasks (group x
// octet half), then an LPT assignment of the tasks to `task_warps` warps so the
// static per-warp schedule inside a CTA is balanced and deterministic.
#include <cub/cub.cuh>

#include "kb_device.cuh"

namespace kbg {

namespace {

struct TaskStats {
    int max_rows, max_h, max_r, too_many_covers;
};

template <class T>
T* talloc(size_t n) {
    T* p = nullptr;
    if (n == 0) n = 1;
    KBG_CUDA(pool_malloc(&p, n * sizeof(T)));
    return p;
}

int64_t scan_total(int64_t* cnt, int64_t* ptr, int64_t n, cudaStream_t st) {
    size_t bytes = 0;
    KBG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, ptr, static_cast<int>(n + 1), st));
    void* tmp = talloc<char>(bytes);
    KBG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, ptr, static_cast<int>(n + 1), st));
    int64_t total = 0;
    KBG_CUDA(cudaMemcpyAsync(&total, ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KBG_CUDA(cudaStreamSynchronize(st));
    pool_free(tmp);
    return total;
}

__device__ __forceinline__ uint16_t sat16(int64_t c) { return static_cast<uint16_t>(c > 65535 ? 65535 : c); }

__global__ void k_tasks(SysParams P, int64_t nblock, const int32_t* __restrict__ blk_ptr,
                        const int32_t* __restrict__ cov_atom, const uint64_t* __restrict__ cov_mask, int64_t* hcnt,
                        int64_t* rcnt, const int64_t* __restrict__ hptr, const int64_t* __restrict__ rptr, Task* hout,
                        Task* rout, TaskStats* st, int32_t* rows_out, int W) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nblock) return;
    const int c0 = blk_ptr[b];
    const int ncov = blk_ptr[b + 1] - c0;
    if (ncov > kMaxCoverPerBlock) {
        atomicMax(&st->too_many_covers, ncov);
        if (hcnt) hcnt[b] = rcnt[b] = 0;
        if (rows_out) rows_out[b] = 0;
        return;
    }
    int norb[kMaxCoverPerBlock], g_first[kMaxCoverPerBlock], g_end[kMaxCoverPerBlock], g_row0[kMaxCoverPerBlock],
        g_rows[kMaxCoverPerBlock], c_row0[kMaxCoverPerBlock], c_group[kMaxCoverPerBlock];
    for (int c = 0; c < ncov; ++c) norb[c] = P.sp[P.spc[cov_atom[c0 + c]]].norb;
    const int ng = make_groups(ncov, [&](int c) { return norb[c]; }, g_first, g_end, g_row0, g_rows, c_row0, c_group);
    int64_t nh = 0, nr = 0;
    for (int g = 0; g < ng; ++g) {
        const int tm = (g_rows[g] + 7) >> 3;
        // H: partners with common quads, paired consecutively when both have
        // <= 16 orbitals and the group <= 16 rows (the pair shares A fragments)
        int pend = -1;
        uint32_t pend_q = 0;
        // point density of a partner: exact common points over the points of the executed quads
        auto dens = [&](int cj, uint32_t q, int64_t& ex, int64_t& pts) {
            uint64_t m = 0;
            for (int ci = g_first[g]; ci < g_end[g] && ci <= cj; ++ci) m |= cov_mask[c0 + ci] & cov_mask[c0 + cj];
            const int tn = (norb[cj] + 7) >> 3;
            ex += static_cast<int64_t>(__popcll(m)) * tn;
            pts += 4LL * __popc(q) * tn;
        };
        auto emit = [&](int c1, uint32_t q1, int c2, uint32_t q2) {
            if (hout) {
                Task t;
                t.g = static_cast<uint8_t>(g);
                t.cj = static_cast<uint8_t>(c1);
                t.half = 0;
                t.pad_ = 0;
                t.qmask = static_cast<uint16_t>(q1);
                int64_t cost = static_cast<int64_t>(__popc(q1)) * tm * ((norb[c1] + 7) >> 3) + 2;
                t.cj2 = 0xFF;
                t.pad2_ = 0;
                t.qmask2 = 0;
                int64_t ex = 0, pts = 0;
                dens(c1, q1, ex, pts);
                if (c2 >= 0) {
                    t.cj2 = static_cast<uint8_t>(c2);
                    t.qmask2 = static_cast<uint16_t>(q2);
                    cost += static_cast<int64_t>(__popc(q2)) * tm * ((norb[c2] + 7) >> 3) + 1;
                    dens(c2, q2, ex, pts);
                }
                // density in 1/255 (A5 switch, KBG_OPT_SPARSE_DFMA): tasks below the threshold run the
                // point-exact FP64 path (kb_gridcore.cuh h_task_dfma) instead of DMMA over whole quads
                t.pad2_ = static_cast<uint8_t>(pts ? (255 * ex + pts / 2) / pts : 255);
                t.cost = sat16(cost);
                hout[hptr[b] + nh] = t;
            }
            ++nh;
        };
        for (int cj = g_first[g]; cj < ncov; ++cj) {
            const uint64_t mj = cov_mask[c0 + cj];
            uint32_t qm = 0;
            for (int ci = g_first[g]; ci < g_end[g] && ci <= cj; ++ci) qm |= quads_of(cov_mask[c0 + ci] & mj);
            if (!qm) continue;
            const bool pairable = g_rows[g] <= 16 && norb[cj] <= 16;
            if (!pairable) {
                emit(cj, qm, -1, 0);
            } else if (pend < 0) {
                pend = cj;
                pend_q = qm;
            } else {
                emit(pend, pend_q, cj, qm);
                pend = -1;
            }
        }
        if (pend >= 0) emit(pend, pend_q, -1, 0);
    }
    // rho tasks: (group, octet half, partner range). Ranges split the partner
    // list so no task exceeds ~1/2 of a warp's average share of the block,
    // which keeps the LPT schedule balanced over W warps.
    int64_t rtotal = 0;
    for (int g = 0; g < ng; ++g)
        for (int cj = g_first[g]; cj < ncov; ++cj) {
            uint32_t om = 0;
            for (int ci = g_first[g]; ci < g_end[g] && ci <= cj; ++ci)
                om |= octets_of(cov_mask[c0 + ci] & cov_mask[c0 + cj]);
            rtotal += __popc(om) * ((g_rows[g] + 7) >> 3) * ((norb[cj] + 3) >> 2);
        }
    const int64_t target = rtotal / (2 * W) > 16 ? rtotal / (2 * W) : 16;
    for (int g = 0; g < ng; ++g) {
        const int tm = (g_rows[g] + 7) >> 3;
        for (int h = 0; h < 8 / kRhoOct; ++h) {
            int64_t cost = 0;
            int start = -1;
            for (int cj = g_first[g]; cj < ncov; ++cj) {
                const uint64_t mj = cov_mask[c0 + cj];
                uint32_t om = 0;
                for (int ci = g_first[g]; ci < g_end[g] && ci <= cj; ++ci) om |= octets_of(cov_mask[c0 + ci] & mj);
                om &= ((1u << kRhoOct) - 1u) << (kRhoOct * h);
                if (om) {
                    if (start < 0) start = cj;
                    cost += __popc(om) * tm * ((norb[cj] + 3) >> 2);
                }
                if (start >= 0 && (cost >= target || cj + 1 == ncov)) {
                    if (rout) {
                        Task t;
                        t.g = static_cast<uint8_t>(g);
                        t.cj = static_cast<uint8_t>(start);  // partner range [cj, qmask)
                        t.half = static_cast<uint8_t>(h);
                        t.pad_ = 0;
                        t.qmask = static_cast<uint16_t>(cj + 1);
                        t.cost = sat16(cost + 8);
                        t.cj2 = 0xFF;
                        t.pad2_ = 0;
                        t.qmask2 = 0;
                        rout[rptr[b] + nr] = t;
                    }
                    ++nr;
                    cost = 0;
                    start = -1;
                }
            }
        }
    }
    if (rows_out) rows_out[b] = ng ? g_row0[ng - 1] + g_rows[ng - 1] : 0;
    if (hcnt) {
        hcnt[b] = nh;
        rcnt[b] = nr;
        atomicMax(&st->max_rows, ng ? g_row0[ng - 1] + g_rows[ng - 1] : 0);
        atomicMax(&st->max_h, static_cast<int>(nh));
        atomicMax(&st->max_r, static_cast<int>(nr));
    }
}

// Sort one block's tasks by cost (descending, stable), assign each to the
// least-loaded of W warps (LPT), emit warp-major into `out`; wptr has a stride
// of kMaxTaskWarps + 1 per block.
__global__ void k_tasks_lpt(int64_t nblock, int W, const int64_t* __restrict__ ptr, Task* tmp, Task* out,
                            int32_t* wptr) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nblock) return;
    const int64_t p0 = ptr[b];
    const int n = static_cast<int>(ptr[b + 1] - p0);
    Task* t = tmp + p0;
    for (int i = 1; i < n; ++i) {  // insertion sort, stable, descending cost
        const Task x = t[i];
        int j = i - 1;
        while (j >= 0 && t[j].cost < x.cost) {
            t[j + 1] = t[j];
            --j;
        }
        t[j + 1] = x;
    }
    int64_t load[kMaxTaskWarps];
    int cnt[kMaxTaskWarps];
    for (int w = 0; w < W; ++w) load[w] = cnt[w] = 0;
    for (int i = 0; i < n; ++i) {
        int best = 0;
        for (int w = 1; w < W; ++w)
            if (load[w] < load[best]) best = w;
        load[best] += t[i].cost;
        t[i].pad_ = static_cast<uint8_t>(best);
        ++cnt[best];
    }
    int pos[kMaxTaskWarps];
    int acc = 0;
    int32_t* wp = wptr + b * (kMaxTaskWarps + 1);
    for (int w = 0; w < W; ++w) {
        wp[w] = acc;
        pos[w] = acc;
        acc += cnt[w];
    }
    for (int w = W; w <= kMaxTaskWarps; ++w) wp[w] = acc;
    for (int i = 0; i < n; ++i) out[p0 + pos[t[i].pad_]++] = t[i];
}

// W == 1 (one task queue per block, the persistent kernels' default): the LPT
// assignment degenerates to a stable sort by descending cost. One warp per
// block ranks its tasks (rank = heavier tasks + equal tasks before it) and
// scatters them -- the same order as k_tasks_lpt, without its serial insertion
// sort through global memory.
__global__ void k_tasks_sort(int64_t nblock, const int64_t* __restrict__ ptr, const Task* __restrict__ tmp, Task* out,
                             int32_t* wptr) {
    const int64_t b = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (b >= nblock) return;
    const int64_t p0 = ptr[b];
    const int n = static_cast<int>(ptr[b + 1] - p0);
    for (int i = lane; i < n; i += 32) {
        Task t = tmp[p0 + i];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            const uint16_t cj = tmp[p0 + j].cost;
            rank += (cj > t.cost) || (cj == t.cost && j < i);
        }
        t.pad_ = 0;
        out[p0 + rank] = t;
    }
    int32_t* wp = wptr + b * (kMaxTaskWarps + 1);
    for (int w = lane; w <= kMaxTaskWarps; w += 32) wp[w] = w == 0 ? 0 : n;
}

}  // namespace

void free_tasks(DevIndex& ix) {
    for (void* p : {static_cast<void*>(ix.ht_ptr), static_cast<void*>(ix.ht), static_cast<void*>(ix.ht_wptr),
                    static_cast<void*>(ix.rt_ptr), static_cast<void*>(ix.rt), static_cast<void*>(ix.rt_wptr)})
        if (p) pool_free(p);
    ix.ht_ptr = ix.rt_ptr = nullptr;
    ix.ht = ix.rt = nullptr;
    ix.ht_wptr = ix.rt_wptr = nullptr;
    if (ix.blk_rows) pool_free(ix.blk_rows);
    ix.blk_rows = nullptr;
}

void build_tasks_device(const SysParams& P, DevIndex& ix, int h_warps, int r_warps, int r_split, cudaStream_t st) {
    free_tasks(ix);
    ix.htask_warps = h_warps;
    ix.rtask_warps = r_warps;
    const int64_t nb = ix.nblock;
    const int T = 128;
    const unsigned grid = static_cast<unsigned>((nb + T - 1) / T);
    int64_t* hcnt = talloc<int64_t>(nb + 1);
    int64_t* rcnt = talloc<int64_t>(nb + 1);
    TaskStats* d_st = talloc<TaskStats>(1);
    KBG_CUDA(cudaMemsetAsync(hcnt, 0, (nb + 1) * sizeof(int64_t), st));
    KBG_CUDA(cudaMemsetAsync(rcnt, 0, (nb + 1) * sizeof(int64_t), st));
    KBG_CUDA(cudaMemsetAsync(d_st, 0, sizeof(TaskStats), st));
    if (!ix.blk_rows) ix.blk_rows = talloc<int32_t>(nb);
    k_tasks<<<grid, T, 0, st>>>(P, nb, ix.blk_ptr, ix.cov_atom, ix.cov_mask, hcnt, rcnt, nullptr, nullptr, nullptr,
                                nullptr, d_st, ix.blk_rows, r_split);
    KBG_CUDA(cudaGetLastError());
    ix.ht_ptr = talloc<int64_t>(nb + 1);
    ix.rt_ptr = talloc<int64_t>(nb + 1);
    ix.nhtask = scan_total(hcnt, ix.ht_ptr, nb, st);
    ix.nrtask = scan_total(rcnt, ix.rt_ptr, nb, st);
    Task* htmp = talloc<Task>(ix.nhtask);
    Task* rtmp = talloc<Task>(ix.nrtask);
    k_tasks<<<grid, T, 0, st>>>(P, nb, ix.blk_ptr, ix.cov_atom, ix.cov_mask, nullptr, nullptr, ix.ht_ptr, ix.rt_ptr,
                                htmp, rtmp, d_st, nullptr, r_split);
    KBG_CUDA(cudaGetLastError());
    ix.ht = talloc<Task>(ix.nhtask);
    ix.rt = talloc<Task>(ix.nrtask);
    ix.ht_wptr = talloc<int32_t>(nb * (kMaxTaskWarps + 1));
    ix.rt_wptr = talloc<int32_t>(nb * (kMaxTaskWarps + 1));
    const unsigned wgrid = static_cast<unsigned>((nb * 32 + 255) / 256);
    if (h_warps == 1)
        k_tasks_sort<<<wgrid, 256, 0, st>>>(nb, ix.ht_ptr, htmp, ix.ht, ix.ht_wptr);
    else
        k_tasks_lpt<<<grid, T, 0, st>>>(nb, h_warps, ix.ht_ptr, htmp, ix.ht, ix.ht_wptr);
    if (r_warps == 1)
        k_tasks_sort<<<wgrid, 256, 0, st>>>(nb, ix.rt_ptr, rtmp, ix.rt, ix.rt_wptr);
    else
        k_tasks_lpt<<<grid, T, 0, st>>>(nb, r_warps, ix.rt_ptr, rtmp, ix.rt, ix.rt_wptr);
    KBG_CUDA(cudaGetLastError());
    TaskStats hs;
    KBG_CUDA(cudaMemcpyAsync(&hs, d_st, sizeof(hs), cudaMemcpyDeviceToHost, st));
    KBG_CUDA(cudaStreamSynchronize(st));
    pool_free(hcnt);
    pool_free(rcnt);
    pool_free(d_st);
    pool_free(htmp);
    pool_free(rtmp);
    if (hs.too_many_covers)
        throw Error(KBG_ERR_DIMENSION, "a grid block is covered by " + std::to_string(hs.too_many_covers) +
                                           " atom images (max " + std::to_string(kMaxCoverPerBlock) + ")");
    ix.max_rows_padded = hs.max_rows;
    ix.max_htask = hs.max_h;
    ix.max_rtask = hs.max_r;
}

}  // namespace kbg
