// Fused H reduction + mirror over NVLink/NVSwitch peer memory (SURVEY.md
// 8(e)): the multi-GPU H step without NCCL.
//
// Every rank accumulates its shard's partial H (canonical pairs only) into its
// own exchange buffer X_r, which every peer has mapped (CUDA IPC). One kernel
// then, on each rank r:
//   1. signals "partials ready" to every peer and waits for all peers
//      (flags in peer memory, system-scope release/acquire);
//   2. for the canonical entries of its slice (contiguous, balanced by size)
//      sums the partials of the ranks whose shard touches the pair (owner
//      masks; the others are exact zeros) in rank order (same bits on every
//      rank), symmetrizes the (a, a, 0) blocks, and stores each result into
//      every rank's buffer -- a reduce-scatter + all-gather in one pass over
//      NVLink; the last CTA signals "slice written";
//   3. once every rank's slice has landed, copies X_r into the caller's H and
//      fills the mirror blocks H_ba(-R) = H_ab(R)^T locally (warp per pair).
// All CTAs fit on the GPU at once (4 per SM, no shared memory) and nothing they
// wait for depends on a later kernel, so the waits cannot deadlock; every wait
// gives up after 10 s anyway (error word, kbg_comm_check).
#include <algorithm>

#include "kb_internal.cuh"

namespace kbg {

namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Thread 0 of every CTA: wait until every rank's flag in this rank's flag
// array lies in [lo, lo + 1] (a peer may already be one phase ahead: it
// signals its next phase once it has seen ours, never two). A flag outside
// that window means the ranks' call sequences drifted apart (e.g. after a
// failed call); a peer that never arrives must not hang the GPU, so the wait
// gives up after 10 s. Either way the error word of EVERY rank is raised
// (flags[kMaxRanks + 1], read by kbg_comm_check on each rank) and the caller
// skips all further reads and writes of peer buffers. Returns false then.
__device__ bool wait_flags(const CommArgs& c, unsigned long long lo) {
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
        const unsigned long long* f = c.flags[c.rank];
        const unsigned long long t0 = globaltimer();
        bool ok = true;
        for (int k = 0; k < c.nranks && ok; ++k)
            for (;;) {
                const unsigned long long v = ld_acquire_sys(f + k);
                if (v == lo || v == lo + 1) break;
                if (v > lo + 1 || globaltimer() - t0 > 10000000000ull) {
                    ok = false;
                    break;
                }
                __nanosleep(64);
            }
        if (!ok)
            for (int k = 0; k < c.nranks; ++k) c.flags[k][kMaxRanks + 1] = 1ull;
        s_ok = ok;
    }
    __syncthreads();
    return s_ok != 0;
}

// Signal `epoch` into slot `rank` of every rank's flag array.
__device__ void signal_flags(const CommArgs& c, unsigned long long epoch) {
    __threadfence_system();
    for (int k = 0; k < c.nranks; ++k) st_release_sys(c.flags[k] + c.rank, epoch);
}

// Copy-out fused with the mirror: one warp per canonical pair block copies the
// block from the exchange buffer into the caller's H and writes its transpose
// into the mirror block H_ba(-R) (the (a, a, 0) blocks arrive symmetrized from
// the reduce and are copied as is). Replaces a full-array copy plus k_mirror.
__device__ __forceinline__ void copy_mirror(const CommArgs& c, int64_t npair, int nspin, int64_t nnz,
                                            const int64_t* __restrict__ poff, const int32_t* __restrict__ mirror,
                                            double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const double* x = c.x[c.rank];
    for (int64_t p = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; p < npair;
         p += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
        if (!c.pair_canon[p]) continue;  // written by its canonical partner
        const int na = c.pair_na[p], nb = c.pair_nb[p];
        const int64_t q = mirror[p];
        for (int s = 0; s < nspin; ++s) {
            // reduced values sit in the hi limb's slot
            const double* src = x + (c.ls == 2 ? det_hi(s, poff[p], nnz) : s * nnz + poff[p]);
            double* dst = out + s * nnz + poff[p];
            double* dq = out + s * nnz + poff[q];
#pragma unroll 4
            for (int e = lane; e < na * nb; e += 32) {
                const double v = src[(KBG_DET_SPLIT || c.ls == 1) ? e : 2 * e];
                dst[e] = v;
                if (q != p) dq[(e % nb) * na + e / nb] = v;
            }
        }
    }
}

// One thread per element of this rank's slice, with the element's two
// offsets precomputed on the host (el0: the canonical entry, el1: its mirror
// entry -- or the transposed entry of an (a,a,0) block, flagged by bit 31 --
// or el0 itself on such a block's diagonal): one coalesced index load, then
// all N partials in flight at once, then the stores.
__global__ void __launch_bounds__(1024, 1) k_reduce_mirror(CommArgs c, int nspin, int64_t nnz, int64_t ne,
                                                       const int32_t* __restrict__ el0,
                                                       const int32_t* __restrict__ el1, unsigned long long epoch,
                                                       int64_t npair, const int64_t* __restrict__ poff,
                                                       const int32_t* __restrict__ pmirror, double* __restrict__ out) {
    if (c.tstamp && blockIdx.x == 0 && threadIdx.x == 0) c.tstamp[0] = globaltimer();
    if (blockIdx.x == 0 && threadIdx.x == 0) signal_flags(c, epoch);
    // on a failed wait this CTA neither reads nor writes peer memory (every rank's error word is set)
    const bool ok = wait_flags(c, epoch);
    if (c.tstamp && threadIdx.x == 0) atomicMax(c.tstamp + 1, globaltimer());
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; ok && t < ne * nspin;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int s = static_cast<int>(t / ne);
        const int64_t el = t - s * ne;
        const int64_t base = s * nnz;
        const int64_t e0 = el0[el];
        const int32_t m = el1[el];
        const bool sym = m < 0;  // (a, a, 0) off-diagonal: (H + H^T) / 2
        const int64_t e1 = m & 0x7fffffff;
        const int64_t o0 = c.ls == 2 ? det_hi(s, e0, nnz) : base + e0;  // result slot: the (hi) value
        const int64_t o1 = c.ls == 2 ? det_hi(s, e1, nnz) : base + e1;
        const int64_t lo = c.ls == 2 ? det_lo(s, e0, nnz) - o0 : 0;     // lo limb offset from hi
        // only the ranks whose shard touches the pair are read: the other partials are exact
        // zeros, so the rank-order sum has the same bits as over all N
        const uint32_t om = c.elm[el];
        double v = 0.0, v2 = 0.0;
        if (c.ls == 2) {
            // two-limb partials (deterministic H): the hi and the lo sums are exact in any order
            // (kb_gridcore.cuh h_scatter), so H = hi + lo has the bits of the single-GPU pass
            // (accumulated as they arrive: any order gives the same bits, and no partials are held,
            // which keeps the kernel at <= 64 registers -- all CTAs must be resident, see launch)
            double hi = 0.0, lo_s = 0.0, hi2 = 0.0, lo2 = 0.0;
#pragma unroll
            for (int k = 0; k < kMaxRanks; ++k) {
                if (k < c.nranks && ((om >> k) & 1u)) {
                    hi += c.x[k][o0];
                    lo_s += c.x[k][o0 + lo];
                    if (sym) {
                        hi2 += c.x[k][o1];
                        lo2 += c.x[k][o1 + lo];
                    }
                }
            }
            v = hi + lo_s;
            v2 = hi2 + lo2;
        } else {
            double part[kMaxRanks], part2[kMaxRanks];
#pragma unroll
            for (int k = 0; k < kMaxRanks; ++k) {
                const bool on = k < c.nranks && ((om >> k) & 1u);
                part[k] = on ? c.x[k][o0] : 0.0;
                part2[k] = (sym && on) ? c.x[k][o1] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < kMaxRanks; ++k) {
                v += part[k];
                v2 += part2[k];
            }
        }
        if (sym) v = 0.5 * (v + v2);  // same expression as k_mirror / k_finalize
        // canonical entries only (and both halves of an (a, a, 0) block): every rank then fills
        // the mirror blocks H_ba(-R) = H_ab(R)^T locally, halving the NVLink writes; the result
        // goes to the first limb's slot
        for (int k = 0; k < c.nranks; ++k) {
            c.x[k][o0] = v;
            if (sym) c.x[k][o1] = v;
        }
    }
    // slice written everywhere: the last CTA signals epoch + 1 (the barrier
    // makes the CTA's stores visible to thread 0, whose system fence is cumulative)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned int done = atomicAdd(c.counter, 1u);
        if (done == gridDim.x - 1) {
            *c.counter = 0u;
            if (c.tstamp) c.tstamp[2] = globaltimer();
            signal_flags(c, epoch + 1);
        }
    }
    if (!out || !ok) return;
    // fused copy-out + mirror (all CTAs are resident): wait until every rank's slice has landed here
    if (c.tstamp && blockIdx.x == 0 && threadIdx.x == 0) c.tstamp[3] = globaltimer();
    if (!wait_flags(c, epoch + 1)) return;
    if (c.tstamp && threadIdx.x == 0) atomicMax(c.tstamp + 4, globaltimer());
    copy_mirror(c, npair, nspin, nnz, poff, pmirror, out);
    if (c.tstamp) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(c.tstamp + 5, globaltimer());
    }
}

__global__ void __launch_bounds__(256) k_comm_copy_out(CommArgs c, int64_t n, int64_t nnz, double* __restrict__ out,
                                                       unsigned long long epoch) {
    if (!wait_flags(c, epoch)) return;
    if (c.ls == 2) {  // reduced values in the hi limbs' slots; n = nspin * nnz, nnz = n_per_spin
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            out[i] = c.x[c.rank][det_hi(static_cast<int>(i / nnz), i % nnz, nnz)];
        return;
    }
    const double2* src = reinterpret_cast<const double2*>(c.x[c.rank]);
    double2* dst = reinterpret_cast<double2*>(out);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n / 2;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[i];
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) out[n - 1] = c.x[c.rank][n - 1];
}

}  // namespace

int launch_reduce_mirror(const CommArgs& c, const DevIndex& ix, const SysParams& sys, int nspin, double* d_out,
                         unsigned long long epoch, cudaStream_t st) {
    int dev = 0, sms = 0;
    KBG_CUDA(cudaGetDevice(&dev));
    KBG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // All CTAs must be resident at once: a CTA that has signalled its slice waits for every other
    // CTA's (the counter) before the copy-out, so a CTA that cannot start would deadlock the rest
    // (until the 10 s timeout). 4 per SM x 256 threads (<= 64 registers, __launch_bounds__) unless the
    // occupancy query says fewer fit; the copy-out phase of large H wants the warps (2 per SM measured
    // 4 % slower at 448 atoms on 4 GPUs).
    int per_sm = 0;
    KBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_reduce_mirror, 256, 0));
    unsigned grid = static_cast<unsigned>(sms) * static_cast<unsigned>(std::max(1, std::min(4, per_sm)));
    unsigned threads = 256;
    if (c.sms > 0 && c.pair_na) {
        // next to the density kernel (KBG_OPT_EXCHANGE_SMS): one 1024-thread CTA per SM (<= 64 registers,
        // __launch_bounds__), so each CTA holds a whole SM and the density kernel's CTAs, which leave
        // that many SMs free, cannot take the SMs the exchange needs resident
        grid = static_cast<unsigned>(std::min(c.sms, sms));
        threads = 1024;
    }
    if (c.pair_na) {  // reduce, then (same kernel) copy-out + mirror once every slice has landed
        k_reduce_mirror<<<grid, threads, 0, st>>>(c, nspin, ix.nnz, c.ne, c.el0, c.el1, epoch, ix.npair, ix.pair_off,
                                                  ix.pair_mirror, d_out);
        KBG_CUDA(cudaGetLastError());
        return 1;
    }
    k_reduce_mirror<<<grid, 256, 0, st>>>(c, nspin, ix.nnz, c.ne, c.el0, c.el1, epoch, 0, nullptr, nullptr, nullptr);
    KBG_CUDA(cudaGetLastError());
    const int64_t n = static_cast<int64_t>(nspin) * ix.nnz;
    k_comm_copy_out<<<grid, 256, 0, st>>>(c, n, ix.nnz, d_out, epoch + 1);
    KBG_CUDA(cudaGetLastError());
    return 2 + launch_mirror(ix, sys, nspin, d_out, st);
}

namespace {
__global__ void k_pair_owners(int64_t nblock, const int64_t* __restrict__ bp_ptr, const BPair* __restrict__ bp,
                              const int64_t* __restrict__ pair_off, int64_t npair, const int64_t* __restrict__ bounds,
                              int nranks, uint32_t* own) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nblock) return;
    int r = 0;
    while (r + 1 < nranks && b >= bounds[r + 1]) ++r;
    for (int64_t e = bp_ptr[b]; e < bp_ptr[b + 1]; ++e) {
        const int64_t off = bp[e].off;
        int64_t lo = 0, hi = npair - 1;  // pair with pair_off[p] == off
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) / 2;
            if (pair_off[mid] <= off)
                lo = mid;
            else
                hi = mid - 1;
        }
        atomicOr(own + lo, 1u << r);
    }
}
}  // namespace

void pair_owners(const DevIndex& ix, const std::vector<int64_t>& bounds, std::vector<uint32_t>& out, cudaStream_t st) {
    const int nranks = static_cast<int>(bounds.size()) - 1;
    out.assign(ix.npair, 0u);
    if (ix.npair == 0) return;
    uint32_t* d_own = nullptr;
    int64_t* d_b = nullptr;
    KBG_CUDA(pool_malloc(&d_own, ix.npair * sizeof(uint32_t)));
    KBG_CUDA(pool_malloc(&d_b, bounds.size() * sizeof(int64_t)));
    KBG_CUDA(cudaMemsetAsync(d_own, 0, ix.npair * sizeof(uint32_t), st));
    KBG_CUDA(cudaMemcpyAsync(d_b, bounds.data(), bounds.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    k_pair_owners<<<static_cast<unsigned>((ix.nblock + 127) / 128), 128, 0, st>>>(ix.nblock, ix.bp_ptr, ix.bp,
                                                                                 ix.pair_off, ix.npair, d_b, nranks,
                                                                                 d_own);
    KBG_CUDA(cudaGetLastError());
    KBG_CUDA(cudaMemcpyAsync(out.data(), d_own, ix.npair * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    KBG_CUDA(cudaStreamSynchronize(st));
    pool_free(d_own);
    pool_free(d_b);
}

}  // namespace kbg
