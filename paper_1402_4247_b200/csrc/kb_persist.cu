// Persistent, warp-specialized grid kernels (one CTA per SM; 1 producer warp +
// kPersistConsumersR = 19 consumer warps for rho, + kPersistConsumersH = 27 for H).
//
// Warp 0 (producer) pulls grid blocks from a global work counter (blocks
// ordered heaviest first, or in grid order for large grids: KBG_OPT_BLOCK_ORDER), waits for a free shared-memory buffer (`empty`
// mbarrier) and stages the block with two TMA bulk copies from the geometry
// cache (kb_cache.cu) -- the block's table image and its Phi rows -- which
// complete on the buffer's `full` mbarrier (expect_tx). For H it also gathers
// w = V dV of the block's 64 points. The other warps (consumers) wait on `full`,
// run their LPT-assigned tasks (DMMA contractions, kb_gridcore.cuh) and move
// on to the next buffer without a CTA-wide barrier; the last consumer to
// finish a block (shared counter) reduces the per-warp rho accumulators in a
// fixed order, writes rho, and arrives on `empty`. Staging of block k+1 thus
// overlaps the DMMA work of block k.
#include "kb_gridcore.cuh"

namespace kbg {

namespace {

using namespace core;

template <bool DENSITY>
struct Cfg {
    static constexpr int NC = DENSITY ? kPersistConsumersR : kPersistConsumersH;
    static constexpr int NT = (kPersistProducers + NC) * 32;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 100000;\n"
        " selp.u32 %0, 1, 0, p;\n"
        "}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Waits for the phase with the given parity; sleeps `ns` between attempts so
// a waiting warp does not take issue slots from the working ones.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, unsigned ns = 32) {
    while (!mbar_try(bar, parity)) __nanosleep(ns);
}
// TMA bulk copy global -> shared, completing `bytes` on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Same with an L2 cache policy (createpolicy): the geometry cache is streamed
// once per pass, so its lines are marked evict_first and do not push the
// gathered operands (repacked DM, H accumulators, V) out of L2.
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Two buffers at byte offsets 0 and bsz of kbg_smem, then the mbarriers.
// Buffer s is selected arithmetically (no dynamically indexed struct arrays,
// which would live in local memory).
// Fixed stride (rho): buffer 1 sits at a compile-time offset (half of the 227 KB
// opt-in maximum), so the buffer select is one multiply by a constant, which the
// compiler rematerializes for free inside the task loops (under register pressure
// it re-derives the buffer base per partner). Measured rho 0.376 -> 0.368 ms (56
// atoms), 2.79 -> 2.73 (448); H is 1-3 % slower with it and keeps the tight stride.
#ifndef KBG_FIXED_STRIDE_R
#define KBG_FIXED_STRIDE_R 1
#endif
#ifndef KBG_FIXED_STRIDE_H
#define KBG_FIXED_STRIDE_H 0
#endif
constexpr uint32_t kBufStride = ((227u * 1024u - 64u) / 2u) & ~15u;

template <bool DENSITY>
struct Buffers {
    static constexpr bool kFixed = DENSITY ? KBG_FIXED_STRIDE_R : KBG_FIXED_STRIDE_H;
    Smem sm0;
    uint32_t bsz;
    uint64_t* full;   // [2]
    uint64_t* empty;  // [2]
    __device__ __forceinline__ Smem buf(int s) const {
        Smem x = sm0;
        x.base = kFixed ? static_cast<uint32_t>(s) * kBufStride : (s ? bsz : 0u);
        return x;
    }
};

template <bool DENSITY>
__device__ __forceinline__ Buffers<DENSITY> carve_all(const GridArgs& g) {
    Buffers<DENSITY> B;
    B.bsz = Buffers<DENSITY>::kFixed ? kBufStride : (g.lay[12] + 15u) & ~15u;
    B.sm0 = carve(0u, g);
    B.full = reinterpret_cast<uint64_t*>(kbg_smem + 2 * B.bsz);
    B.empty = B.full + 2;
    return B;
}

// acc section: H w[nspin][64]; rho per-warp sums [nspin][NC][64] (static
// lists) or per-task sums [nspin][ntask][32] (task queue, task_warps == 1).
__host__ __device__ inline size_t persist_acc(const GridArgs& g, bool density) {
    if (!density) return static_cast<size_t>(g.nspin) * 64;
    if (g.task_warps == 1) return static_cast<size_t>(g.nspin) * g.max_rtasks * 32;
    return static_cast<size_t>(g.nspin) * 64 * kPersistConsumersR;
}

__host__ __device__ inline size_t persist_bytes(const GridArgs& g, bool density) {
    size_t off[12];
    const size_t b = align16(buffer_layout(g, persist_acc(g, density), off));
    if (density ? KBG_FIXED_STRIDE_R : KBG_FIXED_STRIDE_H) return b <= kBufStride ? 2 * static_cast<size_t>(kBufStride) + 64 : 2 * b + 64;
    return 2 * b + 64;
}

// Next non-empty owned block from the work counter (-1: none left); empty
// blocks get rho = 0 on the way.
template <bool DENSITY>
__device__ int64_t next_block(const GridArgs& g, int lane) {
    for (;;) {
        int idx = 0;
        if (lane == 0) idx = atomicAdd(g.counter, 1);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx >= g.norder) return -1;
        const int64_t b = g.order[idx];
        if (g.blk_ptr[b + 1] > g.blk_ptr[b]) return b;
        if (DENSITY) {
            int bi, bj, bk;
            block_decode(g.sys, b, bi, bj, bk);
            for (int p = lane; p < 64; p += 32) {
                bool valid;
                const int64_t pt = slot_point(g.sys, bi, bj, bk, p, valid);
                if (valid)
                    for (int spin = 0; spin < g.nspin; ++spin) g.out[spin * g.npts + pt] = 0.0;
            }
        }
    }
}

__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes, uint64_t pol) {
#if KBG_L2_HINT
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src), "r"(bytes), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
#endif
}

// Producer warp: block k goes to buffer k & 1. The block after the current
// one is fetched early and its cache image prefetched into L2, so the bulk
// copy issued when its buffer frees up is served from L2.
template <bool DENSITY, bool DET>
__device__ void producer(const GridArgs& g, const Buffers<DENSITY>& B, int lane) {
    unsigned long long t_wait = 0, t0 = clock64();
    uint64_t pol = 0;
#if KBG_L2_HINT
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
    auto image = [&](int64_t b, const unsigned char*& tab, const double*& phi, uint32_t& tb, uint32_t& pb) {
        const int64_t i = b - g.blk_begin;
        tab = g.tabs + i * g.tab_bytes;
        phi = g.phis + g.phi_off[i];
        tb = static_cast<uint32_t>(g.tab_bytes);
        pb = static_cast<uint32_t>((g.phi_off[i + 1] - g.phi_off[i]) * sizeof(double));
    };
    // H: w = V dV of a block's points is loaded into registers one block ahead
    // (lane l holds points l and 32 + l of every spin), so the loads -- from
    // HBM, or over PCIe when V is mapped host memory (kbg_grid_pass on pinned
    // buffers) -- are in flight while the producer waits for a free buffer.
    double w_cur[2 * kMaxSpin], w_next[2 * kMaxSpin];
    auto load_w = [&](int64_t b, double (&w)[2 * kMaxSpin]) {
        if (DENSITY || !g.in || b < 0) return;
        int bi, bj, bk;
        block_decode(g.sys, b, bi, bj, bk);
#pragma unroll
        for (int j = 0; j < 2 * kMaxSpin; ++j) {
            const int i = lane + 32 * j;
            bool valid = false;
            const int64_t pt = slot_point(g.sys, bi, bj, bk, i & 63, valid);
            w[j] = (valid && i < g.nspin * 64) ? g.in[(i >> 6) * g.npts + pt] : 0.0;
        }
    };
    int64_t b_next = next_block<DENSITY>(g, lane);
    load_w(b_next, w_next);
    for (int k = 0;; ++k) {
        const int s = k & 1;
        const int64_t b = b_next;
#pragma unroll
        for (int j = 0; j < 2 * kMaxSpin; ++j) w_cur[j] = w_next[j];
        if (b >= 0) {
            b_next = next_block<DENSITY>(g, lane);
            load_w(b_next, w_next);
            if (b_next >= 0 && lane == 0) {
                const unsigned char* tab;
                const double* phi;
                uint32_t tb, pb;
                image(b_next, tab, phi, tb, pb);
                prefetch_l2(tab, tb, pol);
                prefetch_l2(phi, pb, pol);
            }
        }
        if (k >= 2) {
            const unsigned long long tw = clock64();
            mbar_wait(&B.empty[s], ((k >> 1) - 1) & 1, 256);
            t_wait += clock64() - tw;
        }
        const Smem sm = B.buf(s);
        if (b < 0) {
            if (lane == 0) {
                sm.meta()->block = -1;
                mbar_arrive(&B.full[s]);
                if (KBG_EXPERIMENTS && g.dbg) {
                    atomicAdd(&g.dbg[0], t_wait);
                    atomicAdd(&g.dbg[1], clock64() - t0);
                }
            }
            return;
        }
        if (!DENSITY && g.in) {  // w = V dV of the block's points, every spin
            bool fin = true;
#pragma unroll
            for (int j = 0; j < 2 * kMaxSpin; ++j) {
                const int i = lane + 32 * j;
                if (i < g.nspin * 64) sm.acc()[i] = w_cur[j] * (g.dV * g.sign);  // fault hook sign folded into w
                fin = fin && isfinite(w_cur[j]);
            }
            // non-finite V (the deterministic path sees it in its max|V| pass instead): flag it for
            // the host API's KBG_ERR_NONFINITE, like kband's check (householder.cpp:119-123)
            if (!DET && !__all_sync(0xffffffffu, fin) && lane == 0 && g.vbits)
                atomicMax(const_cast<unsigned long long*>(g.vbits), 0x7ff8000000000000ull);
        }
        __syncwarp();
        if (lane == 0) {
            const unsigned char* tab;
            const double* phi;
            uint32_t tb, pb;
            image(b, tab, phi, tb, pb);
            mbar_arrive_tx(&B.full[s], tb + pb);
#if KBG_L2_HINT
            bulk_g2s_hint(sm.meta(), tab, tb, &B.full[s], pol);
            bulk_g2s_hint(sm.phi(), phi, pb, &B.full[s], pol);
#else
            bulk_g2s(sm.meta(), tab, tb, &B.full[s]);
            bulk_g2s(sm.phi(), phi, pb, &B.full[s]);
#endif
            if (KBG_EXPERIMENTS && g.dbg) {  // debug only: copy latency (delays the next fetch)
                const unsigned long long tc = clock64();
                mbar_wait(&B.full[s], (k >> 1) & 1);
                atomicAdd(&g.dbg[7], clock64() - tc);
                atomicAdd(&g.dbg[8], 1ull);
                atomicAdd(&g.dbg[11], static_cast<unsigned long long>(tb + pb));
            }
        }
        __syncwarp();
    }
}

// The block's rho from the per-task partial sums of the rho queue (task order: deterministic). Lane l
// owns slots l (half 0) and 32 + l (half 1); the slots go through the (now idle) Phi rows so each group
// of 4 lanes stores 4 consecutive k in C order -- 32-byte segments instead of the octet layout's 16 (HBM
// sectors; PCIe writes when rho is mapped host memory). The next block's bulk copy rewrites those rows.
__device__ void rho_block_store(const GridArgs& g, const Smem& sm, int ntask, int bi, int bj, int bk, double* out,
                                int lane) {
    double r[kMaxSpin][2];
#pragma unroll
    for (int spin = 0; spin < kMaxSpin; ++spin) {
        r[spin][0] = r[spin][1] = 0.0;
        if (spin >= g.nspin) continue;
        const double* res = sm.acc() + static_cast<size_t>(spin) * ntask * 32;
        for (int e = 0; e < ntask; ++e) {
            const double v = res[e * 32 + lane];
            if (sm.task()[e].half)
                r[spin][1] += v;
            else
                r[spin][0] += v;
        }
    }
    double* tmp = sm.phi();
    __syncwarp();
#pragma unroll
    for (int spin = 0; spin < kMaxSpin; ++spin) {
        tmp[spin * 64 + lane] = r[spin][0];
        tmp[spin * 64 + 32 + lane] = r[spin][1];
    }
    __syncwarp();
    const int lj = (lane >> 2) & 3, lk = lane & 3;
    const int j = bj * 4 + lj, kk = bk * 4 + lk;
    for (int hh = 0; hh < 2; ++hh) {
        const int li = 2 * hh + (lane >> 4);
        const int slot = ((((li >> 1) << 2) | ((lj >> 1) << 1) | (lk >> 1)) << 3) | ((li & 1) << 2) |
                         ((lj & 1) << 1) | (lk & 1);
        const int i = bi * 4 + li;
        if (i < g.sys.N[0] && j < g.sys.N[1] && kk < g.sys.N[2]) {
            const int64_t pt = (static_cast<int64_t>(i) * g.sys.N[1] + j) * g.sys.N[2] + kk;
            for (int spin = 0; spin < g.nspin; ++spin) out[spin * g.npts + pt] = tmp[spin * 64 + slot];
        }
    }
    __syncwarp();
}

template <bool DENSITY, bool DET, bool SPARSE>
__device__ void consumer(const GridArgs& g, const Buffers<DENSITY>& B, int cw, int lane) {
    constexpr int NC = Cfg<DENSITY>::NC;
    unsigned long long t_wait = 0, t_tail = 0, t0 = clock64();
    for (int k = 0;; ++k) {
        const int s = k & 1;
        const unsigned long long tw = clock64();
        mbar_wait(&B.full[s], (k >> 1) & 1);
        const unsigned long long dw = clock64() - tw;
        t_wait += dw;
        if (KBG_EXPERIMENTS && g.dbg && k < 2 && lane == 0) atomicAdd(&g.dbg[6], dw);
        const Smem sm = B.buf(s);
        const int64_t b = sm.meta()->block;
        if (b < 0) {
            t_tail += dw;
            if (KBG_EXPERIMENTS && g.dbg && lane == 0) {
                atomicAdd(&g.dbg[2], t_wait);
                atomicAdd(&g.dbg[3], t_tail);
                atomicAdd(&g.dbg[4], clock64() - t0);
                atomicAdd(&g.dbg[5], static_cast<unsigned long long>(k));
            }
            return;
        }
        const int ncov = sm.meta()->ncov;
        const int ntask = sm.wptr()[1];
        if (g.task_warps == 1) {
            // task queue, heaviest first: (spin, task) pairs pulled one at a time
            for (;;) {
                int q = 0;
                if (lane == 0) q = atomicAdd(&sm.meta()->next, 1);
                q = __shfl_sync(0xffffffffu, q, 0);
                if (q >= g.nspin * ntask) break;
                const int spin = q >= ntask, e = q - spin * ntask;
                const Task t = sm.task()[e];
                if (DENSITY) {
                    // partial sums of this task's octet half, at its own slot
                    double* res = sm.acc() + static_cast<size_t>(q) * 32;
                    res[lane] = 0.0;
                    __syncwarp();
                    rho_task(sm, ncov, t, g.dmr + spin * g.nrep, res - 32 * t.half, lane);
                } else {
                    // timing experiment (KBG_EXPERIMENTS builds, KBG_DFMA_WARPS): the last consumer warps
                    // run every task they pull on the FP64 FMA pipe, next to the DMMA warps
                    const bool dfma_warp = KBG_EXPERIMENTS && SPARSE && cw >= NC - ((g.scatter >> 16) & 0xFF);
                    h_task<DET, SPARSE>(sm, sm.acc() + spin * 64, ncov, t, g.out + spin * g.nnz * (DET ? 2 : 1), g.scatter,
                                        lane, dfma_warp);
                }
            }
        } else
        for (int spin = 0; spin < g.nspin; ++spin) {
            if (DENSITY) {
                const double* Dr = g.dmr + spin * g.nrep;
                double* racc = sm.acc() + (spin * NC + cw) * 64;
                racc[lane] = 0.0;
                racc[lane + 32] = 0.0;
                __syncwarp();
                for (int w = cw; w < g.task_warps; w += NC)
                    for (int e = sm.wptr()[w]; e < sm.wptr()[w + 1]; ++e) rho_task(sm, ncov, sm.task()[e], Dr, racc, lane);
            } else {
                double* Hs = g.out + spin * g.nnz * (DET ? 2 : 1);
                for (int w = cw; w < g.task_warps; w += NC)
                    for (int e = sm.wptr()[w]; e < sm.wptr()[w + 1]; ++e)
                        h_task<DET, SPARSE>(sm, sm.acc() + spin * 64, ncov, sm.task()[e], Hs, g.scatter, lane);
            }
        }
        __syncwarp();
        const unsigned long long t_red = clock64();
        int last = 0;
        if (lane == 0) {
            __threadfence_block();
            last = atomicAdd(&sm.meta()->done, 1) == NC - 1;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
            __threadfence_block();
            if (DENSITY) {
                int bi, bj, bk;
                block_decode(g.sys, b, bi, bj, bk);
                if (g.task_warps == 1) {
                    rho_block_store(g, sm, ntask, bi, bj, bk, g.out, lane);
                } else
                for (int i = lane; i < g.nspin * 64; i += 32) {
                    const int spin = i >> 6, p = i & 63;
                    double r = 0.0;
#pragma unroll
                    for (int w = 0; w < NC; ++w) r += sm.acc()[(spin * NC + w) * 64 + p];
                    bool valid;
                    const int64_t pt = slot_point(g.sys, bi, bj, bk, p, valid);
                    if (valid) g.out[spin * g.npts + pt] = r;
                }
                __syncwarp();
            }
            if (lane == 0) {
                mbar_arrive(&B.empty[s]);
                if (KBG_EXPERIMENTS && g.dbg) atomicAdd(&g.dbg[10], clock64() - t_red);
            }
        }
    }
}

template <bool DENSITY, bool DET, bool SPARSE = false>
__global__ void __launch_bounds__(Cfg<DENSITY>::NT, 1) k_persist(GridArgs g) {
    const Buffers<DENSITY> B = carve_all<DENSITY>(g);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&B.full[s], 1);
            mbar_init(&B.empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (DET) s_hscale = hscale_of(*g.vbits, g.wfac, g.nnz);
    }
    __syncthreads();
    if (warp < kPersistProducers) {
        if (warp == 0) producer<DENSITY, DET>(g, B, lane);
    } else {
        consumer<DENSITY, DET, SPARSE>(g, B, warp - kPersistProducers, lane);
    }
}

// ---- fused rho + H pass ----------------------------------------------------------------
// One persistent kernel for both contractions: a block's Phi is staged once, with the H and the rho
// table images side by side, and the block's rho and H tasks come from one queue, interleaved, so
// the warps of an SM run latency-bound rho tasks and pipe-bound H tasks at the same time. Buffer:
// [H tables | rho tables | w (V dV) | rho per-task sums | Phi], two buffers. Non-deterministic
// FP64-atomic H only; the rho kernel's 19 consumer warps at 96 registers.
struct FusedCfg {
    static constexpr int NC = kPersistConsumersR;
    static constexpr int NT = (kPersistProducers + NC) * 32;
};

struct FusedBuffers {
    Smem sm0;       // H view of buffer 0
    uint32_t T;     // table image bytes: the rho image sits at T
    uint32_t bsz;   // buffer stride
    uint32_t wb;    // bytes of w
    uint64_t* full;
    uint64_t* empty;
    __device__ __forceinline__ Smem h(int s) const {
        Smem x = sm0;
        x.base = static_cast<uint32_t>(s) * bsz;
        return x;
    }
    __device__ __forceinline__ Smem r(int s) const {  // rho view: tables at T, per-task sums after w
        Smem x = sm0;
        x.base = static_cast<uint32_t>(s) * bsz + T;
        x.o_acc = sm0.o_acc - T + wb;
        x.o_phi = sm0.o_phi - T;
        return x;
    }
};

// Host: the fused buffer layout into g.lay (table offsets as one image; acc at 2T; Phi after acc).
__host__ __device__ inline size_t fused_layout(GridArgs& g) {
    size_t off[12];
    const size_t T = tables_layout(g, off);
    const size_t acc = static_cast<size_t>(g.nspin) * 64 + static_cast<size_t>(g.nspin) * g.max_rtasks * 32;
    off[10] = 2 * T;
    off[11] = off[10] + align16(acc * sizeof(double));
    const size_t bytes = off[11] + align16(static_cast<size_t>(g.max_rows) * 64 * sizeof(double));
    for (int i = 0; i < 12; ++i) g.lay[i] = static_cast<uint32_t>(off[i]);
    g.lay[12] = static_cast<uint32_t>(bytes);
    return 2 * align16(bytes) + 64;
}

__device__ __forceinline__ FusedBuffers carve_fused(const GridArgs& g) {
    FusedBuffers B;
    B.sm0 = carve(0u, g);
    B.T = static_cast<uint32_t>(g.tab_bytes);
    B.bsz = (g.lay[12] + 15u) & ~15u;
    B.wb = static_cast<uint32_t>(g.nspin) * 64u * 8u;
    B.full = reinterpret_cast<uint64_t*>(kbg_smem + 2 * B.bsz);
    B.empty = B.full + 2;
    return B;
}

// Next non-empty owned block (-1: none); empty blocks get rho = 0 on the way.
__device__ int64_t next_block_fused(const GridArgs& g, int lane) {
    for (;;) {
        int idx = 0;
        if (lane == 0) idx = atomicAdd(g.counter, 1);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx >= g.norder) return -1;
        const int64_t b = g.order[idx];
        if (g.blk_ptr[b + 1] > g.blk_ptr[b]) return b;
        int bi, bj, bk;
        block_decode(g.sys, b, bi, bj, bk);
        for (int p = lane; p < 64; p += 32) {
            bool valid;
            const int64_t pt = slot_point(g.sys, bi, bj, bk, p, valid);
            if (valid)
                for (int spin = 0; spin < g.nspin; ++spin) g.out2[spin * g.npts + pt] = 0.0;
        }
    }
}

__device__ void producer_fused(const GridArgs& g, const FusedBuffers& B, int lane) {
    uint64_t pol = 0;
#if KBG_L2_HINT
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
    const uint32_t T = B.T;
    auto phi_of = [&](int64_t b, const double*& phi, uint32_t& pb) {
        const int64_t i = b - g.blk_begin;
        phi = g.phis + g.phi_off[i];
        pb = static_cast<uint32_t>((g.phi_off[i + 1] - g.phi_off[i]) * sizeof(double));
    };
    double w_cur[2 * kMaxSpin], w_next[2 * kMaxSpin];
    auto load_w = [&](int64_t b, double (&w)[2 * kMaxSpin]) {
        if (b < 0) return;
        int bi, bj, bk;
        block_decode(g.sys, b, bi, bj, bk);
#pragma unroll
        for (int j = 0; j < 2 * kMaxSpin; ++j) {
            const int i = lane + 32 * j;
            bool valid = false;
            const int64_t pt = slot_point(g.sys, bi, bj, bk, i & 63, valid);
            w[j] = (valid && i < g.nspin * 64) ? g.in[(i >> 6) * g.npts + pt] : 0.0;
        }
    };
    int64_t b_next = next_block_fused(g, lane);
    load_w(b_next, w_next);
    for (int k = 0;; ++k) {
        const int s = k & 1;
        const int64_t b = b_next;
#pragma unroll
        for (int j = 0; j < 2 * kMaxSpin; ++j) w_cur[j] = w_next[j];
        if (b >= 0) {
            b_next = next_block_fused(g, lane);
            load_w(b_next, w_next);
            if (b_next >= 0 && lane == 0) {
                const int64_t i = b_next - g.blk_begin;
                const double* phi;
                uint32_t pb;
                phi_of(b_next, phi, pb);
                prefetch_l2(g.tabs + i * T, T, pol);
                prefetch_l2(g.tabs2 + i * T, T, pol);
                prefetch_l2(phi, pb, pol);
            }
        }
        if (k >= 2) mbar_wait(&B.empty[s], ((k >> 1) - 1) & 1, 256);
        const Smem sh = B.h(s);
        if (b < 0) {
            if (lane == 0) {
                sh.meta()->block = -1;
                mbar_arrive(&B.full[s]);
            }
            return;
        }
        bool fin = true;
#pragma unroll
        for (int j = 0; j < 2 * kMaxSpin; ++j) {
            const int i = lane + 32 * j;
            if (i < g.nspin * 64) sh.acc()[i] = w_cur[j] * (g.dV * g.sign);
            fin = fin && isfinite(w_cur[j]);
        }
        if (!__all_sync(0xffffffffu, fin) && lane == 0 && g.vbits)
            atomicMax(const_cast<unsigned long long*>(g.vbits), 0x7ff8000000000000ull);
        __syncwarp();
        if (lane == 0) {
            const int64_t i = b - g.blk_begin;
            const double* phi;
            uint32_t pb;
            phi_of(b, phi, pb);
            mbar_arrive_tx(&B.full[s], 2 * T + pb);
            bulk_g2s_hint(sh.meta(), g.tabs + i * T, T, &B.full[s], pol);
            bulk_g2s_hint(kbg_smem + sh.base + T, g.tabs2 + i * T, T, &B.full[s], pol);
            bulk_g2s_hint(sh.phi(), phi, pb, &B.full[s], pol);
        }
        __syncwarp();
    }
}

__device__ void consumer_fused(const GridArgs& g, const FusedBuffers& B, int lane) {
    constexpr int NC = FusedCfg::NC;
    for (int k = 0;; ++k) {
        const int s = k & 1;
        mbar_wait(&B.full[s], (k >> 1) & 1);
        const Smem sh = B.h(s), sr = B.r(s);
        const int64_t b = sh.meta()->block;
        if (b < 0) return;
        const int ncov = sh.meta()->ncov;
        const int nh = sh.wptr()[1], nr = sr.wptr()[1];
        const int nht = g.nspin * nh, nrt = g.nspin * nr, m = min(nht, nrt), tot = nht + nrt;
        for (;;) {
            int q = 0;
            if (lane == 0) q = atomicAdd(&sh.meta()->next, 1);
            q = __shfl_sync(0xffffffffu, q, 0);
            if (q >= tot) break;
            // interleaved: rho, H, rho, H, ... while both last, then the longer list's rest
            bool is_rho;
            int e;
            if (q < 2 * m) {
                is_rho = !(q & 1);
                e = q >> 1;
            } else {
                e = q - m;
                is_rho = nrt > nht;
            }
            if (is_rho) {
                const int spin = e >= nr;
                const Task t = sr.task()[e - spin * nr];
                double* res = sr.acc() + static_cast<size_t>(e) * 32;
                res[lane] = 0.0;
                __syncwarp();
                rho_task(sr, ncov, t, g.dmr + spin * g.nrep, res - 32 * t.half, lane);
            } else {
                const int spin = e >= nh;
                const Task t = sh.task()[e - spin * nh];
                h_task<false, false>(sh, sh.acc() + spin * 64, ncov, t, g.out + spin * g.nnz, g.scatter, lane);
            }
        }
        __syncwarp();
        int last = 0;
        if (lane == 0) {
            __threadfence_block();
            last = atomicAdd(&sh.meta()->done, 1) == NC - 1;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
            __threadfence_block();
            int bi, bj, bk;
            block_decode(g.sys, b, bi, bj, bk);
            rho_block_store(g, sr, nr, bi, bj, bk, g.out2, lane);
            if (lane == 0) mbar_arrive(&B.empty[s]);
        }
    }
}

__global__ void __launch_bounds__(FusedCfg::NT, 1) k_fused(GridArgs g) {
    const FusedBuffers B = carve_fused(g);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&B.full[s], 1);
            mbar_init(&B.empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp < kPersistProducers) {
        if (warp == 0) producer_fused(g, B, lane);
    } else {
        consumer_fused(g, B, lane);
    }
}

GridArgs fused_args(const GridArgs& gh, const GridArgs& gr) {
    GridArgs g = gh;
    g.tabs2 = gr.tabs;
    g.out2 = gr.out;
    g.dmr = gr.dmr;
    g.nrep = gr.nrep;
    g.max_rtasks = gr.max_rtasks;
    g.max_tasks = std::max(gh.max_tasks, gr.max_tasks);
    return g;
}

template <class K>
void set_smem(K kernel, size_t bytes) {
    KBG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
}

int launch_persist(const GridArgs& g0, bool density, cudaStream_t st) {
    GridArgs g = g0;
    if (g.norder <= 0) return 0;
    int dev = 0, sms = 0;
    KBG_CUDA(cudaGetDevice(&dev));
    KBG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(sms - g.reserve_sms, g.norder)));
    const size_t smem = persist_bytes(g, density);
    set_layout(g, persist_acc(g, density));
    KBG_CUDA(cudaMemsetAsync(g.counter, 0, sizeof(int), st));
    if (density) {
        set_smem(k_persist<true, false>, smem);
        k_persist<true, false><<<grid, Cfg<true>::NT, smem, st>>>(g);
    } else {
        // deterministic two-limb scatter (KBG_OPT_DETERMINISTIC) x point-exact FP64 path for sparse
        // tasks (KBG_OPT_SPARSE_DFMA): separate instantiations, so the default kernel carries neither
        auto go = [&](auto kernel) {
            set_smem(kernel, smem);
            kernel<<<grid, Cfg<false>::NT, smem, st>>>(g);
        };
        const bool det = g.scatter & 16, sparse = (g.scatter >> 8) != 0;
        if (sparse)
            det ? go(k_persist<false, true, true>) : go(k_persist<false, false, true>);
        else
            det ? go(k_persist<false, true, false>) : go(k_persist<false, false, false>);
    }
    KBG_CUDA(cudaGetLastError());
    return 1;
}

}  // namespace

bool fused_fits(const GridArgs& gh, const GridArgs& gr) {
    if (gh.task_warps != 1 || gr.task_warps != 1 || gh.scatter != 0) return false;
    GridArgs g = fused_args(gh, gr);
    return fused_layout(g) <= 227 * 1024;
}

int launch_fused(const GridArgs& gh, const GridArgs& gr, cudaStream_t st) {
    GridArgs g = fused_args(gh, gr);
    if (g.norder <= 0) return 0;
    const size_t smem = fused_layout(g);
    if (smem > 227 * 1024) return 0;
    int dev = 0, sms = 0;
    KBG_CUDA(cudaGetDevice(&dev));
    KBG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(sms, g.norder)));
    KBG_CUDA(cudaMemsetAsync(g.counter, 0, sizeof(int), st));
    set_smem(k_fused, smem);
    k_fused<<<grid, FusedCfg::NT, smem, st>>>(g);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

bool persist_fits(const GridArgs& g, bool density) { return persist_bytes(g, density) <= 227 * 1024; }
size_t persist_smem(const GridArgs& g, bool density) { return persist_bytes(g, density); }

int launch_density_persist(const GridArgs& g, cudaStream_t st) { return launch_persist(g, true, st); }
int launch_hamiltonian_persist(const GridArgs& g, cudaStream_t st) { return launch_persist(g, false, st); }

}  // namespace kbg
