// One-CTA-per-block grid kernels (fallback when the persistent kernels'
// two shared-memory buffers do not fit), plus the small helper kernels:
// DM repack, H mirror, DM symmetry check, block orbitals. The contraction
// core is in kb_gridcore.cuh.
#include "kb_gridcore.cuh"

namespace kbg {

namespace {

using namespace core;

// Tasks of this warp: its LPT lists, or every NW-th task of a single queue
// (task_warps == 1, the persistent kernels' dynamic schedule) -- a fixed
// assignment either way, so rho stays deterministic.
template <int NW, class F>
__device__ __forceinline__ void for_warp_tasks(const GridArgs& g, const Smem& sm, int warp, F&& f) {
    if (g.task_warps == 1) {
        for (int e = warp; e < sm.wptr()[1]; e += NW) f(e);
    } else {
        for (int w = warp; w < g.task_warps; w += NW)
            for (int e = sm.wptr()[w]; e < sm.wptr()[w + 1]; ++e) f(e);
    }
}

template <int NW, bool DET>
__global__ void __launch_bounds__(NW * 32, 2) k_hamiltonian(GridArgs g) {
    const Smem sm = carve(0u, g);
    const int64_t b = g.blk_begin + blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (DET && tid == 0) s_hscale = hscale_of(*g.vbits, g.wfac, g.nnz);  // stage_block syncs
    const int ncov = stage_block(g, b, sm, tid, NW * 32, [] { __syncthreads(); }, false, NW);
    if (ncov == 0) return;
    for (int spin = 0; spin < g.nspin; ++spin) {
        double* Hs = g.out + spin * g.nnz * (DET ? 2 : 1);
        for_warp_tasks<NW>(g, sm, warp,
                           [&](int e) { h_task<DET, true>(sm, sm.acc() + spin * 64, ncov, sm.task()[e], Hs, g.scatter, lane); });
    }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 2) k_density(GridArgs g) {
    const Smem sm = carve(0u, g);
    const int64_t b = g.blk_begin + blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int bi, bj, bk;
    block_decode(g.sys, b, bi, bj, bk);
    const int ncov = stage_block(g, b, sm, tid, NW * 32, [] { __syncthreads(); }, true, NW);
    if (ncov > 0) {
        for (int spin = 0; spin < g.nspin; ++spin) {
            const double* Dr = g.dmr + spin * g.nrep;
            double* racc = sm.acc() + (spin * NW + warp) * 64;
            for_warp_tasks<NW>(g, sm, warp, [&](int e) { rho_task(sm, ncov, sm.task()[e], Dr, racc, lane); });
        }
        __syncthreads();
    }
    for (int i = tid; i < g.nspin * 64; i += NW * 32) {
        const int spin = i >> 6, p = i & 63;
        double r = 0.0;
        if (ncov > 0)
#pragma unroll
            for (int w = 0; w < NW; ++w) r += sm.acc()[(spin * NW + w) * 64 + p];
        bool valid;
        const int64_t pt = slot_point(g.sys, bi, bj, bk, p, valid);
        if (valid) g.out[spin * g.npts + pt] = r;
    }
}

// Repacked, pre-scaled DM for the rho kernels (see kb_gridcore.cuh gather_a):
// canonical pairs only; row i of pair p at roff[p] + i * 16 * ceil(nb/16);
// column j = 16c + 4s + k stored at position 16c + 4k + s; x2 except (a,a,0).
// With chk != nullptr the same pass validates the DensityMatrices invariant
// DM_ba(-R) = DM_ab(R)^T (what k_dm_check does): per canonical
// pair it compares the block with its mirror block and reduces max|defect|,
// max|DM| and a non-finite flag into chk[0..2] (one atomic per CTA).
__global__ void k_dm_repack(SysParams P, int64_t npair, int nspin, int64_t nnz, int64_t nrep,
                            const int32_t* __restrict__ pa, const int32_t* __restrict__ pb,
                            const int32_t* __restrict__ pR, const int64_t* __restrict__ poff,
                            const int64_t* __restrict__ proff, const int32_t* __restrict__ mirror,
                            const double* __restrict__ dm, double* __restrict__ dmr, unsigned long long* chk,
                            const uint8_t* __restrict__ own) {
    const int lane = threadIdx.x & 31;
    const int64_t p = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    double dmax = 0.0, amax = 0.0;
    bool finite = true;
    bool canon = false;
    int a = 0, b = 0, R0 = 0, R1 = 0, R2 = 0;
    if (p < npair) {
        a = pa[p];
        b = pb[p];
        R0 = pR[3 * p];
        R1 = pR[3 * p + 1];
        R2 = pR[3 * p + 2];
        canon = (a != b) ? a < b : (R0 != 0 ? R0 > 0 : (R1 != 0 ? R1 > 0 : R2 >= 0));
        // shard-local input (kbg_grid_pass on a sharded context): only the pairs this rank's blocks
        // touch are read (dm may be mapped host memory); the others are never used by its rho kernel
        if (own && !own[p]) canon = false;
    }
    const bool chk_p = chk && (!own || (p < npair && (own[p] & 2)));
    if (canon) {
        const double fac = (a == b && R0 == 0 && R1 == 0 && R2 == 0) ? 1.0 : 2.0;
        const int na = P.sp[P.spc[a]].norb, nb = P.sp[P.spc[b]].norb;
        const int stride = 16 * ((nb + 15) >> 4);
        const int64_t q = chk_p ? mirror[p] : p;
        for (int s = 0; s < nspin; ++s) {
            const double* src = dm + s * nnz + poff[p];
            const double* srq = dm + s * nnz + poff[q];  // nb x na
            double* dst = dmr + s * nrep + proff[p];
            // unrolled so several loads per lane are in flight (a pair block is only a few
            // iterations; a rolled loop pays the full load latency each time)
#pragma unroll 4
            for (int e = lane; e < na * stride; e += 32) {
                const int i = e / stride, pos = e % stride;
                const int c = pos >> 4, k = (pos >> 2) & 3, st = pos & 3;
                const int j = 16 * c + 4 * st + k;
                const double v = j < nb ? src[i * nb + j] : 0.0;
                dst[e] = fac * v;
                if (chk_p && j < nb) {
                    const double y = srq[j * na + i];
                    finite &= isfinite(v) && isfinite(y);
                    dmax = fmax(dmax, fabs(v - y));
                    amax = fmax(amax, fmax(fabs(v), fabs(y)));
                }
            }
        }
    }
    if (!chk) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    finite = __all_sync(0xffffffffu, finite);
    __shared__ double s_d[32], s_a[32];
    __shared__ int s_f;
    if (threadIdx.x == 0) s_f = 1;
    __syncthreads();
    if (lane == 0) {
        s_d[threadIdx.x >> 5] = dmax;
        s_a[threadIdx.x >> 5] = amax;
        if (!finite) s_f = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) {
            dmax = fmax(dmax, s_d[k]);
            amax = fmax(amax, s_a[k]);
        }
        atomicMax(chk, static_cast<unsigned long long>(__double_as_longlong(dmax)));
        atomicMax(chk + 1, static_cast<unsigned long long>(__double_as_longlong(amax)));
        if (!s_f) atomicMax(chk + 2, 1ull);
    }
}

#ifndef KBG_REPACK_LIST
#define KBG_REPACK_LIST 1
#endif
// The same repack over the canonical-pair work list (kb_index.cu k_repack_items): one warp per
// item, metadata in one load; for nb <= 16 (one 16-column chunk) lane l always handles repacked
// column l & 15 and rows (l >> 4) + 2k, all loads of an item issued up front.
template <bool CHK>
__global__ void __launch_bounds__(256) k_dm_repack_list(const RepackItem* __restrict__ items,
                                                        const int* __restrict__ count, int nspin, int64_t nnz,
                                                        int64_t nrep, const double* __restrict__ dm,
                                                        double* __restrict__ dmr, unsigned long long* chk,
                                                        const uint8_t* __restrict__ own) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    double dmax = 0.0, amax = 0.0;
    bool finite = true;
    if (w < *count) {
        const RepackItem it = items[w];
        if (!own || own[it.p]) {
            // a shard checks only the pairs it is assigned (own bit 1; it alone holds their mirror blocks)
            const bool chk_p = CHK && (!own || (own[it.p] & 2));
            const double fac = it.fac2 ? 2.0 : 1.0;
            const int na = it.na, nb = it.nb;
            for (int s = 0; s < nspin; ++s) {
                const double* src = dm + s * nnz + it.src;
                const double* srq = dm + s * nnz + it.srq;  // nb x na
                double* dst = dmr + s * nrep + it.dst;
                if (nb <= 16 && na <= 16) {
                    const int pos = lane & 15, i0 = lane >> 4;
                    const int j = 4 * (pos & 3) + ((pos >> 2) & 3);  // column stored at pos
                    double v[8], y[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int i = i0 + 2 * k;
                        v[k] = (i < na && j < nb) ? src[i * nb + j] : 0.0;
                        y[k] = (chk_p && i < na && j < nb) ? srq[j * na + i] : 0.0;
                    }
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int i = i0 + 2 * k;
                        if (i < na) dst[i * 16 + pos] = fac * v[k];
                        if (chk_p && i < na && j < nb) {
                            finite &= isfinite(v[k]) && isfinite(y[k]);
                            dmax = fmax(dmax, fabs(v[k] - y[k]));
                            amax = fmax(amax, fmax(fabs(v[k]), fabs(y[k])));
                        }
                    }
                } else {
                    const int stride = 16 * ((nb + 15) >> 4);
                    for (int e = lane; e < na * stride; e += 32) {
                        const int i = e / stride, pos = e % stride;
                        const int c = pos >> 4, k = (pos >> 2) & 3, st = pos & 3;
                        const int j = 16 * c + 4 * st + k;
                        const double v = j < nb ? src[i * nb + j] : 0.0;
                        dst[e] = fac * v;
                        if (chk_p && j < nb) {
                            const double y = srq[j * na + i];
                            finite &= isfinite(v) && isfinite(y);
                            dmax = fmax(dmax, fabs(v - y));
                            amax = fmax(amax, fmax(fabs(v), fabs(y)));
                        }
                    }
                }
            }
        }
    }
    if (!CHK) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    finite = __all_sync(0xffffffffu, finite);
    __shared__ double s_d[8], s_a[8];
    __shared__ int s_f;
    if (threadIdx.x == 0) s_f = 1;
    __syncthreads();
    if (lane == 0) {
        s_d[threadIdx.x >> 5] = dmax;
        s_a[threadIdx.x >> 5] = amax;
        if (!finite) s_f = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < 8; ++k) {
            dmax = fmax(dmax, s_d[k]);
            amax = fmax(amax, s_a[k]);
        }
        atomicMax(chk, static_cast<unsigned long long>(__double_as_longlong(dmax)));
        atomicMax(chk + 1, static_cast<unsigned long long>(__double_as_longlong(amax)));
        if (!s_f) atomicMax(chk + 2, 1ull);
    }
}

// Shard-local DM input (kbg_grid_pass on a sharded context, DM in pinned host memory): the exact
// [off, len) runs of the pair blocks this rank reads, gathered in place over PCIe into the device
// copy at the same offsets. One warp per run, 8 coalesced loads per lane in flight. Launched on 2
// CTAs ahead of the H kernel (which leaves them their SMs): the fetch overlaps the H pass without a
// copy per run and without the bytes between the runs.
__global__ void __launch_bounds__(1024) k_dm_gather(const int64_t* __restrict__ runs, int64_t nruns, int nspin,
                                                    int64_t nnz, const double* src,
                                                    double* __restrict__ dst) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int s = 0; s < nspin; ++s)
        for (int64_t r = warp; r < nruns; r += nw) {
            const int64_t o = s * nnz + runs[2 * r], n = runs[2 * r + 1];
            for (int64_t e = lane; e < n; e += 32 * 8) {
                double v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    v[k] = 0.0;
                    // plain (coherent) global load: the read-only path does not serve host memory
                    if (e + 32 * k < n) asm volatile("ld.global.f64 %0, [%1];" : "=d"(v[k]) : "l"(src + o + e + 32 * k));
                }
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (e + 32 * k < n) dst[o + e + 32 * k] = v[k];
            }
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
#pragma unroll 4
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
#pragma unroll 4
        for (int e = lane; e < na * nb; e += 32) {
            const int i = e / nb, j = e % nb;
            dst[e] = src[j * na + i];
        }
    }
}

// Mirror over the work list (one warp per item, kb_index.cu k_mirror_items): blocks of <= 16 x 16
// orbitals as two rows per pass, lane = (row parity, column), all loads of an item issued up front;
// the same expressions as k_mirror (bitwise identical result).
__global__ void __launch_bounds__(256) k_mirror_list(const MirrorItem* __restrict__ items,
                                                     const int* __restrict__ count, int nspin, int64_t nnz,
                                                     double* h) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= *count) return;
    const MirrorItem it = items[w];
    const int na = it.na, nb = it.nb;
    const int j = lane & 15, i0 = lane >> 4;
    for (int s = 0; s < nspin; ++s) {
        double* x = h + s * nnz;
        if (it.dst == it.src) {  // (a, a, 0): (H + H^T) / 2 on i < j
            if (na <= 16) {
                double u[8], v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int i = i0 + 2 * k;
                    const bool on = i < j && j < na;
                    u[k] = on ? x[it.dst + i * na + j] : 0.0;
                    v[k] = on ? x[it.dst + j * na + i] : 0.0;
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int i = i0 + 2 * k;
                    if (i < j && j < na) {
                        const double m = 0.5 * (u[k] + v[k]);
                        x[it.dst + i * na + j] = m;
                        x[it.dst + j * na + i] = m;
                    }
                }
            } else {
                for (int e = lane; e < na * na; e += 32) {
                    const int i = e / na, jj = e % na;
                    if (i < jj) {
                        const double m = 0.5 * (x[it.dst + i * na + jj] + x[it.dst + jj * na + i]);
                        x[it.dst + i * na + jj] = m;
                        x[it.dst + jj * na + i] = m;
                    }
                }
            }
        } else if (na <= 16 && nb <= 16) {  // dst(i, j) = src(j, i)
            double u[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = i0 + 2 * k;
                u[k] = (i < na && j < nb) ? x[it.src + j * na + i] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = i0 + 2 * k;
                if (i < na && j < nb) x[it.dst + i * nb + j] = u[k];
            }
        } else {
            for (int e = lane; e < na * nb; e += 32) {
                const int i = e / nb, jj = e % nb;
                x[it.dst + e] = x[it.src + jj * na + i];
            }
        }
    }
}

// ---- deterministic H: max|V| and the final rounding (kb_gridcore.cuh h_scatter) ---
// max|x| over n doubles as the bit pattern of |x| (sign cleared): non-negative
// doubles order like their bits, and NaN > inf > finite, so a non-finite input
// shows up as a maximum above the largest finite double. Order-independent.
__global__ void __launch_bounds__(256) k_absmax(const double* __restrict__ x, int64_t n,
                                                unsigned long long* __restrict__ out) {
    unsigned long long m = 0;
    const int64_t n2 = n >> 1;
    const double2* x2 = reinterpret_cast<const double2*>(x);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n2;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double2 v = x2[i];
        m = max(m, static_cast<unsigned long long>(__double_as_longlong(v.x)) & 0x7fffffffffffffffull);
        m = max(m, static_cast<unsigned long long>(__double_as_longlong(v.y)) & 0x7fffffffffffffffull);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1))
        m = max(m, static_cast<unsigned long long>(__double_as_longlong(x[n - 1])) & 0x7fffffffffffffffull);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// H = hi + lo of the two-limb accumulator (det_hi / det_lo layout), one warp
// per pair. mirror = 0: canonical pair blocks get H, the others 0 (the layout
// kbg_hamiltonian_accumulate_dev returns). mirror = 1: also the mirror blocks
// H_ba(-R) = H_ab(R)^T, and the (a, a, 0) blocks re-symmetrised as
// (H + H^T)/2 -- the same expression as k_mirror and kb_comm.cu's reduction,
// so the result has the same bits on any number of GPUs.
__global__ void k_finalize(SysParams P, int64_t npair, int nspin, int64_t nnz, const int32_t* __restrict__ pa,
                           const int32_t* __restrict__ pb, const int32_t* __restrict__ pR,
                           const int64_t* __restrict__ poff, const int32_t* __restrict__ mirror,
                           const double* __restrict__ acc, double* __restrict__ h, int do_mirror, int limbs) {
    const int lane = threadIdx.x & 31;
    const int64_t p = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (p >= npair) return;
    const int a = pa[p], b = pb[p];
    const int R0 = pR[3 * p], R1 = pR[3 * p + 1], R2 = pR[3 * p + 2];
    const bool canon = (a != b) ? a < b : (R0 != 0 ? R0 > 0 : (R1 != 0 ? R1 > 0 : R2 >= 0));
    const int na = P.sp[P.spc[a]].norb, nb = P.sp[P.spc[b]].norb;
    const int64_t q = mirror[p];
    for (int s = 0; s < nspin; ++s) {
        const int64_t o = poff[p];
        auto val = [&](int e) {
            return limbs == 1 ? acc[s * nnz + o + e] : acc[det_hi(s, o + e, nnz)] + acc[det_lo(s, o + e, nnz)];
        };
        double* dst = h + s * nnz + o;
        if (!canon) {
            if (!do_mirror)
                for (int e = lane; e < na * nb; e += 32) dst[e] = 0.0;
            continue;
        }
        if (q == p && do_mirror) {
#pragma unroll 4
            for (int e = lane; e < na * na; e += 32) {
                const int i = e / na, j = e % na;
                const double v = val(e);
                if (i == j) {
                    dst[e] = v;
                } else {
                    const double w = val(j * na + i);
                    dst[e] = i < j ? 0.5 * (v + w) : 0.5 * (w + v);
                }
            }
            continue;
        }
        double* dq = h + s * nnz + poff[q];
#pragma unroll 4
        for (int e = lane; e < na * nb; e += 32) {
            const double v = val(e);
            dst[e] = v;
            if (do_mirror && q != p) dq[(e % nb) * na + e / nb] = v;
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
    double dmax = 0.0, amax = 0.0;
    bool finite = true;
    const bool live = p < npair;
    const int na = live ? P.sp[P.spc[pa[p]]].norb : 0, nb = live ? P.sp[P.spc[pb[p]]].norb : 0;
    const int64_t q = live ? mirror[p] : 0;
    for (int s = 0; s < nspin && live; ++s) {
        const double* x = dm + s * nnz + poff[p];
        const double* y = dm + s * nnz + poff[q];
#pragma unroll 4
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
    // one atomic per CTA (not per warp: thousands of warps on the same two words serialize in L2)
    __shared__ double s_d[32], s_a[32];
    __shared__ int s_f;
    if (threadIdx.x == 0) s_f = 1;
    __syncthreads();
    const int w = threadIdx.x >> 5;
    if (lane == 0) {
        s_d[w] = dmax;
        s_a[w] = amax;
        if (!finite) s_f = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) {
            dmax = fmax(dmax, s_d[k]);
            amax = fmax(amax, s_a[k]);
        }
        atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(dmax)));
        atomicMax(out + 1, static_cast<unsigned long long>(__double_as_longlong(amax)));
        if (!s_f) atomicMax(out + 2, 1ull);
    }
}

__global__ void k_block_orbitals(GridArgs g, int64_t b, double* out) {
    const Smem sm = carve(0u, g);
    const int ncov = stage_block(g, b, sm, threadIdx.x, blockDim.x, [] { __syncthreads(); }, false, 1);
    // rows in cover order
    int r0 = 0;
    for (int c = 0; c < ncov; ++c) {
        const CoverS& cv = sm.cov()[c];
        for (int i = threadIdx.x; i < cv.norb * 64; i += blockDim.x)
            out[static_cast<size_t>(r0) * 64 + i] = sm.phi()[phi_idx(cv.row0 + (i >> 6), i & 63)];
        r0 += cv.norb;
    }
}

template <class K>
void set_smem(K kernel, size_t bytes) {
    KBG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
}

}  // namespace

size_t grid_smem_bytes(const GridArgs& g, int nwarps, bool density) {
    size_t off[12];
    return core::buffer_layout(g, static_cast<size_t>(g.nspin) * 64 * (density ? nwarps : 1), off);
}

int launch_density(const GridArgs& g0, int64_t nblk, int nwarps, cudaStream_t st) {
    if (nblk <= 0) return 0;
    GridArgs g = g0;
    const size_t smem = grid_smem_bytes(g, nwarps, true);
    set_layout(g, static_cast<size_t>(g.nspin) * 64 * nwarps);
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

int launch_hamiltonian(const GridArgs& g0, int64_t nblk, int nwarps, cudaStream_t st) {
    if (nblk <= 0) return 0;
    GridArgs g = g0;
    const size_t smem = grid_smem_bytes(g, nwarps, false);
    set_layout(g, static_cast<size_t>(g.nspin) * 64);
    const bool det = g.scatter & 16;  // deterministic two-limb scatter (KBG_OPT_DETERMINISTIC)
    auto go = [&](auto kernel, int threads) {
        set_smem(kernel, smem);
        kernel<<<static_cast<unsigned>(nblk), threads, smem, st>>>(g);
    };
    if (nwarps == 4)
        det ? go(k_hamiltonian<4, true>, 128) : go(k_hamiltonian<4, false>, 128);
    else
        det ? go(k_hamiltonian<8, true>, 256) : go(k_hamiltonian<8, false>, 256);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

int launch_dm_gather(const int64_t* d_runs, int64_t nruns, int nspin, int64_t nnz, const double* src, double* dst,
                     cudaStream_t st) {
    if (nruns <= 0) return 0;
    k_dm_gather<<<2, 1024, 0, st>>>(d_runs, nruns, nspin, nnz, src, dst);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(KBG_ERR_CUDA, std::string("k_dm_gather: ") + cudaGetErrorString(e));
    return 1;
}

int launch_mirror(const DevIndex& ix, const SysParams& sys, int nspin, double* h, cudaStream_t st) {
    if (ix.npair == 0) return 0;
    if (ix.mir && ix.nmir > 0) {
        const unsigned grid = static_cast<unsigned>((ix.nmir * 32 + 255) / 256);
        k_mirror_list<<<grid, 256, 0, st>>>(ix.mir, ix.mir_count, nspin, ix.nnz, h);
        KBG_CUDA(cudaGetLastError());
        return 1;
    }
    const unsigned grid = static_cast<unsigned>((ix.npair * 32 + 255) / 256);
    k_mirror<<<grid, 256, 0, st>>>(sys, ix.npair, nspin, ix.nnz, ix.pair_a, ix.pair_b, ix.pair_R, ix.pair_off,
                                   ix.pair_mirror, h);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

int launch_absmax(const double* d_x, int64_t n, unsigned long long* d_out, cudaStream_t st) {
    if (n <= 0) return 0;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(148 * 4, (n / 2 + 255) / 256 + 1));
    k_absmax<<<grid, 256, 0, st>>>(d_x, n, d_out);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

int launch_finalize(const DevIndex& ix, const SysParams& sys, int nspin, const double* acc, double* h, bool mirror,
                    cudaStream_t st, int limbs) {
    if (ix.npair == 0) return 0;
    const unsigned grid = static_cast<unsigned>((ix.npair * 32 + 255) / 256);
    k_finalize<<<grid, 256, 0, st>>>(sys, ix.npair, nspin, ix.nnz, ix.pair_a, ix.pair_b, ix.pair_R, ix.pair_off,
                                     ix.pair_mirror, acc, h, mirror ? 1 : 0, limbs);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

int launch_dm_repack(const DevIndex& ix, const SysParams& sys, int nspin, const double* dm, double* dmr,
                     cudaStream_t st, unsigned long long* chk, const uint8_t* own) {
    if (ix.npair == 0) return 0;
    if (KBG_REPACK_LIST && ix.rep && ix.nrep_items > 0) {
        const unsigned g = static_cast<unsigned>((ix.nrep_items * 32 + 255) / 256);
        if (chk)
            k_dm_repack_list<true><<<g, 256, 0, st>>>(ix.rep, ix.mir_count + 1, nspin, ix.nnz, ix.nrep, dm, dmr, chk,
                                                      own);
        else
            k_dm_repack_list<false><<<g, 256, 0, st>>>(ix.rep, ix.mir_count + 1, nspin, ix.nnz, ix.nrep, dm, dmr,
                                                       chk, own);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw Error(KBG_ERR_CUDA, std::string("k_dm_repack_list: ") + cudaGetErrorString(e));
        return 1;
    }
    const unsigned grid = static_cast<unsigned>((ix.npair * 32 + 255) / 256);
    k_dm_repack<<<grid, 256, 0, st>>>(sys, ix.npair, nspin, ix.nnz, ix.nrep, ix.pair_a, ix.pair_b, ix.pair_R,
                                      ix.pair_off, ix.pair_roff, ix.pair_mirror, dm, dmr, chk, own);
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

int launch_block_orbitals(const GridArgs& g0, int64_t block, double* d_out, cudaStream_t st) {
    GridArgs g = g0;
    const size_t smem = grid_smem_bytes(g, 1, false);
    set_layout(g, static_cast<size_t>(g.nspin) * 64);
    set_smem(k_block_orbitals, smem);
    k_block_orbitals<<<1, 256, smem, st>>>(g, block, d_out);
    KBG_CUDA(cudaGetLastError());
    return 1;
}

}  // namespace kbg
