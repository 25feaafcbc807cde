// Geometry cache for the persistent grid kernels: per owned grid block, the
// orbital values Phi (rows x 64 slots, the kernels' swizzled shared-memory
// layout, + 8 zero tail rows) and the H and rho table images (covers, groups,
// pair offsets, task lists; table_bytes each). Phi depends only on the
// geometry, the grid and the radial tables -- like OpenMX's Orbs_Grid it is
// evaluated once per geometry and reused by every SCF iteration -- so the
// per-pass work is the two contractions; staging a block becomes two TMA bulk
// copies (kb_persist.cu).
#include <cub/cub.cuh>

#include "kb_gridcore.cuh"

namespace kbg {

namespace {

using namespace core;

__global__ void k_phi_count(int64_t b0, int64_t n, const int32_t* __restrict__ rows, const int32_t* __restrict__ blk_ptr,
                            int64_t* cnt) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int64_t b = b0 + i;
    cnt[i] = (blk_ptr[b + 1] > blk_ptr[b]) ? static_cast<int64_t>(rows[b] + 8) * 64 : 0;
}

// Table images (H and rho) of every owned block: stage_block without Phi, so a
// CTA needs only table_bytes of shared memory and many blocks are in flight
// per SM. Thread 0's make_groups is short (<= 64 covers).
__global__ void __launch_bounds__(128) k_build_tables(GridArgs gh, GridArgs gr, unsigned char* htab, unsigned char* rtab) {
    const Smem sm = carve(0u, gh);
    const int64_t i = blockIdx.x;
    const int64_t b = gh.blk_begin + i;
    const int tid = threadIdx.x, nt = blockDim.x;
    auto sync = [] { __syncthreads(); };
    const size_t T = table_bytes(gh);
    stage_block(gh, b, sm, tid, nt, sync, false, 0, false);
    {
        const int4* src = reinterpret_cast<const int4*>(kbg_smem);
        int4* dst = reinterpret_cast<int4*>(htab + i * T);
        for (size_t k = tid; k < T / 16; k += nt) dst[k] = src[k];
    }
    __syncthreads();
    stage_block(gr, b, sm, tid, nt, sync, true, 0, false);
    {
        const int4* src = reinterpret_cast<const int4*>(kbg_smem);
        int4* dst = reinterpret_cast<int4*>(rtab + i * T);
        for (size_t k = tid; k < T / 16; k += nt) dst[k] = src[k];
    }
}

// Phi of the geometry cache (north star (1): radial-table interpolation x real
// solid harmonics per grid block, shared-memory-staged tables, coalesced and
// vectorised HBM stores). Persistent grid; every CTA first stages ALL radial
// tables in shared memory (u, du/dr pairs, as the table array: the cubic-Hermite
// gathers then hit shared memory). One warp per cover (atom image of a block):
// lane l evaluates slots 2l and 2l + 1 and stores each orbital row's two values
// with one 16-byte store, so a warp writes a row's 512 B contiguously (the
// swizzle XOR 4 (row & 3) only permutes 32-byte groups inside the row and keeps
// slots 2l, 2l + 1 adjacent). Covers take their position, mask and first row
// from the block's H table image (k_build_tables); the warp of a block's last
// cover also writes its 8 zero tail rows. Same orbital expressions as
// stage_block (kb_gridcore.cuh).
constexpr int kPhiThreads = 640;

__device__ __forceinline__ void phi_covers(const SysParams& P, const double* __restrict__ tables, int64_t b0,
                                           int64_t c_begin, int64_t c_end, int64_t nblk_end,
                                           const int32_t* __restrict__ blk_ptr, const unsigned char* __restrict__ htab,
                                           int64_t T, uint32_t o_cov, const int64_t* __restrict__ phi_off,
                                           double* phis);

__global__ void __launch_bounds__(kPhiThreads, 1) k_phi_cache(SysParams P, int64_t b0, int64_t c_begin, int64_t c_end,
                                                              int64_t nblk_end, const int32_t* __restrict__ blk_ptr,
                                                              const unsigned char* __restrict__ htab, int64_t T,
                                                              uint32_t o_meta, uint32_t o_cov,
                                                              const int64_t* __restrict__ phi_off, double* phis,
                                                              int64_t ntab_doubles, int smem_tab) {
    extern __shared__ __align__(16) double s_tab[];
    if (smem_tab) {
        const double2* src = reinterpret_cast<const double2*>(P.tables);
        double2* dst = reinterpret_cast<double2*>(s_tab);
        for (int64_t k = threadIdx.x; k < ntab_doubles / 2; k += blockDim.x) dst[k] = src[k];
        __syncthreads();
    }
    if (smem_tab)
        phi_covers(P, s_tab, b0, c_begin, c_end, nblk_end, blk_ptr, htab, T, o_cov, phi_off, phis);
    else
        phi_covers(P, P.tables, b0, c_begin, c_end, nblk_end, blk_ptr, htab, T, o_cov, phi_off, phis);
}

__device__ __forceinline__ void phi_covers(const SysParams& P, const double* __restrict__ tables, int64_t b0,
                                           int64_t c_begin, int64_t c_end, int64_t nblk_end,
                                           const int32_t* __restrict__ blk_ptr, const unsigned char* __restrict__ htab,
                                           int64_t T, uint32_t o_cov, const int64_t* __restrict__ phi_off,
                                           double* phis) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    // one warp per block: the two slots' positions once, then the block's covers
    for (int64_t b = b0 + blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); b < nblk_end;
         b += nwarps) {
        const int first = blk_ptr[b], end = blk_ptr[b + 1];
        if (first == end) continue;
        const unsigned char* img = htab + (b - b0) * T;
        int bi, bj, bk;
        block_decode(P, b, bi, bj, bk);
        double r[2][3];
        slot_pair_pos(P, bi, bj, bk, lane, r);
        double* blk = phis + phi_off[b - b0];
        for (int c = first; c < end; ++c) {
            const CoverS cv = reinterpret_cast<const CoverS*>(img + o_cov)[c - first];
            double* dst = blk + static_cast<int64_t>(cv.row0) * 64;
            phi_slot_pair(P, tables, cv.t, cv.mask, cv.sp, r, lane, [&](int o, double2 v) {
                *reinterpret_cast<double2*>(dst + o * 64 + ((2 * lane) ^ swz(cv.row0 + o))) = v;
            });
            if (c == end - 1) {  // 8 zero tail rows after the block's last cover (DMMA tile overrun)
                double2* tail = reinterpret_cast<double2*>(dst + static_cast<int64_t>(cv.norb) * 64);
                for (int k = lane; k < 8 * 32; k += 32) tail[k] = make_double2(0.0, 0.0);
            }
        }
    }
}

}  // namespace

void free_cache(DevIndex& ix) {
    for (void* p : {static_cast<void*>(ix.htab), static_cast<void*>(ix.rtab), static_cast<void*>(ix.phis),
                    static_cast<void*>(ix.phi_off)})
        if (p) pool_free(p);
    ix.htab = ix.rtab = nullptr;
    ix.phis = nullptr;
    ix.phi_off = nullptr;
    ix.tab_bytes = ix.phi_doubles = 0;
}

void build_cache_device(GridArgs gh, GridArgs gr, DevIndex& ix, cudaStream_t st) {
    free_cache(ix);
    const int64_t b0 = gh.blk_begin, n = ix.norder;  // owned blocks [b0, b0 + n)
    if (n <= 0) return;
    gh.max_tasks = gr.max_tasks = std::max(gh.max_tasks, gr.max_tasks);
    const size_t T = table_bytes(gh);
    int64_t* cnt = nullptr;
    KBG_CUDA(pool_malloc(&cnt, (n + 1) * sizeof(int64_t)));
    KBG_CUDA(pool_malloc(&ix.phi_off, (n + 1) * sizeof(int64_t)));
    KBG_CUDA(cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(int64_t), st));
    k_phi_count<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(b0, n, ix.blk_rows, ix.blk_ptr, cnt);
    KBG_CUDA(cudaGetLastError());
    size_t bytes = 0;
    KBG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, ix.phi_off, static_cast<int>(n + 1), st));
    void* tmp = nullptr;
    KBG_CUDA(pool_malloc(&tmp, std::max<size_t>(bytes, 16)));
    KBG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, ix.phi_off, static_cast<int>(n + 1), st));
    int32_t cov_range[2];
    KBG_CUDA(cudaMemcpyAsync(&ix.phi_doubles, ix.phi_off + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KBG_CUDA(cudaMemcpyAsync(&cov_range[0], ix.blk_ptr + b0, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    KBG_CUDA(cudaMemcpyAsync(&cov_range[1], ix.blk_ptr + b0 + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    KBG_CUDA(cudaStreamSynchronize(st));
    pool_free(tmp);
    pool_free(cnt);
    ix.tab_bytes = static_cast<int64_t>(T);
    KBG_CUDA(pool_malloc(&ix.htab, n * T));
    KBG_CUDA(pool_malloc(&ix.rtab, n * T));
    KBG_CUDA(pool_malloc(&ix.phis, std::max<int64_t>(1, ix.phi_doubles) * sizeof(double)));
    set_layout(gh, 0);
    set_layout(gr, 0);
    // tables only: the Phi and acc sections of the layout are never touched
    const size_t smem_t = std::max<size_t>(T, 16);
    KBG_CUDA(cudaFuncSetAttribute(k_build_tables, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_t)));
    k_build_tables<<<static_cast<unsigned>(n), 128, smem_t, st>>>(gh, gr, ix.htab, ix.rtab);
    KBG_CUDA(cudaGetLastError());
    // Phi: radial tables in shared memory when they fit (all species, 16 B per table point and radial function)
    int64_t ntab = 0;
    for (int t = 0; t < gh.sys.nspecies; ++t)
        ntab = std::max<int64_t>(ntab, gh.sys.sp[t].tab_off + static_cast<int64_t>(gh.sys.sp[t].nrad) * gh.sys.sp[t].ntab * 2);
    ntab = (ntab + 1) & ~int64_t(1);
    const size_t smem_tab = static_cast<size_t>(ntab) * sizeof(double);
    const int use_smem = smem_tab <= 220 * 1024 ? 1 : 0;
    const size_t smem = use_smem ? smem_tab : 0;
    int dev = 0, sms = 0;
    KBG_CUDA(cudaGetDevice(&dev));
    KBG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    KBG_CUDA(cudaFuncSetAttribute(k_phi_cache, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    const int64_t ncov = cov_range[1] - cov_range[0];
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(sms, (ncov + 31) / 32)));
    if (ncov > 0)
        k_phi_cache<<<grid, kPhiThreads, smem, st>>>(gh.sys, b0, cov_range[0], cov_range[1], b0 + n, ix.blk_ptr,
                                                     ix.htab, static_cast<int64_t>(T), gh.lay[0], gh.lay[1],
                                                     ix.phi_off, ix.phis, ntab, use_smem);
    KBG_CUDA(cudaGetLastError());
    KBG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace kbg
