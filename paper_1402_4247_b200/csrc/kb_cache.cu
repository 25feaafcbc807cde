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

__global__ void __launch_bounds__(256) k_build_cache(GridArgs gh, GridArgs gr, const int64_t* __restrict__ phi_off,
                                                     unsigned char* htab, unsigned char* rtab, double* phis) {
    const Smem sm = carve(0u, gh);
    const int64_t i = blockIdx.x;
    const int64_t b = gh.blk_begin + i;
    const int tid = threadIdx.x, nt = blockDim.x;
    auto sync = [] { __syncthreads(); };
    const size_t T = table_bytes(gh);
    const int ncov = stage_block(gh, b, sm, tid, nt, sync, false, 0, true);
    {
        const int4* src = reinterpret_cast<const int4*>(kbg_smem);
        int4* dst = reinterpret_cast<int4*>(htab + i * T);
        for (size_t k = tid; k < T / 16; k += nt) dst[k] = src[k];
    }
    if (ncov > 0) {
        const int64_t n = static_cast<int64_t>(sm.meta()->rows + 8) * 64;
        double* dst = phis + phi_off[i];
        for (int64_t k = tid; k < n; k += nt) dst[k] = sm.phi()[k];
    }
    __syncthreads();
    stage_block(gr, b, sm, tid, nt, sync, true, 0, false);
    {
        const int4* src = reinterpret_cast<const int4*>(kbg_smem);
        int4* dst = reinterpret_cast<int4*>(rtab + i * T);
        for (size_t k = tid; k < T / 16; k += nt) dst[k] = src[k];
    }
}

}  // namespace

void free_cache(DevIndex& ix) {
    for (void* p : {static_cast<void*>(ix.htab), static_cast<void*>(ix.rtab), static_cast<void*>(ix.phis),
                    static_cast<void*>(ix.phi_off)})
        if (p) cudaFree(p);
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
    KBG_CUDA(cudaMalloc(&cnt, (n + 1) * sizeof(int64_t)));
    KBG_CUDA(cudaMalloc(&ix.phi_off, (n + 1) * sizeof(int64_t)));
    KBG_CUDA(cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(int64_t), st));
    k_phi_count<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(b0, n, ix.blk_rows, ix.blk_ptr, cnt);
    KBG_CUDA(cudaGetLastError());
    size_t bytes = 0;
    KBG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, ix.phi_off, static_cast<int>(n + 1), st));
    void* tmp = nullptr;
    KBG_CUDA(cudaMalloc(&tmp, std::max<size_t>(bytes, 16)));
    KBG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, ix.phi_off, static_cast<int>(n + 1), st));
    KBG_CUDA(cudaMemcpyAsync(&ix.phi_doubles, ix.phi_off + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KBG_CUDA(cudaStreamSynchronize(st));
    cudaFree(tmp);
    cudaFree(cnt);
    ix.tab_bytes = static_cast<int64_t>(T);
    KBG_CUDA(cudaMalloc(&ix.htab, n * T));
    KBG_CUDA(cudaMalloc(&ix.rtab, n * T));
    KBG_CUDA(cudaMalloc(&ix.phis, std::max<int64_t>(1, ix.phi_doubles) * sizeof(double)));
    set_layout(gh, 0);
    set_layout(gr, 0);
    const size_t smem = gh.lay[12];
    KBG_CUDA(cudaFuncSetAttribute(k_build_cache, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_build_cache<<<static_cast<unsigned>(n), 256, smem, st>>>(gh, gr, ix.phi_off, ix.htab, ix.rtab, ix.phis);
    KBG_CUDA(cudaGetLastError());
    KBG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace kbg
