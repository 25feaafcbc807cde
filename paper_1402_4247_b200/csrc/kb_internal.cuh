// Internal declarations of libkbgrid (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "kbgrid.h"

namespace kbg {

constexpr int kMaxSpecies = 8;
constexpr int kMaxRad = 16;
constexpr int kMaxSpin = 2;  // nspin is 1 or 2 (check_nspin)
// Two-limb H accumulator of the deterministic scatter (kb_gridcore.cuh h_scatter):
// KBG_DET_SPLIT 1 = [nspin][2][nnz] (per spin the hi limbs, then the lo limbs: a
// warp's RED of one limb touches as many L2 sectors as a plain FP64 scatter),
// 0 = [nspin][nnz][2] interleaved.
#ifndef KBG_DET_SPLIT
#define KBG_DET_SPLIT 1
#endif
__host__ __device__ __forceinline__ int64_t det_hi(int s, int64_t e, int64_t nnz) {
    return KBG_DET_SPLIT ? 2 * s * nnz + e : 2 * (s * nnz + e);
}
__host__ __device__ __forceinline__ int64_t det_lo(int s, int64_t e, int64_t nnz) {
    return KBG_DET_SPLIT ? 2 * s * nnz + nnz + e : 2 * (s * nnz + e) + 1;
}
constexpr int kGroupRows = 16;  // covers are packed into row groups of <= 16 orbitals (2 DMMA row tiles)
constexpr int kMaxTaskWarps = 32;  // task lists are LPT-balanced over <= 24 consumer warps
// Timing-experiment paths (KBG_OPT_SCATTER_STORE bits, KBG_OPT_DEBUG_COUNTERS, KBG_DFMA_WARPS) exist only
// in builds with -DKBG_EXPERIMENTS=1 (tools/build_variants.sh): the product kernels carry no runtime checks.
#ifndef KBG_EXPERIMENTS
#define KBG_EXPERIMENTS 0
#endif

constexpr int kMaxCoverPerBlock = 64;
constexpr int kRhoOct = 4;  // octets per rho task (4: halves of the block, 2: quarters; halves measured faster)

// Error taxonomy of kband (common.hpp:21-38) carried as a status code.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define KBG_CUDA(call)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            throw ::kbg::Error(KBG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct DevSpecies {
    int nrad;
    int norb;
    int ntab;
    int pad_;
    double rc;
    double rc2;     // rc*rc (host-rounded, identical to the oracle's)
    double h;       // rc / (ntab-1)
    double inv_h;
    int l[kMaxRad];
    long long tab_off;  // offset (doubles) of this species' table in the table array
};

struct SysParams {
    double A[9];
    double Ainv[9];
    int N[3];
    int nblk[3];
    int natom;
    int nspecies;
    const double* tau;    // [natom*3]
    const int* spc;       // [natom]
    const double* tables; // concatenated radial tables
    DevSpecies sp[kMaxSpecies];
};

// One canonical work item of a grid block: covers (ci <= cj, block-local),
// value offset of the pair block (a_ci, a_cj, R_cj - R_ci).
struct BPair {
    int32_t cicj;  // ci | (cj << 16)
    int32_t roff;  // offset of the pair in the repacked density matrix (see kb_grid.cu: k_dm_repack)
    int64_t off;   // value offset of the pair block (a_ci, a_cj, R_cj - R_ci)
};

// One warp task of a grid block. H: rows of group g x columns of cover cj over
// the quads in qmask, and optionally of a second cover cj2 (quads qmask2;
// cj2 = 0xFF: none) sharing the group's A fragments. rho: rows of group g,
// octet half `half`, partner covers in [cj, qmask).
struct Task {
    uint8_t g;
    uint8_t cj;
    uint8_t half;
    uint8_t pad_;  // LPT warp during the build
    uint16_t qmask;
    uint16_t cost;
    uint8_t cj2;
    uint8_t pad2_;
    uint16_t qmask2;
};

struct Candidate {
    int32_t atom;
    int32_t R[3];
    int32_t lo[3];
    int32_t hi[3];
};

// Device-resident index.
struct MirrorItem {
    int64_t dst, src;  // pair-block offsets in H (dst = src: an (a, a, 0) block)
    int32_t na, nb;    // dst block is na x nb (src nb x na)
};

struct RepackItem {
    int64_t src, dst, srq;  // DM block (na x nb), its repacked block, the mirror DM block (nb x na)
    int32_t p;              // pair index (shard ownership)
    int32_t na, nb;         // orbitals
    int32_t fac2;           // 1: x2 (off the (a, a, 0) blocks)
};

struct DevIndex {
    int64_t nblock = 0, ncover = 0, npair = 0, nnz = 0, nbpair = 0;
    int32_t* blk_ptr = nullptr;
    int32_t* cov_atom = nullptr;
    int32_t* cov_R = nullptr;
    uint64_t* cov_mask = nullptr;
    int32_t* pair_a = nullptr;
    int32_t* pair_b = nullptr;
    int32_t* pair_R = nullptr;
    int64_t* pair_off = nullptr;
    int64_t* pair_key = nullptr;
    int64_t* pair_roff = nullptr;  // [npair+1] repacked-DM offsets (canonical pairs only)
    int64_t nrep = 0;              // repacked DM doubles per spin
    int32_t* pair_mirror = nullptr;
    // mirror work list (k_mirror_list): one item per non-canonical pair (filled from its canonical
    // mirror) and per (a, a, 0) pair (re-symmetrised); nmir items, count also at mir_count[0]
    MirrorItem* mir = nullptr;
    RepackItem* rep = nullptr;  // canonical pairs (k_dm_repack_list), nrep_items of them (count at mir_count[1])
    int64_t nrep_items = 0;
    int* mir_count = nullptr;
    int64_t nmir = 0;
    int64_t* bp_ptr = nullptr;
    BPair* bp = nullptr;
    int64_t* blk_cost = nullptr;
    // per-block warp task lists (kb_tasks.cu): tasks of block b are
    // [t_ptr[b], t_ptr[b+1]), warp w's tasks start at t_ptr[b] + t_wptr[b*9+w]
    int64_t* ht_ptr = nullptr;
    Task* ht = nullptr;
    int32_t* ht_wptr = nullptr;
    int64_t* rt_ptr = nullptr;
    Task* rt = nullptr;
    int32_t* rt_wptr = nullptr;
    int64_t nhtask = 0, nrtask = 0;
    int max_rows_padded = 0;  // max Phi rows of a block (groups padded to 8-row tiles)
    int max_htask = 0, max_rtask = 0;
    int htask_warps = 0, rtask_warps = 0;  // warps the H / rho task lists are LPT-balanced over
    int32_t* blk_rows = nullptr;  // Phi rows of each block (without the 8 tail rows)
    // geometry cache (kb_cache.cu): per block the H / rho table images
    // (table_bytes each) and Phi ((rows + 8) x 64 doubles at phi_off[b])
    unsigned char* htab = nullptr;
    unsigned char* rtab = nullptr;
    double* phis = nullptr;
    int64_t* phi_off = nullptr;
    int64_t tab_bytes = 0;
    int64_t phi_doubles = 0;
    int64_t* order = nullptr;   // owned blocks, heaviest first (persistent scheduling)
    int64_t norder = 0;
    int max_phi = 0;     // (unused)
    int max_cover = 0;   // max covers per block
    int max_bpairs = 0;  // max work items per block
    int64_t natompt = 0;
    double sum_m = 0, sum_m2 = 0;
};

// Host copies for kbg_index_view.
struct HostIndex {
    std::vector<int32_t> blk_ptr, cov_atom, cov_R, pair_a, pair_b, pair_R, pair_mirror;
    std::vector<uint64_t> cov_mask;
    std::vector<int64_t> pair_off;
    bool valid = false;
};

struct GridArgs {
    SysParams sys;
    const int32_t* blk_ptr;
    const int32_t* cov_atom;
    const int32_t* cov_R;
    const uint64_t* cov_mask;
    const int64_t* bp_ptr;
    const BPair* bp;
    const int64_t* t_ptr;   // task lists of this kernel (H or rho)
    const Task* tasks;
    const int32_t* t_wptr;
    int task_warps;
    const double* dmr;      // density: repacked DM [nspin][nrep]
    int64_t nrep;
    const int64_t* order;   // persistent kernels: block order
    int64_t norder;
    int* counter;           // persistent kernels: work counter (zeroed per launch)
    unsigned long long* dbg;    // optional timing counters (KBG_OPT_DEBUG_COUNTERS), else nullptr
    const unsigned char* tabs;  // geometry cache: this kernel's table images
    int64_t tab_bytes;
    const double* phis;
    const int64_t* phi_off;
    int64_t blk_begin;  // first owned block
    int max_rows;       // Phi rows allocated (padded groups + 8 pad rows)
    int max_cover;
    int max_bpairs;
    int max_tasks;      // table layout (shared by the H and rho images): max over both task kinds
    int max_rtasks;     // rho tasks of a block (per-task partial sums of the rho queue)
    int nspin;
    int64_t nnz;
    int64_t npts;
    double dV;
    double sign;        // +1, or -1 under the fault hook
    int scatter;        // 0: FP64 atomic scatter; 1: plain stores (timing experiment only, wrong H);
                        // bit value 16: deterministic two-limb scatter into out [nspin][2][nnz]
    const unsigned long long* vbits;  // H, deterministic: bit pattern of max|V| (written by a preceding kernel)
    double wfac;        // H, deterministic: |dV| * hbound (kb_gridcore.cuh hscale_of)
    const double* in;   // dm [nspin][nnz] or veff [nspin][npts]
    double* out;        // rho [nspin][npts] or h [nspin][nnz]
    // Shared-memory buffer layout of this launch (core::set_layout, by the
    // launcher): section byte offsets [0, 12), buffer size [12]. Kernel
    // parameters, so the compiler reloads them from the constant bank instead
    // of recomputing the layout arithmetic under register pressure.
    uint32_t lay[13];
    int reserve_sms;    // persistent kernels: SMs left free (a concurrent exchange, KBG_OPT_EXCHANGE_SMS)
    // fused rho + H pass (k_fused): the rho table images and the rho output next to H's
    const unsigned char* tabs2;
    double* out2;
};

// Allocations of the once-per-geometry build (index, task lists, geometry cache,
// comm tables): stream-ordered from the device's default memory pool with an
// unlimited release threshold, on the stream set by BuildStream (the context's
// stream), so a rebuild re-uses the pool without cudaMalloc/cudaFree round
// trips and implicit device synchronizations.
struct BuildStream {
    explicit BuildStream(cudaStream_t st);
    ~BuildStream();
    cudaStream_t prev;
};
cudaError_t pool_malloc_bytes(void** p, size_t bytes);
void pool_free(void* p);
template <class T>
cudaError_t pool_malloc(T** p, size_t bytes) {
    return pool_malloc_bytes(reinterpret_cast<void**>(p), bytes);
}

// Index build (kb_index.cu). Fills `ix` (device) and returns host stats.
void build_index_device(const SysParams& sys, DevIndex& ix, cudaStream_t st);
void free_index(DevIndex& ix);
// ix.order = owned blocks [b0, b1), by descending blk_cost (stable) or in block order.
void block_order_device(DevIndex& ix, int64_t b0, int64_t b1, bool heaviest_first, cudaStream_t st);
void copy_index_to_host(const DevIndex& ix, HostIndex& h, cudaStream_t st);

// Orbital / offset tables of the format converters (kb_formats.cu), built
// lazily from the host index: orbital row of atom a, orbital i = orb_off[a] + i.
struct FormatIndex {
    int n = 0, natom = 0, nR = 0;
    std::vector<int32_t> R;           // distinct pair offsets, sorted, 3 per entry
    int32_t* orb_atom = nullptr;      // [n] atom of each orbital row
    int32_t* orb_off = nullptr;       // [natom + 1]
    int32_t* run = nullptr;           // [natom * natom][2] pair range of atom pair (a, b), sorted by R
    int32_t* rid = nullptr;           // [npair] index of pair_R[p] in R
    int32_t* runs = nullptr;          // [nrun + 1] first pair of each distinct (a, b), pairs sorted by (a, b, R)
    int nrun = 0;
    bool valid = false;
};
void free_formats(FormatIndex& f);
int launch_phase(int nk, int64_t npair, const double* d_kpts, const int32_t* pair_R, double sign, double2* d_phase,
                 cudaStream_t st);
int launch_bloch(const FormatIndex& f, const DevIndex& ix, int nk, const double* d_M, const double2* d_phase,
                 double* d_out, cudaStream_t st);
int launch_fold(const FormatIndex& f, const DevIndex& ix, int nk, const double* d_w, const double2* d_phase,
                const double* d_rho_k, double* d_out, unsigned long long* d_max_imag, cudaStream_t st);
int launch_realspace(const FormatIndex& f, const DevIndex& ix, bool to_dense, double* d_sparse, double* d_dense,
                     cudaStream_t st);
int launch_scale_states(int n, int m, const double* d_C, const double* d_w, double* d_D, cudaStream_t st);
// V_eff from rho (kb_veff.cu): cuFFT plans + work, per context.
struct VeffPlan {
    bool planned = false;
    int fwd = 0, inv = 0;  // cufftHandle
    double* work = nullptr;
    double* B = nullptr;   // reciprocal basis rows (device)
    void release();
};
int run_veff(VeffPlan& vp, const int N[3], const double Ainv[9], int nspin, int xc, const double* d_rho,
             const double* d_vloc, double dV, double* d_veff, double* d_energy, cudaStream_t st,
             unsigned int* d_bad = nullptr);

// Fused H reduction + mirror over peer memory (kb_comm.cu).
constexpr int kMaxRanks = 8;
struct CommArgs {
    int nranks = 0, rank = 0;
    double* x[kMaxRanks] = {};                  // exchange buffers [2][nnz], peer-mapped (CUDA IPC)
    unsigned long long* flags[kMaxRanks] = {};  // flag array [kMaxRanks] at the tail of each buffer
    unsigned int* counter = nullptr;            // local CTA counter
    // this rank's slice of the canonical entries: el0 = entry offset, el1 =
    // mirror offset (bit 31: transposed entry of an (a,a,0) block, averaged)
    const int32_t* el0 = nullptr;
    const int32_t* el1 = nullptr;
    const uint8_t* elm = nullptr;  // ranks whose partial of the entry can be nonzero (bit k: rank k)
    int64_t ne = 0;
    // per pair: orbital counts and canonical flag (fused copy-out + mirror)
    const int32_t* pair_na = nullptr;
    const int32_t* pair_nb = nullptr;
    const uint8_t* pair_canon = nullptr;
    unsigned long long* tstamp = nullptr;  // KBG_COMM_TIMING: globaltimer stamps of the exchange phases [8]
    int ls = 1;  // doubles per entry of the partials: 2 = two-limb deterministic accumulators, 1 = FP64
    int sms = 0;  // > 0: run as this many whole-SM CTAs (concurrent with the density pass), else the GPU
};
// Per pair, the ranks (bit k) whose block range [bounds[k], bounds[k + 1]) holds
// a canonical (block, cover pair) work item of that pair.
void pair_owners(const DevIndex& ix, const std::vector<int64_t>& bounds, std::vector<uint32_t>& out, cudaStream_t st);
int launch_reduce_mirror(const CommArgs& c, const DevIndex& ix, const SysParams& sys, int nspin, double* d_out,
                         unsigned long long epoch, cudaStream_t st);

// Eigen_HH (kb_eigen.cu). Complex arrays interleaved.
size_t hh_tridiag_smem(int n);
// Tridiagonal eigensolver (kb_tridiag.cu): eigenvalues ascending into d_w, eigenvectors as the
// columns of d_z [n][n]; d_scr holds tridiag_scratch_doubles(n, vectors).
size_t tridiag_scratch_doubles(int n, bool vectors);
int launch_tridiag_solve(int n, const double* d_d, const double* d_e, bool vectors, double* d_w, double* d_z,
                         double* d_scr, cudaStream_t st);
int launch_hermitian_repair(int n, double* d_A, unsigned long long* d_defect, bool apply, cudaStream_t st);
int launch_hh_tridiagonalize(int n, double* d_B, double* d_p, double* d, double* e, double* u, double* h, double* s,
                             double* ph, double sign, cudaStream_t st);
int launch_hh_back_transform(int n, int m, const double* d_Y, const double* d_U, const double* d_h,
                             const double* d_ph, double* d_dph, double* d_W, cudaStream_t st);
// Blocked (compact WY, cuBLAS ZGEMM) variant of the same W = Q Y; d_scr holds
// hh_back_transform_wy_scratch(n, m) doubles. Used from n >= kWyMinN.
int launch_hh_back_transform_wy(int n, int m, const double* d_Y, const double* d_U, const double* d_h,
                                const double* d_ph, double* d_dph, double* d_W, double* d_scr, cudaStream_t st);
size_t hh_back_transform_wy_scratch(int n, int m);
constexpr int kWyMinN = 1024;  // measured crossover vs the per-column kernel (profiles/eigen_wy*.jsonl)
int launch_hh_normalize_columns(int64_t n, int64_t m, double* d_C, int* d_zero, cudaStream_t st);
// HBM probe (kb_probe.cu): x[v][:] /= ||x[v]|| for nvec rows of len doubles.
int launch_normalize(double* d_x, int64_t nvec, int64_t len, cudaStream_t st);

// Grid kernels (kb_grid.cu). Return number of kernel launches.
size_t grid_smem_bytes(const GridArgs& g, int nwarps, bool density);
// Task lists (kb_tasks.cu), built after the index.
// h_warps / r_warps: warps the H / rho lists are LPT-balanced over (1: one
// queue, heaviest first); r_split: rho partner ranges are cut for this many warps.
void build_tasks_device(const SysParams& sys, DevIndex& ix, int h_warps, int r_warps, int r_split, cudaStream_t st);
void free_tasks(DevIndex& ix);
int launch_density(const GridArgs& g, int64_t nblk_owned, int nwarps, cudaStream_t st);
int launch_hamiltonian(const GridArgs& g, int64_t nblk_owned, int nwarps, cudaStream_t st);
int launch_dm_repack(const DevIndex& ix, const SysParams& sys, int nspin, const double* dm, double* dmr,
                     cudaStream_t st, unsigned long long* chk = nullptr, const uint8_t* own = nullptr);
// Persistent warp-specialized kernels (kb_persist.cu): kPersistProducers
// producer warps stage block k+1 while kPersistConsumers consumer warps work
// on block k (two shared-memory buffers). persist_fits() says whether two
// buffers fit in shared memory for this index.
constexpr int kPersistProducers = 1;
#ifndef KBG_CONSUMERS_R
#define KBG_CONSUMERS_R 19
#endif
#ifndef KBG_CONSUMERS_H
#define KBG_CONSUMERS_H 27
#endif
constexpr int kPersistConsumersR = KBG_CONSUMERS_R;  // rho: 20 warps with the producer (96 registers)
constexpr int kPersistConsumersH = KBG_CONSUMERS_H;  // H: 28 warps with the producer (72 registers)
// Geometry cache (kb_cache.cu): Phi and the per-block tables, built once per
// geometry after the task lists.
void build_cache_device(GridArgs gh, GridArgs gr, DevIndex& ix, cudaStream_t st);
void free_cache(DevIndex& ix);
bool persist_fits(const GridArgs& g, bool density);
size_t persist_smem(const GridArgs& g, bool density);
int launch_density_persist(const GridArgs& g, cudaStream_t st);
// Fused rho + H pass (one persistent kernel, a block's Phi staged once, both task queues interleaved):
// gh = the H launch's args (in = V, out = H accumulator), gr = the rho launch's (dmr, out = rho).
// Returns 0 (nothing launched) when the fused buffers do not fit shared memory.
bool fused_fits(const GridArgs& gh, const GridArgs& gr);
int launch_fused(const GridArgs& gh, const GridArgs& gr, cudaStream_t st);
int launch_hamiltonian_persist(const GridArgs& g, cudaStream_t st);
int launch_dm_gather(const int64_t* d_runs, int64_t nruns, int nspin, int64_t nnz, const double* src, double* dst,
                     cudaStream_t st);
int launch_mirror(const DevIndex& ix, const SysParams& sys, int nspin, double* h, cudaStream_t st);
// Deterministic H (kb_gridcore.cuh h_scatter): max|x| as a bit pattern (atomicMax into *d_out, which the
// caller zeroes), and H = hi + lo of the two-limb accumulator [nspin][nnz][2] (+ mirror blocks).
int launch_absmax(const double* d_x, int64_t n, unsigned long long* d_out, cudaStream_t st);
int launch_finalize(const DevIndex& ix, const SysParams& sys, int nspin, const double* acc, double* h, bool mirror,
                    cudaStream_t st, int limbs = 2);
int launch_dm_check(const DevIndex& ix, const SysParams& sys, int nspin, const double* dm,
                    unsigned long long* d_maxdiff_maxabs, cudaStream_t st);
int launch_block_orbitals(const GridArgs& g, int64_t block, double* d_out, cudaStream_t st);

}  // namespace kbg
