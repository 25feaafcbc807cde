// C-ABI of libkbgrid (include/kbgrid.h): context, validation, host/device
// entry points. Errors follow the kband taxonomy (common.hpp:21-38) as status
// codes with a message naming the failing field (kbg_last_error).
#include <algorithm>
#include <chrono>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <cstdio>
#include <string>
#include <vector>

#include <cublas_v2.h>
#include <unistd.h>

#include "kb_device.cuh"

struct kbg_ctx {
    int device = 0;
    int rank = 0, nranks = 1;
    kbg::SysParams P{};
    double* d_tau = nullptr;
    int* d_spc = nullptr;
    double* d_tables = nullptr;
    kbg::DevIndex ix;
    kbg::HostIndex hix;
    bool built = false;
    int64_t blk_begin = 0, blk_end = 0;
    int nwarps = 8;
    bool persist_ok = false;   // two staging buffers fit: persistent kernels
    int persist = 1;           // option: use the persistent kernels when they fit
    int schedule = 3;          // KBG_OPT_SCHEDULE
    int block_order = 2;       // KBG_OPT_BLOCK_ORDER (2: by blocks per SM)
    int xc = 0;                // KBG_OPT_XC
    int plan_schedule = -1;    // schedule / rho split the task lists were built with (kbg_plan_info)
    int plan_split = 0;
    double* d_dmr = nullptr;   // repacked DM scratch
    size_t cap_dmr = 0;
    int* d_counter = nullptr;  // persistent work counters: [0] density, [1] H (the two may run concurrently)
    double sign = 1.0;
    int scatter = 0;
    unsigned long long* d_dbg = nullptr;  // KBG_OPT_DEBUG_COUNTERS
    cudaStream_t stream = nullptr;
    double* d_in = nullptr;
    size_t cap_in = 0;
    double* d_out = nullptr;
    size_t cap_out = 0;
    unsigned long long* d_check = nullptr;
    int last_launches = 0;
    kbg_tally tally{0, 0};
    std::string err;
    int64_t npts = 0;
    std::vector<int> h_spc;
    // format converters (kb_formats.cu)
    kbg::FormatIndex fmt;
    double* d_fa = nullptr;  // host-API staging: pairs / dense side
    size_t cap_fa = 0;
    double* d_fb = nullptr;
    size_t cap_fb = 0;
    double* d_phase = nullptr;  // [nk][npair] double2
    size_t cap_phase = 0;
    double* d_kw = nullptr;  // kpts (3 nk) then weights (nk)
    size_t cap_kw = 0;
    double* h_kw = nullptr;  // pinned staging of d_kw (async copy); h_kw_done: its last copy finished
    size_t cap_hkw = 0;
    cudaEvent_t h_kw_done = nullptr;
    cublasHandle_t blas = nullptr;  // Part 6 density matrix (ZGEMM)
    // fused H reduction over peer memory (kb_comm.cu)
    kbg::CommArgs comm;
    double* d_xbuf = nullptr;           // own exchange buffer [2][nnz] + flags + counter
    unsigned char* d_pairtab = nullptr; // per-pair na, nb, canonical flag (fused copy-out + mirror)
    std::vector<void*> ipc_opened;      // peer buffers opened with cudaIpcOpenMemHandle
    int32_t* d_canon = nullptr;
    kbg::VeffPlan veff;  // kbg_veff (cuFFT plans)
    // kbg_grid_pass: second stream and buffers for the H half
    cudaStream_t stream2 = nullptr;
    cudaEvent_t ev_pass = nullptr;
    cudaEvent_t ev_rho = nullptr;  // sharded kbg_grid_pass: density kernel done (the exchange waits for it)
    double* d_in2 = nullptr;
    size_t cap_in2 = 0;
    double* d_out2 = nullptr;
    size_t cap_out2 = 0;
    int64_t* d_cpre = nullptr;
    unsigned long long epoch = 0;
    bool comm_ready = false;
    double* d_states = nullptr;     // scaled states scratch
    size_t cap_states = 0;
    // deterministic H (KBG_OPT_DETERMINISTIC, kb_gridcore.cuh h_scatter)
    int det = 0;  // KBG_OPT_DETERMINISTIC (off by default: +68 % H time on 56 atoms)
    double hbound = 0.0;            // >= sum over r of |phi_i(r) phi_j(r)| for any orbital pair (h_bound)
    double* d_hacc = nullptr;       // two-limb accumulator [nspin][nnz][2]
    size_t cap_hacc = 0;
    unsigned long long* d_vbits = nullptr;  // max|V| bit pattern of the current H pass
    // shard-local host transfers of kbg_grid_pass on a sharded context (KBG_OPT_SHARD_IO)
    int shard_io = 1;
    int sparse_thr = 0;  // KBG_OPT_SPARSE_DFMA (0: every task on DMMA)
    int xsms = 8;        // KBG_OPT_EXCHANGE_SMS (0: exchange on the whole GPU, not overlapped)
    int fused = 2;       // KBG_OPT_FUSED_PASS: 0 separate, 1 fused, 2 auto (fused while DM' + H fit kFusedAutoBytes)
    int pending_nspin = 0;  // kbg_hamiltonian_partial_dev done, exchange pending
    uint8_t* d_pown = nullptr;      // per pair: 1 if this rank's blocks touch it (kbg_comm_open)
    std::vector<int64_t> dm_runs;   // [off, len] pairs: DM ranges (per spin) covering the pairs the repack reads
    int64_t* d_xruns = nullptr;     // the exact [off, len] runs of the needed pair blocks (k_dm_gather)
    unsigned long long* h_flags = nullptr;  // pinned: kbg_grid_pass's DM check words and V flag
    int64_t dm_xruns_n = 0;
    int64_t dm_read_copy = 0;       // doubles per spin the memcpy runs move (pageable DM)
    int64_t io[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // kbg_shard_io
};

// rho partner ranges are cut at 1/(2 KBG_RHO_SPLIT) of a block's work
// (kb_tasks.cu). With the per-block task queue, long tasks win: measured
// density pass 0.421 ms (19), 0.392 (10), 0.376 (6), 0.379 (4 .. 1, no cuts).
#ifndef KBG_RHO_SPLIT
#define KBG_RHO_SPLIT 6
#endif

namespace kbg {
namespace {
thread_local cudaStream_t g_build_stream = nullptr;
}
BuildStream::BuildStream(cudaStream_t st) : prev(g_build_stream) {
    g_build_stream = st;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
}
BuildStream::~BuildStream() { g_build_stream = prev; }
cudaError_t pool_malloc_bytes(void** p, size_t bytes) {
    return cudaMallocAsync(p, bytes ? bytes : 1, g_build_stream);
}
void pool_free(void* p) {
    if (p) cudaFreeAsync(p, g_build_stream);
}
}  // namespace kbg

namespace {

using kbg::Error;

template <class F>
int guard(kbg_ctx* ctx, F&& fn) {
    try {
        fn();
        if (ctx) ctx->err.clear();
        return KBG_OK;
    } catch (const Error& e) {
        if (ctx) ctx->err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        return KBG_ERR_CONSISTENCY;
    }
}

// Bound used by the deterministic H accumulation (kb_gridcore.cuh h_scatter):
// hbound >= sum over the grid of |phi_i(r)| |phi_j(r)| for any two orbitals,
// so max|V| |dV| hbound bounds the sum of |contributions| of every H entry.
// |phi| <= umax rc^l A_l with umax bounding the cubic-Hermite interpolant
// (|h00|+|h01| = 1, |h10|, |h11| <= 4/27 on [0, 1]) and A_l the largest real
// solid-harmonic prefactor; an orbital is nonzero on at most P grid points,
// P <= volume(ball of radius rc + cell diameter) / dV + 1.
double h_bound(const kbg::SysParams& P, const kbg_system& s) {
    const double* A = P.A;
    const double det = std::fabs(A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
                                 A[2] * (A[3] * A[7] - A[4] * A[6]));
    const double dv = det / (static_cast<double>(s.grid[0]) * s.grid[1] * s.grid[2]);
    double diam = 0.0;
    for (int sg = 0; sg < 8; ++sg) {
        double d[3] = {0, 0, 0};
        for (int i = 0; i < 3; ++i) {
            const double f = ((sg >> i) & 1 ? -1.0 : 1.0) / s.grid[i];
            for (int q = 0; q < 3; ++q) d[q] += f * A[3 * i + q];
        }
        diam = std::max(diam, std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]));
    }
    const double Al[3] = {0.28209479177387814, 0.4886025119029199, 0.6307831305050401};
    double phimax = 0.0, pmax = 0.0;
    for (int t = 0; t < s.nspecies; ++t) {
        const kbg_species& sp = s.spec[t];
        const double h = sp.rc / (sp.ntab - 1);
        for (int r = 0; r < sp.nrad; ++r) {
            double u = 0.0, du = 0.0;
            for (int k = 0; k < sp.ntab; ++k) {
                u = std::max(u, std::fabs(sp.table[2 * (static_cast<size_t>(r) * sp.ntab + k)]));
                du = std::max(du, std::fabs(sp.table[2 * (static_cast<size_t>(r) * sp.ntab + k) + 1]));
            }
            const double umax = u + (8.0 / 27.0) * h * du;
            phimax = std::max(phimax, umax * std::pow(sp.rc, sp.l[r]) * Al[sp.l[r]]);
        }
        const double rr = sp.rc + diam;
        pmax = std::max(pmax, std::floor(4.18879020478639 * rr * rr * rr / dv) + 1.0);
    }
    return pmax * phimax * phimax * (1.0 + 1e-12);
}

void validate_and_load(kbg_ctx* c, const kbg_system& s) {
    if (s.natom < 1) throw Error(KBG_ERR_CONFIG, "system: natom must be >= 1");
    if (s.nspecies < 1 || !s.spec) throw Error(KBG_ERR_CONFIG, "system: no species");
    if (s.nspecies > kbg::kMaxSpecies) throw Error(KBG_ERR_CONFIG, "system: too many species (max 8)");
    if (!s.species || !s.tau) throw Error(KBG_ERR_CONFIG, "system: null species/tau");
    for (int i = 0; i < 3; ++i)
        if (s.grid[i] < 1) throw Error(KBG_ERR_DIMENSION, "system: grid[" + std::to_string(i) + "] < 1");
    kbg::SysParams& P = c->P;
    std::memcpy(P.A, s.lattice, sizeof(P.A));
    const double* A = P.A;
    const double det = A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
                       A[2] * (A[3] * A[7] - A[4] * A[6]);
    if (!(std::fabs(det) > 1e-12)) throw Error(KBG_ERR_CONFIG, "system: singular lattice");
    P.Ainv[0] = (A[4] * A[8] - A[5] * A[7]) / det;
    P.Ainv[1] = (A[2] * A[7] - A[1] * A[8]) / det;
    P.Ainv[2] = (A[1] * A[5] - A[2] * A[4]) / det;
    P.Ainv[3] = (A[5] * A[6] - A[3] * A[8]) / det;
    P.Ainv[4] = (A[0] * A[8] - A[2] * A[6]) / det;
    P.Ainv[5] = (A[2] * A[3] - A[0] * A[5]) / det;
    P.Ainv[6] = (A[3] * A[7] - A[4] * A[6]) / det;
    P.Ainv[7] = (A[1] * A[6] - A[0] * A[7]) / det;
    P.Ainv[8] = (A[0] * A[4] - A[1] * A[3]) / det;
    for (int i = 0; i < 3; ++i) {
        P.N[i] = s.grid[i];
        P.nblk[i] = (s.grid[i] + KBG_BLOCK_EDGE - 1) / KBG_BLOCK_EDGE;
    }
    P.natom = s.natom;
    P.nspecies = s.nspecies;
    std::vector<double> tables;
    for (int t = 0; t < s.nspecies; ++t) {
        const kbg_species& in = s.spec[t];
        const std::string who = "species " + std::to_string(t);
        if (in.nrad < 1 || !in.l || !in.table) throw Error(KBG_ERR_CONFIG, who + ": empty radial list");
        if (in.nrad > kbg::kMaxRad) throw Error(KBG_ERR_CONFIG, who + ": too many radial functions");
        if (!(in.rc > 0)) throw Error(KBG_ERR_CONFIG, who + ": rc <= 0");
        if (in.ntab < 4) throw Error(KBG_ERR_CONFIG, who + ": ntab < 4");
        kbg::DevSpecies& d = P.sp[t];
        d.nrad = in.nrad;
        d.ntab = in.ntab;
        d.rc = in.rc;
        d.rc2 = in.rc * in.rc;
        d.h = in.rc / (in.ntab - 1);
        d.inv_h = 1.0 / d.h;
        d.norb = 0;
        for (int r = 0; r < in.nrad; ++r) {
            if (in.l[r] < 0 || in.l[r] > KBG_MAX_L) throw Error(KBG_ERR_CONFIG, who + ": l out of range");
            d.l[r] = in.l[r];
            d.norb += 2 * in.l[r] + 1;
        }
        if (d.norb > KBG_MAX_ORB_PER_ATOM) throw Error(KBG_ERR_CONFIG, who + ": too many orbitals");
        d.tab_off = static_cast<long long>(tables.size());
        const size_t n = static_cast<size_t>(in.nrad) * in.ntab * 2;
        for (size_t i = 0; i < n; ++i) {
            if (!std::isfinite(in.table[i])) throw Error(KBG_ERR_NONFINITE, who + ": non-finite radial table");
            tables.push_back(in.table[i]);
        }
    }
    for (int a = 0; a < s.natom; ++a) {
        if (s.species[a] < 0 || s.species[a] >= s.nspecies)
            throw Error(KBG_ERR_CONFIG, "atom " + std::to_string(a) + ": bad species id");
        for (int q = 0; q < 3; ++q)
            if (!std::isfinite(s.tau[3 * a + q]))
                throw Error(KBG_ERR_NONFINITE, "atom " + std::to_string(a) + ": non-finite position");
    }
    c->npts = static_cast<int64_t>(s.grid[0]) * s.grid[1] * s.grid[2];
    c->hbound = h_bound(P, s);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw Error(KBG_ERR_CUDA, "no CUDA device available (libkbgrid has no CPU fallback)");
    if (c->device < 0 || c->device >= ndev) throw Error(KBG_ERR_CUDA, "device index out of range");
    KBG_CUDA(cudaSetDevice(c->device));
    KBG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    KBG_CUDA(cudaMalloc(&c->d_tau, sizeof(double) * 3 * s.natom));
    KBG_CUDA(cudaMalloc(&c->d_spc, sizeof(int) * s.natom));
    KBG_CUDA(cudaMalloc(&c->d_tables, sizeof(double) * tables.size()));
    KBG_CUDA(cudaMalloc(&c->d_check, sizeof(unsigned long long) * 4));
    KBG_CUDA(cudaMalloc(&c->d_vbits, sizeof(unsigned long long) * 2));
    KBG_CUDA(cudaMemcpy(c->d_tau, s.tau, sizeof(double) * 3 * s.natom, cudaMemcpyHostToDevice));
    KBG_CUDA(cudaMemcpy(c->d_spc, s.species, sizeof(int) * s.natom, cudaMemcpyHostToDevice));
    KBG_CUDA(cudaMemcpy(c->d_tables, tables.data(), sizeof(double) * tables.size(), cudaMemcpyHostToDevice));
    c->h_spc.assign(s.species, s.species + s.natom);
    P.tau = c->d_tau;
    P.spc = c->d_spc;
    P.tables = c->d_tables;
}

void ensure(double*& buf, size_t& cap, size_t n) {
    if (cap >= n) return;
    if (buf) cudaFree(buf);
    buf = nullptr;
    KBG_CUDA(cudaMalloc(&buf, n * sizeof(double)));
    cap = n;
}

void require_index(kbg_ctx* c) {
    if (!c->built) throw Error(KBG_ERR_CONFIG, "index not built (call kbg_build_index first)");
}

void check_nspin(int nspin) {
    if (nspin < 1 || nspin > 2) throw Error(KBG_ERR_CONFIG, "nspin must be 1 or 2");
}

kbg::GridArgs grid_args(kbg_ctx* c, int nspin, double dV, const double* in, double* out, bool density) {
    kbg::GridArgs g{};
    g.sys = c->P;
    g.blk_ptr = c->ix.blk_ptr;
    g.cov_atom = c->ix.cov_atom;
    g.cov_R = c->ix.cov_R;
    g.cov_mask = c->ix.cov_mask;
    g.bp_ptr = c->ix.bp_ptr;
    g.bp = c->ix.bp;
    g.blk_begin = c->blk_begin;
    g.max_rows = c->ix.max_rows_padded + 8;
    g.max_cover = c->ix.max_cover > 0 ? c->ix.max_cover : 1;
    g.max_bpairs = c->ix.max_bpairs > 0 ? c->ix.max_bpairs : 1;
    g.task_warps = density ? c->ix.rtask_warps : c->ix.htask_warps;
    g.order = c->ix.order;
    g.norder = c->ix.norder;
    g.counter = c->d_counter + (density ? 0 : 1);
    // the density kernel of a sharded context leaves the exchange's SMs free (KBG_OPT_EXCHANGE_SMS)
    g.reserve_sms = density && c->comm_ready ? c->xsms : 0;
    g.nrep = c->ix.nrep;
    g.t_ptr = density ? c->ix.rt_ptr : c->ix.ht_ptr;
    g.tasks = density ? c->ix.rt : c->ix.ht;
    g.t_wptr = density ? c->ix.rt_wptr : c->ix.ht_wptr;
    g.max_tasks = std::max(1, std::max(c->ix.max_rtask, c->ix.max_htask));
    g.max_rtasks = std::max(1, c->ix.max_rtask);
    g.tabs = density ? c->ix.rtab : c->ix.htab;
    g.tab_bytes = c->ix.tab_bytes;
    g.phis = c->ix.phis;
    g.phi_off = c->ix.phi_off;
    g.nspin = nspin;
    g.nnz = c->ix.nnz;
    g.npts = c->npts;
    g.dV = dV;
    g.sign = c->sign;
    g.scatter = c->scatter;
    g.dbg = c->d_dbg;
    g.in = in;
    g.out = out;
    if (!density) {
        g.scatter |= c->sparse_thr << 8;  // A5 switch: tasks below this point density (1/255) run DFMA
        if (KBG_EXPERIMENTS && std::getenv("KBG_DFMA_WARPS"))  // timing experiment: DFMA-only warps
            g.scatter |= (std::atoi(std::getenv("KBG_DFMA_WARPS")) << 16) | (1 << 8);
        g.vbits = c->d_vbits;  // deterministic: max|V| (k_absmax); legacy: non-finite flag of the kernels
        if (c->det) {
            g.scatter |= 16;  // deterministic two-limb scatter (kb_gridcore.cuh h_scatter)
            g.wfac = std::fabs(dV) * c->hbound;
        }
    }
    if (g.max_cover > 32 * c->nwarps || g.max_cover > kbg::kMaxCoverPerBlock)
        throw Error(KBG_ERR_DIMENSION, "a grid block is covered by too many atom images");
    const size_t smem = kbg::grid_smem_bytes(g, c->nwarps, density);
    if (smem > 227 * 1024)
        throw Error(KBG_ERR_DIMENSION, "grid block needs " + std::to_string(smem) +
                                           " B of shared memory (> 227 KB): too many orbitals per block");
    return g;
}

int run_density(kbg_ctx* c, int nspin, const double* d_dm, double* d_rho, cudaStream_t st,
                unsigned long long* chk = nullptr, const uint8_t* own = nullptr) {
    ensure(c->d_dmr, c->cap_dmr, static_cast<size_t>(nspin) * std::max<int64_t>(1, c->ix.nrep));
    int n = kbg::launch_dm_repack(c->ix, c->P, nspin, d_dm, c->d_dmr, st, chk, own);
    kbg::GridArgs g = grid_args(c, nspin, 0.0, d_dm, d_rho, true);
    g.dmr = c->d_dmr;
    if (c->persist_ok && c->persist && c->ix.phis) {
        if (kbg::persist_fits(g, true)) return n + kbg::launch_density_persist(g, st);
        // accumulators for every spin do not fit: one persistent launch per spin
        for (int s = 0; s < nspin; ++s) {
            kbg::GridArgs g1 = grid_args(c, 1, 0.0, d_dm + s * c->ix.nnz, d_rho + s * c->npts, true);
            g1.dmr = c->d_dmr + s * c->ix.nrep;
            if (!kbg::persist_fits(g1, true)) break;
            n += kbg::launch_density_persist(g1, st);
            if (s + 1 == nspin) return n;
        }
    }
    return n + kbg::launch_density(g, c->blk_end - c->blk_begin, c->nwarps, st);
}

// Reads and clears this rank's exchange error word (kb_comm.cu wait_flags); after a synchronize.
void comm_check(kbg_ctx* c) {
    unsigned long long* err = c->comm.flags[c->rank] + kbg::kMaxRanks + 1;
    unsigned long long v = 0;
    KBG_CUDA(cudaMemcpy(&v, err, sizeof(v), cudaMemcpyDeviceToHost));
    if (v) {
        const unsigned long long zero = 0;
        KBG_CUDA(cudaMemcpy(err, &zero, sizeof(zero), cudaMemcpyHostToDevice));
        throw Error(KBG_ERR_NCCL, "peer-memory H exchange: a peer did not arrive within 10 s (H invalid)");
    }
}

// Doubles per H entry of the accumulator (deterministic: hi and lo limbs).
int h_limbs(const kbg_ctx* c) { return c->det ? 2 : 1; }

int run_hamiltonian(kbg_ctx* c, int nspin, double dV, const double* d_veff, double* d_h, cudaStream_t st) {
    const kbg::GridArgs g = grid_args(c, nspin, dV, d_veff, d_h, false);
    if (c->persist_ok && c->persist && c->ix.phis) {
        if (kbg::persist_fits(g, false)) return kbg::launch_hamiltonian_persist(g, st);
        int n = 0;
        for (int s = 0; s < nspin; ++s) {
            const kbg::GridArgs g1 =
                grid_args(c, 1, dV, d_veff + s * c->npts, d_h + s * c->ix.nnz * h_limbs(c), false);
            if (!kbg::persist_fits(g1, false)) break;
            n += kbg::launch_hamiltonian_persist(g1, st);
            if (s + 1 == nspin) return n;
        }
    }
    return kbg::launch_hamiltonian(g, c->blk_end - c->blk_begin, c->nwarps, st);
}

// One H accumulation into `acc`: deterministic (default) -- zero the two-limb
// accumulator [nspin][nnz][2] and the max|V| word, reduce max|V| over every
// point of the device-resident V, accumulate; legacy -- zero [nspin][nnz] and
// accumulate with FP64 atomics. The caller finalizes (launch_finalize) or
// reduces across ranks (kb_comm.cu).
int h_accumulate(kbg_ctx* c, int nspin, double dV, const double* d_veff, double* acc, cudaStream_t st) {
    int n = 0;
    const size_t ne = static_cast<size_t>(nspin) * c->ix.nnz * h_limbs(c);
    KBG_CUDA(cudaMemsetAsync(acc, 0, ne * sizeof(double), st));
    KBG_CUDA(cudaMemsetAsync(c->d_vbits, 0, sizeof(unsigned long long), st));
    if (c->det) n += kbg::launch_absmax(d_veff, static_cast<int64_t>(nspin) * c->npts, c->d_vbits, st);
    return n + run_hamiltonian(c, nspin, dV, d_veff, acc, st);
}

// Accumulator of the single-rank H paths: the context's two-limb scratch when
// deterministic, else the output itself.
double* h_acc_buffer(kbg_ctx* c, int nspin, double* d_out) {
    if (!c->det) return d_out;
    ensure(c->d_hacc, c->cap_hacc, static_cast<size_t>(2) * nspin * std::max<int64_t>(1, c->ix.nnz));
    return c->d_hacc;
}

// Max|V| of the last H pass (legacy path: only the non-finite flag): non-finite V -> KBG_ERR_NONFINITE
// (kband raises on non-finite values, householder.cpp:119-123). Host API only
// (after its synchronize).
void check_vbits(kbg_ctx* c, const char* who) {
    unsigned long long v = 0;
    KBG_CUDA(cudaMemcpy(&v, c->d_vbits, sizeof(v), cudaMemcpyDeviceToHost));
    if (v >= 0x7ff0000000000000ull)
        throw Error(KBG_ERR_NONFINITE, std::string(who) + ": non-finite V_eff (outputs invalid)");
}

// Device alias of a caller's host buffer that the GPU can read in place (pinned
// or registered, hence mapped under UVA), else nullptr. Only the persistent H
// kernel reads its input this way: its producer warp loads a block's 64 V
// values one block ahead, so the PCIe reads hide behind the DMMA work and the
// pass does not wait for a whole-array H2D copy first.
const double* mapped_input(const kbg_ctx* c, const double* host) {
    if (!(c->persist_ok && c->persist && c->ix.phis) || std::getenv("KBG_NO_ZERO_COPY")) return nullptr;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
        (void)cudaGetLastError();
        return nullptr;
    }
    if (a.type != cudaMemoryTypeHost || !a.devicePointer) return nullptr;
    return static_cast<const double*>(a.devicePointer);
}

// Same for an output: the persistent density kernel stores each finished
// block's 64 points in C order (32-byte segments), so with rho in pinned host
// memory the result streams over PCIe during the kernel instead of in one D2H
// copy after it. Single-rank contexts only (a shard must zero foreign points).
double* mapped_output(const kbg_ctx* c, double* host) {
    if ((c->nranks > 1 && !(c->comm_ready && c->shard_io)) || std::getenv("KBG_NO_ZERO_COPY_OUT")) return nullptr;
    return const_cast<double*>(mapped_input(c, host));
}

// Block ranges of every rank: rank r owns [bounds[r], bounds[r + 1]).
std::vector<int64_t> shard_bounds(kbg_ctx* c) {
    const int64_t nb = c->ix.nblock;
    std::vector<int64_t> out(c->nranks + 1, nb);
    out[0] = 0;
    if (c->nranks == 1) return out;
    std::vector<int64_t> cost(nb);
    KBG_CUDA(cudaMemcpy(cost.data(), c->ix.blk_cost, nb * sizeof(int64_t), cudaMemcpyDeviceToHost));
    // Contiguous cost-balanced split; mirrors
    // paper_1402_4247_b200/shard.py:partition: weights cost+1 (empty blocks
    // count), bound(r) = first b with prefix(b) * nranks >= total * r (exact
    // integer arithmetic).
    std::vector<int64_t> pre(nb + 1, 0);
    for (int64_t b = 0; b < nb; ++b) pre[b + 1] = pre[b] + cost[b] + 1;
    auto bound = [&](int r) -> int64_t {
        if (r <= 0) return 0;
        if (r >= c->nranks) return nb;
        const __int128 target = static_cast<__int128>(pre[nb]) * r;
        int64_t lo = 0, hi = nb;
        while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if (static_cast<__int128>(pre[mid]) * c->nranks < target)
                lo = mid + 1;
            else
                hi = mid;
        }
        return lo;
    };
    for (int r = 0; r <= c->nranks; ++r) out[r] = bound(r);
    return out;
}

void shard(kbg_ctx* c) {
    const std::vector<int64_t> b = shard_bounds(c);
    c->blk_begin = b[c->rank];
    c->blk_end = b[c->rank + 1];
}

}  // namespace

extern "C" {

const char* kbg_version(void) { return "kbgrid 0.1 sm_100a"; }

const char* kbg_status_string(int status) {
    switch (status) {
        case KBG_OK: return "ok";
        case KBG_ERR_CONFIG: return "config error";
        case KBG_ERR_DIMENSION: return "dimension error";
        case KBG_ERR_CONSISTENCY: return "consistency error";
        case KBG_ERR_NONFINITE: return "non-finite value";
        case KBG_ERR_CUDA: return "cuda error";
        case KBG_ERR_NCCL: return "collective error";
        default: return "unknown status";
    }
}

int kbg_create_sharded(const kbg_system* sys, int device, int rank, int nranks, kbg_ctx** out) {
    if (!out) return KBG_ERR_CONFIG;
    *out = nullptr;
    if (!sys) return KBG_ERR_CONFIG;
    if (nranks < 1 || rank < 0 || rank >= nranks) return KBG_ERR_CONFIG;
    auto* c = new kbg_ctx();
    c->device = device;
    c->rank = rank;
    c->nranks = nranks;
    const int st = guard(c, [&] { validate_and_load(c, *sys); });
    if (st != KBG_OK) {
        std::fprintf(stderr, "kbg_create: %s\n", c->err.c_str());
        kbg_destroy(c);
        return st;
    }
    *out = c;
    return KBG_OK;
}

int kbg_create(const kbg_system* sys, int device, kbg_ctx** out) { return kbg_create_sharded(sys, device, 0, 1, out); }

int kbg_build_index(kbg_ctx* c) {
    if (!c) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        KBG_CUDA(cudaSetDevice(c->device));
        // the previous geometry's arrays go back to the pool in stream order; nothing else may still
        // be reading them
        if (c->stream2) KBG_CUDA(cudaStreamSynchronize(c->stream2));
        kbg::BuildStream bs(c->stream);
        c->built = false;
        c->hix = kbg::HostIndex();
        kbg::free_formats(c->fmt);
        kbg::build_index_device(c->P, c->ix, c->stream);
        // persistent kernels: one task queue (1 "warp") or LPT lists per consumer warp
        auto persist_tasks = [&](int sched, int split) {
            c->plan_schedule = sched;
            c->plan_split = split;
            kbg::build_tasks_device(c->P, c->ix, (sched & 1) ? 1 : kbg::kPersistConsumersH,
                                    (sched & 2) ? 1 : kbg::kPersistConsumersR, split, c->stream);
            const kbg::GridArgs gd = grid_args(c, 1, 0.0, nullptr, nullptr, true);
            const kbg::GridArgs gh = grid_args(c, 1, 0.0, nullptr, nullptr, false);
            return kbg::persist_fits(gd, true) && kbg::persist_fits(gh, false);
        };
        c->built = true;
        shard(c);
        c->persist_ok = persist_tasks(c->schedule, KBG_RHO_SPLIT);
        // The rho queue keeps per-task partial sums in shared memory (max_rtasks x 32 doubles per
        // buffer); if they do not fit next to the largest block's Phi rows, fall back to static
        // per-warp lists (~30 % slower rho).
        if (!c->persist_ok && (c->schedule & 2)) c->persist_ok = persist_tasks(c->schedule & 1, KBG_RHO_SPLIT);
        if (!c->persist_ok) kbg::build_tasks_device(c->P, c->ix, 8, 8, 8, c->stream);
        // owned blocks, heaviest first (stable: ties in block order), for the persistent kernels'
        // work counter -- a stable device radix sort, no host round trip
        kbg::pool_free(c->ix.order);
        c->ix.order = nullptr;
        c->ix.norder = c->blk_end - c->blk_begin;
        bool heavy_first = c->block_order == 0;
        if (c->block_order == 2) {
            int sms = 148;
            KBG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
            heavy_first = c->blk_end - c->blk_begin <= static_cast<int64_t>(500) * sms;
        }
        kbg::block_order_device(c->ix, c->blk_begin, c->blk_end, heavy_first, c->stream);
        if (!c->d_counter) KBG_CUDA(cudaMalloc(&c->d_counter, 2 * sizeof(int)));
        if (c->persist_ok) {
            kbg::build_cache_device(grid_args(c, 1, 0.0, nullptr, nullptr, false),
                                    grid_args(c, 1, 0.0, nullptr, nullptr, true), c->ix, c->stream);
        }
    });
}

int kbg_plan_info(const kbg_ctx* c, int64_t info[8]) {
    if (!c || !info) return KBG_ERR_CONFIG;
    if (!c->built) return KBG_ERR_CONFIG;
    kbg_ctx* m = const_cast<kbg_ctx*>(c);
    info[0] = c->persist_ok ? 1 : 0;
    info[1] = c->plan_schedule;
    info[2] = c->plan_split;
    info[3] = c->ix.max_rows_padded;
    info[4] = c->ix.max_htask;
    info[5] = c->ix.max_rtask;
    info[6] = static_cast<int64_t>(kbg::persist_smem(grid_args(m, 1, 0.0, nullptr, nullptr, false), false));
    info[7] = static_cast<int64_t>(kbg::persist_smem(grid_args(m, 1, 0.0, nullptr, nullptr, true), true));
    return KBG_OK;
}

int kbg_index_view(kbg_ctx* c, kbg_index* out) {
    if (!c || !out) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        require_index(c);
        KBG_CUDA(cudaSetDevice(c->device));
        if (!c->hix.valid) kbg::copy_index_to_host(c->ix, c->hix, c->stream);
        std::memset(out, 0, sizeof(*out));
        out->npts = c->npts;
        for (int i = 0; i < 3; ++i) out->nblk[i] = c->P.nblk[i];
        out->nblock = c->ix.nblock;
        out->ncover = c->ix.ncover;
        out->blk_ptr = c->hix.blk_ptr.data();
        out->cov_atom = c->hix.cov_atom.data();
        out->cov_R = c->hix.cov_R.data();
        out->cov_mask = c->hix.cov_mask.data();
        out->npair = c->ix.npair;
        out->pair_a = c->hix.pair_a.data();
        out->pair_b = c->hix.pair_b.data();
        out->pair_R = c->hix.pair_R.data();
        out->pair_off = c->hix.pair_off.data();
        out->pair_mirror = c->hix.pair_mirror.data();
        out->nnz = c->ix.nnz;
        out->nbpair = c->ix.nbpair;
        out->natompt = c->ix.natompt;
        out->sum_m = c->ix.sum_m;
        out->sum_m2 = c->ix.sum_m2;
    });
}

int kbg_shard_range(const kbg_ctx* c, int64_t* b0, int64_t* b1) {
    if (!c || !b0 || !b1) return KBG_ERR_CONFIG;
    if (!c->built) return KBG_ERR_CONFIG;
    *b0 = c->blk_begin;
    *b1 = c->blk_end;
    return KBG_OK;
}

int kbg_density_dev(kbg_ctx* c, int nspin, const double* d_dm, double* d_rho, void* stream) {
    if (!c || !d_dm || !d_rho) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nspin(nspin);
        require_index(c);
        KBG_CUDA(cudaSetDevice(c->device));
        c->last_launches = run_density(c, nspin, d_dm, d_rho, static_cast<cudaStream_t>(stream));
        c->tally.flops = nspin * (2.0 * c->ix.sum_m2 + 2.0 * c->ix.sum_m);
        c->tally.bytes = 8.0 * nspin * (c->ix.nnz + c->npts);
    });
}

int kbg_hamiltonian_accumulate_dev(kbg_ctx* c, int nspin, const double* d_veff, double dV, double* d_h,
                                   void* stream) {
    if (!c || !d_veff || !d_h) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nspin(nspin);
        require_index(c);
        KBG_CUDA(cudaSetDevice(c->device));
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        double* acc = h_acc_buffer(c, nspin, d_h);
        c->last_launches = h_accumulate(c, nspin, dV, d_veff, acc, st);
        if (c->det) c->last_launches += kbg::launch_finalize(c->ix, c->P, nspin, acc, d_h, false, st, h_limbs(c));
        c->tally.flops = nspin * 2.0 * c->ix.sum_m2;
        c->tally.bytes = 8.0 * nspin * (c->ix.nnz + c->npts);
    });
}

// KBG_OPT_FUSED_PASS = 2 (auto): the fused pass while nspin * (repacked DM + H) stays below this
constexpr double kFusedAutoBytes = 24.0 * (1 << 20);

int kbg_grid_pass_dev(kbg_ctx* c, int nspin, const double* d_dm, const double* d_veff, double dV, double* d_rho,
                      double* d_h, void* stream) {
    if (!c || !d_dm || !d_veff || !d_rho || !d_h) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nspin(nspin);
        require_index(c);
        KBG_CUDA(cudaSetDevice(c->device));
        if (c->nranks > 1) throw Error(KBG_ERR_CONFIG, "grid_pass_dev: single-rank contexts only");
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        int n = 0;
        // auto: the fused kernel wins while the repacked DM and the H accumulator share L2 without
        // contention (56 atoms 0.649 vs 0.660 ms) and loses once they do not (448 atoms, 2 x 30 MB: 5.53 vs 4.89)
        const double fused_bytes = 8.0 * nspin * static_cast<double>(c->ix.nrep + c->ix.nnz);
        const bool fused_want = c->fused == 1 || (c->fused == 2 && fused_bytes <= kFusedAutoBytes);
        const bool fused_ok = fused_want && c->persist_ok && c->persist && c->ix.phis && !c->det &&
                              c->sparse_thr == 0 && c->scatter == 0;
        kbg::GridArgs gh = grid_args(c, nspin, dV, d_veff, d_h, false);
        kbg::GridArgs gr = grid_args(c, nspin, 0.0, d_dm, d_rho, true);
        if (fused_ok && kbg::fused_fits(gh, gr)) {
            ensure(c->d_dmr, c->cap_dmr, static_cast<size_t>(nspin) * std::max<int64_t>(1, c->ix.nrep));
            gr.dmr = c->d_dmr;
            n += kbg::launch_dm_repack(c->ix, c->P, nspin, d_dm, c->d_dmr, st);
            KBG_CUDA(cudaMemsetAsync(d_h, 0, static_cast<size_t>(nspin) * c->ix.nnz * sizeof(double), st));
            KBG_CUDA(cudaMemsetAsync(c->d_vbits, 0, sizeof(unsigned long long), st));
            n += kbg::launch_fused(gh, gr, st);
        } else {
            n += run_density(c, nspin, d_dm, d_rho, st);
            double* acc = h_acc_buffer(c, nspin, d_h);
            n += h_accumulate(c, nspin, dV, d_veff, acc, st);
            if (c->det) {
                n += kbg::launch_finalize(c->ix, c->P, nspin, acc, d_h, true, st, h_limbs(c));
                c->last_launches = n;
                return;
            }
        }
        n += kbg::launch_mirror(c->ix, c->P, nspin, d_h, st);
        c->last_launches = n;
        c->tally.flops = nspin * (4.0 * c->ix.sum_m2 + 2.0 * c->ix.sum_m);
        c->tally.bytes = 16.0 * nspin * (c->ix.nnz + c->npts);
    });
}

int kbg_hamiltonian_mirror_dev(kbg_ctx* c, int nspin, double* d_h, void* stream) {
    if (!c || !d_h) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nspin(nspin);
        require_index(c);
        KBG_CUDA(cudaSetDevice(c->device));
        c->last_launches = kbg::launch_mirror(c->ix, c->P, nspin, d_h, static_cast<cudaStream_t>(stream));
    });
}

int kbg_hamiltonian_dev(kbg_ctx* c, int nspin, const double* d_veff, double dV, double* d_h, void* stream) {
    if (c && c->det) {  // accumulate + one fused finalize/mirror kernel
        if (!d_veff || !d_h) return KBG_ERR_CONFIG;
        return guard(c, [&] {
            check_nspin(nspin);
            require_index(c);
            KBG_CUDA(cudaSetDevice(c->device));
            const cudaStream_t st = static_cast<cudaStream_t>(stream);
            double* acc = h_acc_buffer(c, nspin, d_h);
            c->last_launches = h_accumulate(c, nspin, dV, d_veff, acc, st);
            c->last_launches += kbg::launch_finalize(c->ix, c->P, nspin, acc, d_h, true, st, h_limbs(c));
            c->tally.flops = nspin * 2.0 * c->ix.sum_m2;
            c->tally.bytes = 8.0 * nspin * (c->ix.nnz + c->npts);
        });
    }
    int st = kbg_hamiltonian_accumulate_dev(c, nspin, d_veff, dV, d_h, stream);
    if (st != KBG_OK) return st;
    const int n1 = c->last_launches;
    const kbg_tally t = c->tally;
    st = kbg_hamiltonian_mirror_dev(c, nspin, d_h, stream);
    if (st != KBG_OK) return st;
    c->last_launches += n1;
    c->tally = t;
    return KBG_OK;
}

int kbg_density(kbg_ctx* c, int nspin, const double* dm, double* rho) {
    if (!c || !dm || !rho) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nspin(nspin);
        require_index(c);
        KBG_CUDA(cudaSetDevice(c->device));
        const size_t nin = static_cast<size_t>(nspin) * c->ix.nnz, nout = static_cast<size_t>(nspin) * c->npts;
        ensure(c->d_in, c->cap_in, nin);
        ensure(c->d_out, c->cap_out, nout);
        KBG_CUDA(cudaMemcpyAsync(c->d_in, dm, nin * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        KBG_CUDA(cudaMemsetAsync(c->d_check, 0, 4 * sizeof(unsigned long long), c->stream));
        kbg::launch_dm_check(c->ix, c->P, nspin, c->d_in, c->d_check, c->stream);
        unsigned long long chk[4];
        KBG_CUDA(cudaMemcpyAsync(chk, c->d_check, sizeof(chk), cudaMemcpyDeviceToHost, c->stream));
        KBG_CUDA(cudaStreamSynchronize(c->stream));
        double dmax, amax;
        std::memcpy(&dmax, &chk[0], 8);
        std::memcpy(&amax, &chk[1], 8);
        if (chk[2]) throw Error(KBG_ERR_NONFINITE, "density: non-finite density-matrix entry");
        if (dmax > 1e-13 * amax)
            throw Error(KBG_ERR_CONSISTENCY, "density: DM violates DM_ba(-R) = DM_ab(R)^T by " + std::to_string(dmax));
        if (c->nranks > 1) KBG_CUDA(cudaMemsetAsync(c->d_out, 0, nout * sizeof(double), c->stream));
        c->last_launches = 1 + run_density(c, nspin, c->d_in, c->d_out, c->stream);
        KBG_CUDA(cudaMemcpyAsync(rho, c->d_out, nout * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        KBG_CUDA(cudaStreamSynchronize(c->stream));
        c->tally.flops = nspin * (2.0 * c->ix.sum_m2 + 2.0 * c->ix.sum_m);
        c->tally.bytes = 8.0 * nspin * (c->ix.nnz + c->npts);
    });
}

int kbg_hamiltonian(kbg_ctx* c, int nspin, const double* veff, double dV, double* h) {
    if (!c || !veff || !h) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nspin(nspin);
        require_index(c);
        if (!std::isfinite(dV)) throw Error(KBG_ERR_NONFINITE, "hamiltonian: non-finite dV");
        KBG_CUDA(cudaSetDevice(c->device));
        const size_t nin = static_cast<size_t>(nspin) * c->npts, nout = static_cast<size_t>(nspin) * c->ix.nnz;
        ensure(c->d_in, c->cap_in, nin);
        ensure(c->d_out, c->cap_out, nout);
        // deterministic H needs max|V| before the first contribution: V goes to the device first
        const double* v_map = c->det ? nullptr : mapped_input(c, veff);
        if (!v_map) KBG_CUDA(cudaMemcpyAsync(c->d_in, veff, nin * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        double* acc = h_acc_buffer(c, nspin, c->d_out);
        int n = h_accumulate(c, nspin, dV, v_map ? v_map : c->d_in, acc, c->stream);
        if (c->det)
            n += kbg::launch_finalize(c->ix, c->P, nspin, acc, c->d_out, true, c->stream, h_limbs(c));
        else
            n += kbg::launch_mirror(c->ix, c->P, nspin, c->d_out, c->stream);
        c->last_launches = n;
        KBG_CUDA(cudaMemcpyAsync(h, c->d_out, nout * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        KBG_CUDA(cudaStreamSynchronize(c->stream));
        check_vbits(c, "hamiltonian");
        c->tally.flops = nspin * 2.0 * c->ix.sum_m2;
        c->tally.bytes = 8.0 * nspin * (c->ix.nnz + c->npts);
    });
}

namespace {
// Host-to-device copy of the DM pair blocks a shard reads (c->dm_runs, per spin): one cudaMemcpyAsync
// per run on c->stream (copy engine; overlaps the H kernel on the other stream). kbg_comm_open merges
// the runs to at most kMaxDmRuns, so the host issues only a few dozen copies per call.
void dm_run_copy(kbg_ctx* c, int nspin, const double* dm) {
    const size_t nr = c->dm_runs.size() / 2;
    for (int s = 0; s < nspin; ++s)
        for (size_t r = 0; r < nr; ++r) {
            const int64_t o = s * c->ix.nnz + c->dm_runs[2 * r];
            KBG_CUDA(cudaMemcpyAsync(c->d_in + o, dm + o, static_cast<size_t>(c->dm_runs[2 * r + 1]) * sizeof(double),
                                     cudaMemcpyHostToDevice, c->stream));
        }
}
}  // namespace

int kbg_grid_pass(kbg_ctx* c, int nspin, const double* dm, const double* veff, double dV, double* rho, double* h) {
    if (!c || !dm || !veff || !rho || !h) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nspin(nspin);
        require_index(c);
        if (!std::isfinite(dV)) throw Error(KBG_ERR_NONFINITE, "grid_pass: non-finite dV");
        KBG_CUDA(cudaSetDevice(c->device));
        if (!c->stream2) KBG_CUDA(cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking));
        if (!c->ev_pass) KBG_CUDA(cudaEventCreateWithFlags(&c->ev_pass, cudaEventDisableTiming));
        if (!c->ev_rho) KBG_CUDA(cudaEventCreateWithFlags(&c->ev_rho, cudaEventDisableTiming));
        const size_t ndm = static_cast<size_t>(nspin) * c->ix.nnz, npt = static_cast<size_t>(nspin) * c->npts;
        ensure(c->d_in, c->cap_in, ndm);
        ensure(c->d_out, c->cap_out, npt);
        ensure(c->d_in2, c->cap_in2, npt);
        ensure(c->d_out2, c->cap_out2, ndm);
        if (!c->h_flags) KBG_CUDA(cudaMallocHost(&c->h_flags, 8 * sizeof(unsigned long long)));
        // stream 2: V in -> H -> mirror -> H out; stream 1: DM in -> symmetry check -> rho -> rho out.
        // The copies of one half overlap the kernels of the other. H goes first: its input (npts) is the
        // smaller one to wait for and rho (npts) the smaller output left after the last kernel. The DM
        // check is read at the end.
        int n = 0;
        // KBG_PHASE_TIMING=1 (diagnostic): events at the phase boundaries of both streams, printed to stderr
        static const bool kPhase = std::getenv("KBG_PHASE_TIMING") != nullptr;
        const auto t_entry = std::chrono::steady_clock::now();
        std::vector<std::pair<const char*, cudaEvent_t>> ph;
        auto mark = [&](const char* what, cudaStream_t s) {
            if (!kPhase) return;
            cudaEvent_t e;
            KBG_CUDA(cudaEventCreate(&e));
            KBG_CUDA(cudaEventRecord(e, s));
            ph.emplace_back(what, e);
        };
        mark("start", c->stream2);
        // Legacy H: V from pinned host memory is read in place by the H kernel (mapped_input), so the
        // first DMMAs do not wait for a whole-array copy. Deterministic H needs max|V| before the
        // first contribution: V is copied first, at the full PCIe bandwidth (the DM copy waits for
        // it, ev_pass), then the H pass runs while the DM crosses.
        const double* v_map = c->det ? nullptr : mapped_input(c, veff);
        double* rho_map = mapped_output(c, rho);
        // Shard-local host transfers (sharded context with the peer exchange open, KBG_OPT_SHARD_IO):
        // the repack reads only the DM pairs this rank's blocks touch (in place from pinned memory),
        // rho is written only at the rank's points (in place when pinned, else the D2H covers just
        // its plane range), and H -- complete on every rank after the fused reduction -- leaves only
        // the rank's slice [io[4], io[5]) of each spin. kbg_shard_io reports the ranges.
        const bool sio = c->comm_ready && c->shard_io;
        // exchange right after the H accumulate (default; KBG_XCHG_FIRST=0: after the density pass)
        const char* xf_env = std::getenv("KBG_XCHG_FIRST");
        const bool xfirst = !(xf_env && xf_env[0] == '0');
        // pinned DM on a shard: its pair blocks are gathered in place (KBG_NO_DM_GATHER: memcpy runs)
        const char* ng_env = std::getenv("KBG_NO_DM_GATHER");
        const double* dm_map = sio && c->d_xruns && !(ng_env && ng_env[0] == '1') ? mapped_input(c, dm) : nullptr;
        const bool dm_gathered = dm_map != nullptr;
        auto rho_half = [&](bool after_exchange) {
            if (c->det) KBG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_pass, 0));
            // the DM crosses on the copy engine while the H kernel computes; a shard copies only the pair
            // blocks its rho reads (a few dozen copies of their merged contiguous runs)
            mark("s1 start", c->stream);
            if (dm_gathered) {
                // the pair blocks were fetched in place by k_dm_gather (launched ahead of the H kernel)
            } else if (sio && !c->dm_runs.empty())
                dm_run_copy(c, nspin, dm);
            else
                KBG_CUDA(cudaMemcpyAsync(c->d_in, dm, ndm * sizeof(double), cudaMemcpyHostToDevice, c->stream));
            mark("s1 dm copied", c->stream);
            KBG_CUDA(cudaMemsetAsync(c->d_check, 0, 4 * sizeof(unsigned long long), c->stream));
            if (c->nranks > 1 && !rho_map) KBG_CUDA(cudaMemsetAsync(c->d_out, 0, npt * sizeof(double), c->stream));
            if (after_exchange) KBG_CUDA(cudaStreamWaitEvent(c->stream, c->ev_rho, 0));
            // the DM symmetry check rides along in the repack pass (no separate k_dm_check)
            n += run_density(c, nspin, c->d_in, rho_map ? rho_map : c->d_out, c->stream, c->d_check,
                             sio ? c->d_pown : nullptr);
            mark("s1 density done", c->stream);
            if (!rho_map) {
                if (sio) {
                    const int64_t p0 = c->io[2], p1 = c->io[3];
                    for (int s = 0; s < nspin; ++s)
                        if (p1 > p0)
                            KBG_CUDA(cudaMemcpyAsync(rho + s * c->npts + p0, c->d_out + s * c->npts + p0,
                                                     (p1 - p0) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
                } else {
                    KBG_CUDA(cudaMemcpyAsync(rho, c->d_out, npt * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
                }
            }
            mark("s1 rho out", c->stream);
        };
        auto h_half = [&] {
            if (!v_map)
                KBG_CUDA(cudaMemcpyAsync(c->d_in2, veff, npt * sizeof(double), cudaMemcpyHostToDevice, c->stream2));
            KBG_CUDA(cudaEventRecord(c->ev_pass, c->stream2));
            const double* vin = v_map ? v_map : c->d_in2;
            if (c->comm_ready) {
                // sharded: partials into the peer-mapped exchange buffer, then the fused reduce +
                // mirror over NVLink (kb_comm.cu) -- the full H on every rank. The reduce waits for this
                // rank's density kernel (ev_rho): the rank spread and the flag round trip hide behind it,
                // and its spinning CTAs never keep the density kernel off the SMs.
                if (dm_gathered) n += kbg::launch_dm_gather(c->d_xruns, c->dm_xruns_n, nspin, c->ix.nnz, dm_map, c->d_in,
                                                            c->stream);
                n += h_accumulate(c, nspin, dV, vin, c->d_xbuf, c->stream2);
                mark("s2 h accumulated", c->stream2);
                if (xfirst) {
                    // exchange right after the accumulate, then the density pass (it waits for the
                    // exchange's CTAs to leave the SMs): the H slice's D2H overlaps the density kernel
                    c->epoch += 2;
                    c->comm.ls = h_limbs(c);
                    c->comm.sms = c->xsms;  // > 0: on its own SMs, next to the density kernel
                    n += kbg::launch_reduce_mirror(c->comm, c->ix, c->P, nspin, c->d_out2, c->epoch - 1, c->stream2);
                    KBG_CUDA(cudaEventRecord(c->ev_rho, c->stream2));
                    mark("s2 exchanged", c->stream2);
                    rho_half(c->xsms == 0);
                } else {
                    rho_half(false);
                    KBG_CUDA(cudaEventRecord(c->ev_rho, c->stream));
                    KBG_CUDA(cudaStreamWaitEvent(c->stream2, c->ev_rho, 0));
                    c->epoch += 2;
                    c->comm.ls = h_limbs(c);
                    c->comm.sms = 0;
                    n += kbg::launch_reduce_mirror(c->comm, c->ix, c->P, nspin, c->d_out2, c->epoch - 1, c->stream2);
                    mark("s2 exchanged", c->stream2);
                }
            } else {
                double* acc = h_acc_buffer(c, nspin, c->d_out2);
                n += h_accumulate(c, nspin, dV, vin, acc, c->stream2);
                if (c->det)
                    n += kbg::launch_finalize(c->ix, c->P, nspin, acc, c->d_out2, true, c->stream2, h_limbs(c));
                else
                    n += kbg::launch_mirror(c->ix, c->P, nspin, c->d_out2, c->stream2);
                // the density kernel starts after the mirror: otherwise its CTAs take every SM the
                // moment the H kernel ends, the mirror waits for the whole density pass and the H
                // D2H trails it (~80 us at 56 atoms); this way the D2H overlaps the density pass
                KBG_CUDA(cudaEventRecord(c->ev_rho, c->stream2));
            }
            if (sio) {
                const int64_t h0 = c->io[4], h1 = c->io[5];
                for (int s = 0; s < nspin; ++s)
                    if (h1 > h0)
                        KBG_CUDA(cudaMemcpyAsync(h + s * c->ix.nnz + h0, c->d_out2 + s * c->ix.nnz + h0,
                                                 (h1 - h0) * sizeof(double), cudaMemcpyDeviceToHost, c->stream2));
            } else {
                KBG_CUDA(cudaMemcpyAsync(h, c->d_out2, ndm * sizeof(double), cudaMemcpyDeviceToHost, c->stream2));
            }
            mark("s2 h out", c->stream2);
        };
        h_half();
        if (!c->comm_ready) rho_half(true);  // sharded: h_half runs rho_half itself
        // the DM check words and the non-finite-V flag land in pinned scratch (allocated before the
        // first launch: an allocation may synchronize, and a sharded pass must not wait on itself)
        unsigned long long* chk = c->h_flags;
        KBG_CUDA(cudaMemcpyAsync(chk, c->d_check, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
        KBG_CUDA(cudaMemcpyAsync(chk + 4, c->d_vbits, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream2));
        const auto t_issued = std::chrono::steady_clock::now();
        KBG_CUDA(cudaStreamSynchronize(c->stream2));
        KBG_CUDA(cudaStreamSynchronize(c->stream));
        const auto t_synced = std::chrono::steady_clock::now();
        if (kPhase && !ph.empty()) {
            auto us = [&](auto t) { return std::to_string(static_cast<long>(
                std::chrono::duration_cast<std::chrono::microseconds>(t - t_entry).count())); };
            std::string line = "kbg_grid_pass host (us from entry): issued " + us(t_issued) + ", synced " +
                               us(t_synced) + "; phases (us from start):";
            for (auto& e : ph) {
                float ms = 0.f;
                KBG_CUDA(cudaEventElapsedTime(&ms, ph[0].second, e.second));
                line += std::string(" [") + e.first + " " + std::to_string(static_cast<int>(ms * 1e3f)) + "]";
            }
            for (auto& e : ph) KBG_CUDA(cudaEventDestroy(e.second));
            std::fprintf(stderr, "%s\n", line.c_str());
        }
        if (c->comm_ready) comm_check(c);
        if (chk[4] >= 0x7ff0000000000000ull)
            throw Error(KBG_ERR_NONFINITE, "grid_pass: non-finite V_eff (outputs invalid)");
        c->last_launches = n;
        double dmax, amax;
        std::memcpy(&dmax, &chk[0], 8);
        std::memcpy(&amax, &chk[1], 8);
        if (chk[2]) throw Error(KBG_ERR_NONFINITE, "grid_pass: non-finite density-matrix entry (outputs invalid)");
        if (dmax > 1e-13 * amax)
            throw Error(KBG_ERR_CONSISTENCY,
                        "grid_pass: DM violates DM_ba(-R) = DM_ab(R)^T by " + std::to_string(dmax) + " (outputs invalid)");
        c->tally.flops = nspin * (4.0 * c->ix.sum_m2 + 2.0 * c->ix.sum_m);
        c->tally.bytes = 16.0 * nspin * (c->ix.nnz + c->npts);
    });
}

namespace {
double cell_dV(const kbg_ctx* c) {
    const double* A = c->P.A;
    const double det = A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
                       A[2] * (A[3] * A[7] - A[4] * A[6]);
    return std::fabs(det) / static_cast<double>(c->npts);
}
}  // namespace

int kbg_veff_dev(kbg_ctx* c, int nspin, const double* d_rho, const double* d_vloc, double* d_veff, double* d_energy,
                 void* stream) {
    if (!c || !d_rho || !d_veff) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nspin(nspin);
        KBG_CUDA(cudaSetDevice(c->device));
        c->last_launches = kbg::run_veff(c->veff, c->P.N, c->P.Ainv, nspin, c->xc, d_rho, d_vloc, cell_dV(c), d_veff,
                                         d_energy,
                                         static_cast<cudaStream_t>(stream));
        c->tally.flops = 0.0;
        c->tally.bytes = 8.0 * c->npts * (2.0 * nspin + (d_vloc ? 1.0 : 0.0));
    });
}

int kbg_veff(kbg_ctx* c, int nspin, const double* rho, const double* vloc, double* veff, double* energy) {
    if (!c || !rho || !veff) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nspin(nspin);
        KBG_CUDA(cudaSetDevice(c->device));
        const size_t n = static_cast<size_t>(c->npts);
        ensure(c->d_in2, c->cap_in2, 2 * n * nspin + n + 2);
        double* d_rho = c->d_in2;
        double* d_v = d_rho + n * nspin;
        double* d_vloc = vloc ? d_v + n * nspin : nullptr;
        double* d_e = d_v + n * nspin + n;
        KBG_CUDA(cudaMemcpyAsync(d_rho, rho, n * nspin * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        if (vloc) KBG_CUDA(cudaMemcpyAsync(d_vloc, vloc, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        // every rho value is checked on the device (k_rho_total) -- kband raises on any non-finite
        // input (householder.cpp:119-123)
        unsigned int* d_bad = reinterpret_cast<unsigned int*>(c->d_check + 3);
        KBG_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(unsigned int), c->stream));
        c->last_launches = kbg::run_veff(c->veff, c->P.N, c->P.Ainv, nspin, c->xc, d_rho, d_vloc, cell_dV(c), d_v, d_e,
                                         c->stream, d_bad);
        KBG_CUDA(cudaMemcpyAsync(veff, d_v, n * nspin * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        double e[2];
        unsigned int bad = 0;
        KBG_CUDA(cudaMemcpyAsync(e, d_e, sizeof(e), cudaMemcpyDeviceToHost, c->stream));
        KBG_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, c->stream));
        KBG_CUDA(cudaStreamSynchronize(c->stream));
        if (bad) throw Error(KBG_ERR_NONFINITE, "veff: non-finite rho (outputs invalid)");
        if (energy) std::memcpy(energy, e, sizeof(e));
    });
}

int kbg_block_orbitals(kbg_ctx* c, int64_t block, double* out, int64_t cap, int* m_out) {
    if (!c || !out || !m_out) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        require_index(c);
        if (block < 0 || block >= c->ix.nblock) throw Error(KBG_ERR_DIMENSION, "block_orbitals: bad block");
        KBG_CUDA(cudaSetDevice(c->device));
        if (!c->hix.valid) kbg::copy_index_to_host(c->ix, c->hix, c->stream);
        int M = 0;
        for (int e = c->hix.blk_ptr[block]; e < c->hix.blk_ptr[block + 1]; ++e)
            M += c->P.sp[c->h_spc[c->hix.cov_atom[e]]].norb;
        *m_out = M;
        if (static_cast<int64_t>(M) * 64 > cap) throw Error(KBG_ERR_DIMENSION, "block_orbitals: cap too small");
        if (M == 0) return;
        ensure(c->d_out, c->cap_out, static_cast<size_t>(M) * 64);
        const kbg::GridArgs g = grid_args(c, 1, 0.0, nullptr, nullptr, false);
        kbg::launch_block_orbitals(g, block, c->d_out, c->stream);
        KBG_CUDA(cudaMemcpyAsync(out, c->d_out, sizeof(double) * M * 64, cudaMemcpyDeviceToHost, c->stream));
        KBG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int kbg_last_launches(const kbg_ctx* c) { return c ? c->last_launches : 0; }

int kbg_debug_counters(kbg_ctx* c, int64_t* out, int n) {
    if (!c || !out || n < 0) return KBG_ERR_CONFIG;
    for (int i = 0; i < n; ++i) out[i] = 0;
    if (!c->d_dbg) return KBG_OK;
    unsigned long long h[16];
    if (cudaMemcpy(h, c->d_dbg, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return KBG_ERR_CUDA;
    for (int i = 0; i < n && i < 16; ++i) out[i] = static_cast<int64_t>(h[i]);
    return KBG_OK;
}

// ---- formats either side of the grid pass (kb_formats.cu) -------------------
namespace {

const kbg::FormatIndex& formats(kbg_ctx* c) {
    require_index(c);
    kbg::FormatIndex& f = c->fmt;
    if (f.valid) return f;
    if (!c->hix.valid) kbg::copy_index_to_host(c->ix, c->hix, c->stream);
    const kbg::HostIndex& h = c->hix;
    const int natom = c->P.natom;
    std::vector<int32_t> off(natom + 1, 0), atom;
    for (int a = 0; a < natom; ++a) off[a + 1] = off[a] + c->P.sp[c->h_spc[a]].norb;
    for (int a = 0; a < natom; ++a) atom.insert(atom.end(), off[a + 1] - off[a], a);
    const int64_t npair = c->ix.npair;
    std::vector<std::array<int32_t, 3>> R(npair);
    for (int64_t p = 0; p < npair; ++p) R[p] = {h.pair_R[3 * p], h.pair_R[3 * p + 1], h.pair_R[3 * p + 2]};
    std::vector<std::array<int32_t, 3>> uniq = R;
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    std::vector<int32_t> rid(npair), run(2 * static_cast<size_t>(natom) * natom, 0), runs;
    for (int64_t p = 0; p < npair; ++p) {
        rid[p] = static_cast<int32_t>(std::lower_bound(uniq.begin(), uniq.end(), R[p]) - uniq.begin());
        const size_t ab = static_cast<size_t>(h.pair_a[p]) * natom + h.pair_b[p];
        if (run[2 * ab] == run[2 * ab + 1]) {  // pairs sorted by (a, b, R): first pair of a run
            run[2 * ab] = static_cast<int32_t>(p);
            runs.push_back(static_cast<int32_t>(p));
        }
        run[2 * ab + 1] = static_cast<int32_t>(p + 1);
    }
    runs.push_back(static_cast<int32_t>(npair));
    f.n = off[natom];
    f.natom = natom;
    f.nR = static_cast<int>(uniq.size());
    f.R.clear();
    for (const auto& r : uniq) f.R.insert(f.R.end(), r.begin(), r.end());
    auto up = [&](int32_t*& d, const std::vector<int32_t>& v) {
        KBG_CUDA(cudaMalloc(&d, std::max<size_t>(1, v.size()) * sizeof(int32_t)));
        if (!v.empty()) KBG_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    };
    up(f.orb_atom, atom);
    up(f.orb_off, off);
    up(f.run, run);
    up(f.rid, rid);
    up(f.runs, runs);
    f.nrun = static_cast<int>(runs.size()) - 1;
    f.valid = true;
    return f;
}

void check_nk(int nk, const double* kpts) {
    if (nk < 1) throw Error(KBG_ERR_CONFIG, "nk must be >= 1");
    if (!kpts) throw Error(KBG_ERR_CONFIG, "null k points");
    for (int i = 0; i < 3 * nk; ++i)
        if (!std::isfinite(kpts[i])) throw Error(KBG_ERR_NONFINITE, "k point " + std::to_string(i / 3) + " is not finite");
}

// k points (and weights) to the device, phases exp(sign 2 pi i k.R_p) per (k, pair)
const double2* phases(kbg_ctx* c, int nk, const double* kpts, const double* w, double sign, cudaStream_t st) {
    const size_t nkw = 4 * static_cast<size_t>(nk);
    ensure(c->d_kw, c->cap_kw, nkw);
    if (!c->h_kw_done) KBG_CUDA(cudaEventCreateWithFlags(&c->h_kw_done, cudaEventDisableTiming));
    KBG_CUDA(cudaEventSynchronize(c->h_kw_done));  // previous copy out of the staging buffer is done
    if (c->cap_hkw < nkw) {
        if (c->h_kw) cudaFreeHost(c->h_kw);
        c->h_kw = nullptr;
        KBG_CUDA(cudaMallocHost(&c->h_kw, nkw * sizeof(double)));
        c->cap_hkw = nkw;
    }
    std::copy(kpts, kpts + 3 * nk, c->h_kw);
    if (w) std::copy(w, w + nk, c->h_kw + 3 * nk);
    KBG_CUDA(cudaMemcpyAsync(c->d_kw, c->h_kw, nkw * sizeof(double), cudaMemcpyHostToDevice, st));
    KBG_CUDA(cudaEventRecord(c->h_kw_done, st));
    ensure(c->d_phase, c->cap_phase, 2 * static_cast<size_t>(nk) * std::max<int64_t>(1, c->ix.npair));
    c->last_launches =
        kbg::launch_phase(nk, c->ix.npair, c->d_kw, c->ix.pair_R, sign, reinterpret_cast<double2*>(c->d_phase), st);
    return reinterpret_cast<const double2*>(c->d_phase);
}

// M_{-R} = M_R^T check of one matrix already on the device (host API only);
// names the first offending pair.
void check_hermitian(kbg_ctx* c, const double* d_pairs, const double* h_pairs, const char* who) {
    KBG_CUDA(cudaMemsetAsync(c->d_check, 0, 4 * sizeof(unsigned long long), c->stream));
    kbg::launch_dm_check(c->ix, c->P, 1, d_pairs, c->d_check, c->stream);
    unsigned long long chk[4];
    KBG_CUDA(cudaMemcpyAsync(chk, c->d_check, sizeof(chk), cudaMemcpyDeviceToHost, c->stream));
    KBG_CUDA(cudaStreamSynchronize(c->stream));
    double dmax, amax;
    std::memcpy(&dmax, &chk[0], 8);
    std::memcpy(&amax, &chk[1], 8);
    if (chk[2]) throw Error(KBG_ERR_NONFINITE, std::string(who) + ": non-finite entry");
    if (dmax <= 1e-13 * amax) return;
    if (!c->hix.valid) kbg::copy_index_to_host(c->ix, c->hix, c->stream);
    const kbg::HostIndex& h = c->hix;
    for (int64_t p = 0; p < c->ix.npair; ++p) {
        const int na = c->P.sp[c->h_spc[h.pair_a[p]]].norb, nb = c->P.sp[c->h_spc[h.pair_b[p]]].norb;
        const int64_t q = h.pair_mirror[p];
        for (int i = 0; i < na; ++i)
            for (int j = 0; j < nb; ++j)
                if (std::fabs(h_pairs[h.pair_off[p] + i * nb + j] - h_pairs[h.pair_off[q] + j * na + i]) > 1e-13 * amax)
                    throw Error(KBG_ERR_CONSISTENCY,
                                std::string(who) + ": M_{-R} != M_R^T at pair " + std::to_string(p) + " (a=" +
                                    std::to_string(h.pair_a[p]) + ", b=" + std::to_string(h.pair_b[p]) + ", R=(" +
                                    std::to_string(h.pair_R[3 * p]) + "," + std::to_string(h.pair_R[3 * p + 1]) + "," +
                                    std::to_string(h.pair_R[3 * p + 2]) + ")) by " + std::to_string(dmax));
    }
}

}  // namespace

int kbg_offsets(kbg_ctx* c, int* nR, int32_t* R) {
    if (!c || !nR) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        KBG_CUDA(cudaSetDevice(c->device));
        const kbg::FormatIndex& f = formats(c);
        *nR = f.nR;
        if (R) std::copy(f.R.begin(), f.R.end(), R);
    });
}

int kbg_to_realspace_dev(kbg_ctx* c, const double* d_pairs, double* d_blocks, void* stream) {
    if (!c || !d_pairs || !d_blocks) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        KBG_CUDA(cudaSetDevice(c->device));
        const kbg::FormatIndex& f = formats(c);
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        KBG_CUDA(cudaMemsetAsync(d_blocks, 0, sizeof(double) * f.nR * f.n * f.n, st));
        c->last_launches = kbg::launch_realspace(f, c->ix, true, const_cast<double*>(d_pairs), d_blocks, st);
    });
}

int kbg_from_realspace_dev(kbg_ctx* c, const double* d_blocks, double* d_pairs, void* stream) {
    if (!c || !d_pairs || !d_blocks) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        KBG_CUDA(cudaSetDevice(c->device));
        const kbg::FormatIndex& f = formats(c);
        c->last_launches = kbg::launch_realspace(f, c->ix, false, d_pairs, const_cast<double*>(d_blocks),
                                                 static_cast<cudaStream_t>(stream));
    });
}

int kbg_to_realspace(kbg_ctx* c, const double* pairs, double* blocks) {
    if (!c || !pairs || !blocks) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        KBG_CUDA(cudaSetDevice(c->device));
        const kbg::FormatIndex& f = formats(c);
        const size_t nd = static_cast<size_t>(f.nR) * f.n * f.n;
        ensure(c->d_fa, c->cap_fa, c->ix.nnz);
        ensure(c->d_fb, c->cap_fb, nd);
        KBG_CUDA(cudaMemcpyAsync(c->d_fa, pairs, c->ix.nnz * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        KBG_CUDA(cudaMemsetAsync(c->d_fb, 0, nd * sizeof(double), c->stream));
        c->last_launches = kbg::launch_realspace(f, c->ix, true, c->d_fa, c->d_fb, c->stream);
        KBG_CUDA(cudaMemcpyAsync(blocks, c->d_fb, nd * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        KBG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int kbg_from_realspace(kbg_ctx* c, const double* blocks, double* pairs) {
    if (!c || !pairs || !blocks) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        KBG_CUDA(cudaSetDevice(c->device));
        const kbg::FormatIndex& f = formats(c);
        const size_t nd = static_cast<size_t>(f.nR) * f.n * f.n;
        ensure(c->d_fa, c->cap_fa, c->ix.nnz);
        ensure(c->d_fb, c->cap_fb, nd);
        KBG_CUDA(cudaMemcpyAsync(c->d_fb, blocks, nd * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        c->last_launches = kbg::launch_realspace(f, c->ix, false, c->d_fa, c->d_fb, c->stream);
        KBG_CUDA(cudaMemcpyAsync(pairs, c->d_fa, c->ix.nnz * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        KBG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int kbg_bloch_dev(kbg_ctx* c, const double* d_pairs, int nk, const double* kpts, double* d_out, void* stream) {
    if (!c || !d_pairs || !d_out) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nk(nk, kpts);
        KBG_CUDA(cudaSetDevice(c->device));
        const kbg::FormatIndex& f = formats(c);
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        const double2* ph = phases(c, nk, kpts, nullptr, 1.0, st);
        c->last_launches += kbg::launch_bloch(f, c->ix, nk, d_pairs, ph, d_out, st);
        c->tally.flops = 4.0 * nk * c->ix.nnz;
        c->tally.bytes = 8.0 * c->ix.nnz + 16.0 * nk * f.n * f.n;
    });
}

int kbg_bloch(kbg_ctx* c, const double* pairs, int nk, const double* kpts, double* out) {
    if (!c || !pairs || !out) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nk(nk, kpts);
        KBG_CUDA(cudaSetDevice(c->device));
        const kbg::FormatIndex& f = formats(c);
        const size_t nd = 2 * static_cast<size_t>(nk) * f.n * f.n;
        ensure(c->d_fa, c->cap_fa, c->ix.nnz);
        ensure(c->d_fb, c->cap_fb, nd);
        KBG_CUDA(cudaMemcpyAsync(c->d_fa, pairs, c->ix.nnz * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        check_hermitian(c, c->d_fa, pairs, "bloch");
        const double2* ph = phases(c, nk, kpts, nullptr, 1.0, c->stream);
        c->last_launches += 1 + kbg::launch_bloch(f, c->ix, nk, c->d_fa, ph, c->d_fb, c->stream);
        KBG_CUDA(cudaMemcpyAsync(out, c->d_fb, nd * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        KBG_CUDA(cudaStreamSynchronize(c->stream));
        c->tally.flops = 4.0 * nk * c->ix.nnz;
        c->tally.bytes = 8.0 * c->ix.nnz + 16.0 * nk * f.n * f.n;
    });
}

int kbg_fold_dev(kbg_ctx* c, int nk, const double* kpts, const double* w, const double* d_rho_k, double* d_pairs,
                 void* stream) {
    if (!c || !w || !d_rho_k || !d_pairs) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nk(nk, kpts);
        KBG_CUDA(cudaSetDevice(c->device));
        const kbg::FormatIndex& f = formats(c);
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        const double2* ph = phases(c, nk, kpts, w, -1.0, st);
        c->last_launches += kbg::launch_fold(f, c->ix, nk, c->d_kw + 3 * nk, ph, d_rho_k, d_pairs, nullptr, st);
        c->tally.flops = 8.0 * nk * c->ix.nnz;
        c->tally.bytes = 8.0 * c->ix.nnz + 16.0 * nk * c->ix.nnz;
    });
}

int kbg_fold(kbg_ctx* c, int nk, const double* kpts, const double* w, const double* rho_k, double* pairs,
             double* max_imag) {
    if (!c || !w || !rho_k || !pairs) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nk(nk, kpts);
        for (int k = 0; k < nk; ++k)
            if (!std::isfinite(w[k])) throw Error(KBG_ERR_NONFINITE, "fold: weight " + std::to_string(k) + " is not finite");
        KBG_CUDA(cudaSetDevice(c->device));
        const kbg::FormatIndex& f = formats(c);
        const size_t nd = 2 * static_cast<size_t>(nk) * f.n * f.n;
        ensure(c->d_fa, c->cap_fa, c->ix.nnz);
        ensure(c->d_fb, c->cap_fb, nd);
        KBG_CUDA(cudaMemcpyAsync(c->d_fb, rho_k, nd * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        const double2* ph = phases(c, nk, kpts, w, -1.0, c->stream);
        KBG_CUDA(cudaMemsetAsync(c->d_check, 0, 4 * sizeof(unsigned long long), c->stream));
        c->last_launches +=
            kbg::launch_fold(f, c->ix, nk, c->d_kw + 3 * nk, ph, c->d_fb, c->d_fa, c->d_check, c->stream);
        unsigned long long mi = 0;
        KBG_CUDA(cudaMemcpyAsync(pairs, c->d_fa, c->ix.nnz * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        KBG_CUDA(cudaMemcpyAsync(&mi, c->d_check, sizeof(mi), cudaMemcpyDeviceToHost, c->stream));
        KBG_CUDA(cudaStreamSynchronize(c->stream));
        if (max_imag) std::memcpy(max_imag, &mi, sizeof(double));
        c->tally.flops = 8.0 * nk * c->ix.nnz;
        c->tally.bytes = 8.0 * c->ix.nnz + 16.0 * nk * c->ix.nnz;
    });
}

namespace {

void density_matrix_k(kbg_ctx* c, int m, const double* d_C, const double* d_w, double* d_rho, cudaStream_t st) {
    const int n = formats(c).n;
    if (m < 1 || m > n) throw Error(KBG_ERR_DIMENSION, "density_matrix_k: m = " + std::to_string(m) +
                                                           " states for n = " + std::to_string(n) + " orbitals");
    if (!c->blas && cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) throw Error(KBG_ERR_CUDA, "cublasCreate failed");
    ensure(c->d_states, c->cap_states, 2 * static_cast<size_t>(n) * m);
    c->last_launches = kbg::launch_scale_states(n, m, d_C, d_w, c->d_states, st);
    // row-major C (n x m) is column-major Ct = C^T (m x n, ld m); row-major
    // rho = column-major rho^T = Ct^H (W Ct): one ZGEMM
    const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
    if (cublasSetStream(c->blas, st) != CUBLAS_STATUS_SUCCESS ||
        cublasZgemm(c->blas, CUBLAS_OP_C, CUBLAS_OP_N, n, n, m, &one, reinterpret_cast<const cuDoubleComplex*>(d_C), m,
                    reinterpret_cast<const cuDoubleComplex*>(c->d_states), m, &zero,
                    reinterpret_cast<cuDoubleComplex*>(d_rho), n) != CUBLAS_STATUS_SUCCESS)
        throw Error(KBG_ERR_CUDA, "density_matrix_k: cublasZgemm failed");
    c->last_launches += 1;
    c->tally.flops = 8.0 * n * n * m;
    c->tally.bytes = 16.0 * (static_cast<double>(n) * m + static_cast<double>(n) * n);
}

}  // namespace

int kbg_density_matrix_k_dev(kbg_ctx* c, int m, const double* d_C, const double* d_w, double* d_rho, void* stream) {
    if (!c || !d_C || !d_w || !d_rho) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        KBG_CUDA(cudaSetDevice(c->device));
        density_matrix_k(c, m, d_C, d_w, d_rho, static_cast<cudaStream_t>(stream));
    });
}

int kbg_density_matrix_k(kbg_ctx* c, int m, const double* C, const double* w, double* rho) {
    if (!c || !C || !w || !rho) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        KBG_CUDA(cudaSetDevice(c->device));
        const int n = formats(c).n;
        if (m < 1 || m > n) throw Error(KBG_ERR_DIMENSION, "density_matrix_k: m = " + std::to_string(m));
        for (int i = 0; i < m; ++i)
            if (!std::isfinite(w[i])) throw Error(KBG_ERR_NONFINITE, "density_matrix_k: weight " + std::to_string(i));
        const size_t nc = 2 * static_cast<size_t>(n) * m, nr = 2 * static_cast<size_t>(n) * n;
        ensure(c->d_fa, c->cap_fa, nc + m);
        ensure(c->d_fb, c->cap_fb, nr);
        KBG_CUDA(cudaMemcpyAsync(c->d_fa, C, nc * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        KBG_CUDA(cudaMemcpyAsync(c->d_fa + nc, w, m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        density_matrix_k(c, m, c->d_fa, c->d_fa + nc, c->d_fb, c->stream);
        KBG_CUDA(cudaMemcpyAsync(rho, c->d_fb, nr * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        KBG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int kbg_normalize_rows_dev(double* d_x, int64_t nvec, int64_t len, void* stream) {
    if (!d_x || nvec < 0 || len < 0) return KBG_ERR_CONFIG;
    return guard(nullptr, [&] { kbg::launch_normalize(d_x, nvec, len, static_cast<cudaStream_t>(stream)); });
}

int kbg_normalize_rows(double* x, int64_t nvec, int64_t len) {
    if (!x || nvec < 0 || len < 0) return KBG_ERR_CONFIG;
    return guard(nullptr, [&] {
        const size_t n = static_cast<size_t>(nvec) * len;
        if (n == 0) return;
        double* d = nullptr;
        KBG_CUDA(cudaMalloc(&d, n * sizeof(double)));
        struct Free {
            double* p;
            ~Free() { cudaFree(p); }
        } guard_d{d};
        KBG_CUDA(cudaMemcpy(d, x, n * sizeof(double), cudaMemcpyHostToDevice));
        kbg::launch_normalize(d, nvec, len, nullptr);
        KBG_CUDA(cudaMemcpy(x, d, n * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

// ---- fused H reduction + mirror over peer memory (kb_comm.cu) ----------------
namespace {

struct CommBlob {
    cudaIpcMemHandle_t h;
    uint64_t ptr;
    int64_t pid;
    int32_t device;  // CUDA ordinal of the owner (same-process peers must be reachable from this device)
};
static_assert(sizeof(CommBlob) <= KBG_COMM_HANDLE_BYTES, "comm handle size");

// [nspin <= 2][nnz][2 limbs] (the legacy FP64 path uses the first half as [nspin][nnz])
size_t xbuf_doubles(const kbg_ctx* c) { return 4 * static_cast<size_t>(std::max<int64_t>(1, c->ix.nnz)); }

}  // namespace

int kbg_comm_handle(kbg_ctx* c, void* out) {
    if (!c || !out) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        require_index(c);
        KBG_CUDA(cudaSetDevice(c->device));
        if (!c->d_xbuf) {
            const size_t bytes = xbuf_doubles(c) * sizeof(double) + 8 * kbg::kMaxRanks + 64;
            KBG_CUDA(cudaMalloc(&c->d_xbuf, bytes));
            KBG_CUDA(cudaMemset(c->d_xbuf, 0, bytes));
        }
        CommBlob b{};
        KBG_CUDA(cudaIpcGetMemHandle(&b.h, c->d_xbuf));
        b.ptr = reinterpret_cast<uint64_t>(c->d_xbuf);
        b.pid = static_cast<int64_t>(getpid());
        b.device = c->device;
        std::memset(out, 0, KBG_COMM_HANDLE_BYTES);
        std::memcpy(out, &b, sizeof(b));
    });
}

int kbg_comm_open(kbg_ctx* c, const void* handles) {
    if (!c || !handles) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        require_index(c);
        if (!c->d_xbuf) throw Error(KBG_ERR_CONFIG, "comm_open: call kbg_comm_handle first");
        if (c->nranks > kbg::kMaxRanks) throw Error(KBG_ERR_CONFIG, "comm_open: more than 8 ranks");
        KBG_CUDA(cudaSetDevice(c->device));
        kbg::CommArgs& cm = c->comm;
        cm.nranks = c->nranks;
        cm.rank = c->rank;
        const size_t nd = xbuf_doubles(c);
        for (int k = 0; k < c->nranks; ++k) {
            CommBlob b;
            std::memcpy(&b, static_cast<const char*>(handles) + k * KBG_COMM_HANDLE_BYTES, sizeof(b));
            double* x = nullptr;
            if (k == c->rank) {
                x = c->d_xbuf;
            } else if (b.pid == static_cast<int64_t>(getpid())) {
                // same process: direct pointer, valid from this device only on the same device or with peer access
                if (b.device != c->device) {
                    int can = 0;
                    KBG_CUDA(cudaDeviceCanAccessPeer(&can, c->device, b.device));
                    if (!can)
                        throw Error(KBG_ERR_CONFIG, "comm_open: rank " + std::to_string(k) + " lives on device " +
                                                        std::to_string(b.device) + " in this process, which device " +
                                                        std::to_string(c->device) + " cannot access (no P2P)");
                    const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled)
                        (void)cudaGetLastError();
                    else
                        KBG_CUDA(e);
                }
                x = reinterpret_cast<double*>(b.ptr);
            } else {
                void* q = nullptr;
                KBG_CUDA(cudaIpcOpenMemHandle(&q, b.h, cudaIpcMemLazyEnablePeerAccess));
                c->ipc_opened.push_back(q);
                x = static_cast<double*>(q);
            }
            cm.x[k] = x;
            cm.flags[k] = reinterpret_cast<unsigned long long*>(x + nd);
        }
        cm.counter = reinterpret_cast<unsigned int*>(cm.flags[c->rank] + kbg::kMaxRanks);
        // canonical pairs, contiguous slices balanced by block size
        if (!c->hix.valid) kbg::copy_index_to_host(c->ix, c->hix, c->stream);
        const kbg::HostIndex& h = c->hix;
        std::vector<int32_t> canon;
        std::vector<int64_t> pre{0};
        for (int64_t p = 0; p < c->ix.npair; ++p) {
            const int a = h.pair_a[p], b = h.pair_b[p];
            const int R0 = h.pair_R[3 * p], R1 = h.pair_R[3 * p + 1], R2 = h.pair_R[3 * p + 2];
            const bool can = (a != b) ? a < b : (R0 != 0 ? R0 > 0 : (R1 != 0 ? R1 > 0 : R2 >= 0));
            if (!can) continue;
            canon.push_back(static_cast<int32_t>(p));
            pre.push_back(pre.back() + (h.pair_off[p + 1] - h.pair_off[p]));
        }
        auto bound = [&](int r) -> int64_t {
            const int64_t target = (pre.back() * r + c->nranks - 1) / c->nranks;
            return std::lower_bound(pre.begin(), pre.end(), target) - pre.begin();
        };
        const int64_t w0 = std::min<int64_t>(bound(c->rank), static_cast<int64_t>(canon.size()));
        const int64_t w1 = c->rank + 1 == c->nranks ? static_cast<int64_t>(canon.size())
                                                     : std::min<int64_t>(bound(c->rank + 1), static_cast<int64_t>(canon.size()));
        if (c->ix.nnz >= (int64_t(1) << 31)) throw Error(KBG_ERR_DIMENSION, "comm_open: nnz >= 2^31");
        // ranks whose shard accumulates into each pair (the others' partials are exact zeros)
        std::vector<uint32_t> owners;
        {
            kbg::BuildStream bs(c->stream);
            kbg::pair_owners(c->ix, shard_bounds(c), owners, c->stream);
        }
        {
            // pairs this rank's blocks touch: the DM it reads in kbg_grid_pass (shard-local input)
            // bit 0: the rank's blocks touch pair p (its repack reads it); bit 1: the rank checks p's DM
            // symmetry -- every pair is checked by exactly one rank, its lowest owner, which alone reads
            // the mirror block (each mirror crosses PCIe once in total, not once per owner)
            std::vector<uint8_t> mine(std::max<int64_t>(1, c->ix.npair), 0), need(std::max<int64_t>(1, c->ix.npair), 0);
            for (int64_t p = 0; p < c->ix.npair; ++p) {
                const uint32_t o = owners[p];
                if ((o >> c->rank) & 1u) mine[p] = 1;
                if (o && __builtin_ctz(o) == c->rank) mine[p] |= 2;
                if (mine[p]) need[p] = 1;
                if (mine[p] & 2) need[h.pair_mirror[p]] = 1;
            }
            // contiguous runs of the needed pair blocks, then the smallest gaps merged until at most
            // kMaxDmRuns copies remain (448 atoms on 4 GPUs: 2.5 k runs, 42 % of the DM)
            std::vector<int64_t> runs;
            for (int64_t p = 0; p < c->ix.npair; ++p) {
                if (!need[p]) continue;
                const int64_t o = h.pair_off[p], n = h.pair_off[p + 1] - o;
                if (!runs.empty() && runs[runs.size() - 2] + runs.back() == o)
                    runs.back() += n;
                else {
                    runs.push_back(o);
                    runs.push_back(n);
                }
            }
            // exact runs for the in-place gather (k_dm_gather, pinned DM: no bytes beyond the blocks)
            c->dm_xruns_n = static_cast<int64_t>(runs.size() / 2);
            if (c->d_xruns) cudaFree(c->d_xruns);
            c->d_xruns = nullptr;
            KBG_CUDA(cudaMalloc(&c->d_xruns, std::max<size_t>(1, runs.size()) * sizeof(int64_t)));
            if (!runs.empty())
                KBG_CUDA(cudaMemcpy(c->d_xruns, runs.data(), runs.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
            int64_t dm_exact = 0;
            for (size_t r = 0; r < runs.size() / 2; ++r) dm_exact += runs[2 * r + 1];
            // memcpy runs (pageable DM): a copy costs the host a few us to issue: about one per 4 MB of DM, at most 48 (56 atoms:
            // a single copy of the whole 3.8 MB DM; 448 atoms: 7; 1512 atoms: 24)
            const size_t kMaxDmRuns = static_cast<size_t>(
                std::max<int64_t>(1, std::min<int64_t>(48, c->ix.nnz * 8 / (4 << 20))));
            if (runs.size() / 2 > kMaxDmRuns) {
                std::vector<int64_t> gaps;
                for (size_t r = 1; r < runs.size() / 2; ++r) gaps.push_back(runs[2 * r] - runs[2 * r - 2] - runs[2 * r - 1]);
                std::nth_element(gaps.begin(), gaps.begin() + (gaps.size() - (kMaxDmRuns - 1)), gaps.end());
                const int64_t gmax = gaps[gaps.size() - (kMaxDmRuns - 1)];  // gaps below this are bridged
                std::vector<int64_t> merged{runs[0], runs[1]};
                for (size_t r = 1; r < runs.size() / 2; ++r) {
                    const int64_t gap = runs[2 * r] - merged[merged.size() - 2] - merged.back();
                    if (gap < gmax) {
                        merged.back() = runs[2 * r] + runs[2 * r + 1] - merged[merged.size() - 2];
                    } else {
                        merged.push_back(runs[2 * r]);
                        merged.push_back(runs[2 * r + 1]);
                    }
                }
                runs.swap(merged);
            }
            c->dm_runs = runs;
            int64_t dm_read = 0;
            for (size_t r = 0; r < runs.size() / 2; ++r) dm_read += runs[2 * r + 1];
            c->dm_read_copy = dm_read;
            dm_read = dm_exact;  // io[6]: the pinned (gather) path; kbg_shard_io reports the copy path's if pageable
            if (c->d_pown) cudaFree(c->d_pown);
            c->d_pown = nullptr;
            KBG_CUDA(cudaMalloc(&c->d_pown, mine.size()));
            KBG_CUDA(cudaMemcpy(c->d_pown, mine.data(), mine.size(), cudaMemcpyHostToDevice));
            // io ranges: blocks, the rank's grid-plane range (C order, i outermost), its H output slice
            const int64_t nb12 = static_cast<int64_t>(c->P.nblk[1]) * c->P.nblk[2];
            const int64_t plane = static_cast<int64_t>(c->P.N[1]) * c->P.N[2];
            c->io[0] = c->blk_begin;
            c->io[1] = c->blk_end;
            c->io[2] = c->blk_end > c->blk_begin ? std::min<int64_t>(c->P.N[0], 4 * (c->blk_begin / nb12)) * plane : 0;
            c->io[3] = c->blk_end > c->blk_begin
                           ? std::min<int64_t>(c->P.N[0], 4 * ((c->blk_end - 1) / nb12 + 1)) * plane : 0;
            c->io[4] = c->ix.nnz * c->rank / c->nranks;
            c->io[5] = c->ix.nnz * (c->rank + 1) / c->nranks;
            c->io[6] = dm_read;
            c->io[7] = c->io[3] - c->io[2];
        }
        std::vector<int32_t> e0, e1;
        std::vector<uint8_t> em;
        for (int64_t w = w0; w < w1; ++w) {
            const int64_t p = canon[w], q = h.pair_mirror[p];
            const uint8_t om = static_cast<uint8_t>(owners[p]);
            const int na = c->P.sp[c->h_spc[h.pair_a[p]]].norb, nb = c->P.sp[c->h_spc[h.pair_b[p]]].norb;
            for (int i = 0; i < na; ++i)
                for (int j = 0; j < nb; ++j) {
                    if (q == p && i > j) continue;  // (a, a, 0): the upper triangle carries both entries
                    e0.push_back(static_cast<int32_t>(h.pair_off[p] + i * nb + j));
                    em.push_back(om);
                    if (q == p)
                        e1.push_back(static_cast<int32_t>(h.pair_off[p] + j * na + i) | (i < j ? INT32_MIN : 0));
                    else
                        e1.push_back(static_cast<int32_t>(h.pair_off[q] + j * na + i));
                }
        }
        if (c->d_canon) cudaFree(c->d_canon);
        c->d_canon = nullptr;
        KBG_CUDA(cudaMalloc(&c->d_canon, std::max<size_t>(1, 2 * e0.size() + (e0.size() + 3) / 4) * sizeof(int32_t)));
        if (!e0.empty()) {
            KBG_CUDA(cudaMemcpy(c->d_canon, e0.data(), e0.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
            KBG_CUDA(cudaMemcpy(c->d_canon + e0.size(), e1.data(), e1.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
            KBG_CUDA(cudaMemcpy(c->d_canon + 2 * e0.size(), em.data(), em.size(), cudaMemcpyHostToDevice));
        }
        // per-pair tables of the fused copy-out + mirror
        {
            const int64_t np = c->ix.npair;
            std::vector<int32_t> na(np), nb(np);
            std::vector<uint8_t> cf(np);
            for (int64_t p = 0; p < np; ++p) {
                const int a = h.pair_a[p], b = h.pair_b[p];
                const int R0 = h.pair_R[3 * p], R1 = h.pair_R[3 * p + 1], R2 = h.pair_R[3 * p + 2];
                na[p] = c->P.sp[c->h_spc[a]].norb;
                nb[p] = c->P.sp[c->h_spc[b]].norb;
                cf[p] = (a != b) ? a < b : (R0 != 0 ? R0 > 0 : (R1 != 0 ? R1 > 0 : R2 >= 0));
            }
            if (c->d_pairtab) cudaFree(c->d_pairtab);
            c->d_pairtab = nullptr;
            KBG_CUDA(cudaMalloc(&c->d_pairtab, std::max<size_t>(1, 9 * np)));
            if (np) {
                KBG_CUDA(cudaMemcpy(c->d_pairtab, na.data(), 4 * np, cudaMemcpyHostToDevice));
                KBG_CUDA(cudaMemcpy(c->d_pairtab + 4 * np, nb.data(), 4 * np, cudaMemcpyHostToDevice));
                KBG_CUDA(cudaMemcpy(c->d_pairtab + 8 * np, cf.data(), np, cudaMemcpyHostToDevice));
            }
            cm.pair_na = reinterpret_cast<const int32_t*>(c->d_pairtab);
            cm.pair_nb = reinterpret_cast<const int32_t*>(c->d_pairtab + 4 * np);
            cm.pair_canon = reinterpret_cast<const uint8_t*>(c->d_pairtab + 8 * np);
        }
        if (std::getenv("KBG_COMM_TIMING") && !cm.tstamp) {
            KBG_CUDA(cudaMalloc(&cm.tstamp, 8 * sizeof(unsigned long long)));
            KBG_CUDA(cudaMemset(cm.tstamp, 0, 8 * sizeof(unsigned long long)));
        }
        cm.el0 = c->d_canon;
        cm.el1 = c->d_canon + e0.size();
        cm.elm = reinterpret_cast<const uint8_t*>(c->d_canon + 2 * e0.size());
        cm.ne = static_cast<int64_t>(e0.size());
        // Everything kbg_grid_pass allocates, for up to kMaxSpin spins, now: an allocation (or the free
        // of a growing buffer) inside a sharded pass may synchronize the device while a peer's exchange
        // waits for this rank's -- a deadlock until the 10 s timeout when the ranks share a process.
        {
            const size_t ndm = static_cast<size_t>(kbg::kMaxSpin) * std::max<int64_t>(1, c->ix.nnz);
            const size_t npt = static_cast<size_t>(kbg::kMaxSpin) * std::max<int64_t>(1, c->npts);
            ensure(c->d_in, c->cap_in, ndm);
            ensure(c->d_out, c->cap_out, npt);
            ensure(c->d_in2, c->cap_in2, npt);
            ensure(c->d_out2, c->cap_out2, ndm);
            ensure(c->d_dmr, c->cap_dmr, static_cast<size_t>(kbg::kMaxSpin) * std::max<int64_t>(1, c->ix.nrep));
            if (!c->stream2) KBG_CUDA(cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking));
            if (!c->ev_pass) KBG_CUDA(cudaEventCreateWithFlags(&c->ev_pass, cudaEventDisableTiming));
            if (!c->ev_rho) KBG_CUDA(cudaEventCreateWithFlags(&c->ev_rho, cudaEventDisableTiming));
            if (!c->h_flags) KBG_CUDA(cudaMallocHost(&c->h_flags, 8 * sizeof(unsigned long long)));
        }
        c->comm_ready = true;
    });
}


// Timing aid (KBG_COMM_TIMING set at kbg_comm_open): the last exchange's phase stamps in ns relative to
// the reduce kernel's start: [0] all partials ready, [1] slice reduced and signalled, [2] copy kernel start,
// [3] all slices landed, [4] copy + mirror done. Returns KBG_ERR_CONFIG when timing is off.
int kbg_comm_timing(kbg_ctx* c, double* out5) {
    if (!c || !out5 || !c->comm.tstamp) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        KBG_CUDA(cudaSetDevice(c->device));
        unsigned long long t[8];
        KBG_CUDA(cudaMemcpy(t, c->comm.tstamp, sizeof(t), cudaMemcpyDeviceToHost));
        for (int i = 0; i < 5; ++i) out5[i] = static_cast<double>(t[i + 1]) - static_cast<double>(t[0]);
        KBG_CUDA(cudaMemset(c->comm.tstamp, 0, sizeof(t)));
    });
}

int kbg_shard_io(const kbg_ctx* c, int64_t out[8]) {
    if (!c || !out) return KBG_ERR_CONFIG;
    if (!c->comm_ready) return KBG_ERR_CONFIG;
    for (int i = 0; i < 8; ++i) out[i] = c->io[i];
    return KBG_OK;
}

int kbg_comm_check(kbg_ctx* c) {
    if (!c) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        if (!c->comm_ready) throw Error(KBG_ERR_CONFIG, "comm_check: call kbg_comm_open first");
        KBG_CUDA(cudaSetDevice(c->device));
        comm_check(c);
    });
}

int kbg_hamiltonian_allreduce_dev(kbg_ctx* c, int nspin, const double* d_veff, double dV, double* d_h, void* stream) {
    if (!c || !d_veff || !d_h) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nspin(nspin);
        require_index(c);
        if (!c->comm_ready) throw Error(KBG_ERR_CONFIG, "hamiltonian_allreduce: call kbg_comm_open first");
        KBG_CUDA(cudaSetDevice(c->device));
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        int n = h_accumulate(c, nspin, dV, d_veff, c->d_xbuf, st);
        c->epoch += 2;
        c->comm.ls = h_limbs(c);
        c->comm.sms = 0;  // nothing runs next to it here: the whole GPU
        n += kbg::launch_reduce_mirror(c->comm, c->ix, c->P, nspin, d_h, c->epoch - 1, st);
        c->last_launches = n;
        c->tally.flops = nspin * 2.0 * c->ix.sum_m2 / c->nranks;
        c->tally.bytes = 8.0 * nspin * (c->ix.nnz + c->npts);
    });
}

// The two halves of kbg_hamiltonian_allreduce_dev, so a caller can put independent work (the density
// pass) between them: the exchange then finds every peer's partials ready instead of spinning on the
// slowest rank, and the rank spread and flag latency hide behind that work.
int kbg_hamiltonian_partial_dev(kbg_ctx* c, int nspin, const double* d_veff, double dV, void* stream) {
    if (!c || !d_veff) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nspin(nspin);
        require_index(c);
        if (!c->comm_ready) throw Error(KBG_ERR_CONFIG, "hamiltonian_partial: call kbg_comm_open first");
        KBG_CUDA(cudaSetDevice(c->device));
        c->last_launches = h_accumulate(c, nspin, dV, d_veff, c->d_xbuf, static_cast<cudaStream_t>(stream));
        c->pending_nspin = nspin;
        c->tally.flops = nspin * 2.0 * c->ix.sum_m2 / c->nranks;
        c->tally.bytes = 8.0 * nspin * (c->ix.nnz + c->npts);
    });
}

int kbg_hamiltonian_exchange_dev(kbg_ctx* c, int nspin, double* d_h, void* stream) {
    if (!c || !d_h) return KBG_ERR_CONFIG;
    return guard(c, [&] {
        check_nspin(nspin);
        require_index(c);
        if (!c->comm_ready) throw Error(KBG_ERR_CONFIG, "hamiltonian_exchange: call kbg_comm_open first");
        if (c->pending_nspin != nspin)
            throw Error(KBG_ERR_CONFIG, "hamiltonian_exchange: no kbg_hamiltonian_partial_dev with this nspin before");
        KBG_CUDA(cudaSetDevice(c->device));
        c->pending_nspin = 0;
        c->epoch += 2;
        c->comm.ls = h_limbs(c);
        c->comm.sms = c->xsms;
        c->last_launches = kbg::launch_reduce_mirror(c->comm, c->ix, c->P, nspin, d_h, c->epoch - 1,
                                                     static_cast<cudaStream_t>(stream));
    });
}

// ---- Eigen_HH on the GPU (kb_eigen.cu) ------------------
namespace {

thread_local std::string g_hh_err;

int hh_guard(const std::function<void()>& fn) {
    try {
        fn();
        g_hh_err.clear();
        return KBG_OK;
    } catch (const Error& e) {
        g_hh_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_hh_err = e.what();
        return KBG_ERR_CONSISTENCY;
    }
}

// Stream-ordered device scratch freed at scope exit.
// Stream-ordered allocations come from the device's default pool; keep freed memory in the pool
// (release threshold: unlimited) so repeated calls do not re-map hundreds of MB each time.
void keep_pool() {
    static thread_local int done_dev = -1;
    int dev = 0;
    KBG_CUDA(cudaGetDevice(&dev));
    if (done_dev == dev) return;
    cudaMemPool_t pool;
    KBG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = UINT64_MAX;
    KBG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    done_dev = dev;
}

struct DevBuf {
    double* p = nullptr;
    cudaStream_t st = nullptr;
    DevBuf(size_t n, cudaStream_t s) : st(s) {
        keep_pool();
        KBG_CUDA(cudaMallocAsync(&p, std::max<size_t>(1, n) * sizeof(double), s));
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// W = Q Y on the device: per-column reflector chain for small n, blocked compact WY (ZGEMMs) from
// kWyMinN (set KBG_BT_WY=0 to force the per-column kernel, =1 to force WY).
void back_transform_dev(int64_t n, int64_t m, const double* Y, const double* U, const double* H, const double* P,
                        double* W, cudaStream_t st) {
    DevBuf dph(2 * n, st);
    const char* env = std::getenv("KBG_BT_WY");
    const bool wy = env ? env[0] == '1' : n >= kbg::kWyMinN;
    if (wy && n > 1) {
        DevBuf scr(kbg::hh_back_transform_wy_scratch(static_cast<int>(n), static_cast<int>(m)), st);
        kbg::launch_hh_back_transform_wy(static_cast<int>(n), static_cast<int>(m), Y, U, H, P, dph.p, W, scr.p, st);
    } else {
        kbg::launch_hh_back_transform(static_cast<int>(n), static_cast<int>(m), Y, U, H, P, dph.p, W, st);
    }
}

void hh_check_n(int64_t n) {
    if (n < 1) throw Error(KBG_ERR_DIMENSION, "tridiagonalize: empty matrix");
    if (n > 4800) throw Error(KBG_ERR_DIMENSION, "tridiagonalize: n = " + std::to_string(n) + " > 4800 (shared-memory reflectors)");
}

// HermitianMatrix::from on the device (linalg.cpp:44-63): reject a defect above tol, then symmetrize.
void hermitian_from(int64_t n, double* d_A, cudaStream_t st, double tol = 1e-13) {
    DevBuf def(1, st);
    KBG_CUDA(cudaMemsetAsync(def.p, 0, sizeof(double), st));
    kbg::launch_hermitian_repair(static_cast<int>(n), d_A, reinterpret_cast<unsigned long long*>(def.p), false, st);
    double defect = 0.0;
    KBG_CUDA(cudaMemcpyAsync(&defect, def.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    KBG_CUDA(cudaStreamSynchronize(st));
    if (!std::isfinite(defect)) throw Error(KBG_ERR_CONSISTENCY, "HermitianMatrix: non-finite entries");
    if (defect > tol)
        throw Error(KBG_ERR_CONSISTENCY, "HermitianMatrix: defect " + std::to_string(defect) + " exceeds tolerance " +
                                             std::to_string(tol));
    kbg::launch_hermitian_repair(static_cast<int>(n), d_A, nullptr, true, st);
}

void tridiag_dev(int64_t n, double* d_work, int fault_sign, double* d, double* e, double* u, double* h, double* s,
                 double* ph, cudaStream_t st) {
    DevBuf p(4 * n, st);  // double-buffered p (complex)
    kbg::launch_hh_tridiagonalize(static_cast<int>(n), d_work, p.p, d, e, u, h, s, ph, fault_sign ? 1.0 : -1.0, st);
}

}  // namespace

const char* kbg_hh_last_error(void) { return g_hh_err.c_str(); }

int kbg_hh_tridiagonalize_dev(int64_t n, double* d_a, int fault_sign, double* d_d, double* d_e, double* d_u,
                              double* d_h, double* d_s, double* d_phase, void* stream) {
    if (!d_a || !d_d || !d_e || !d_u || !d_h || !d_s || !d_phase) return KBG_ERR_CONFIG;
    return hh_guard([&] {
        hh_check_n(n);
        tridiag_dev(n, d_a, fault_sign, d_d, d_e, d_u, d_h, d_s, d_phase, static_cast<cudaStream_t>(stream));
    });
}

int kbg_hh_tridiagonalize(int64_t n, const double* a, int fault_sign, double* d, double* e, double* u, double* h,
                          double* s, double* phase) {
    if (!a || !d || !e || !u || !h || !s || !phase) return KBG_ERR_CONFIG;
    return hh_guard([&] {
        hh_check_n(n);
        const cudaStream_t st = nullptr;
        const size_t nn = static_cast<size_t>(n) * n, nr = static_cast<size_t>(n - 1);
        DevBuf A(2 * nn, st), D(n, st), E(std::max<size_t>(1, nr), st), U(2 * nr * n, st), H(nr, st), S(nr, st),
            P(2 * nr, st);
        KBG_CUDA(cudaMemcpyAsync(A.p, a, 2 * nn * sizeof(double), cudaMemcpyHostToDevice, st));
        hermitian_from(n, A.p, st);
        tridiag_dev(n, A.p, fault_sign, D.p, E.p, U.p, H.p, S.p, P.p, st);
        KBG_CUDA(cudaMemcpyAsync(d, D.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
        if (nr) {
            KBG_CUDA(cudaMemcpyAsync(e, E.p, nr * sizeof(double), cudaMemcpyDeviceToHost, st));
            KBG_CUDA(cudaMemcpyAsync(u, U.p, 2 * nr * n * sizeof(double), cudaMemcpyDeviceToHost, st));
            KBG_CUDA(cudaMemcpyAsync(h, H.p, nr * sizeof(double), cudaMemcpyDeviceToHost, st));
            KBG_CUDA(cudaMemcpyAsync(s, S.p, nr * sizeof(double), cudaMemcpyDeviceToHost, st));
            KBG_CUDA(cudaMemcpyAsync(phase, P.p, 2 * nr * sizeof(double), cudaMemcpyDeviceToHost, st));
        }
        KBG_CUDA(cudaStreamSynchronize(st));
        for (size_t i = 0; i < nr; ++i)
            if (!std::isfinite(s[i]) || !std::isfinite(h[i]))
                throw Error(KBG_ERR_NONFINITE, "tridiagonalize: non-finite reflector at stage " + std::to_string(i));
    });
}

int kbg_hh_back_transform_dev(int64_t n, int64_t m, const double* d_u, const double* d_h, const double* d_phase,
                              const double* d_y, double* d_w, void* stream) {
    if (!d_u || !d_h || !d_phase || !d_y || !d_w) return KBG_ERR_CONFIG;
    return hh_guard([&] {
        hh_check_n(n);
        if (m < 1) throw Error(KBG_ERR_DIMENSION, "back_transform: no columns");
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        back_transform_dev(n, m, d_y, d_u, d_h, d_phase, d_w, st);
    });
}

int kbg_hh_back_transform(int64_t n, int64_t m, const double* u, const double* h, const double* phase,
                          const double* y, double* w) {
    if (!u || !h || !phase || !y || !w) return KBG_ERR_CONFIG;
    return hh_guard([&] {
        hh_check_n(n);
        if (m < 1) throw Error(KBG_ERR_DIMENSION, "back_transform: no columns");
        const cudaStream_t st = nullptr;
        const size_t nr = static_cast<size_t>(n - 1);
        DevBuf U(2 * nr * n, st), H(nr, st), P(2 * nr, st), Y(static_cast<size_t>(n) * m, st),
            W(2 * static_cast<size_t>(n) * m, st), dph(2 * n, st);
        if (nr) {
            KBG_CUDA(cudaMemcpyAsync(U.p, u, 2 * nr * n * sizeof(double), cudaMemcpyHostToDevice, st));
            KBG_CUDA(cudaMemcpyAsync(H.p, h, nr * sizeof(double), cudaMemcpyHostToDevice, st));
            KBG_CUDA(cudaMemcpyAsync(P.p, phase, 2 * nr * sizeof(double), cudaMemcpyHostToDevice, st));
        }
        KBG_CUDA(cudaMemcpyAsync(Y.p, y, static_cast<size_t>(n) * m * sizeof(double), cudaMemcpyHostToDevice, st));
        back_transform_dev(n, m, Y.p, U.p, H.p, P.p, W.p, st);
        KBG_CUDA(cudaMemcpyAsync(w, W.p, 2 * static_cast<size_t>(n) * m * sizeof(double), cudaMemcpyDeviceToHost, st));
        KBG_CUDA(cudaStreamSynchronize(st));
    });
}

// kband::triple_product (linalg.cpp:112-120): C = T^H H T with two ZGEMMs, then HermitianMatrix::from_scaled
// (defect <= 1e-13 max(1, ||C||_F), symmetrized). Row-major buffers are their column-major transposes:
// C^T = t h t^H with t = T^T (m x n), h = H^T.
int kbg_hh_triple_product(int64_t n, int64_t m, const double* t, const double* h, double* c_out) {
    if (!t || !h || !c_out || n < 1 || m < 1) return KBG_ERR_CONFIG;
    return hh_guard([&] {
        const cudaStream_t st = nullptr;
        DevBuf T(2 * static_cast<size_t>(n) * m, st), H(2 * static_cast<size_t>(n) * n, st),
            X(2 * static_cast<size_t>(n) * m, st), C(2 * static_cast<size_t>(m) * m, st);
        KBG_CUDA(cudaMemcpyAsync(T.p, t, 2 * static_cast<size_t>(n) * m * sizeof(double), cudaMemcpyHostToDevice, st));
        KBG_CUDA(cudaMemcpyAsync(H.p, h, 2 * static_cast<size_t>(n) * n * sizeof(double), cudaMemcpyHostToDevice, st));
        cublasHandle_t bh = nullptr;
        if (cublasCreate(&bh) != CUBLAS_STATUS_SUCCESS) throw Error(KBG_ERR_CUDA, "cublasCreate failed");
        struct Destroy {
            cublasHandle_t h;
            ~Destroy() { cublasDestroy(h); }
        } destroy{bh};
        const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
        auto z = [](double* p) { return reinterpret_cast<cuDoubleComplex*>(p); };
        const int N = static_cast<int>(n), M = static_cast<int>(m);
        if (cublasSetStream(bh, st) != CUBLAS_STATUS_SUCCESS ||
            cublasZgemm(bh, CUBLAS_OP_N, CUBLAS_OP_C, N, M, N, &one, z(H.p), N, z(T.p), M, &zero, z(X.p), N) !=
                CUBLAS_STATUS_SUCCESS ||
            cublasZgemm(bh, CUBLAS_OP_N, CUBLAS_OP_N, M, M, N, &one, z(T.p), M, z(X.p), N, &zero, z(C.p), M) !=
                CUBLAS_STATUS_SUCCESS)
            throw Error(KBG_ERR_CUDA, "triple_product: cublasZgemm failed");
        double fro = 0.0;
        if (cublasDznrm2(bh, M * M, z(C.p), 1, &fro) != CUBLAS_STATUS_SUCCESS)
            throw Error(KBG_ERR_CUDA, "triple_product: cublasDznrm2 failed");
        hermitian_from(m, C.p, st, 1e-13 * std::max(1.0, fro));
        KBG_CUDA(cudaMemcpyAsync(c_out, C.p, 2 * static_cast<size_t>(m) * m * sizeof(double), cudaMemcpyDeviceToHost, st));
        KBG_CUDA(cudaStreamSynchronize(st));
    });
}

int kbg_hh_normalize_columns_dev(int64_t n, int64_t m, double* d_c, void* stream) {
    if (!d_c) return KBG_ERR_CONFIG;
    return hh_guard([&] {
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        DevBuf z(1, st);
        const int big = 0x7fffffff;
        KBG_CUDA(cudaMemcpyAsync(z.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
        kbg::launch_hh_normalize_columns(n, m, d_c, reinterpret_cast<int*>(z.p), st);
        int zero = big;
        KBG_CUDA(cudaMemcpyAsync(&zero, z.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        KBG_CUDA(cudaStreamSynchronize(st));
        if (zero != big) throw Error(KBG_ERR_CONSISTENCY, "normalize_columns: zero column " + std::to_string(zero));
    });
}

int kbg_hh_normalize_columns(int64_t n, int64_t m, double* c) {
    if (!c) return KBG_ERR_CONFIG;
    return hh_guard([&] {
        const size_t nm = 2 * static_cast<size_t>(n) * m;
        DevBuf C(nm, nullptr);
        KBG_CUDA(cudaMemcpyAsync(C.p, c, nm * sizeof(double), cudaMemcpyHostToDevice, nullptr));
        const int st = kbg_hh_normalize_columns_dev(n, m, C.p, nullptr);
        if (st != KBG_OK) throw Error(st, g_hh_err);
        KBG_CUDA(cudaMemcpy(c, C.p, nm * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

// kband::eigen_hh (householder.cpp:333-351) device-resident end to end: Hermitian check,
// tridiagonalize, tridiagonal solve, back transform, column normalization; only A in and
// (w, C) out cross PCIe.
int kbg_hh_eigen(int64_t n, const double* a, int want_vectors, double* w, double* c) {
    if (!a || !w || (want_vectors && !c)) return KBG_ERR_CONFIG;
    return hh_guard([&] {
        hh_check_n(n);
        const cudaStream_t st = nullptr;
        const size_t nn = static_cast<size_t>(n) * n, nr = static_cast<size_t>(n - 1);
        DevBuf A(2 * nn, st), D(n, st), E(std::max<size_t>(1, nr), st), U(2 * std::max<size_t>(1, nr) * n, st),
            H(std::max<size_t>(1, nr), st), S(std::max<size_t>(1, nr), st), P(2 * std::max<size_t>(1, nr), st),
            W(n, st), Y(want_vectors ? nn : 1, st), scr(kbg::tridiag_scratch_doubles(static_cast<int>(n), want_vectors != 0), st);
        KBG_CUDA(cudaMemcpyAsync(A.p, a, 2 * nn * sizeof(double), cudaMemcpyHostToDevice, st));
        hermitian_from(n, A.p, st);
        tridiag_dev(n, A.p, 0, D.p, E.p, U.p, H.p, S.p, P.p, st);
        kbg::launch_tridiag_solve(static_cast<int>(n), D.p, n > 1 ? E.p : D.p, want_vectors != 0, W.p, Y.p, scr.p, st);
        KBG_CUDA(cudaMemcpyAsync(w, W.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
        if (want_vectors) {
            double* C = A.p;  // the working matrix is free again
            if (n == 1) {
                const double one[2] = {1.0, 0.0};
                KBG_CUDA(cudaMemcpyAsync(C, one, sizeof(one), cudaMemcpyHostToDevice, st));
            } else {
                back_transform_dev(n, n, Y.p, U.p, H.p, P.p, C, st);
            }
            const int stn = kbg_hh_normalize_columns_dev(n, n, C, st);
            if (stn != KBG_OK) throw Error(stn, g_hh_err);
            KBG_CUDA(cudaMemcpyAsync(c, C, 2 * nn * sizeof(double), cudaMemcpyDeviceToHost, st));
        }
        KBG_CUDA(cudaStreamSynchronize(st));
        for (int64_t i = 0; i < n; ++i)
            if (!std::isfinite(w[i])) throw Error(KBG_ERR_NONFINITE, "eigen_hh: non-finite eigenvalue " + std::to_string(i));
    });
}

int kbg_tridiag_solve_dev(int64_t n, const double* d_d, const double* d_e, int want_vectors, double* d_w,
                          double* d_z, void* stream) {
    if (!d_d || !d_w || (n > 1 && !d_e) || (want_vectors && !d_z)) return KBG_ERR_CONFIG;
    return hh_guard([&] {
        if (n < 1) throw Error(KBG_ERR_DIMENSION, "solve_tridiag: empty problem");
        if (n > 12000) throw Error(KBG_ERR_DIMENSION, "solve_tridiag: n = " + std::to_string(n) + " > 12000");
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        DevBuf scr(kbg::tridiag_scratch_doubles(static_cast<int>(n), want_vectors != 0), st);
        kbg::launch_tridiag_solve(static_cast<int>(n), d_d, n > 1 ? d_e : d_d, want_vectors != 0, d_w, d_z, scr.p,
                                  st);
    });
}

int kbg_tridiag_solve(int64_t n, const double* d, const double* e, int want_vectors, double* w, double* z) {
    if (!d || !w || (n > 1 && !e) || (want_vectors && !z)) return KBG_ERR_CONFIG;
    return hh_guard([&] {
        if (n < 1) throw Error(KBG_ERR_DIMENSION, "solve_tridiag: empty problem");
        for (int64_t i = 0; i < n; ++i)
            if (!std::isfinite(d[i]) || (i + 1 < n && !std::isfinite(e[i])))
                throw Error(KBG_ERR_NONFINITE, "solve_tridiag: non-finite entry at index " + std::to_string(i));
        DevBuf D(n, nullptr), E(std::max<int64_t>(1, n - 1), nullptr), W(n, nullptr),
            Z(want_vectors ? n * n : 1, nullptr);
        KBG_CUDA(cudaMemcpyAsync(D.p, d, n * sizeof(double), cudaMemcpyHostToDevice, nullptr));
        if (n > 1) KBG_CUDA(cudaMemcpyAsync(E.p, e, (n - 1) * sizeof(double), cudaMemcpyHostToDevice, nullptr));
        const int st = kbg_tridiag_solve_dev(n, D.p, E.p, want_vectors, W.p, Z.p, nullptr);
        if (st != KBG_OK) throw Error(st, g_hh_err);
        KBG_CUDA(cudaMemcpy(w, W.p, n * sizeof(double), cudaMemcpyDeviceToHost));
        if (want_vectors) KBG_CUDA(cudaMemcpy(z, Z.p, n * n * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int kbg_last_tally(const kbg_ctx* c, kbg_tally* out) {
    if (!c || !out) return KBG_ERR_CONFIG;
    *out = c->tally;
    return KBG_OK;
}

int kbg_set_option(kbg_ctx* c, int option, int64_t value) {
    if (!c) return KBG_ERR_CONFIG;
    switch (option) {
        case KBG_OPT_WARPS:
            if (value != 4 && value != 8) {
                c->err = "set_option: warps must be 4 or 8";
                return KBG_ERR_CONFIG;
            }
            c->nwarps = static_cast<int>(value);
            return KBG_OK;
        case KBG_OPT_FAULT_SIGN:
            c->sign = value ? -1.0 : 1.0;
            return KBG_OK;
        case KBG_OPT_SCATTER_STORE:  // bit 0: stores; bits 1-3: timing experiments (see kb_gridcore.cuh)
            c->scatter = static_cast<int>(value & 15);
            return KBG_OK;
        case KBG_OPT_PERSIST:
            c->persist = value ? 1 : 0;
            return KBG_OK;
        case KBG_OPT_XC:
            if (value < 0 || value > 1) {
                c->err = "set_option: xc must be 0 (exchange only) or 1 (LSDA, PW92 correlation)";
                return KBG_ERR_CONFIG;
            }
            c->xc = static_cast<int>(value);
            return KBG_OK;
        case KBG_OPT_BLOCK_ORDER:
            if (value < 0 || value > 2) {
                c->err = "set_option: block order must be 0, 1 or 2";
                return KBG_ERR_CONFIG;
            }
            c->block_order = static_cast<int>(value);
            return KBG_OK;
        case KBG_OPT_SCHEDULE:
            if (value < 0 || value > 3) {
                c->err = "set_option: schedule must be 0..3";
                return KBG_ERR_CONFIG;
            }
            c->schedule = static_cast<int>(value);
            return KBG_OK;
        case KBG_OPT_DETERMINISTIC:
            c->det = value ? 1 : 0;
            return KBG_OK;
        case KBG_OPT_SHARD_IO:
            c->shard_io = value ? 1 : 0;
            return KBG_OK;
        case KBG_OPT_FUSED_PASS:
            if (value < 0 || value > 2) {
                c->err = "set_option: fused pass must be 0, 1 or 2";
                return KBG_ERR_CONFIG;
            }
            c->fused = static_cast<int>(value);
            return KBG_OK;
        case KBG_OPT_EXCHANGE_SMS:
            if (value < 0 || value > 32) {
                c->err = "set_option: exchange SMs must be 0..32";
                return KBG_ERR_CONFIG;
            }
            c->xsms = static_cast<int>(value);
            return KBG_OK;
        case KBG_OPT_SPARSE_DFMA:
            if (value < 0 || value > 255) {
                c->err = "set_option: sparse-DFMA threshold must be 0..255 (point density x 255)";
                return KBG_ERR_CONFIG;
            }
            c->sparse_thr = static_cast<int>(value);
            return KBG_OK;
        case KBG_OPT_DEBUG_COUNTERS:
            if (value && !c->d_dbg) {
                if (cudaMalloc(&c->d_dbg, 16 * sizeof(unsigned long long)) != cudaSuccess) return KBG_ERR_CUDA;
            }
            if (c->d_dbg) cudaMemset(c->d_dbg, 0, 16 * sizeof(unsigned long long));
            return KBG_OK;
        default:
            c->err = "set_option: unknown option";
            return KBG_ERR_CONFIG;
    }
}

const char* kbg_last_error(const kbg_ctx* c) { return c ? c->err.c_str() : "null context"; }

void kbg_destroy(kbg_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->stream2) cudaStreamSynchronize(c->stream2);
    {
        kbg::BuildStream bs(c->stream);
        kbg::free_index(c->ix);
    }
    if (c->stream) cudaStreamSynchronize(c->stream);
    kbg::free_formats(c->fmt);
    for (double* p : {c->d_fa, c->d_fb, c->d_phase, c->d_kw})
        if (p) cudaFree(p);
    if (c->h_kw) cudaFreeHost(c->h_kw);
    if (c->d_states) cudaFree(c->d_states);
    for (void* q : c->ipc_opened) cudaIpcCloseMemHandle(q);
    if (c->d_xbuf) cudaFree(c->d_xbuf);
    if (c->d_canon) cudaFree(c->d_canon);
    if (c->d_pairtab) cudaFree(c->d_pairtab);
    if (c->d_pown) cudaFree(c->d_pown);
    if (c->d_xruns) cudaFree(c->d_xruns);
    if (c->h_flags) cudaFreeHost(c->h_flags);
    if (c->comm.tstamp) cudaFree(c->comm.tstamp);
    if (c->d_cpre) cudaFree(c->d_cpre);
    c->veff.release();
    if (c->d_in2) cudaFree(c->d_in2);
    if (c->d_out2) cudaFree(c->d_out2);
    if (c->ev_pass) cudaEventDestroy(c->ev_pass);
    if (c->ev_rho) cudaEventDestroy(c->ev_rho);
    if (c->stream2) cudaStreamDestroy(c->stream2);
    if (c->blas) cublasDestroy(c->blas);
    if (c->h_kw_done) cudaEventDestroy(c->h_kw_done);
    if (c->d_tau) cudaFree(c->d_tau);
    if (c->d_spc) cudaFree(c->d_spc);
    if (c->d_tables) cudaFree(c->d_tables);
    if (c->d_in) cudaFree(c->d_in);
    if (c->d_out) cudaFree(c->d_out);
    if (c->d_check) cudaFree(c->d_check);
    if (c->d_dmr) cudaFree(c->d_dmr);
    if (c->d_counter) cudaFree(c->d_counter);
    if (c->d_dbg) cudaFree(c->d_dbg);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

}  // extern "C"
