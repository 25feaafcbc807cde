/*
 * kbgrid.h -- C-ABI of the B200 NAO real-space grid pass (libkbgrid.so).
 *
 * The grid pass of an NAO-DFT SCF iteration:
 *   (G1) index      : which (atom, lattice image) spheres cover which grid points,
 *                     and the sparse atom-pair list (a, b, R) that carries DM and H;
 *   (G2) orbitals   : phi_{a,l zeta m}(r) = u_{l zeta}(|r - t_a|) * P_lm(r - t_a)
 *                     (u = radial table R(r)/r^l, P_lm = real solid harmonic);
 *   (G3) density    : rho(r)  = sum_{ab} sum_ij phi_ai(r) DM_ab(R)_ij phi_bj(r);
 *   (G4) hamiltonian: H_ab(R)_ij += sum_r phi_ai(r) V(r) dV phi_bj(r).
 *
 * Reference anchor.  arxiv/paper_1402_4247 ships no code for this path
 * (/root/reference/SPEC.md:9 and :318 put it out of scope).
 * The entry points below are what the reference's Band_DFT_Col pipeline would
 * bind between Part 6 (density_matrices, producing
 * DensityMatrices) and Part 1 (bloch_transform, SPEC.md:235-243,
 * consuming RealSpaceOperator).  They follow the reference's
 * conventions:
 *   - status codes mirror the kband::Error taxonomy
 *     (/root/reference/proj/include/kband/common.hpp:21-38);
 *   - an optional work tally mirrors kband::WorkTally (common.hpp:43-56);
 *   - errors carry a message naming the failing index, like
 *     householder.cpp:119-123 / :312-316 (kbg_last_error).
 *   - pure, reentrant operations on caller-owned buffers; one
 *     host thread per context (ThreadTeam single-job rule, common.hpp:84-93).
 *
 * Conventions (shared bit-for-bit with the CPU oracle in oracle/):
 *   lattice[3*i + c]  = Cartesian component c of lattice vector a_i (bohr).
 *   grid point (i,j,k), 0 <= i < N0 ...; linear index p = (i*N1 + j)*N2 + k.
 *   position r_c = (fi*A[0][c] + fj*A[1][c]) + fk*A[2][c], fi = (double)i/N0,
 *   image centre t_c = tau_c + ((R0*A[0][c] + R1*A[1][c]) + R2*A[2][c]),
 *   d = r - t,  d2 = (d0*d0 + d1*d1) + d2*d2 (no fused multiply-add),
 *   sphere membership  d2 < rc*rc  (strict).
 *   Pair (a, b, R) exists iff |t_b(R) - tau_a|^2 < (rc_a + rc_b)^2, same
 *   expression order.  Pairs sorted lexicographically by (a, b, R0, R1, R2);
 *   the block of pair p is n_a x n_b doubles, row-major, at pair_off[p].
 *   Grid blocks are 4x4x4 points, block id = (bi*nb1 + bj)*nb2 + bk; within
 *   a block point (li,lj,lk) has slot
 *     ((((li>>1)*2 + (lj>>1))*2 + (lk>>1)) * 8) + ((li&1)*2 + (lj&1))*2 + (lk&1)
 *   and bit `slot` of a cover mask is set iff that point lies in the sphere.
 *   Orbital order inside an atom: species radial list order; within l:
 *     s; p_x p_y p_z; d_z2, d_x2-y2, d_xy, d_xz, d_yz.
 *   Radial table of (species, radial fn r): table[(r*ntab + k)*2 + {0,1}] =
 *     (u(r_k), du/dr(r_k)), r_k = k*rc/(ntab-1), u = R(r)/r^l; cubic Hermite.
 *   Spin-major arrays: dm/h [nspin][nnz], rho/veff [nspin][npts].
 */
#ifndef KBGRID_H
#define KBGRID_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KBG_OK 0
#define KBG_ERR_CONFIG 1      /* kband::ConfigError      */
#define KBG_ERR_DIMENSION 2   /* kband::DimensionError   */
#define KBG_ERR_CONSISTENCY 3 /* kband::ConsistencyError */
#define KBG_ERR_NONFINITE 4   /* kband::ConvergenceError (non-finite values) */
#define KBG_ERR_CUDA 5        /* CUDA runtime failure / no device */
#define KBG_ERR_NCCL 6        /* collective failure (host-side reduction) */

#define KBG_BLOCK_EDGE 4      /* grid block = 4x4x4 points = 64 slots */
#define KBG_MAX_L 2           /* s, p, d */
#define KBG_MAX_ORB_PER_ATOM 32

typedef struct kbg_species {
    int nrad;            /* number of radial functions                       */
    const int* l;        /* [nrad] angular momentum, 0..KBG_MAX_L            */
    double rc;           /* cutoff radius (bohr), > 0                        */
    int ntab;            /* radial table points, >= 4                        */
    const double* table; /* [nrad][ntab][2] (u, du/dr)                       */
} kbg_species;

typedef struct kbg_system {
    double lattice[9];        /* rows = lattice vectors (bohr)                */
    int grid[3];              /* N0, N1, N2                                   */
    int natom;
    const int* species;       /* [natom] species id                           */
    const double* tau;        /* [natom*3] Cartesian positions (bohr)         */
    int nspecies;
    const kbg_species* spec;  /* [nspecies]                                   */
} kbg_system;

/* Host view of the integer index (bit-exact parity surface). Pointers are
 * owned by the context and stay valid until the next kbg_build_index or
 * kbg_destroy. */
typedef struct kbg_index {
    int64_t npts;
    int nblk[3];
    int64_t nblock;
    int64_t ncover;
    const int32_t* blk_ptr;   /* [nblock+1] CSR into the cover arrays         */
    const int32_t* cov_atom;  /* [ncover]                                     */
    const int32_t* cov_R;     /* [ncover*3] lattice image of the atom         */
    const uint64_t* cov_mask; /* [ncover] slot mask                           */
    int64_t npair;
    const int32_t* pair_a;    /* [npair]                                      */
    const int32_t* pair_b;    /* [npair]                                      */
    const int32_t* pair_R;    /* [npair*3]                                    */
    const int64_t* pair_off;  /* [npair+1] value offsets                      */
    const int32_t* pair_mirror; /* [npair] index of (b, a, -R)                */
    int64_t nnz;              /* pair_off[npair]                              */
    int64_t nbpair;           /* canonical (block, cover-pair) work items     */
    int64_t natompt;          /* sum of popcount(cov_mask)                    */
    double sum_m;             /* sum_r m(r)   (m = nonzero orbitals at r)     */
    double sum_m2;            /* sum_r m(r)^2                                 */
} kbg_index;

/* Work accounting (kband::WorkTally analogue): algorithmic flops and
 * compulsory bytes of the last call, SURVEY.md section 8(d) formulas. */
typedef struct kbg_tally {
    double flops;
    double bytes;
} kbg_tally;

typedef struct kbg_ctx kbg_ctx;

/* Create a context on CUDA device `device`; copies the system (the caller's
 * arrays may be freed afterwards). Validates the system (ConfigError /
 * DimensionError with a message naming the bad field). */
int kbg_create(const kbg_system* sys, int device, kbg_ctx** out);

/* Sharded context for multi-GPU: this rank owns a contiguous, cost-balanced
 * range of grid blocks. rho is produced for owned points only; H holds this
 * rank's partial sums -- the caller sums it across ranks (ncclAllReduce,
 * see INTEGRATION.md). */
int kbg_create_sharded(const kbg_system* sys, int device, int rank, int nranks, kbg_ctx** out);

/* Build the integer index on the device (once per geometry). */
int kbg_build_index(kbg_ctx* ctx);

/* Host copies of the index lists (for bit-exact parity and for callers that
 * lay out DM / H in pair order). */
int kbg_index_view(kbg_ctx* ctx, kbg_index* out);

/* Execution plan chosen by kbg_build_index (diagnostics): info[0] persistent kernels in use (1/0),
 * [1] intra-block schedule (KBG_OPT_SCHEDULE bits actually used), [2] rho partner-range split,
 * [3] max padded Phi rows of a block, [4] max H tasks, [5] max rho tasks of a block,
 * [6] / [7] dynamic shared memory per CTA of the H / rho persistent kernel (bytes). */
int kbg_plan_info(const kbg_ctx* ctx, int64_t info[8]);

/* Owned block range [blk_begin, blk_end) of this context (sharded or not). */
int kbg_shard_range(const kbg_ctx* ctx, int64_t* blk_begin, int64_t* blk_end);

/* Host-pointer drop-in entry points: copies in, computes, copies out.
 * dm: [nspin][nnz]; rho: [nspin][npts] (every point written; points outside
 * this shard are written as 0 in a sharded context). DM must satisfy
 * DM_ba(-R) = DM_ab(R)^T (DensityMatrices invariant); violations
 * above 1e-13 * max|DM| return KBG_ERR_CONSISTENCY. */
int kbg_density(kbg_ctx* ctx, int nspin, const double* dm, double* rho);
/* veff: [nspin][npts]; h: [nspin][nnz], overwritten with sum_r phi V dV phi. */
int kbg_hamiltonian(kbg_ctx* ctx, int nspin, const double* veff, double dV, double* h);

/* One SCF grid pass through host buffers: rho from dm and h from veff in one
 * call (the drop-in an SCF loop makes per iteration). The two halves run on
 * two streams so each half's host<->device copies overlap the other half's
 * kernels (pinned host buffers make the copies asynchronous). DM is checked
 * like kbg_density; on a violation the status is KBG_ERR_CONSISTENCY and the
 * outputs are invalid. Pinned (mapped) host veff / rho are read / written in
 * place by the kernels, without staging copies. On a sharded context after
 * kbg_comm_open, h is the full H on every rank (fused NVLink reduction; every
 * rank must make the call) and rho holds this rank's points. */
int kbg_grid_pass(kbg_ctx* ctx, int nspin, const double* dm, const double* veff, double dV, double* rho,
                  double* h);

/* Device-pointer variants (timing path). `stream` is a cudaStream_t (0 =
 * legacy default). No host synchronisation, no validation. */
int kbg_density_dev(kbg_ctx* ctx, int nspin, const double* d_dm, double* d_rho, void* stream);
int kbg_hamiltonian_dev(kbg_ctx* ctx, int nspin, const double* d_veff, double dV, double* d_h,
                        void* stream);

/* Phase split of kbg_hamiltonian_dev for timing: accumulate canonical pair
 * blocks (hot kernel), then mirror H_ba(-R) = H_ab(R)^T. */
int kbg_hamiltonian_accumulate_dev(kbg_ctx* ctx, int nspin, const double* d_veff, double dV,
                                   double* d_h, void* stream);
int kbg_hamiltonian_mirror_dev(kbg_ctx* ctx, int nspin, double* d_h, void* stream);

/* (new) One SCF grid pass on device buffers: rho and the mirrored H, on a single-rank context: density
 * then Hamiltonian, or with KBG_OPT_FUSED_PASS (FP64-atomic H, persistent kernels) ONE fused
 * persistent kernel -- each block's Phi staged once, its rho and H tasks interleaved on the same SM
 * (56 atoms 1.7 % faster, 448 atoms 13 % slower: DESIGN.md). No host synchronisation. */
int kbg_grid_pass_dev(kbg_ctx* ctx, int nspin, const double* d_dm, const double* d_veff, double dV, double* d_rho,
                      double* d_h, void* stream);

/* Orbital values phi on all grid points of one block, [ncover_blk][64] rows
 * in cover order (testing surface for G2). out must hold M*64 doubles where
 * M = total orbitals of the block's covers; *m_out receives M. */
int kbg_block_orbitals(kbg_ctx* ctx, int64_t block, double* out, int64_t cap, int* m_out);

/* Number of kernel launches made by the last kbg_density_dev /
 * kbg_hamiltonian_dev call (evidence for gpu_launches). */
int kbg_last_launches(const kbg_ctx* ctx);

/* Persistent-kernel timing counters (clock64 cycles summed over warps/CTAs
 * since the last KBG_OPT_DEBUG_COUNTERS reset): [0] producer wait on empty,
 * [1] producer total, [2] consumer wait on full, [3] consumer wait at the end,
 * [4] consumer total, [5] blocks seen by consumers, [6] consumer wait on the
 * first two blocks, [7] producer-measured copy latency (the producer waits for
 * each copy when counters are on), [8] copies, [10] last-consumer reduce +
 * release, [11] bytes copied. Profiling aid. */
int kbg_debug_counters(kbg_ctx* ctx, int64_t* out, int n);

/* Work tally of the last density / hamiltonian call. */
int kbg_last_tally(const kbg_ctx* ctx, kbg_tally* out);

/* Options. KBG_OPT_WARPS: warps per CTA of the grid kernels (4 or 8). */
#define KBG_OPT_WARPS 1
#define KBG_OPT_FAULT_SIGN 2 /* test hook: flip the sign of the H accumulate (kband fault_proc6_sign analogue) */
#define KBG_OPT_SCATTER_STORE 3 /* timing experiment: plain stores instead of atomics (H is WRONG) */
#define KBG_OPT_PERSIST 4 /* 1 (default): persistent warp-specialized kernels when they fit; 0: one CTA per block */
#define KBG_OPT_DEBUG_COUNTERS 5 /* nonzero: enable + reset the persistent kernels' timing counters */
/* Intra-block schedule of the persistent kernels, read by kbg_build_index: bit 0 (H) / bit 1 (rho) set = the
 * block's tasks, heaviest first, form one queue the consumer warps pull from; clear = static LPT lists per
 * warp. Default 3. rho stays bitwise deterministic either way (per-task partial sums, fixed-order reduce). */
#define KBG_OPT_SCHEDULE 6
/* Order in which the persistent kernels pull grid blocks, read by kbg_build_index: 0 heaviest first (load
 * balance of the tail); 1 natural (i, j, k) block order (neighbouring blocks in flight share their atom
 * pairs' DM / H entries in L1/L2); 2 (default) natural when the rank owns more than 500 blocks per SM
 * (the tail is then negligible and the locality pays: 1512 atoms rho 8.68 -> 8.44 ms), else heaviest
 * first. */
#define KBG_OPT_BLOCK_ORDER 7
/* Exchange-correlation of kbg_veff: 0 (default) Slater exchange only; 1 LSDA = exchange + Perdew-Wang 1992
 * correlation (energy[1] is then E_xc). */
#define KBG_OPT_XC 8
/* H accumulation: 1 deterministic -- every H contribution is split into two parts on fixed power-of-two
 * grids derived from max|V_eff| (one extra max-reduction over V per H pass) and added with exact FP64
 * atomics, so H has the same bits on every run, with every kernel/schedule, and on any number of GPUs
 * (the multi-GPU reduction adds the limbs the same way); 0 (default) plain FP64 atomics, ~1.4x faster on
 * the 56-atom cell, whose last bits depend on the order of arrival (<= 1e-15 relative run to run).
 * Either way a non-finite V_eff gives KBG_ERR_NONFINITE from the host API. */
#define KBG_OPT_DETERMINISTIC 9
/* kbg_grid_pass on a sharded context after kbg_comm_open: 1 (default) shard-local host transfers -- the
 * rank copies in only the DM ranges holding the pairs its blocks touch, reads V at its points, writes
 * rho only at the points of its blocks and H only in its slice of each spin's entries (kbg_shard_io);
 * the other entries of the caller's buffers are left as they were. 0: every rank reads everything and
 * returns the full H and a full-size rho (zeros outside its blocks). */
#define KBG_OPT_SHARD_IO 10
/* A5's "dense enough" switch: H tasks whose point density (exact common points / points of the quads the
 * DMMA path executes, x 255) is below this threshold run point-exact FP64 FMAs instead of DMMA over whole
 * quads. 0 (default): every task on the FP64 tensor path (measured faster at every cutoff). */
#define KBG_OPT_SPARSE_DFMA 11
/* Sharded contexts: SMs the peer-memory H exchange runs on while the density pass runs on the others
 * (0..32). k > 0 (default 8): the exchange runs as k whole-SM CTAs concurrently with the density kernel,
 * which leaves those k SMs free -- in kbg_grid_pass, and for a caller that runs
 * kbg_hamiltonian_exchange_dev on a second stream next to kbg_density_dev. 0: the exchange takes the
 * whole GPU before (kbg_grid_pass) or after (the split device API on one stream) the density pass. */
#define KBG_OPT_EXCHANGE_SMS 12
/* kbg_grid_pass_dev: 1 = one fused rho + H persistent kernel (see there), 0 = separate kernels,
 * 2 (default) = fused while nspin x (repacked DM + H) <= 24 MB (the two share L2 without contention). */
#define KBG_OPT_FUSED_PASS 13
int kbg_set_option(kbg_ctx* ctx, int option, int64_t value);

const char* kbg_last_error(const kbg_ctx* ctx);
const char* kbg_status_string(int status);
void kbg_destroy(kbg_ctx* ctx);

/* ---- V_eff from rho ----------------------------------------
 * The step between the density and the Hamiltonian pass of one SCF iteration:
 * V_eff,s = V_H[rho] + V_x,s[rho_s] + V_loc with V_H from the periodic Poisson
 * equation in G space (4 pi rho(G)/|G|^2, G = 0 dropped: neutralizing
 * background; cuFFT) and exchange-only local spin density (Slater) V_x,s =
 * -(6 rho_s/pi)^(1/3) (nspin 1: rho_s = rho/2). Hartree atomic units; grids
 * [nspin][npts] C-order as the density pass writes them; vloc [npts] may be
 * NULL; energy (may be NULL) receives E_H = 1/2 int V_H rho, E_x (E_xc with
 * KBG_OPT_XC = 1: + PW92 correlation). Does not need the index. */
int kbg_veff(kbg_ctx* ctx, int nspin, const double* rho, const double* vloc, double* veff, double* energy);
int kbg_veff_dev(kbg_ctx* ctx, int nspin, const double* d_rho, const double* d_vloc, double* d_veff,
                 double* d_energy, void* stream);

/* ---- Multi-GPU H without NCCL --------------------------------
 * Sharded contexts (one per GPU / process) exchange their H partials through
 * peer memory: each rank publishes an exchange buffer (kbg_comm_handle, a
 * KBG_COMM_HANDLE_BYTES blob to all-gather, e.g. with torch.distributed),
 * opens every peer's (kbg_comm_open, blobs in rank order), and
 * kbg_hamiltonian_allreduce_dev then leaves the FULL mirrored H on every rank:
 * accumulate the shard into the own buffer, one kernel that waits for all
 * partials (flags in peer memory), sums its slice of the canonical pairs in
 * rank order, mirrors it and stores it into every rank's buffer over
 * NVLink, and a copy-out once all slices have landed. Replaces
 * hamiltonian_dev + ncclAllReduce; same bits on every rank. */
#define KBG_COMM_HANDLE_BYTES 96
int kbg_comm_handle(kbg_ctx* ctx, void* handle_out);
int kbg_comm_open(kbg_ctx* ctx, const void* handles);
int kbg_hamiltonian_allreduce_dev(kbg_ctx* ctx, int nspin, const double* d_veff, double dV, double* d_h,
                                  void* stream);
/* The two halves of kbg_hamiltonian_allreduce_dev: accumulate this rank's partial H into its exchange
 * buffer, then (same nspin, later on the stream, after any independent work such as the density pass)
 * the fused reduce + mirror that leaves the full H in d_h. Placing the density pass between them lets
 * the exchange find every peer ready instead of waiting for the slowest rank. */
int kbg_hamiltonian_partial_dev(kbg_ctx* ctx, int nspin, const double* d_veff, double dV, void* stream);
int kbg_hamiltonian_exchange_dev(kbg_ctx* ctx, int nspin, double* d_h, void* stream);
/* After synchronizing a kbg_hamiltonian_allreduce_dev: KBG_ERR_NCCL if a peer
 * never arrived (the kernels give up after 10 s instead of hanging the GPU;
 * the H of that call is invalid), else KBG_OK. Clears the flag. kbg_grid_pass
 * on a sharded context checks it itself. */
int kbg_comm_check(kbg_ctx* ctx);
/* Shard-local I/O ranges of this rank (after kbg_comm_open): out[0..1] its blocks [b0, b1), out[2..3] the
 * points [p0, p1) of its grid-plane range in C order (kbg_grid_pass writes rho at the points of its blocks;
 * with a pageable rho buffer the D2H covers [p0, p1) and the other points there become 0), out[4..5] its
 * slice [h0, h1) of each spin's H entries, out[6] DM doubles per spin it copies in (ranges covering the
 * pairs its blocks touch and their mirror blocks, for the symmetry check), out[7] = p1 - p0. */
int kbg_shard_io(const kbg_ctx* ctx, int64_t out[8]);
/* Timing aid: with KBG_COMM_TIMING set in the environment at kbg_comm_open, the
 * phase times (ns from the reduce kernel's start) of the last exchange: all
 * partials ready, slice reduced, copy kernel start, all slices landed, done. */
int kbg_comm_timing(kbg_ctx* ctx, double* out5);

/* ---- Formats either side of the grid pass ----------------
 * The pair-sparse blocks of kbg_index (grid-pass DM input, H output) against
 * the reference's band-pipeline types: RealSpaceOperator (dense n x n block
 * M_R per lattice offset R), its Bloch image
 * (Part 1 bloch_transform) and the real-space folding of
 * k-resolved density matrices (Part 6 density_matrices).
 * Orbital row of atom a, orbital i: orb_off[a] + i with orb_off the prefix sum
 * of the atoms' orbital counts (n = nbasis). k points are fractional
 * (reciprocal-lattice) coordinates, R integer lattice offsets. Complex
 * matrices are row-major n x n of interleaved (re, im) doubles. One matrix
 * (one spin) per call; `pairs` holds nnz values. The index must be built. */

/* Distinct lattice offsets of the pair list, sorted lexicographically
 * (R = 0 included): *nR receives the count; R (3 * nR ints) may be NULL. */
int kbg_offsets(kbg_ctx* ctx, int* nR, int32_t* R);

/* pair-sparse -> RealSpaceOperator blocks [nR][n][n] in kbg_offsets order
 * (entries outside the pair list are 0), and back (extracts the pair-list
 * entries of dense blocks). */
int kbg_to_realspace(kbg_ctx* ctx, const double* pairs, double* blocks);
int kbg_from_realspace(kbg_ctx* ctx, const double* blocks, double* pairs);
int kbg_to_realspace_dev(kbg_ctx* ctx, const double* d_pairs, double* d_blocks, void* stream);
int kbg_from_realspace_dev(kbg_ctx* ctx, const double* d_blocks, double* d_pairs, void* stream);

/* Bloch transform M(k) = sum_R exp(+2 pi i k.R) M_R for nk k points
 * (kpts: 3 * nk host doubles); out: [nk][n][n] complex. The host variant
 * validates M_{-R} = M_R^T (the RealSpaceOperator invariant) first and
 * returns KBG_ERR_CONSISTENCY naming the offending pair and R. */
int kbg_bloch(kbg_ctx* ctx, const double* pairs, int nk, const double* kpts, double* out);
int kbg_bloch_dev(kbg_ctx* ctx, const double* d_pairs, int nk, const double* kpts, double* d_out, void* stream);

/* Real-space folding DM_R = sum_k w_k exp(-2 pi i k.R) rho_k onto the pair
 * list (real part; for a time-reversal-symmetric k set the imaginary part
 * vanishes -- its largest magnitude is returned in *max_imag, may be NULL).
 * rho_k: [nk][n][n] complex; w: nk host weights. */
int kbg_fold(kbg_ctx* ctx, int nk, const double* kpts, const double* w, const double* rho_k, double* pairs,
             double* max_imag);
int kbg_fold_dev(kbg_ctx* ctx, int nk, const double* kpts, const double* w, const double* d_rho_k, double* d_pairs,
                 void* stream);

/* Part 6 density matrix at one k from the states of the eigenvector pass
 * (SPEC.md:279): rho_k = sum_i w_i c_i c_i^H, C: [n][m] complex row-major
 * (column i = state i), w: m real weights -- occupations f_i for the charge
 * density matrix, eps_i f_i for the energy density matrix. out: [n][n]
 * complex. One ZGEMM (cuBLAS; a plain library GEMM) after a weight kernel. */
int kbg_density_matrix_k(kbg_ctx* ctx, int m, const double* C, const double* w, double* rho);
int kbg_density_matrix_k_dev(kbg_ctx* ctx, int m, const double* d_C, const double* d_w, double* d_rho,
                             void* stream);

/* HBM calibration probe (the paper's Table 2 experiment,
 * PAPER.md:56): divide each of nvec vectors of len doubles
 * (row-major, contiguous) by its Euclidean norm; zero vectors stay zero.
 * Context-free; device is the current CUDA device. Host variant copies in and
 * out through the library's own staging buffers (times the transfers the
 * paper's Table 2 discussion is about). */
int kbg_normalize_rows_dev(double* d_x, int64_t nvec, int64_t len, void* stream);
int kbg_normalize_rows(double* x, int64_t nvec, int64_t len);

/* ---- Eigen_HH on the GPU ----------------------------------
 * The reference's Householder eigensolver pieces (kband, /root/reference/proj/
 * include/kband/householder.hpp:56-82), context-free. Complex arrays are
 * interleaved (re, im) doubles, row-major. The tridiagonal QL solve between
 * tridiagonalize and back_transform stays with the caller (kband::
 * solve_tridiag, tridiag.hpp:18-21; the paper runs LAPACK on the CPUs there).
 * Errors: kband taxonomy status codes, message from kbg_hh_last_error(). */

/* kband::tridiagonalize (householder.hpp:65-67): a [n][n] Hermitian (defect
 * <= 1e-13, symmetrized like HermitianMatrix::from); out d [n], e [n-1] and the
 * stage records: u [n-1][n] complex (reflector of stage i, zero above i+1 and
 * for skipped stages), h, s [n-1], phase [n-1] complex. fault_sign != 0 flips
 * the procedure-6 sign (ProcedurePlan::fault_proc6_sign). n <= 4800. The _dev
 * variant destroys d_a (working matrix) and skips the Hermitian check. */
int kbg_hh_tridiagonalize(int64_t n, const double* a, int fault_sign, double* d, double* e, double* u, double* h,
                          double* s, double* phase);
int kbg_hh_tridiagonalize_dev(int64_t n, double* d_a, int fault_sign, double* d_d, double* d_e, double* d_u,
                              double* d_h, double* d_s, double* d_phase, void* stream);

/* kband::back_transform (householder.hpp:69-72): W [n][m] complex = Q Y for the
 * real tridiagonal-basis eigenvectors Y [n][m] (columns). */
int kbg_hh_back_transform(int64_t n, int64_t m, const double* u, const double* h, const double* phase,
                          const double* y, double* w);
int kbg_hh_back_transform_dev(int64_t n, int64_t m, const double* d_u, const double* d_h, const double* d_phase,
                              const double* d_y, double* d_w, void* stream);

/* kband::normalize_columns (householder.hpp:74-76): columns of c [n][m]
 * complex to unit 2-norm in place; a zero column is KBG_ERR_CONSISTENCY. */
int kbg_hh_normalize_columns(int64_t n, int64_t m, double* c);
int kbg_hh_normalize_columns_dev(int64_t n, int64_t m, double* d_c, void* stream);
/* kband::triple_product (linalg.hpp:82-84, Part 3 S^H H S): c [m][m] = T^H H T
 * for T [n][m], H [n][n] Hermitian, re-symmetrized and validated Hermitian
 * (defect <= 1e-13 max(1, ||C||_F)). Two ZGEMMs (cuBLAS: plain library GEMMs). */
int kbg_hh_triple_product(int64_t n, int64_t m, const double* t, const double* h, double* c);
/* The tridiagonal eigensolve between tridiagonalize and back_transform
 * (kband::solve_tridiag, tridiag.hpp:18-21: implicit QL on the host in the
 * reference, LAPACK on the CPUs in the paper) on the GPU: multisection on
 * kband's Sturm count for the eigenvalues (ascending into w [n]), inverse
 * iteration with re-orthogonalization inside clusters (gaps < 1e-3 ||T||_1)
 * for the eigenvectors (columns of z [n][n], row-major; want_vectors = 0 leaves
 * z untouched). d [n], e [n-1]. n <= 12000. */
int kbg_tridiag_solve(int64_t n, const double* d, const double* e, int want_vectors, double* w, double* z);
int kbg_tridiag_solve_dev(int64_t n, const double* d_d, const double* d_e, int want_vectors, double* d_w, double* d_z,
                          void* stream);
/* kband::eigen_hh (householder.hpp:78-80) on the device end to end: a [n][n]
 * Hermitian (defect <= 1e-13) -> eigenvalues ascending w [n] and, if
 * want_vectors, normalized eigenvectors as the columns of c [n][n] complex;
 * tridiagonalize, kbg_tridiag_solve, back_transform and normalize_columns with
 * the data resident on the GPU (only a in and w, c out cross PCIe). n <= 4800. */
int kbg_hh_eigen(int64_t n, const double* a, int want_vectors, double* w, double* c);
const char* kbg_hh_last_error(void);

/* Library identification: "kbgrid <version> sm_100a". */
const char* kbg_version(void);

#ifdef __cplusplus
}
#endif

#endif /* KBGRID_H */
