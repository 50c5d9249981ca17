/*
 * chk_pcg.h -- C ABI of the B200-native PCG hot path for the periodic 3-D
 * checkerboard problem of arXiv 2007.06524 (reference package `checkerhom`,
 * /root/reference/pkg/src/checkerhom).
 *
 * Plain pointers and sizes only.  All double arrays passed to the compute
 * entry points are DEVICE pointers (cudaMalloc / torch CUDA tensors) unless a
 * comment says "host".  Grid vectors are fp64, C order, axis 0 slowest
 * (operators.py:374-381): idx = (x0*n + x1)*n + x2.  A batch of B
 * realizations is stored back to back ([B][n^3]).  `stream` is a
 * cudaStream_t (NULL = legacy default stream); every call is stream-ordered
 * with respect to it.
 *
 * Return codes (mirroring the reference error taxonomy, errors.py:4-38):
 *   CHK_OK           0
 *   CHK_EINVAL       1  bad argument / size mismatch      -> ValueError
 *                       (operators.py:304-305, spectral.py:107-108, lowrank.py:187-188)
 *   CHK_EUNSUPPORTED 2  unsupported grid (d != 3; n not n0*L with n <= 720;
 *                       slab entry points: n not a power of two in [8, 512])
 *                                                         -> ValueError
 * Grid sizes: n = n0*L with n0 a power of two >= 4 and any L >= 1, as the
 * reference (lattice.py:117-123,156-159).  Powers of two 8..512 (the BASELINE
 * configurations) run the fused kernels; every other n <= 720 (e.g. 12, 20,
 * 24, 96) runs plain device kernels with the same semantics and results.
 *   CHK_ECUDA        3  CUDA runtime failure              -> RuntimeError
 * chk_last_error() returns a thread-local message for the last failure.
 *
 * Per-realization PCG status (PcgReport semantics, solver.py:61-70,161-194):
 *   CHK_CONVERGED 0, CHK_NOT_CONVERGED 1, CHK_BREAKDOWN 2 (-> SolverBreakdown,
 *   solver.py:164-165,172-173).
 */
#ifndef CHK_PCG_H
#define CHK_PCG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CHK_OK 0
#define CHK_EINVAL 1
#define CHK_EUNSUPPORTED 2
#define CHK_ECUDA 3

#define CHK_CONVERGED 0
#define CHK_NOT_CONVERGED 1
#define CHK_BREAKDOWN 2

/* Preconditioner kinds (solver.py:29 PRECONDITIONERS). */
#define CHK_PRECOND_FOURIER 0     /* exact pseudo-inverse, spectral.py:77-87,98-112 */
#define CHK_PRECOND_LKR 1         /* low Kronecker rank, lowrank.py:141-192 */
#define CHK_PRECOND_REGULARIZED 2 /* 1/(g+delta), spectral.py:90-95 */

/* Grid / lattice geometry of one realization batch (lattice.py:82-166).
 * n = n0*L; k = 2*alpha*n0 h-cells of the sub-cell per axis, starting at
 * `offset` inside each cell; lam = background conductivity lambda. */
typedef struct chk_grid {
  int32_t d;      /* must be 3 */
  int32_t n;      /* grid nodes per axis */
  int32_t L;      /* cells per axis */
  int32_t n0;     /* h-cells per cell (power of two >= 4) */
  int32_t k;      /* sub-cell width in h-cells */
  int32_t offset; /* sub-cell start inside its cell */
  double lam;     /* lambda in (0, 1] */
} chk_grid;

typedef struct chk_precond_plan chk_precond_plan; /* opaque, immutable after create */

/* Options of one batched solve (SolveOptions, solver.py:32-58). */
typedef struct chk_pcg_opts {
  double tol;
  int32_t max_iter;
  int32_t precond_residual_stopping; /* solver.py:181-183 */
} chk_pcg_opts;

int32_t chk_abi_version(void);
const char* chk_last_error(void);

/* ---------------------------------------------------------------------------
 * Stiffness matvec: y = A x for B realizations (replaces the CSR product
 * `A.matrix() @ x`, solver.py:150,162 / operators.py:122-131, equal to the
 * edge-weighted stencil of tests/oracles.py:35-82).
 *   beta : device [B][L^3] per-cell contrast (0 for uncovered cells)
 *   x, y : device [B][n^3]
 *   xy   : device [B] receives <x, y> (p'Ap of solver.py:163) or NULL
 * ------------------------------------------------------------------------- */
int32_t chk_stencil_apply(const chk_grid* grid, const double* beta, const double* x, double* y,
                          double* xy, int32_t B, void* stream);

/* Corrector right-hand side on the device: f = scale * 1/2 (c[x+e_i] - c[x-e_i])
 * with c the nodal 2^3-cell average of the cell field (homogenize.py:75-89,
 * lattice.py:326-345).  direction in {1,2,3}; scale = h^(d-1) reproduces
 * corrector_rhs, h^(d-1)*h^(2-d) = h the PCG load of homogenize.py:110. */
int32_t chk_corrector_rhs(const chk_grid* grid, const double* beta, double* f, int32_t B,
                          int32_t direction, double scale, void* stream);

/* ---------------------------------------------------------------------------
 * Preconditioner plans (replace _cached_preconditioner, solver.py:79-93).
 * factors: HOST [3][r1][n] fp64, the CanonicalTensor factors produced by
 * dc_correction(canonical_reciprocal(...)) (lowrank.py:129,147-180), consumed
 * as-is; only read for CHK_PRECOND_LKR (pass NULL/0 otherwise).
 * eigenvalues: HOST [n], fourier_eigenvalues(n).values (spectral.py:56-68);
 * read for FOURIER / REGULARIZED (may be NULL for LKR).
 * ------------------------------------------------------------------------- */
int32_t chk_precond_plan_create(int32_t kind, int32_t n, int32_t r1, const double* factors,
                                const double* eigenvalues, double delta,
                                chk_precond_plan** out);
int32_t chk_precond_plan_destroy(chk_precond_plan* plan);

/* Device workspace (bytes) a chk_precond_apply of B vectors needs. */
size_t chk_precond_workspace_bytes(const chk_precond_plan* plan, int32_t B);

/* z = Re ifftn(D * fftn(r)) for B vectors (apply_lkr_preconditioner,
 * lowrank.py:183-192, and apply_fourier_preconditioner, spectral.py:98-112).
 * The zero-frequency term is kept exactly as the reference computes it. */
int32_t chk_precond_apply(const chk_precond_plan* plan, const double* r, double* z, int32_t B,
                          void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Batched mean-projected PCG (pcg_solve, solver.py:118-194), B independent
 * realizations sharing one grid shape and one preconditioner.
 *   beta       device [B][L^3]
 *   f          device [B][n^3]   right-hand sides (not modified)
 *   u          device [B][n^3]   solutions (output, mean zero)
 *   iterations HOST   [B]        PcgReport.iterations
 *   final_rel  HOST   [B]        PcgReport.final_residual
 *   status     HOST   [B]        CHK_CONVERGED / CHK_NOT_CONVERGED / CHK_BREAKDOWN
 *   rhs_projected HOST [B]       PcgReport.rhs_projected
 *   history    HOST   [B][max_iter] relative residuals (PcgReport.residuals) or NULL
 *   workspace  device buffer of chk_pcg_workspace_bytes(...) bytes
 * The call returns after the solve completed (it synchronizes internally on
 * a convergence poll every few iterations).
 * ------------------------------------------------------------------------- */
size_t chk_pcg_workspace_bytes(const chk_grid* grid, const chk_precond_plan* plan, int32_t B,
                               int32_t max_iter);
int32_t chk_pcg_solve_batched(const chk_grid* grid, const chk_precond_plan* plan,
                              const double* beta, const double* f, double* u, int32_t B,
                              const chk_pcg_opts* opts, int32_t* iterations, double* final_rel,
                              int32_t* status, int32_t* rhs_projected, double* history,
                              void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * The same batched solve from HOST buffers (the reference-facing call: numpy
 * in, numpy out).  beta_host [B][L^3], f_host [B][n^3] in, u_host [B][n^3]
 * out; pinned host memory makes the copies asynchronous.  The batch runs in
 * chunks of `chunk` realizations on three lanes (host threads with their own
 * stream, device slot and solver workspace, alternate chunks): one lane's
 * uploads, downloads and convergence tail overlap the other lanes' solves.
 * Per-realization results are identical to chk_pcg_solve_batched.
 * workspace: device buffer of chk_pcg_host_workspace_bytes bytes.
 * ------------------------------------------------------------------------- */
size_t chk_pcg_host_workspace_bytes(const chk_grid* grid, const chk_precond_plan* plan, int32_t chunk,
                                    int32_t max_iter);
int32_t chk_pcg_solve_host(const chk_grid* grid, const chk_precond_plan* plan, const double* beta_host,
                           const double* f_host, double* u_host, int32_t B, int32_t chunk,
                           const chk_pcg_opts* opts, int32_t* iterations, double* final_rel,
                           int32_t* status, int32_t* rhs_projected, double* history,
                           void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Realizations drawn on the device (sample_realization, lattice.py:284-311).
 * keys: [B][2] Philox4x64 keys of the realizations' streams, i.e.
 * SeedSequence(seed).generate_state(2, uint64) of each seed (lattice.py:279-281;
 * the hash stays on the host).  Cell c (C order) is covered iff the c-th
 * Generator.random() draw is < coverage_prob; its contrast is beta0
 * (CHK_CONTRAST_FIXED: the caller passes 1 - lam) or, CHK_CONTRAST_TWO_VALUE,
 * beta0 / beta1 by the (L^3 + c)-th draw < 1/2.  beta: device [B][L^3] out,
 * bit-identical to the reference's realization.  (The layered contrast stays on
 * the host path.)
 * ------------------------------------------------------------------------- */
#define CHK_CONTRAST_FIXED 0
#define CHK_CONTRAST_TWO_VALUE 1
int32_t chk_sample_cells(const chk_grid* grid, const uint64_t* keys, double coverage_prob, int32_t contrast_kind,
                         double beta0, double beta1, double* beta, int32_t B, void* stream);

/* Seeds-to-solutions pipeline: chk_pcg_solve_host with the realizations drawn
 * on the device from HOST keys_host [B][2] (as chk_sample_cells) and the load
 * either the device corrector RHS along rhs_direction (f_host NULL; the PCG
 * load of homogenize.py:110) or HOST f_host [B][n^3].  u_host and the reports
 * out as chk_pcg_solve_host; same workspace (chk_pcg_host_workspace_bytes). */
int32_t chk_pcg_solve_seeds(const chk_grid* grid, const chk_precond_plan* plan, const uint64_t* keys_host,
                            double coverage_prob, int32_t contrast_kind, double beta0, double beta1,
                            const double* f_host, int32_t rhs_direction, double* u_host, int32_t B, int32_t chunk,
                            const chk_pcg_opts* opts, int32_t* iterations, double* final_rel, int32_t* status,
                            int32_t* rhs_projected, double* history, void* workspace, size_t workspace_bytes,
                            void* stream);

/* ---------------------------------------------------------------------------
 * Slab decomposition of one grid over `nranks` GPUs (the
 * realization loop of ensemble_run, homogenize.py:133-182, shards instead).
 * Rank r owns planes x0 in [r n/P, (r+1) n/P) of p, u, f and one chunk of the
 * spectral columns.  The caller drives the iteration phase by phase and runs
 * the collectives in between (torch.distributed / NCCL):
 *   STATS, allreduce(red), STATS_DECIDE, FWD_INIT, all_to_all(xa -> xb),
 *   MID(0), allreduce(red), MID_DECIDE(0), all_to_all(xb -> xa), INV(0),
 *   then per iteration k: halo exchange of p (first/last local planes),
 *   FWD_Q(k), allreduce(red), ALPHA_DECIDE(k), all_to_all(xa -> xb), MID(k),
 *   allreduce(red), MID_DECIDE(k), all_to_all(xb -> xa), INV(k); finally
 *   MEANU, allreduce(red), MEANU_APPLY.
 * xa / xb: device exchange buffers of chk_slab_exchange_elems complex128
 * laid out [chunk s][b][local plane][x1 group][ncols]; all_to_all with equal
 * splits maps x0 slabs <-> column chunks.  red: device [B][4] doubles; phases
 * that produce rank-local sums zero it first; allreduce(SUM) it over ranks.
 * halo_lo / halo_hi: device [B][n*n] planes x0 = r n/P - 1 and (r+1) n/P.
 * ------------------------------------------------------------------------- */
typedef struct chk_slab {
  int32_t nranks; /* P: must divide n and the middle-pass tile count */
  int32_t rank;
} chk_slab;

#define CHK_SLAB_STATS 0
#define CHK_SLAB_STATS_DECIDE 1
#define CHK_SLAB_FWD_INIT 2
#define CHK_SLAB_MID 3
#define CHK_SLAB_MID_DECIDE 4
#define CHK_SLAB_INV 5
#define CHK_SLAB_FWD_Q 6
#define CHK_SLAB_ALPHA_DECIDE 7
#define CHK_SLAB_MEANU 8
#define CHK_SLAB_MEANU_APPLY 9

size_t chk_slab_exchange_elems(const chk_grid* grid, const chk_slab* slab, int32_t B);
size_t chk_slab_workspace_bytes(const chk_grid* grid, const chk_precond_plan* plan, const chk_slab* slab,
                                int32_t B, int32_t max_iter);
int32_t chk_slab_phase(const chk_grid* grid, const chk_precond_plan* plan, const chk_slab* slab,
                       int32_t phase, int32_t it, const double* beta, const double* f, double* u, double* p,
                       void* xa, void* xb, const double* halo_lo, const double* halo_hi, double* red,
                       int32_t B, const chk_pcg_opts* opts, void* workspace, size_t workspace_bytes,
                       void* stream);
/* The plane phases (FWD_INIT, FWD_Q, INV) over local planes [plane_begin,
 * plane_begin + plane_count) only: a phase split into plane chunks lets the
 * all_to_all of chunk k (rows of those planes, contiguous per destination in
 * xa / xb) overlap the kernels of chunk k+1.  The chunks of one phase must run
 * in plane order on one stream; plane_count < 0 means "to the last plane". */
int32_t chk_slab_phase_planes(const chk_grid* grid, const chk_precond_plan* plan, const chk_slab* slab,
                              int32_t phase, int32_t it, int32_t plane_begin, int32_t plane_count,
                              const double* beta, const double* f, double* u, double* p, void* xa, void* xb,
                              const double* halo_lo, const double* halo_hi, double* red, int32_t B,
                              const chk_pcg_opts* opts, void* workspace, size_t workspace_bytes, void* stream);
/* Stream-ordered copy of the B per-realization status words (3 = still active)
 * into `status` ([B] int32, pinned host or device): the convergence poll without
 * a host synchronisation. */
int32_t chk_slab_status_async(const chk_grid* grid, const chk_slab* slab, int32_t B, int32_t max_iter,
                              void* workspace, int32_t* status, void* stream);
/* Per-realization status words (device -> host, synchronous on `stream`). */
int32_t chk_slab_read_state(const chk_grid* grid, const chk_slab* slab, int32_t B, int32_t max_iter,
                            void* workspace, int32_t* iterations, double* final_rel, int32_t* status,
                            int32_t* rhs_projected, double* history, void* stream);

/* Number of kernels launched by the last chk_pcg_solve_batched on this thread
 * (the bench's gpu_launches evidence). */
int64_t chk_last_launch_count(void);

/* Per-kernel-class device timing (CUDA events on the launching stream) for the
 * calling thread: classes 0 stencil_dot, 1 fwd_plane, 2 mid_column,
 * 3 inv_plane, 4 other.  Enabling resets the accumulators; read returns the
 * summed milliseconds and launch counts of the solves since. */
int32_t chk_profile_enable(int32_t on);
int32_t chk_profile_read(double* ms /* [5] */, int64_t* launches /* [5] */);

#ifdef __cplusplus
}
#endif
#endif /* CHK_PCG_H */
