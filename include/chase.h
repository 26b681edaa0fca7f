/* chase.h -- C ABI of the B200-native ChASE library (libchase_b200.so).
 *
 * Problem (§2; Alg. 1 Require/Ensure): for a Hermitian
 * H (N x N, complex double), find the nev lowest ("extreme", ledger #17) eigenpairs
 * H y = lambda y by Chebyshev-filtered subspace iteration with search space nev+nex.
 *
 * Data layout (§3.2):
 *   - Ranks form an r x c grid, rank = i + j*r (column-major numbering).
 *   - Rows of H are split into r blocks, columns into c blocks; the first (N mod r) row blocks
 *     (resp. (N mod c) column blocks) get one extra row (ledger #19).  Rank (i,j) owns the shard
 *     H_ij = H[row0_i : row0_i+p_i, col0_j : col0_j+q_j], column-major, leading dim ldh >= p_i,
 *     complex double interleaved (re, im) == torch.complex128, ON THE DEVICE.
 *   - "V-layout" blocks are q_j x ncols, rows [col0_j, col0_j+q_j), replicated over
 *     the column communicator j.  "W-layout" blocks are p_i x ncols, rows
 *     [row0_i, row0_i+p_i), replicated over the row communicator i.
 *
 * Ownership: the caller owns H and every buffer passed in; the library never frees them.  The
 * library owns its workspace (allocated in chase_init, sized from N, nev_max+nex_max)
 * and its CUDA stream/events and NCCL communicators.
 *
 * Collectives: chase_init, chase_solve, chase_filter, chase_hemm_step, chase_lanczos,
 * chase_finalize must be called by all r*c ranks with identical scalar arguments.  Arguments are
 * validated collectively (allreduce of an error flag) so every rank returns the same status.
 * chase_set_option must be called identically on all ranks; chase_local_layout and
 * chase_last_error are local.
 *
 * Errors: every call returns a chase_status; the message of the last failure is available from
 * chase_last_error.  CUDA/NCCL errors leave the handle unusable (finalize it).
 * All calls are synchronous with respect to the host (they synchronize the library stream
 * before returning), except where stated.
 */
#ifndef CHASE_B200_H
#define CHASE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct chase_handle chase_handle;

typedef enum {
  CHASE_OK = 0,
  CHASE_E_USAGE = 2,    /* invalid arguments (S:596 exit code 2) */
  CHASE_E_NUMERIC = 3,  /* Lanczos breakdown, CholQR failure after fallback, Jacobi non-convergence */
  CHASE_E_IO = 4,
  CHASE_E_CUDA = 5,
  CHASE_E_NCCL = 6,
  CHASE_E_NOMEM = 7,    /* workspace does not fit (memory check) */
  CHASE_E_MAXITER = 8   /* max_iter reached; `locked` pairs in the report are valid */
} chase_status;

typedef enum {
  CHASE_C128 = 0, /* complex<double>, interleaved (re, im): Hermitian H -- the north_star path */
  CHASE_C64 = 1,  /* complex<float> interleaved: Hermitian H in complex single; every product with
                     H runs on the tcgen05 tensor cores (TF32 with the 3xTF32 split, FP32-class
                     accuracy) or, for Lanczos, an FP64-accumulated skinny kernel.  chase_solve
                     iterates QR / RR / residuals in complex double on the library's workspace and
                     returns complex<float> vectors (approx input likewise).  Layout limits of the
                     TMA operands: q % 4 == 0, p even, ldh even, 16-byte aligned H.  The library
                     keeps the 3xTF32 lo part of H (one extra shard-sized buffer). */
  CHASE_R64 = 2   /* double: real symmetric H, the paper's own experimental field.
                     Every buffer argument is then real double with the same layouts. */
} chase_dtype;

typedef struct {
  chase_dtype dtype;              /* CHASE_C128, CHASE_C64 or CHASE_R64 */
  int64_t N;                      /* matrix order */
  int32_t nev_max, nex_max;       /* workspace sizing */
  int32_t grid_rows, grid_cols;   /* r, c; 0,0 = auto: r * c = world, r <= c, |r - c| minimal
                                     (ledger #19).  world_size == 1 with r*c > 1 selects
                                     the emulated-grid mode: the handle owns shard `rank` of an
                                     r x c grid and all cross-rank sums are skipped (each call
                                     returns this rank's partial) -- for single-GPU testing. */
  int32_t rank, world_size;       /* rank = i + j*r */
  const void* nccl_unique_id;     /* 128-byte ncclUniqueId, identical on all ranks; NULL if world_size == 1 */
  int32_t cuda_device;
  void* cuda_stream;              /* cudaStream_t the caller produces inputs on (e.g. torch's current
                                     stream); every call waits for work already queued on it.
                                     NULL = the legacy default stream. */
  int32_t colocated;              /* 0: one process per rank, NCCL communicators (production).
                                     1: the world_size ranks are threads of THIS process, each with
                                     its own handle (usually all on one device, which NCCL refuses):
                                     the communicators are an in-process group keyed by the 128
                                     bytes at nccl_unique_id (any bytes shared by the ranks), sums
                                     taken in rank order (replicas bitwise identical), and the fused
                                     f1 reduction uses the co-located handles' own device pointers.
                                     Every collective call must then be made concurrently by all
                                     ranks' threads.  For single-GPU testing of the grid data plane. */
} chase_init_args;

typedef struct {
  int32_t iterations, locked;
  int64_t matvecs;                /* sum over filter calls of sum_a m_a (P:729-731 footnote) */
  double filter_flops;            /* 8 N^2 matvecs (complex) or 2 N^2 matvecs (real) */
  double t_all, t_lanczos, t_filter, t_qr, t_rr, t_resid;   /* seconds, Table 2 columns P:646-655 */
  double b_sup, mu_1, mu_ne, nu, max_resid;
} chase_report;

/* Create a handle: selects the device, builds the r x c grid and NCCL world/row/col
 * communicators (row comm: color i, key j; column comm: color j, key i), allocates workspace. */
chase_status chase_init(chase_handle** out, const chase_init_args* args);

/* Options (defaults): deg_max=36, max_iter=0 (auto: iterate while the solve progresses -- a new
 * locked pair or the smallest active residual below 0.99 x its best so far -- and return
 * CHASE_E_MAXITER after stall_iter=100 iterations without progress, or 5000 in all; a value > 0
 * is a hard cap), deg_extra=2 (degrees added to the optimal-degree estimate before the cap --
 * the estimate aims exactly at tol and otherwise lets columns just above tol creep),
 * lanczos_steps=25, lanczos_runs=4, seed_v=2,
 * seed_lanczos=3, largest=0, approx=0 (1: ritz_vectors holds an initial V-hat on entry),
 * gemm3m=1 (filter and H*Q products use the 3M complex product -- 3 real DMMAs per complex
 * multiply-add instead of 4; normwise-stable; 0 selects the 4M kernel),
 * mixed_filter=0 (CHASE_C128 only: a value r > 0 runs the filter of an iteration on a
 * complex-single shadow of the shard -- the tcgen05 3xTF32 path, ~3.5x the FP64 filter rate --
 * while every active column's residual is above r, with degrees aimed at max(tol, 1e-5); later
 * iterations use the FP64 filter, so the returned pairs meet tol as usual.  Costs one extra
 * shard-sized buffer (the complex64 shadow and its 3xTF32 low part)),
 * fused_reduce=1 (on a grid the complex-double filter steps sum their partial products
 * inside the GEMM epilogue over peer memory -- CUDA IPC over NVLink -- instead of ncclAllReduce),
 * fused_reduce_c64=0 (the same for the complex-single filter; off by default: measured slower
 * than ncclAllReduce + local format rebuild at N = 170000 on 2x2),
 * peer_timeout=120 (seconds a rank's fused-reduce wait tolerates a peer that stopped arriving;
 * then CHASE_E_NCCL on every rank and no further fused steps are issued; each fused filter call
 * also starts with a world barrier so host-side skew between calls does not count),
 * comm_timeout=0 (host waits poll ncclCommGetAsyncError; a value > 0 also fails a wait that
 * exceeds it, e.g. when a peer died -- its communicators are aborted on CUDA/NCCL errors),
 * fp64_emulation=7 (CHASE_C128 / CHASE_R64: the filter's H products run on the INT8 tensor cores
 * as an Ozaki-scheme emulation of FP64 with exact int32 sums; 0 selects the
 * FP64 DMMA kernels and the fused f1 epilogue), oz_crt=1 (scheme II: the 52-bit scaled operands'
 * residues modulo 16 coprime moduli, 16 int8 GEMMs per real product and an exact Chinese-
 * remainder reconstruction -- one FP64 rounding per product; 48 B of residues per complex
 * element of H; when they do not fit, or with oz_crt=0, the slice scheme: fp64_emulation 7-bit
 * slices, 3..8, 28 int8 GEMMs per real product at 7, error ~2^-49 ||H|| ||X||, 21 B per element), oz_gemm_min=4e9 and oz_gemm_kmin=12288 (with the emulation on, the
 * plain GEMMs of the iteration -- the CGS projection against the locked block, the CholQR Gram,
 * Rayleigh-Ritz Q^H (HQ), Q Z, (HQ) Z -- whose M N K and contraction length K reach these also
 * run on it; short-K products are faster on DMMA, each emulated launch rewrites the FP64 result).
 * Complex-double grids fall back from the fused reduction to ncclAllReduce when a step would have
 * more tiles than the 2^17 arrival counters per communicator. */
chase_status chase_set_option(chase_handle* h, const char* key, double value);

/* Read an option or the path in effect: key "ozaki_scheme" -> 0 (FP64 DMMA products: emulation
 * off, complex single, or no room for it), 1 (7-slice Ozaki scheme), 2 (Ozaki scheme II, CRT);
 * also oz_crt, fp64_emulation, deg_max, deg_extra, max_iter, mixed_filter (the current values,
 * after any fallback).  *value is written on CHASE_OK; unknown key -> CHASE_E_USAGE.  Local. */
chase_status chase_get_option(chase_handle* h, const char* key, double* value);

/* This rank's shard: rows [row0, row0+p) and columns [col0, col0+q) of H. */
chase_status chase_local_layout(const chase_handle* h, int64_t* row0, int64_t* p, int64_t* col0,
                                int64_t* q);

/* Alg. 1.  H_shard: p x q, ldh >= p, read-only; device memory, or host memory
 * (pinned or pageable), in which case this call copies it into a library-owned device buffer
 * (one shard-sized allocation, kept for later calls).  ritz_values: host, nev doubles, ascending.
 * ritz_vectors: V-layout q x (nev) with leading dim ldv >= q, device or host memory (if approx=1
 * it must hold >= nev+nex columns with the initial V-hat on entry).  report may be NULL.
 * Returns CHASE_E_MAXITER with the locked pairs valid if max_iter is reached. */
chase_status chase_solve(chase_handle* h, const void* H_shard, int64_t ldh, int64_t N, int32_t nev,
                         int32_t nex, int32_t deg, double tol, double* ritz_values,
                         void* ritz_vectors, int64_t ldv, chase_report* report);

/* ---- hot-path rows exposed for parity tests and benchmarks ------------------ */

/* (a2)/(a4) + (a3)/(a5): one fused distributed step of the three-term recurrence:
 *   dir = 0 (forward,  Eq. w=av):  Y_i = alpha (H_ij X_j - gamma E_ij X_j) [+ beta Y_i on j = j*(i)],
 *           X V-layout (q x ncols, ldx), Y W-layout (p x ncols, ldy); sum over the row comm.
 *   dir = 1 (backward, Eq. v=aw):  Y_j = alpha (H_ij^H X_i - gamma E_ij^T X_i) [+ beta Y_j on i = i*(j)],
 *           X W-layout, Y V-layout; sum over the column comm.
 * E_ij is the restriction of I_N to the shard (nonzero on the global-diagonal crossing I_ij);
 * H is never modified.  On return Y holds the full result, replicated.  ncols = 0 is a no-op
 * (CHASE_OK; pointers may be NULL, nothing is read or written). */
chase_status chase_hemm_step(chase_handle* h, int32_t dir, const void* H_shard, int64_t ldh,
                             const void* X, int64_t ldx, void* Y, int64_t ldy, int32_t ncols,
                             double alpha, double beta, double gamma);

/* (a1)-(a5): V <- Filter(A, b_sup, mu_1, mu_ne, V, m) (Alg. 1 line 4).  V: device
 * V-layout q x ncols (ldv); W: device W-layout workspace p x ncols (ldw), overwritten.
 * degrees: host, ncols even integers >= 0 sorted ascending (Alg. 1 line 14).  Column a
 * receives the damped scaled Chebyshev polynomial of degree m_a (ledger #1), ends in V-layout.
 * matvecs (may be NULL) receives sum_a m_a.  On a multi-GPU grid with fused_reduce=1
 * (complex double / real) the block is staged through the library's V / W workspace, whose
 * replicas the step kernels sum into over peer memory (f1); W is then not written.  CHASE_C64
 * uses internal operand formats (W unused).  Errors: CHASE_E_USAGE for unsorted / odd degrees,
 * an empty interval (b_sup <= mu_ne) or bad leading dimensions; CHASE_E_NCCL if a peer stops
 * arriving in the fused all-reduce (20 s).  ncols = 0 is a no-op (CHASE_OK, *matvecs = 0, no
 * argument is read). */
chase_status chase_filter(chase_handle* h, const void* H_shard, int64_t ldh, void* V, int64_t ldv,
                          void* W, int64_t ldw, int32_t ncols, const int32_t* degrees,
                          double b_sup, double mu_1, double mu_ne, int64_t* matvecs);

/* (a6): spectral bounds by repeated Lanczos + DoS (Alg. 1 line 2; ledger #14).
 * Outputs (host): b_sup >= lambda_max estimate, mu_1, mu_ne (DoS quantile n_e/N), nu = max |Ritz|. */
chase_status chase_lanczos(chase_handle* h, const void* H_shard, int64_t ldh, int32_t n_e,
                           double* b_sup, double* mu_1, double* mu_ne, double* nu);

/* Fill a V-layout block (q x ncols, ldv) with the counter-based start block (Philox4x32-10 keyed
 * by (seed, global row, column, stream)).  ncols = 0 is a
 * no-op. */
chase_status chase_random_block(chase_handle* h, void* V, int64_t ldv, int32_t col0, int32_t ncols,
                                uint64_t seed, uint32_t stream);

chase_status chase_finalize(chase_handle* h);
const char* chase_last_error(const chase_handle* h);

/* Utility (the Rayleigh-Ritz eigensolver of row a8, exposed for parity tests): Hermitian
 * eigendecomposition G = Z diag(theta) Z^H of a device n x n matrix (ld) by the library's
 * block-cyclic Jacobi.  G is destroyed; theta (device, n doubles) ascending; Z device n x n (ldz).
 * *sweeps (may be NULL) receives the number of outer sweeps.  Local (no communication). */
chase_status chase_heev(chase_handle* h, void* G, int64_t ld, int32_t n, double* theta, void* Z,
                        int64_t ldz, int32_t* sweeps);

/* Library build/version string (for diagnostics). */
const char* chase_version(void);

/* Fill a 128-byte buffer with a fresh ncclUniqueId (call on rank 0, broadcast to all ranks
 * out of band, pass as chase_init_args.nccl_unique_id).  Local. */
chase_status chase_nccl_unique_id(void* out128);

/* Number of CUDA kernels this process has launched through the library so far (diagnostic;
 * used by the benchmark to report how many of its own kernels ran in the timed region). */
unsigned long long chase_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* CHASE_B200_H */
