/*
 * mpjacobi.h -- C ABI of the B200-native mixed-precision Jacobi eigensolver /
 * one-sided Jacobi SVD (Zhang & Bai, arXiv 2211.03339).
 *
 * Citation keys: P:n = line n of the paper's LaTeX source.
 *   Problem statement, EVD:  A = P Lambda P^T, A real symmetric
 *   Alg. 3 (mixed-precision Jacobi EVD)
 *   Alg. 5 (mixed-precision one-sided Jacobi SVD)
 *   Lemma 3.1 (rotation), Eq. (3.1) J(i,j;theta)
 *   Lemma 5.1 (one-sided rotation)
 *   Tolerances eps = 0.1 omega, nu = 20 omega (EVD), nu = omega and
 *   the 2e-4 early stop (SVD); upsilon = 2^-24, omega = 2^-53
 *   Parallel (merry-go-round) ordering
 *
 * Conventions (all entry points):
 *   - Matrices are IEEE binary64 (or binary32 where stated), COLUMN-MAJOR,
 *     with a leading dimension >= rows.  Indices are 0-based.
 *   - Unless stated otherwise, pointers are DEVICE pointers (cudaMalloc /
 *     torch CUDA tensors) on the current device, and all work is enqueued on
 *     `stream` (a cudaStream_t passed as void*; NULL = legacy default
 *     stream).  The call returns after the result is written (it
 *     synchronises `stream` once per sweep to evaluate the stop test).
 *   - The caller owns every buffer.  `workspace` may be NULL, in which case
 *     the library allocates it stream-ordered (cudaMallocAsync) and frees it
 *     before returning; otherwise it must hold at least the size returned by
 *     the matching *_workspace() query, 256-byte aligned.
 *   - Errors: the return value is an mpj_status; mpjacobi_last_error() gives
 *     a thread-local message.  On MPJ_ERR_NOCONV the outputs hold the last
 *     iterate.  Invalid sizes return MPJ_ERR_INVALID before any work.
 *   - Thread safety: calls on distinct streams with distinct buffers may run
 *     concurrently.
 *   - The GPU code path is the only path: there is no CPU fallback.  A call
 *     on a machine without an sm_100 device returns MPJ_ERR_CUDA.
 */
#ifndef MPJACOBI_H
#define MPJACOBI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPJ_ABI_VERSION 1

typedef enum {
    MPJ_OK = 0,
    MPJ_ERR_INVALID = 1,    /* bad size / pointer / config                        */
    MPJ_ERR_NOCONV = 2,     /* max_sweeps reached before ||off|| <= eps ||A||_F    */
    MPJ_ERR_RANKDEF = 3,    /* SVD: some sigma_j <= n omega ||A||_F; MGS breakdown */
    MPJ_ERR_NONFINITE = 4,  /* NaN/Inf in the input                               */
    MPJ_ERR_CUDA = 5,       /* CUDA runtime error (message in last_error)         */
    MPJ_ERR_NCCL = 6,       /* NCCL error (multi-GPU entry points)                */
    MPJ_ERR_NOMEM = 7       /* workspace too small / allocation failed            */
} mpj_status;

/* Jacobi sweep implementation. */
enum {
    MPJ_VARIANT_AUTO = 0,   /* block (b = 32) for n >= 32, scalar rounds below     */
    MPJ_VARIANT_SCALAR = 1, /* one launch pair per round, bit-exact with the oracle */
    MPJ_VARIANT_BLOCK = 2,  /* 2b x 2b block solves + fp64 tensor-core (DMMA) apply */
    MPJ_VARIANT_BLOCK_FULL = 3  /* classic block Jacobi (reading R26):
                                   each 2b x 2b block pair fully diagonalised by inner
                                   sweeps before the DMMA apply; a different ordering,
                                   so different sweep counts than the scalar rounds    */
};

typedef struct mpj_config {
    double eps_factor;        /* eps = eps_factor * omega; default 0.1            */
    double nu_factor;         /* nu = nu_factor * omega; default 20 (EVD), 1 (SVD)       */
    double eps_low_factor;    /* low stage: eps_low = f * upsilon; <= 0: the rule
                                 max(10, 1.25 sqrt(n)) of DESIGN.md reading R12 (EVD
                                 default); SVD default 10 (SPEC's value)           */
    double nu_low_factor;     /* low stage: nu_low = f * upsilon; default 20 EVD, 1 SVD  */
    double early_stop_ratio;  /* SVD: stop after a sweep with rotations/N below this;
                                 default 2e-4; 0 disables                        */
    int max_sweeps;           /* fp64 stage cap; default 60                               */
    int max_sweeps_low;       /* fp32 stage cap; default 60                               */
    int stop_rule;            /* 0: |t_pq| <= nu min(|t_pp|,|t_qq|);
                                 1: |t_pq| <= nu sqrt(t_pp t_qq) (Remark 3.1)      */
    int variant;              /* MPJ_VARIANT_*                                             */
    int block_b;              /* ordering block size b (1 or even); 0 = auto (32)        */
    int low_solver;           /* EVD step 1 (reading R12'): MPJ_LOW_*             */
    int orth;                 /* EVD step 2: MPJ_ORTH_*                            */
} mpj_config;

/* Orthogonaliser of Alg. 3 step 2 (both give the unique QR factor Q of Z with
 * a positive diagonal of R, the MGS Q; reading R10). */
enum {
    MPJ_ORTH_AUTO = 0,        /* default: MPJ_ORTH_SERIES for n <= 2048, else MPJ_ORTH_CGS */
    MPJ_ORTH_HOUSEHOLDER = 1, /* blocked Householder QR (the paper's GPU choice)     */
    MPJ_ORTH_CGS = 2,         /* blocked CGS (twice-is-enough) + panel CholeskyQR2          */
    MPJ_ORTH_SERIES = 3       /* Cholesky QR with the factor from a fixed-point series on
                                 DMMA GEMMs (reading R10b; needs ||Z^T Z - I||_F <= 1e-4,
                                 else CGS runs)                                             */
};

/* Low-precision eigensolver of Alg. 3 step 1 (mpjacobi_eig / _eig_z). */
enum {
    MPJ_LOW_AUTO = 0,         /* = MPJ_LOW_SYMQR                                          */
    MPJ_LOW_JACOBI = 1,       /* the fp32 parallel Jacobi (the same sweep kernels on
                                 binary32; eps_low / nu_low / max_sweeps_low apply)      */
    MPJ_LOW_SYMQR = 2         /* "symmetric QR factorization in low precision":
                                 binary32 Householder tridiagonalisation, the
                                 tridiagonal's eigenpairs (bisection + twisted
                                 factorisation, binary64), back-transformation        */
};

/* Fill *cfg with the paper's EVD / SVD settings.  The multi-GPU and
 * batched entry points and the SVD always use a Jacobi low stage. */
void mpj_config_default_eig(mpj_config *cfg);
void mpj_config_default_svd(mpj_config *cfg);

typedef struct mpj_report {
    int sweeps;               /* fp64 sweeps executed (the paper's SP)             */
    int sweeps_low;           /* fp32 (low-precision stage) sweeps                        */
    int status;               /* mpj_status of the fp64 stage                             */
    int status_low;           /* mpj_status of the fp32 stage (NOCONV there is benign)    */
    long long rotations;      /* applied fp64 rotations (the paper's JU x N)              */
    long long rotations_low;  /* applied fp32 rotations                                   */
    double norm_a;            /* ||A||_F of the symmetrised input                          */
    double off0;              /* ||off(Q^T A Q)||_F (EVD) / ||off((AQ)^T AQ)||_F (SVD)     */
    double off_hist[64];      /* ||off(T)||_F before fp64 sweep k (first 64)              */
    double t_low, t_orth, t_precond, t_jacobi, t_extract, t_total; /* seconds (events)    */
    int n_padded;             /* n rounded up to a multiple of 2b                         */
    int block_b;              /* ordering block size used                                 */
    int variant;              /* MPJ_VARIANT_SCALAR or MPJ_VARIANT_BLOCK                  */
    long long launches;       /* kernels launched by the call                             */
    double off_hist_low[64];  /* ||off(T32)||_F before fp32 sweep k (first 64)            */
    long long rot_hist[64];   /* rotations applied in fp64 sweep k+1 (k < sweeps, first 64) */
} mpj_report;

/* ------------------------------------------------------------------------
 * Alg. 3 end to end: fp32 Jacobi EVD of fl32(A) -> Z, Q = MGS(Z)
 * in fp64 (blocked CGS2), T = Q^T A Q (fp64 DMMA GEMMs, symmetrised),
 * parallel-ordered fp64 Jacobi sweeps on T accumulating V = Q J1 J2 ...,
 * then Lambda = diag(T) sorted descending (stable) with V's columns alike.
 *
 *   A       in:  n x n, lda >= n; symmetrised internally ((A + A^T)/2); not
 *                modified.  HOST or DEVICE pointer (host buffers are staged
 *                through the workspace with cudaMemcpyAsync on `stream`).
 *   Lambda  out: n eigenvalues, descending.  Host or device.
 *   V       out: n x n eigenvectors (column k <-> Lambda[k]), ldv >= n.
 *                Host or device.
 *   sweeps  out: fp64 sweeps (may be NULL; host pointer).
 *   rep     out: telemetry (may be NULL; host pointer).
 * Returns MPJ_OK, MPJ_ERR_NOCONV, MPJ_ERR_NONFINITE, MPJ_ERR_RANKDEF (MGS
 * breakdown), MPJ_ERR_INVALID, MPJ_ERR_NOMEM or MPJ_ERR_CUDA.
 * n <= 64 with cfg->variant == MPJ_VARIANT_AUTO and the default step 1
 * (MPJ_LOW_SYMQR) runs the same algorithm on the single-CTA kernels of
 * mpjacobi_eig_batched (batch 1; the workspace is not used, a small staging
 * buffer is allocated on `stream`); rep then carries sweeps, sweeps_low,
 * variant, n_padded, block_b, launches and t_total only.  Environment
 * MPJ_SMALL_BATCHED=0 selects the general path.
 * ---------------------------------------------------------------------- */
size_t mpjacobi_eig_workspace(int64_t n, const mpj_config *cfg);
mpj_status mpjacobi_eig(const double *A, int64_t n, int64_t lda, double *Lambda, double *V,
                        int64_t ldv, int *sweeps, void *workspace, size_t ws_bytes, void *stream,
                        const mpj_config *cfg, mpj_report *rep);

/* Alg. 3 with step 1's output supplied or exported ("Compute the
 * spectral decomposition in low precision ... A = Z Lambda Z^T"; the paper's
 * own step 1 was a library SSYEV / cusolverDnSsyevd):
 *   Z_in   in:  NULL -> run the low-precision stage (fp32 Jacobi, reading
 *               R12); otherwise an n x n binary32 matrix (column-major,
 *               ld = ldz >= n; host or device) used as Z in step 2, and the
 *               low-precision stage is skipped (rep->sweeps_low = 0).
 *   Z_out  out: NULL, or n x n binary32 (ld = ldz; host or device) that
 *               receives the Z step 2 consumed (the fp32 stage's V, or Z_in).
 * Feeding the same Z to this call and to the oracle isolates the fp64 stage:
 * its sweep count must then be identical.  Other arguments,
 * outputs and errors as mpjacobi_eig (MPJ_ERR_INVALID if ldz < n while Z_in or
 * Z_out is given). */
mpj_status mpjacobi_eig_z(const double *A, int64_t n, int64_t lda, const float *Z_in, float *Z_out, int64_t ldz,
                          double *Lambda, double *V, int64_t ldv, int *sweeps, void *workspace, size_t ws_bytes,
                          void *stream, const mpj_config *cfg, mpj_report *rep);

/* Alg. 2 from T = A, P = I: "plain" fp64 parallel Jacobi with the
 * same kernels and ordering (the baseline of BASELINE.json config 2).  Same
 * arguments and outputs as mpjacobi_eig. */
mpj_status mpjacobi_eig_plain(const double *A, int64_t n, int64_t lda, double *Lambda, double *V,
                              int64_t ldv, int *sweeps, void *workspace, size_t ws_bytes,
                              void *stream, const mpj_config *cfg, mpj_report *rep);

/* ------------------------------------------------------------------------
 * The Jacobi loop of Alg. 2 / Alg. 3 steps 4-11 on a given T
 * with accumulation into a given V: the hot path of the method.
 *   T  in/out: n x n symmetric (must be exactly symmetric), ldt >= n, DEVICE.
 *   V  in/out: n x n, ldv >= n, DEVICE; V <- V J_1 J_2 ... (right rotations).
 *   tol: the while test is ||off(T)||_F > tol (pass eps * ||A||_F).
 *   nu:  threshold of the test |t_pq| <= nu min(|t_pp|,|t_qq|).
 *   max_sweeps: cap; max_rounds >= 0 stops after that many rounds in total
 *        (round-level parity tests), -1 = no limit.  With the block variant
 *        the limit must fall on a block-round boundary: block round 0 of a
 *        sweep holds 2b-1 rounds, each later one b (reading R1); otherwise
 *        MPJ_ERR_INVALID.
 *   The f32 variant runs the identical algorithm in binary32 (the
 *   low-precision stage, reading R12).  Only cfg->variant, cfg->block_b and
 *   cfg->stop_rule are read from cfg (may be NULL).
 *   sweeps / rotations (host pointers, may be NULL) receive SP and JU*N.
 * ---------------------------------------------------------------------- */
mpj_status mpjacobi_jacobi_f64(double *T, int64_t ldt, double *V, int64_t ldv, int64_t n,
                               double tol, double nu, int max_sweeps, int64_t max_rounds,
                               int *sweeps, long long *rotations, double *off_hist64,
                               void *stream, const mpj_config *cfg);
mpj_status mpjacobi_jacobi_f32(float *T, int64_t ldt, float *V, int64_t ldv, int64_t n,
                               double tol, double nu, int max_sweeps, int64_t max_rounds,
                               int *sweeps, long long *rotations, double *off_hist64,
                               void *stream, const mpj_config *cfg);

/* Alg. 3 step 2: Q = orth(Z) in fp64 by blocked classical
 * Gram-Schmidt with reorthogonalisation (CGS2, reading R10); Z, Q: n x n,
 * DEVICE, ld = n.  Returns MPJ_ERR_RANKDEF on a zero column. */
mpj_status mpjacobi_orth(const double *Z, double *Q, int64_t n, void *stream);

/* The stages of Alg. 3 step 1 by symmetric QR (reading R12'), for
 * stage-level parity tests:
 *   mpjacobi_sytrd: Householder tridiagonalisation in binary32 (GvL Alg.
 *     8.3.1 blocked as LAPACK ssytrd, lower): A (n x n symmetric, lda >= n a
 *     multiple of 4, DEVICE) is overwritten with the reflectors in the LAPACK layout
 *     (v_j(2:) below the subdiagonal of column j; H_j = I - tau_j v_j v_j^T,
 *     v_j(1) = 1, beta = -sign(alpha) ||x||); d (n), e (n-1), tau (n) DEVICE
 *     receive T's diagonal, subdiagonal and the reflector scalars.
 *   mpjacobi_tridiag_eig: the eigenpairs of the symmetric tridiagonal (d, e)
 *     (binary32 in, DEVICE) in binary64: lam (n) descending, Y (n x n, ldy)
 *     the unit eigenvectors alike (columns' signs unspecified).  Bisection on
 *     Sturm counts + one twisted-factorisation solve per eigenvalue; the
 *     matrix is split where |e_i| <= omega sqrt(|d_i d_{i+1}|).  n <= 65536.
 * Both synchronise `stream` before returning. */
mpj_status mpjacobi_sytrd(float *A, int64_t n, int64_t lda, float *d, float *e, float *tau, void *stream);
mpj_status mpjacobi_tridiag_eig(const float *d, const float *e, int64_t n, double *lam, double *Y, int64_t ldy,
                                void *stream);

/* Alg. 3 step 2 by blocked Householder QR: Q =
 * H_0 ... H_{n-1} with the columns' signs making diag(R) positive.  Z, Q: n x n
 * DEVICE, ld = n.  Returns MPJ_ERR_RANKDEF on a zero diagonal of R. */
mpj_status mpjacobi_orth_householder(const double *Z, double *Q, int64_t n, void *stream);
/* Step 2 by Cholesky QR with the factor from a fixed-point series (reading
 * R10b): Q = Z (I + U)^{-1}, U = Phi(E - U^T U), E = Z^T Z - I, six n^3 DMMA
 * GEMMs; the same unique Q (positive diag R) as MGS to O(||E||^4 + n omega).
 * Z, Q: n x n column-major DEVICE.  MPJ_ERR_NOCONV (Q untouched) when
 * ||E||_F > 1e-4 -- a Z that needs CGS. */
mpj_status mpjacobi_orth_series(const double *Z, double *Q, int64_t n, void *stream);

/* Alg. 3 step 3: T = Q^T A Q, symmetrised; A, Q, T: n x n DEVICE,
 * ld = n.  fp64 tensor-core (DMMA) GEMMs. */
mpj_status mpjacobi_precond(const double *A, const double *Q, double *T, int64_t n, void *stream);

/* C (m x n) = op(A) (m x k) * B (k x n), fp64, DEVICE, column-major with
 * ld = rows; transa = 1 means A is stored k x m.  (The DMMA GEMM that the
 * preconditioner and the SVD's C = A Q use; exported for parity tests.) */
mpj_status mpjacobi_dgemm(int transa, const double *A, const double *B, double *C, int64_t m,
                          int64_t n, int64_t k, void *stream);

/* ------------------------------------------------------------------------
 * Alg. 5 end to end: fp32 one-sided Jacobi on fl32(A) -> Z,
 * Q = orth(Z), C = A Q, V = Q, fp64 one-sided sweeps (rotate iff
 * |c_p^T c_q| > nu ||c_p|| ||c_q||), stop when ||off(C^T C)||_F <=
 * eps ||C^T C||_F or a sweep's rotations / N < early_stop_ratio;
 * then sort columns by ||c_j|| descending, sigma_j = ||c_j||, u_j = c_j/sigma_j.
 *   A: m x n, m >= n, lda >= m (host or device); Sigma: n; U: m x n (ldu >= m);
 *   V: n x n (ldv >= n).  MPJ_ERR_RANKDEF if some sigma_j <= n omega ||A||_F.
 * ---------------------------------------------------------------------- */
size_t mpjacobi_svd_workspace(int64_t m, int64_t n, const mpj_config *cfg);
mpj_status mpjacobi_svd(const double *A, int64_t m, int64_t n, int64_t lda, double *Sigma,
                        double *U, int64_t ldu, double *V, int64_t ldv, int *sweeps,
                        void *workspace, size_t ws_bytes, void *stream, const mpj_config *cfg,
                        mpj_report *rep);

/* Alg. 5 with step 1's output (the n x n right singular vector estimate Z of
 * the low-precision SVD) supplied (Z_in) or exported
 * (Z_out), as mpjacobi_eig_z: binary32, n x n, ld = ldz >= n, host or device. */
mpj_status mpjacobi_svd_z(const double *A, int64_t m, int64_t n, int64_t lda, const float *Z_in, float *Z_out,
                          int64_t ldz, double *Sigma, double *U, int64_t ldu, double *V, int64_t ldv, int *sweeps,
                          void *workspace, size_t ws_bytes, void *stream, const mpj_config *cfg, mpj_report *rep);

/* ------------------------------------------------------------------------
 * Multi-GPU Alg. 5 (the column partition of Alg. 5's
 * one-sided rotations): one call per rank (NCCL communicator from
 * mpjacobi_nccl_unique_id, as mpjacobi_eig_mg), or emulate_ranks = G ranks
 * inside one process (nccl_id NULL; device copies instead of NCCL).  Rank g
 * runs the block-pair slots [g mb/G, (g+1) mb/G) of every block round (mb =
 * n_p/64); the 32-column blocks that move to another rank's slot are sent
 * there (ncclSend / ncclRecv), every block is broadcast from its owner before
 * each sweep's stop test; steps 2-3 (Q = orth(Z), C = A Q) are replicated.
 * Bit-identical to mpjacobi_svd when n is a multiple of 64 G (same padding).
 *   A: m x n (lda >= m), host or device, the same bits on every rank;
 *   Sigma (n), U (m x n, ldu), V (n x n, ldv): DEVICE, replicated on every
 *   rank.  Errors as mpjacobi_svd; MPJ_ERR_NCCL from NCCL. */
mpj_status mpjacobi_svd_mg(const double *A, int64_t m, int64_t n, int64_t lda, double *Sigma, double *U,
                           int64_t ldu, double *V, int64_t ldv, int *sweeps, const void *nccl_id, int rank,
                           int nranks, int emulate_ranks, void *stream, const mpj_config *cfg, mpj_report *rep);

/* Host-only view of mpjacobi_svd_mg's partition (no GPU needed): the padded
 * order n_p (multiple of 64 nranks), the block rounds per sweep, the 32-column
 * block pairs of every round (pairs: rounds x n_p/64 x 2 ints; slot k belongs
 * to rank k / (n_p / 64 / nranks)) and the blocks that change rank between
 * consecutive rounds (moves: (rounds - 1) x 4 nranks x 3 ints (block, src,
 * dst); nmoves: rounds - 1).  Any output pointer may be NULL. */
mpj_status mpjacobi_svd_mg_plan(int64_t n, int nranks, int *np_out, int *rounds_out, int *pairs, int *moves,
                                int *nmoves);

/* ------------------------------------------------------------------------
 * Batched Alg. 3: `batch` independent n x n matrices, contiguous with stride
 * n*n (each column-major), one matrix per CTA (n <= 64).  Lambda: batch x n;
 * V: batch x n x n (each column-major); sweeps / sweeps_low: batch ints
 * (DEVICE, may be NULL).  All pointers DEVICE.  Step 1 follows
 * cfg->low_solver: symmetric QR in binary32 by default (reading R12'),
 * the fp32 Jacobi with MPJ_LOW_JACOBI (R12; sweeps_low is 0 for symmetric QR).
 * Returns MPJ_ERR_NONFINITE if some matrix holds a NaN / Inf,
 * MPJ_ERR_RANKDEF if some Z is rank deficient in step 2, MPJ_ERR_NOCONV if
 * any matrix hit max_sweeps.
 * ---------------------------------------------------------------------- */
mpj_status mpjacobi_eig_batched(const double *A, int64_t n, int64_t batch, double *Lambda,
                                double *V, int *sweeps, int *sweeps_low, void *stream,
                                const mpj_config *cfg);

/* Batched Alg. 3 with step 1's output supplied (Z_in: step 1 is skipped) or
 * exported (Z_out), as mpjacobi_eig_z: batch x n x n binary32, each n x n
 * column-major (stride n*n), DEVICE; either may be NULL.  A shared Z isolates
 * the fp64 stage (sweep parity with the oracle). */
mpj_status mpjacobi_eig_batched_z(const double *A, int64_t n, int64_t batch, const float *Z_in, float *Z_out,
                                  double *Lambda, double *V, int *sweeps, int *sweeps_low, void *stream,
                                  const mpj_config *cfg);

/* ------------------------------------------------------------------------
 * Multi-GPU Alg. 3, one process per GPU: the block-pair slots
 * of the block merry-go-round (and the columns of T and V they own) are
 * split over `nranks` ranks; per block round the 64 x 64 rotation blocks are
 * all-gathered and the column blocks that cross rank boundaries exchanged
 * over NCCL (NVLink); the off-norm is all-reduced per sweep.
 *   A       in: the full n x n matrix on EVERY rank (host or device, lda >= n).
 *   Lambda, V  out: replicated on every rank (host or device), as mpjacobi_eig.
 *   nccl_id 128 bytes from mpjacobi_nccl_unique_id() on rank 0, broadcast to
 *           all ranks (e.g. torch.distributed); NULL -> single process.
 *   rank, nranks  this rank and the world size (nranks must divide n_p/64;
 *           n is padded to a multiple of 64 * nranks).
 *   emulate_ranks  with nccl_id == NULL: run that many ranks inside this
 *           process on this GPU (device copies instead of NCCL) -- a testing
 *           mode for the partitioned algorithm on one GPU.
 * Every rank must call it with the same n, config and id.
 * ---------------------------------------------------------------------- */
mpj_status mpjacobi_eig_mg(const double *A, int64_t n, int64_t lda, double *Lambda, double *V, int64_t ldv,
                           int *sweeps, const void *nccl_id, int rank, int nranks, int emulate_ranks,
                           void *stream, const mpj_config *cfg, mpj_report *rep);

/* Host-only: the partition plan of one sweep of mpjacobi_eig_mg (no GPU
 * needed; used by the CPU multi-rank tests).  Pass NULL arrays to query
 * n_p and the number of block rounds.  slots: rounds x mb x 4 (top block,
 * bottom block, physical position of each on its rank; mb = n_p/64), xfers:
 * rounds x (4 nranks) x 4 (src rank, src position, dst rank, dst position),
 * nxfer: rounds.  Positions count blocks of 32 columns. */
mpj_status mpjacobi_mg_plan(int64_t n, int nranks, int *np_out, int *rounds_out, int *slots, int *xfers,
                            int *nxfer);

/* ncclGetUniqueId into out (>= 128 bytes). */
mpj_status mpjacobi_nccl_unique_id(void *out, size_t bytes);

/* Kernel timing (diagnostics for the bench's roofline numbers).  While
 * enabled, the library brackets each launch of its dominant kernels with CUDA
 * events ON THE STREAM IT LAUNCHES THEM ON and accumulates their durations per
 * kernel name: "block_apply_f64|f32", "block_solve_f64|f32" (and
 * "block_apply_*.sweep1": the first sweep's launches alone), "round_apply_*",
 * "svd_gram_*", "svd_solve_*", "svd_apply_*", "mg_apply_*", "mg_solve_*",
 * "batched_evd".  Counters without a time (seconds = 0, launches = count):
 * "block_apply_*.items" (work items), ".skipped_t" / ".skipped_v" (T / V tiles
 * skipped because their rotation blocks are exactly I), ".half_t" (T tiles
 * with one identity block: one product), ".identity_blocks", and the same
 * with ".sweep1".  Process-wide; not for concurrent calls.  get() returns 0
 * launches for unknown names. */
void mpjacobi_profile_enable(int on);
void mpjacobi_profile_reset(void);
void mpjacobi_profile_get(const char *kernel, double *seconds, long long *launches);

/* Thread-local description of the last error ("" if none). */
const char *mpjacobi_last_error(void);

/* Number of kernels this thread has launched through the library (the bench
 * reports it as gpu_launches). */
long long mpjacobi_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MPJACOBI_H */
