// mpj_internal.h -- host-side declarations shared by the library's .cu files.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/mpjacobi.h"

namespace mpj {

// launch with programmatic stream serialisation (PDL): the kernel may be
// scheduled while its predecessor drains; it must execute griddepcontrol.wait
// before touching data the predecessor writes
template <typename... KA, typename... A>
inline cudaError_t launch_pdl_k(void (*k)(KA...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

struct Sched;

// ---- error / launch bookkeeping --------------------------------------------
void set_error(const std::string &msg);
void count_launch(long long k = 1);
// kernel timing (mpjacobi_profile_*): events recorded on the launch stream
bool prof_on();
void prof_mark(const char *name, cudaStream_t st, bool begin);
void prof_flush();   // after the stream has been synchronised
void prof_add(const std::string &name, long long n);   // a counter (launches field only)

// Opt a kernel into `bytes` of dynamic shared memory on the CURRENT device
// (the attribute is per device context) and return its resident CTAs per SM
// for `threads` threads (per_sm may be NULL).  Thread-safe; the attribute is
// set once per (kernel, device, size).
cudaError_t smem_optin(const void *func, size_t bytes, int threads, int *per_sm);

#define MPJ_CK(expr)                                                                    \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            ::mpj::set_error(std::string(#expr) + ": " + cudaGetErrorString(e_));       \
            return MPJ_ERR_CUDA;                                                        \
        }                                                                               \
    } while (0)

#define MPJ_CK_VOID(expr)                                                               \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess) ::mpj::set_error(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define MPJ_TRY(expr)                                                                   \
    do {                                                                                \
        mpj_status s_ = (expr);                                                         \
        if (s_ != MPJ_OK) return s_;                                                    \
    } while (0)

// low-stage stop tolerance factor (reading R12)
double eps_low_factor(const mpj_config &cfg, int64_t n);

// ---- ordering (host side) --------------------------------------------------
struct HostSchedule {
    int n = 0, b = 1, np = 0, nb = 0, mb = 0, rounds = 0;
    std::vector<int2> bsched;   // (nb-1) x mb
    std::vector<int2> lsched;   // (b-1) x (b/2)
};
int padded_n(int64_t n, int b);
void build_schedule(int64_t n, int b, HostSchedule &hs);

struct DevSched {
    int2 *bsched = nullptr, *lsched = nullptr;
    int b = 1, nb = 0, np = 0, rounds = 0;
};

// ---- launchers (k_rounds.cu) ------------------------------------------------
template <typename R>
void launch_round_params(const R *T, int64_t ldt, const DevSched &S, int r, R nu, int rule,
                         int2 *pq, R *t, R *s, R *u, unsigned long long *cnt, cudaStream_t st,
                         int *pos = nullptr);
// T and V of one round in one coalesced pass (pos: row -> slot | is_q << 30,
// written by launch_round_params)
template <typename R>
void launch_round_apply_fused_oop(const R *T, R *Tout, int64_t ldt, R *V, int64_t ldv, int vrows, int np,
                                  const int2 *pq, const int *pos, const R *t, const R *s, const R *u,
                                  cudaStream_t st);
template <typename R>
void launch_round_apply(R *T, int64_t ldt, const int2 *pq, const R *t, const R *s, const R *u,
                        int h, cudaStream_t st);
template <typename R>
void launch_round_apply_v(R *V, int64_t ldv, int vrows, const int2 *pq, const R *s, const R *u,
                          int h, cudaStream_t st);

// ---- batched path (k_batched.cu): batch contiguous n x n matrices (n <= 64),
// device pointers; sweeps / sweeps_low device arrays of `batch` ints ----------
mpj_status batched_evd(const double *A, int64_t n, int64_t batch, double *Lambda, double *V, int *sweeps,
                       int *sweeps_low, const float *Zin, float *Zout, cudaStream_t st, const mpj_config &cfg);

// ---- block variant pieces (k_block.cu) ---------------------------------------
template <typename R>
cudaError_t launch_block_apply_cols(R *M, int64_t ld, int rows, const DevSched &ds, int Rb, const R *Ubuf,
                             cudaStream_t st, const int *uid = nullptr, const int *nid = nullptr, int *ctr = nullptr);

// ---- utilities (k_util.cu) --------------------------------------------------
// out[0] = sqrt(sum_{i != j} T_ij^2) (offdiag) or sqrt(sum T_ij^2) over an m x n
// matrix; deterministic two-stage reduction; `partial` holds >= kRedBlocks doubles.
constexpr int kRedBlocks = 296;
template <typename R>
void launch_norm(const R *T, int64_t ld, int m, int n, bool offdiag, double *partial,
                 double *out, cudaStream_t st);
// the same two norms of a symmetric n x n matrix read from its upper triangle
// only (strict upper entries counted twice); the lower triangle is not read.
void launch_norm_sym_upper(const double *T, int64_t ld, int n, bool offdiag, double *partial,
                           double *out, cudaStream_t st);
// copy an m x n block between leading dimensions, zero-filling dst rows/cols
// beyond (m, n) up to (mp, np_)
template <typename Rs, typename Rd>
void launch_copy_pad(const Rs *src, int64_t lds, int m, int n, Rd *dst, int64_t ldd, int mp, int np_,
                     cudaStream_t st);
// dst = (src + src^T)/2 into a padded n_p x n_p buffer (zero pad)
void launch_symmetrize(const double *src, int64_t lds, int n, double *dst, int64_t ldd, int np_,
                       cudaStream_t st);
// dst (in place) = (dst + dst^T)/2 for an n x n matrix, or (mirror_upper) the
// upper triangle copied onto the lower one
void launch_symmetrize_inplace(double *T, int64_t ld, int n, cudaStream_t st, bool mirror_upper = false);
template <typename R>
void launch_identity(R *V, int64_t ld, int m, int n, cudaStream_t st);
// nonfinite check: flag[0] = 1 if any entry is NaN/Inf
void launch_check_finite(const double *A, int64_t ld, int m, int n, int *flag, cudaStream_t st);
// eigen-extraction: lam[rank[i]] = T[i,i]; Vout[:, rank[i]] = V[:, i] (stable descending)
void launch_extract_evd(const double *T, int64_t ldt, const double *V, int64_t ldv, int n,
                        int vrows, double *lam, double *Vout, int64_t ldvo, int *rank,
                        cudaStream_t st);

// ---- GEMM (k_gemm.cu) ----------------------------------------------------------
// C = alpha * op(A) op(B) + beta * C, fp64 DMMA (mma.sync m8n8k4).  All column-major.
void launch_dgemm(bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha,
                  const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                  double *C, int64_t ldc, cudaStream_t st, double *scratch = nullptr,
                  size_t scratch_elems = 0, bool upper_only = false, const int *skip = nullptr,
                  int min_splits = 1);
// upper_only: only the 64 x 64 tiles of C that meet its upper triangle are
// computed (a symmetric product such as C^T C); the rest of C is left as is.
// skip (device int, may be NULL): the product is skipped when *skip != 0.
// split-K scratch the library reserves for tall-skinny products (doubles)
size_t dgemm_scratch_elems(int64_t m, int64_t n);

// ---- orthogonalisation (k_orth.cu) ------------------------------------------------
size_t orth_workspace(int64_t n);
mpj_status orth_cgs2(const double *Z, int64_t ldz, double *Q, int64_t ldq, int64_t m, int64_t n,
                     void *ws, cudaStream_t st);

// ---- orthogonalisation by Householder QR (k_hqr.cu) ---------------------------
size_t hqr_workspace(int64_t m, int64_t n);
mpj_status orth_series(const double *Z, int64_t ldz, double *Q, int64_t ldq, int64_t n, cudaStream_t st);
mpj_status orth_householder(const double *Z, int64_t ldz, double *Q, int64_t ldq, int64_t m, int64_t n, void *ws,
                            cudaStream_t st);

// ---- low-precision stage by symmetric QR (k_tridiag.cu, reading R12') ---------
size_t symqr_workspace(int64_t np);
mpj_status low_evd_symqr(float *A32, int64_t lda, int n, float *Z32, int64_t ldz, double *Y, int64_t ldy,
                         double *Dp, double *Dm, void *ws, cudaStream_t st);

}  // namespace mpj
