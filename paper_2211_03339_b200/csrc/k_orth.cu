// k_orth.cu -- Alg. 3 step 2: Q = orth(Z) in fp64.
//
// Reading R10: the paper's MGS (Lemma 2.1) -- and the
// Householder QR its GPU code used -- both compute the QR factor Q of
// Z, which is unique (positive diag(R)) and, since Z is orthogonal to
// O(upsilon), perfectly conditioned.  We compute it by left-looking
// blocked Gram-Schmidt with reorthogonalisation, panel width 64:
//   for each panel X = Z(:, p0:p0+64):
//     twice:  R = Q(:, :p0)^T X ;  X = X - Q(:, :p0) R        (CGS2, DMMA GEMMs)
//     twice:  G = X^T X ; G = R^T R (Cholesky) ; X = X R^{-1} (CholeskyQR2)
// Every step is a dense fp64 tensor-core product except the 64 x 64
// Cholesky / triangular inverse (one CTA).  Orthogonality O(omega), same Q as
// MGS to O(n omega) (tests/test_gpu_parity.py::test_orth_cgs2_matches_mgs).
#include "mpj_device.cuh"
#include "mpj_internal.h"

#include <algorithm>

namespace mpj {

namespace {
constexpr int kPanel = 64;
constexpr int kLDG = kPanel + 1;

// G (w x w, ld w) -> Rinv (w x w, ld w) with G = R^T R, R upper, Rinv = R^{-1};
// fail = 1 on a non-positive pivot.
__global__ void __launch_bounds__(256) k_chol_inv(const double *__restrict__ G, int w, double *__restrict__ Rinv,
                                                  int *__restrict__ fail)
{
    __shared__ double A[kPanel * kLDG];    // working copy, upper triangle -> R
    const int tid = threadIdx.x;
    for (int e = tid; e < w * w; e += blockDim.x) {
        const int i = e % w, j = e / w;
        A[i + j * kLDG] = 0.5 * (G[i + j * w] + G[j + i * w]);
        Rinv[i + j * w] = 0.0;
    }
    __syncthreads();
    __shared__ int bad;
    if (tid == 0) bad = 0;
    __syncthreads();
    for (int k = 0; k < w; ++k) {
        // pivot
        const double d = A[k + k * kLDG];
        if (!(d > 0.0)) { if (tid == 0) bad = 1; }
        const double r = sqrt(fmax(d, 1e-300));
        __syncthreads();
        // row k of R:  R(k, j) = A(k, j) / r, j >= k
        for (int j = k + tid; j < w; j += blockDim.x) A[k + j * kLDG] = (j == k) ? r : A[k + j * kLDG] / r;
        __syncthreads();
        // trailing update A(i, j) -= R(k, i) R(k, j), k < i <= j
        for (int e = tid; e < w * w; e += blockDim.x) {
            const int i = e % w, j = e / w;
            if (i > k && j >= i) A[i + j * kLDG] = __fma_rn(-A[k + i * kLDG], A[k + j * kLDG], A[i + j * kLDG]);
        }
        __syncthreads();
    }
    // R^{-1}: column j by back substitution (thread j), into the strictly lower
    // part of A (transposed: X(i, j) stored at A(j, i), i < j) and the diagonal buffer
    __shared__ double dinv[kPanel];
    if (tid < w) dinv[tid] = 1.0 / A[tid + tid * kLDG];
    __syncthreads();
    if (tid < w) {
        const int j = tid;
        for (int i = j - 1; i >= 0; --i) {
            double acc = A[i + j * kLDG] * dinv[j];   // k = j term: R(i,j) X(j,j)
            for (int k = i + 1; k < j; ++k) acc = __fma_rn(A[i + k * kLDG], A[j + k * kLDG], acc);
            A[j + i * kLDG] = -acc * dinv[i];          // X(i, j) = -acc / R(i,i)
        }
    }
    __syncthreads();
    for (int e = tid; e < w * w; e += blockDim.x) {
        const int i = e % w, j = e / w;
        if (i < j) Rinv[i + j * w] = A[j + i * kLDG];
        else if (i == j) Rinv[i + j * w] = dinv[i];
    }
    if (tid == 0 && bad) *fail = 1;
}
}  // namespace

size_t dgemm_scratch_elems(int64_t m, int64_t n)
{
    (void)m; (void)n;
    return (size_t)300 * 64 * 64;
}

size_t orth_workspace(int64_t n)
{
    // R (n x 64) + S (n x 64) + split-K scratch + G + Rinv + flag
    return ((size_t)2 * n * kPanel + dgemm_scratch_elems(n, kPanel) + 2 * kPanel * kPanel + 64) * sizeof(double);
}

mpj_status orth_cgs2(const double *Z, int64_t ldz, double *Q, int64_t ldq, int64_t m, int64_t n,
                     void *ws, cudaStream_t st)
{
    double *R = (double *)ws;
    double *S = R + (size_t)n * kPanel;
    double *scratch = S + (size_t)m * kPanel;
    const size_t scratch_elems = dgemm_scratch_elems(n, kPanel);
    double *G = scratch + scratch_elems;
    double *Rinv = G + kPanel * kPanel;
    int *fail = (int *)(Rinv + kPanel * kPanel);

    MPJ_CK(cudaMemsetAsync(fail, 0, sizeof(int), st));
    if (Q != Z || ldq != ldz) launch_copy_pad<double, double>(Z, ldz, (int)m, (int)n, Q, ldq, (int)m, (int)n, st);

    for (int64_t p0 = 0; p0 < n; p0 += kPanel) {
        const int w = (int)std::min<int64_t>(kPanel, n - p0);
        double *X = Q + p0 * ldq;
        if (p0 > 0) {
            for (int rep = 0; rep < 2; ++rep) {
                launch_dgemm(true, false, p0, w, m, 1.0, Q, ldq, X, ldq, 0.0, R, p0, st, scratch, scratch_elems);
                launch_dgemm(false, false, m, w, p0, -1.0, Q, ldq, R, p0, 1.0, X, ldq, st, scratch,
                             scratch_elems);
            }
        }
        // CholeskyQR2 of the panel: X -> S -> X
        for (int rep = 0; rep < 2; ++rep) {
            const double *src = rep == 0 ? X : S;
            const int64_t lds = rep == 0 ? ldq : m;
            double *dst = rep == 0 ? S : X;
            const int64_t ldd = rep == 0 ? m : ldq;
            launch_dgemm(true, false, w, w, m, 1.0, src, lds, src, lds, 0.0, G, w, st, scratch, scratch_elems);
            k_chol_inv<<<1, 256, 0, st>>>(G, w, Rinv, fail);
            count_launch();
            launch_dgemm(false, false, m, w, w, 1.0, src, lds, Rinv, w, 0.0, dst, ldd, st);
        }
    }
    int h_fail = 0;
    MPJ_CK(cudaMemcpyAsync(&h_fail, fail, sizeof(int), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaStreamSynchronize(st));
    if (h_fail) {
        set_error("orth: non-positive Cholesky pivot (rank deficient Z)");
        return MPJ_ERR_RANKDEF;
    }
    return MPJ_OK;
}

}  // namespace mpj
