// k_orth.cu -- Alg. 3 step 2: Q = orth(Z) in fp64.
//
// Reading R10: the paper's MGS (Lemma 2.1) -- and the
// Householder QR its GPU code used -- both compute the QR factor Q of
// Z, which is unique (positive diag(R)) and, since Z is orthogonal to
// O(upsilon), perfectly conditioned.  We compute it by left-looking
// blocked classical Gram-Schmidt, panel width 64:
//   for each panel X = Z(:, p0:p0+64):
//     once:   R = Q(:, :p0)^T X ;  X = X - Q(:, :p0) R        (CGS, DMMA GEMMs)
//             -- twice (CGS2) if any column kept less than half its norm
//             ("twice is enough"; checked on the panel Gram, the whole Q
//             is then recomputed with two passes)
//     G = X^T X ; G = R^T R (Cholesky) ; X = X R^{-1} (CholeskyQR, the last
//             step as a row-parallel triangular solve) -- a second pass
//             (CholeskyQR2) only when the first G was not within 1e-3 of I
//             (device-side decision: the pass's kernels read a flag)
// Every step is a dense fp64 tensor-core product except the 64 x 64
// Cholesky (one CTA) and the row-wise forward substitution.  Orthogonality O(omega), same Q as
// MGS to O(n omega) (tests/test_gpu_parity.py::test_orth_cgs2_matches_mgs).
#include "mpj_device.cuh"
#include "mpj_internal.h"

#include <algorithm>

namespace mpj {

namespace {
constexpr int kPanel = 64;
constexpr int kLDG = kPanel + 1;
constexpr int kCholNT = 1024;   // threads of the panel Cholesky: 16 rows of the update per column

// Cholesky G = R^T R of a w x w panel Gram matrix (w <= 64): R upper (ld w,
// zero below the diagonal); fail = 1 on a non-positive pivot.  Right-looking;
// thread t owns column j = t % 64 and rows i = t / 64 (mod 4) of the trailing
// triangle, so a step is a few FMAs per thread and two barriers (k_chol_inv's
// flat loop over all w^2 entries with an integer division per entry made it
// issue-bound: 150 us per call, 1% of an n = 8192 EVD).
__global__ void __launch_bounds__(kCholNT) k_chol(const double *__restrict__ G, int w, double *__restrict__ Rf,
                                              int *__restrict__ fail, const double *__restrict__ pre,
                                              int *__restrict__ reorth, int *__restrict__ single,
                                              const int *__restrict__ skip)
{
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL)
    __shared__ double A[kPanel * kLDG];
    __shared__ int far_from_I;
    if (skip && *skip) return;
    const int tid = threadIdx.x, cj = tid & (kPanel - 1), ri = tid >> 6;   // ri < kCholNT / 64
    // single: the panel is orthonormal to 1e-3 (max |G - I|), so one CholeskyQR
    // pass already gives an O(omega kappa^2) = O(omega) orthogonality and the
    // second pass is skipped (the caller's conditional kernels read *single)
    if (single) {
        if (tid == 0) far_from_I = 0;
        __syncthreads();
        if (cj < w)
            for (int i = ri; i < w; i += kCholNT / 64)
                if (!(fabs(G[i + cj * w] - (i == cj ? 1.0 : 0.0)) <= 1e-3)) far_from_I = 1;
        __syncthreads();
        if (tid == 0) *single = far_from_I ? 0 : 1;
    }
    // one projection pass lost more than half of a column's norm: "twice is
    // enough" (Kahan, Parlett) asks for the second pass (the caller redoes Q with CGS2)
    if (pre && reorth && ri == 0 && cj < w && G[cj + cj * w] < 0.25 * pre[cj]) *reorth = 1;
    if (cj < w)
        for (int i = ri; i <= cj; i += kCholNT / 64) A[i + cj * kLDG] = 0.5 * (G[i + cj * w] + G[cj + i * w]);
    __syncthreads();
    bool bad = false;
    for (int k = 0; k < w; ++k) {
        const double d = A[k + k * kLDG];
        const double r = sqrt(fmax(d, 1e-300));
        bad |= !(d > 0.0);
        if (ri == 0 && cj > k && cj < w) A[k + cj * kLDG] /= r;      // row k of R (A(k,k) is written below)
        __syncthreads();
        if (cj > k && cj < w) {                                       // A(i, j) -= R(k, i) R(k, j), k < i <= j
            const double rkj = A[k + cj * kLDG];
            for (int i = k + 1 + ri; i <= cj; i += kCholNT / 64) A[i + cj * kLDG] = __fma_rn(-A[k + i * kLDG], rkj, A[i + cj * kLDG]);
        }
        if (ri == 0 && cj == k) A[k + k * kLDG] = r;
        __syncthreads();
    }
    if (cj < w)
        for (int i = ri; i < w; i += kCholNT / 64) Rf[i + cj * w] = (i <= cj) ? A[i + cj * kLDG] : 0.0;
    if (tid == 0 && bad) *fail = 1;
}

// X(:, 0:w) = S(:, 0:w) when *run (the panel's single CholeskyQR pass sufficed)
__global__ void k_copy_panel_if(const double *__restrict__ S, int64_t lds, int64_t m, double *__restrict__ X,
                                int64_t ldx, const int *__restrict__ run)
{
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL)
    if (!*run) return;
    const int j = blockIdx.y;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        X[i + j * ldx] = S[i + j * lds];
}

// pre[j] = ||X(:, j)||^2 for the w columns of a panel (one CTA per column)
__global__ void k_colnorm2(const double *__restrict__ X, int64_t ldx, int64_t m, double *__restrict__ pre)
{
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL)
    __shared__ double red[256 / 32];
    const double *x = X + (size_t)blockIdx.x * ldx;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += 256) acc = __fma_rn(x[i], x[i], acc);
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int k = 0; k < 256 / 32; ++k) s += red[k];
        pre[blockIdx.x] = s;
    }
}

// Q(r, :) = X(r, :) R^{-1} for every row r (forward substitution
// q_j = (x_j - sum_{k<j} q_k R(k, j)) / R(j, j)): one thread per row, the row in
// registers, R broadcast from shared memory.  Replaces R^{-1} + a GEMM.
template <int W>
__global__ void __launch_bounds__(64) k_trsm_rows(const double *__restrict__ X, int64_t ldx, int64_t m,
                                                  const double *__restrict__ Rf, double *__restrict__ Q, int64_t ldq,
                                                  const int *__restrict__ skip)
{
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL)
    __shared__ double R[W * W];
    if (skip && *skip) return;
    for (int e = threadIdx.x; e < W * W; e += blockDim.x) R[e] = Rf[e];
    __syncthreads();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    double q[W];
    #pragma unroll
    for (int j = 0; j < W; ++j) q[j] = X[r + j * ldx];
    #pragma unroll
    for (int j = 0; j < W; ++j) {
        double acc = q[j];
        #pragma unroll
        for (int k = 0; k < j; ++k) acc = __fma_rn(-q[k], R[k + j * W], acc);
        q[j] = __ddiv_rn(acc, R[j + j * W]);
        Q[r + j * ldq] = q[j];
    }
}

// the same for a narrow last panel (w < 64)
__global__ void __launch_bounds__(64) k_trsm_rows_w(const double *__restrict__ X, int64_t ldx, int64_t m, int w,
                                                    const double *__restrict__ Rf, double *__restrict__ Q, int64_t ldq,
                                                    const int *__restrict__ skip)
{
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL)
    __shared__ double R[kPanel * kPanel];
    if (skip && *skip) return;
    for (int e = threadIdx.x; e < w * w; e += blockDim.x) R[e] = Rf[e];
    __syncthreads();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    for (int j = 0; j < w; ++j) {
        double acc = X[r + j * ldx];
        for (int k = 0; k < j; ++k) acc = __fma_rn(-Q[r + k * ldq], R[k + j * w], acc);
        Q[r + j * ldq] = __ddiv_rn(acc, R[j + j * w]);
    }
}
}  // namespace

size_t dgemm_scratch_elems(int64_t m, int64_t n)
{
    (void)m; (void)n;
    return (size_t)300 * 64 * 64;
}

size_t orth_workspace(int64_t n)
{
    // R (n x 64) + S (n x 64) + split-K scratch + G + the Cholesky factor + flag
    return ((size_t)2 * n * kPanel + dgemm_scratch_elems(n, kPanel) + 3 * kPanel * kPanel + 64) * sizeof(double);
}

// one left-looking sweep over the panels with `passes` projection passes (1:
// CGS with the twice-is-enough check recorded in *reorth; 2: CGS2)
static mpj_status orth_sweep(const double *Z, int64_t ldz, double *Q, int64_t ldq, int64_t m, int64_t n, void *ws,
                             int passes, cudaStream_t st)
{
    double *R = (double *)ws;
    double *S = R + (size_t)n * kPanel;
    double *scratch = S + (size_t)m * kPanel;
    const size_t scratch_elems = dgemm_scratch_elems(n, kPanel);
    double *G = scratch + scratch_elems;
    double *Rf = G + kPanel * kPanel;      // Cholesky factor of the panel Gram matrix
    double *pre = Rf + kPanel * kPanel;    // panel column norms^2 before the projection
    int *fail = (int *)(pre + kPanel);
    int *reorth = fail + 1;
    int *single = fail + 2;

    MPJ_CK(cudaMemsetAsync(fail, 0, 3 * sizeof(int), st));
    if (Q != Z || ldq != ldz) launch_copy_pad<double, double>(Z, ldz, (int)m, (int)n, Q, ldq, (int)m, (int)n, st);

    for (int64_t p0 = 0; p0 < n; p0 += kPanel) {
        const int w = (int)std::min<int64_t>(kPanel, n - p0);
        double *X = Q + p0 * ldq;
        const bool check = passes == 1 && p0 > 0;
        if (check) {
            launch_pdl_k(k_colnorm2, dim3(w), dim3(256), 0, st, (const double *)X, ldq, m, pre);
            count_launch();
        }
        if (p0 > 0) {
            for (int rep = 0; rep < passes; ++rep) {
                launch_dgemm(true, false, p0, w, m, 1.0, Q, ldq, X, ldq, 0.0, R, p0, st, scratch, scratch_elems);
                launch_dgemm(false, false, m, w, p0, -1.0, Q, ldq, R, p0, 1.0, X, ldq, st, scratch,
                             scratch_elems);
            }
        }
        // CholeskyQR of the panel X -> S; the second pass S -> X only if the
        // first Gram was not within 1e-3 of I (device-side decision), else S -> X
        const int nblk = (int)((m + 63) / 64);
        for (int rep = 0; rep < 2; ++rep) {
            const double *src = rep == 0 ? X : S;
            const int64_t lds = rep == 0 ? ldq : m;
            double *dst = rep == 0 ? S : X;
            const int64_t ldd = rep == 0 ? m : ldq;
            const int *skip = rep == 1 ? single : nullptr;
            // the panel Gram (one 64 x 64 tile, K = m): split K into 64-row slices, one CTA each
            launch_dgemm(true, false, w, w, m, 1.0, src, lds, src, lds, 0.0, G, w, st, scratch, scratch_elems, false,
                         skip, (int)std::min<int64_t>(128, m / 64));
            launch_pdl_k(k_chol, dim3(1), dim3(kCholNT), 0, st, (const double *)G, w, Rf, fail,
                         (const double *)((check && rep == 0) ? pre : nullptr), reorth, rep == 0 ? single : nullptr,
                         skip);
            if (w == kPanel)
                launch_pdl_k(k_trsm_rows<kPanel>, dim3(nblk), dim3(64), 0, st, src, lds, m, (const double *)Rf, dst, ldd,
                             skip);
            else
                launch_pdl_k(k_trsm_rows_w, dim3(nblk), dim3(64), 0, st, src, lds, m, w, (const double *)Rf, dst, ldd,
                             skip);
            count_launch(2);
        }
        launch_pdl_k(k_copy_panel_if, dim3((unsigned)std::min<int64_t>(64, (m + 255) / 256), w), dim3(256), 0, st,
                     (const double *)S, m, m, X, ldq, (const int *)single);
        count_launch();
    }
    int h[2] = {0, 0};
    MPJ_CK(cudaMemcpyAsync(h, fail, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaStreamSynchronize(st));
    if (h[0]) {
        set_error("orth: non-positive Cholesky pivot (rank deficient Z)");
        return MPJ_ERR_RANKDEF;
    }
    return h[1] ? MPJ_ERR_NOCONV : MPJ_OK;    // NOCONV here: a projection needs its second pass
}

mpj_status orth_cgs2(const double *Z, int64_t ldz, double *Q, int64_t ldq, int64_t m, int64_t n,
                     void *ws, cudaStream_t st)
{
    // Step 1's Z is orthogonal to O(upsilon): one classical projection
    // pass loses no significant part of a column, and CGS's loss of
    // orthogonality is then O(omega kappa(Z)^2) = O(omega).  The sweep checks
    // that (no column kept less than half its norm); otherwise Q is redone
    // with the second pass everywhere (CGS2, reading R10).
    const bool z_alias = (Z == Q);
    if (!z_alias) {
        mpj_status s = orth_sweep(Z, ldz, Q, ldq, m, n, ws, 1, st);
        if (s != MPJ_ERR_NOCONV) return s;
    }
    return orth_sweep(Z, ldz, Q, ldq, m, n, ws, 2, st);
}

// ---------------------------------------------------------------------------
// Step 2 by Cholesky QR with a fixed-point Cholesky factor (reading R10b, the
// batched path's step 2 at full size): G = Z^T Z = I + E; R = chol(G) = I + U
// with U = Phi(E - U^T U) (Phi: strict upper part plus half the diagonal),
// two corrections after U0 = Phi(E) leave O(||E||^4); Q = Z R^{-1} =
// Z (I - U + U^2 - U^3) + O(||E||^4).  Six n^3 DMMA GEMMs and no sequential
// panel chain: for n <= ~2048, where CGS's 64-column panels are a chain of
// small launches, it is several times faster; above, CGS's 2n^3 flops win.
// Needs ||E||_F <= 1e-4 (binary32 step 1 gives ~1e-6); returns MPJ_ERR_NOCONV
// (nothing written) otherwise, and the caller takes CGS.
// ---------------------------------------------------------------------------
namespace {
// E = G - I (n x n), U = Phi(E)
__global__ void k_series_init(const double *__restrict__ G, int n, double *E, double *U)
{
    const int j = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double e = G[i + (size_t)j * n] - (i == j ? 1.0 : 0.0);
        E[i + (size_t)j * n] = e;
        U[i + (size_t)j * n] = i < j ? e : (i == j ? 0.5 * e : 0.0);
    }
}
// U = Phi(E - P)
__global__ void k_series_phi(const double *__restrict__ E, const double *__restrict__ P, int n, double *U)
{
    const int j = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double x = E[i + (size_t)j * n] - P[i + (size_t)j * n];
        U[i + (size_t)j * n] = i < j ? x : (i == j ? 0.5 * x : 0.0);
    }
}
// Q(:, j) += a Y(:, j)
__global__ void k_series_axpy(double *Q, int64_t ldq, const double *__restrict__ Y, int n, double a)
{
    const int j = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        Q[i + (size_t)j * ldq] = __fma_rn(a, Y[i + (size_t)j * n], Q[i + (size_t)j * ldq]);
}
}  // namespace

mpj_status orth_series(const double *Z, int64_t ldz, double *Q, int64_t ldq, int64_t n, cudaStream_t st)
{
    if (n < 1) return MPJ_OK;
    const size_t nn = (size_t)n * n;
    double *buf = nullptr;
    MPJ_CK(cudaMallocAsync(&buf, (4 * nn + kRedBlocks + 8) * sizeof(double), st));
    struct F { double *p; cudaStream_t st; ~F() { cudaFreeAsync(p, st); } } fr{buf, st};
    double *E = buf, *U = E + nn, *P = U + nn, *Y = P + nn, *red = Y + nn;
    const dim3 g2((unsigned)std::max<int64_t>(1, std::min<int64_t>(8, (n + 255) / 256)), (unsigned)n);
    launch_dgemm(true, false, n, n, n, 1.0, Z, ldz, Z, ldz, 0.0, P, n, st);          // G = Z^T Z
    k_series_init<<<g2, 256, 0, st>>>(P, (int)n, E, U);
    count_launch();
    launch_norm<double>(E, n, (int)n, (int)n, false, red, red + kRedBlocks, st);
    double h = 0.0;
    MPJ_CK(cudaMemcpyAsync(&h, red + kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaStreamSynchronize(st));
    if (!(h <= 1e-4)) return MPJ_ERR_NOCONV;
    for (int it = 0; it < 2; ++it) {
        launch_dgemm(true, false, n, n, n, 1.0, U, n, U, n, 0.0, P, n, st);          // P = U^T U
        k_series_phi<<<g2, 256, 0, st>>>(E, P, (int)n, U);
        count_launch();
    }
    // Q = Z - Z U + (Z U) U - ((Z U) U) U
    launch_copy_pad<double, double>(Z, ldz, (int)n, (int)n, Q, ldq, (int)n, (int)n, st);
    double *Yc = Y, *Yn = P;
    launch_dgemm(false, false, n, n, n, 1.0, Z, ldz, U, n, 0.0, Yc, n, st);          // Y1 = Z U
    for (int t = 1; t <= 3; ++t) {
        k_series_axpy<<<g2, 256, 0, st>>>(Q, ldq, Yc, (int)n, (t & 1) ? -1.0 : 1.0);
        count_launch();
        if (t < 3) {
            launch_dgemm(false, false, n, n, n, 1.0, Yc, n, U, n, 0.0, Yn, n, st);   // Y_{t+1} = Y_t U
            std::swap(Yc, Yn);
        }
    }
    MPJ_CK(cudaGetLastError());
    return MPJ_OK;
}

}  // namespace mpj
