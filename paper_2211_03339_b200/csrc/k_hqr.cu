// k_hqr.cu -- Alg. 3 step 2 by Householder QR (the paper's GPU code
// orthogonalised with Householder QR; the algorithm states MGS, P:189;
// SURVEY 8(f) row 3).  Both give the unique QR factor Q of Z with a positive
// diagonal of R (reading R10), so this is an alternative to the CGS path of
// k_orth.cu, selected with mpj_config.orth = MPJ_ORTH_HOUSEHOLDER.
//
//   for each 64-column panel P = Z(k:, k:k+64):
//     one CTA factors P column by column (LAPACK dgeqr2: beta = -sign(alpha)
//       ||x||, tau = (beta - alpha)/beta, v = x / (alpha - beta), v(0) = 1);
//     the trailing columns get Z(k:, k+64:) -= V T^T (V^T Z(k:, k+64:)) (WY
//       form, T from dlarft; three fp64 DMMA GEMMs);
//   Q = H_0 H_1 ... H_{n-1} formed by backward accumulation on the identity,
//   then column j scaled by sign(R_jj) (positive diag R: the MGS Q).
#include "mpj_device.cuh"
#include "mpj_internal.h"

#include <algorithm>

namespace mpj {

namespace {

constexpr int HB = 64;          // panel width
constexpr int HNT = 1024;       // threads of the panel kernel

__device__ __forceinline__ double block_sum(double v, double *red)
{
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    for (int i = 0; i < HNT / 32; ++i) r += red[i];   // fixed order
    return r;
}

// Householder QR of the m x w panel P (ld), in place: R on and above the
// diagonal, v_j(1:) below it; tau[j], beta (the diagonal of R) in rdiag[j].
__global__ void __launch_bounds__(HNT) k_hqr_panel(double *P, int64_t ld, int m, int w, double *tau, double *rdiag)
{
    __shared__ double red[HNT / 32];
    __shared__ double wv[HB];
    __shared__ double sc[4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int j = 0; j < w && j < m; ++j) {
        double *x = P + (size_t)j * ld;
        double s = 0.0;
        for (int i = j + 1 + tid; i < m; i += HNT) s = __fma_rn(x[i], x[i], s);
        s = block_sum(s, red);
        const double alpha = x[j];
        double beta, t, scal;
        if (s == 0.0) { beta = alpha; t = 0.0; scal = 0.0; }
        else {
            const double nrm = sqrt(__fma_rn(alpha, alpha, s));
            beta = alpha >= 0.0 ? -nrm : nrm;
            t = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        __syncthreads();
        for (int i = j + 1 + tid; i < m; i += HNT) x[i] *= scal;
        if (tid == 0) { tau[j] = t; rdiag[j] = beta; x[j] = beta; }
        __syncthreads();
        // w_c = P(j, c) + sum_{i > j} v_i P(i, c), c = j+1 .. w-1 (a warp per column)
        for (int c = j + 1 + warp; c < w; c += HNT / 32) {
            const double *pc = P + (size_t)c * ld;
            double acc = 0.0;
            for (int i = j + 1 + lane; i < m; i += 32) acc = __fma_rn(x[i], pc[i], acc);
            #pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) wv[c] = pc[j] + acc;
        }
        __syncthreads();
        // P(i, c) -= tau v_i w_c  (v_j = 1)
        for (int c = j + 1; c < w; ++c) {
            double *pc = P + (size_t)c * ld;
            const double tw = t * wv[c];
            if (tid == 0) pc[j] -= tw;
            for (int i = j + 1 + tid; i < m; i += HNT) pc[i] = __fma_rn(-tw, x[i], pc[i]);
        }
        __syncthreads();
    }
    (void)sc;
}

// Vp (rows k0 .. m-1, ld ldv) of the panel's reflectors (column t: 0 above its
// row k0 + t, 1 there, v below), zero columns t >= w
__global__ void k_hqr_vp(const double *__restrict__ Z, int64_t ldz, int m, int k0, int w, double *Vp, int64_t ldv)
{
    const int t = blockIdx.y;
    for (int i = k0 + blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        double v = 0.0;
        if (t < w) {
            const int j = k0 + t;
            v = i < j ? 0.0 : (i == j ? 1.0 : Z[i + (size_t)j * ldz]);
        }
        Vp[(i - k0) + (size_t)t * ldv] = v;
    }
}

// T (HB x HB, ld HB) of H_0 ... H_{w-1} = I - V T V^T from G = V^T V (dlarft)
__global__ void __launch_bounds__(128) k_hqr_t(const double *__restrict__ G, const double *__restrict__ tau, int w,
                                               double *Tm)
{
    __shared__ double T[HB * (HB + 1)];
    __shared__ double z[HB];
    const int tid = threadIdx.x;
    for (int e = tid; e < HB * (HB + 1); e += 128) T[e] = 0.0;
    __syncthreads();
    for (int t = 0; t < w; ++t) {
        const double ta = tau[t];
        if (tid < t) z[tid] = -ta * G[tid + t * HB];
        __syncthreads();
        if (tid < t) {
            double acc = 0.0;
            for (int u = tid; u < t; ++u) acc = __fma_rn(T[tid + u * (HB + 1)], z[u], acc);
            T[tid + t * (HB + 1)] = acc;
        }
        if (tid == 0) T[t + t * (HB + 1)] = ta;
        __syncthreads();
    }
    for (int e = tid; e < HB * HB; e += 128) Tm[e] = T[(e % HB) + (e / HB) * (HB + 1)];
}

__global__ void k_identity_d(double *Q, int64_t ld, int m, int n)
{
    const int j = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        Q[i + (size_t)j * ld] = (i == j) ? 1.0 : 0.0;
}

// Q(:, j) *= sign(R_jj) (positive diagonal of R); flag a zero pivot
__global__ void k_hqr_sign(double *Q, int64_t ld, int m, const double *__restrict__ rdiag, int *fail)
{
    const int j = blockIdx.y;
    const double r = rdiag[j];
    if (blockIdx.x == 0 && threadIdx.x == 0 && !(r != 0.0)) *fail = 1;
    if (r < 0.0)
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
            Q[i + (size_t)j * ld] = -Q[i + (size_t)j * ld];
}

}  // namespace

size_t hqr_workspace(int64_t m, int64_t n)
{
    // Zw (m x n), Vp (m x HB), G, T (HB x HB), W1, W2 (HB x n), tau, rdiag (n), split-K scratch, flag
    return ((size_t)m * n + (size_t)m * HB + 2 * HB * HB + 2 * (size_t)HB * n + 2 * (size_t)n +
            dgemm_scratch_elems(n, HB) + 64) * sizeof(double) + 1024;
}

// Q = the Householder QR factor of Z (m x n, m >= n) with positive diag(R)
mpj_status orth_householder(const double *Z, int64_t ldz, double *Q, int64_t ldq, int64_t m, int64_t n, void *ws,
                            cudaStream_t st)
{
    double *Zw = (double *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    double *Vp = Zw + (size_t)m * n;
    double *G = Vp + (size_t)m * HB, *Tm = G + HB * HB;
    double *W1 = Tm + HB * HB, *W2 = W1 + (size_t)HB * n;
    double *tau = W2 + (size_t)HB * n, *rdiag = tau + n;
    double *skw = rdiag + n;
    const size_t ske = dgemm_scratch_elems(n, HB);
    int *fail = (int *)(skw + ske);
    MPJ_CK(cudaMemsetAsync(fail, 0, sizeof(int), st));
    launch_copy_pad<double, double>(Z, ldz, (int)m, (int)n, Zw, m, (int)m, (int)n, st);
    // factorisation
    for (int64_t k0 = 0; k0 < n; k0 += HB) {
        const int w = (int)std::min<int64_t>(HB, n - k0);
        const int mr = (int)(m - k0);
        k_hqr_panel<<<1, HNT, 0, st>>>(Zw + k0 + k0 * m, m, mr, w, tau + k0, rdiag + k0);
        count_launch();
        if (k0 + w < n) {
            k_hqr_vp<<<dim3(std::max(1, std::min(32, (mr + 255) / 256)), HB), 256, 0, st>>>(Zw, m, (int)m, (int)k0, w,
                                                                                             Vp, m);
            count_launch();
            launch_dgemm(true, false, HB, HB, mr, 1.0, Vp, m, Vp, m, 0.0, G, HB, st, skw, ske);
            k_hqr_t<<<1, 128, 0, st>>>(G, tau + k0, w, Tm);
            count_launch();
            const int nc = (int)(n - k0 - w);
            double *Ct = Zw + k0 + (k0 + w) * m;
            // C -= V T^T (V^T C)
            launch_dgemm(true, false, HB, nc, mr, 1.0, Vp, m, Ct, m, 0.0, W1, HB, st, skw, ske);
            launch_dgemm(true, false, HB, nc, HB, 1.0, Tm, HB, W1, HB, 0.0, W2, HB, st);
            launch_dgemm(false, false, mr, nc, HB, -1.0, Vp, m, W2, HB, 1.0, Ct, m, st);
        }
    }
    // Q = H_0 ... H_{n-1} I(:, 1:n), backward
    k_identity_d<<<dim3(std::max<int64_t>(1, std::min<int64_t>(32, (m + 255) / 256)), (unsigned)n), 256, 0, st>>>(
        Q, ldq, (int)m, (int)n);
    count_launch();
    for (int64_t k0 = ((n - 1) / HB) * HB; k0 >= 0; k0 -= HB) {
        const int w = (int)std::min<int64_t>(HB, n - k0);
        const int mr = (int)(m - k0), nc = (int)(n - k0);
        k_hqr_vp<<<dim3(std::max(1, std::min(32, (mr + 255) / 256)), HB), 256, 0, st>>>(Zw, m, (int)m, (int)k0, w, Vp,
                                                                                         m);
        count_launch();
        launch_dgemm(true, false, HB, HB, mr, 1.0, Vp, m, Vp, m, 0.0, G, HB, st, skw, ske);
        k_hqr_t<<<1, 128, 0, st>>>(G, tau + k0, w, Tm);
        count_launch();
        double *Qt = Q + k0 + k0 * ldq;
        // Q(k0:, k0:) -= V T (V^T Q(k0:, k0:))
        launch_dgemm(true, false, HB, nc, mr, 1.0, Vp, m, Qt, ldq, 0.0, W1, HB, st, skw, ske);
        launch_dgemm(false, false, HB, nc, HB, 1.0, Tm, HB, W1, HB, 0.0, W2, HB, st);
        launch_dgemm(false, false, mr, nc, HB, -1.0, Vp, m, W2, HB, 1.0, Qt, ldq, st);
    }
    k_hqr_sign<<<dim3(std::max<int64_t>(1, std::min<int64_t>(32, (m + 255) / 256)), (unsigned)n), 256, 0, st>>>(
        Q, ldq, (int)m, rdiag, fail);
    count_launch();
    int h = 0;
    MPJ_CK(cudaMemcpyAsync(&h, fail, sizeof(int), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaStreamSynchronize(st));
    if (h) {
        set_error("orth (Householder): zero diagonal of R (rank deficient Z)");
        return MPJ_ERR_RANKDEF;
    }
    return MPJ_OK;
}

}  // namespace mpj
