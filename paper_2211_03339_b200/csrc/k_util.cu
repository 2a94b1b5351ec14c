// k_util.cu -- norms, padding, symmetrisation and extraction kernels.
//   off(T) = sqrt(sum_{i != j} t_ij^2), summed directly (reading R9; the
//   ||T||^2 - sum t_ii^2 form cancels), deterministic two-stage reduction.
//   Extraction (Alg. 3 output; P:39 descending order): stable rank.
#include "mpj_device.cuh"
#include "mpj_internal.h"

namespace mpj {

template <typename R>
__global__ void __launch_bounds__(256) k_norm_partial(const R *__restrict__ T, int64_t ld, int m,
                                                      int n, int offdiag, double *__restrict__ part)
{
    __shared__ double sh[32];
    double acc = 0.0;
    const int64_t total = (int64_t)m * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e / m), i = (int)(e - (int64_t)j * m);
        if (offdiag && i == j) continue;
        const double x = (double)T[i + j * ld];
        acc = __fma_rn(x, x, acc);
    }
    const double s = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_norm_final(const double *__restrict__ part, int nparts, double *__restrict__ out)
{
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc += part[i];
    const double s = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) out[0] = sqrt(s);
}

template <typename R>
void launch_norm(const R *T, int64_t ld, int m, int n, bool offdiag, double *partial, double *out,
                 cudaStream_t st)
{
    k_norm_partial<R><<<kRedBlocks, 256, 0, st>>>(T, ld, m, n, offdiag ? 1 : 0, partial);
    k_norm_final<<<1, 256, 0, st>>>(partial, kRedBlocks, out);
    count_launch(2);
}
template void launch_norm<double>(const double *, int64_t, int, int, bool, double *, double *, cudaStream_t);

// sum over i <= j of w_ij T_ij^2 with w = 2 above the diagonal, 1 on it (0 if
// offdiag): the full sums of launch_norm for a symmetric T, lower half unread
__global__ void __launch_bounds__(256) k_norm_sym_upper(const double *__restrict__ T, int64_t ld, int n,
                                                        int offdiag, double *__restrict__ part)
{
    __shared__ double sh[32];
    double acc = 0.0;
    const int64_t total = (int64_t)n * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e / n), i = (int)(e - (int64_t)j * n);
        if (i > j || (offdiag && i == j)) continue;
        const double x = T[i + j * ld];
        acc = __fma_rn(i < j ? 2.0 * x : x, x, acc);
    }
    const double s = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

void launch_norm_sym_upper(const double *T, int64_t ld, int n, bool offdiag, double *partial, double *out,
                           cudaStream_t st)
{
    k_norm_sym_upper<<<kRedBlocks, 256, 0, st>>>(T, ld, n, offdiag ? 1 : 0, partial);
    k_norm_final<<<1, 256, 0, st>>>(partial, kRedBlocks, out);
    count_launch(2);
}
template void launch_norm<float>(const float *, int64_t, int, int, bool, double *, double *, cudaStream_t);

template <typename Rs, typename Rd>
__global__ void k_copy_pad(const Rs *__restrict__ src, int64_t lds, int m, int n,
                           Rd *__restrict__ dst, int64_t ldd, int mp, int np_)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= mp || j >= np_) return;
    dst[i + j * ldd] = (i < m && j < n) ? (Rd)src[i + j * lds] : Rd(0);
}

template <typename Rs, typename Rd>
void launch_copy_pad(const Rs *src, int64_t lds, int m, int n, Rd *dst, int64_t ldd, int mp, int np_,
                     cudaStream_t st)
{
    dim3 grd((mp + 255) / 256, np_);
    k_copy_pad<Rs, Rd><<<grd, 256, 0, st>>>(src, lds, m, n, dst, ldd, mp, np_);
    count_launch();
}
template void launch_copy_pad<double, double>(const double *, int64_t, int, int, double *, int64_t, int, int, cudaStream_t);
template void launch_copy_pad<double, float>(const double *, int64_t, int, int, float *, int64_t, int, int, cudaStream_t);
template void launch_copy_pad<float, double>(const float *, int64_t, int, int, double *, int64_t, int, int, cudaStream_t);
template void launch_copy_pad<float, float>(const float *, int64_t, int, int, float *, int64_t, int, int, cudaStream_t);

// (A + A^T)/2 as (a_ij + a_ji) * 0.5 (reading R14), zero padding beyond n.
__global__ void k_symmetrize(const double *__restrict__ src, int64_t lds, int n,
                             double *__restrict__ dst, int64_t ldd, int np_)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= np_ || j >= np_) return;
    double v = 0.0;
    if (i < n && j < n) v = (src[i + j * lds] + src[j + i * lds]) * 0.5;
    dst[i + j * ldd] = v;
}

void launch_symmetrize(const double *src, int64_t lds, int n, double *dst, int64_t ldd, int np_,
                       cudaStream_t st)
{
    dim3 grd((np_ + 255) / 256, np_);
    k_symmetrize<<<grd, 256, 0, st>>>(src, lds, n, dst, ldd, np_);
    count_launch();
}

// In place: each (i<j) couple handled by one thread; 32x32 tiles through smem
// keep both the read of a_ij and of a_ji coalesced.
__global__ void k_symmetrize_inplace(double *__restrict__ T, int64_t ld, int n, int mirror)
{
    __shared__ double up[32][33], lo[32][33];
    const int bi = blockIdx.x, bj = blockIdx.y;
    if (bi > bj) return;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        const int i = bi * 32 + tx, j = bj * 32 + r;      // (i, j) in tile (bi, bj)
        up[r][tx] = (i < n && j < n) ? T[i + (int64_t)j * ld] : 0.0;
        const int i2 = bj * 32 + tx, j2 = bi * 32 + r;    // (i2, j2) in tile (bj, bi)
        lo[r][tx] = (i2 < n && j2 < n) ? T[i2 + (int64_t)j2 * ld] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        // element (bi*32+tx, bj*32+r) pairs with (bj*32+r, bi*32+tx) = lo[tx][r]
        const int i = bi * 32 + tx, j = bj * 32 + r;
        const int i2 = bj * 32 + tx, j2 = bi * 32 + r;
        // mirror: the upper triangle (i <= j) is the source; else the average
        const double v = mirror ? (i <= j ? up[r][tx] : lo[tx][r]) : (up[r][tx] + lo[tx][r]) * 0.5;
        if (i < n && j < n) T[i + (int64_t)j * ld] = v;
        const double w = mirror ? (i2 <= j2 ? lo[r][tx] : up[tx][r]) : (lo[r][tx] + up[tx][r]) * 0.5;
        if (i2 < n && j2 < n) T[i2 + (int64_t)j2 * ld] = w;
    }
}

void launch_symmetrize_inplace(double *T, int64_t ld, int n, cudaStream_t st, bool mirror_upper)
{
    const int nt = (n + 31) / 32;
    k_symmetrize_inplace<<<dim3(nt, nt), dim3(32, 8), 0, st>>>(T, ld, n, mirror_upper ? 1 : 0);
    count_launch();
}

template <typename R>
__global__ void k_identity(R *__restrict__ V, int64_t ld, int m, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= m || j >= n) return;
    V[i + j * ld] = (i == j) ? R(1) : R(0);
}

template <typename R>
void launch_identity(R *V, int64_t ld, int m, int n, cudaStream_t st)
{
    k_identity<R><<<dim3((m + 255) / 256, n), 256, 0, st>>>(V, ld, m, n);
    count_launch();
}
template void launch_identity<double>(double *, int64_t, int, int, cudaStream_t);
template void launch_identity<float>(float *, int64_t, int, int, cudaStream_t);

__global__ void k_check_finite(const double *__restrict__ A, int64_t ld, int m, int n,
                               int *__restrict__ flag)
{
    const int64_t total = (int64_t)m * n;
    int bad = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e / m), i = (int)(e - (int64_t)j * m);
        if (!isfinite(A[i + j * ld])) bad = 1;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

void launch_check_finite(const double *A, int64_t ld, int m, int n, int *flag, cudaStream_t st)
{
    k_check_finite<<<kRedBlocks, 256, 0, st>>>(A, ld, m, n, flag);
    count_launch();
}

// rank[i] = #{j : d_j > d_i} + #{j < i : d_j == d_i}  (stable descending order)
__global__ void k_rank_desc(const double *__restrict__ T, int64_t ldt, int n, int *__restrict__ rank,
                            double *__restrict__ lam)
{
    extern __shared__ double dsh[];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const double di = (i < n) ? T[i + (int64_t)i * ldt] : 0.0;
    int cnt = 0;
    for (int base = 0; base < n; base += 1024) {
        const int lim = min(1024, n - base);
        __syncthreads();
        for (int t = threadIdx.x; t < lim; t += blockDim.x) dsh[t] = T[(base + t) + (int64_t)(base + t) * ldt];
        __syncthreads();
        if (i < n)
            for (int t = 0; t < lim; ++t) {
                const double dj = dsh[t];
                cnt += (dj > di) || (dj == di && base + t < i);
            }
    }
    if (i < n) { rank[i] = cnt; lam[cnt] = di; }
}

__global__ void k_permute_cols(const double *__restrict__ V, int64_t ldv, int vrows,
                               const int *__restrict__ rank, double *__restrict__ Vout, int64_t ldvo)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= vrows) return;
    Vout[i + (int64_t)rank[j] * ldvo] = V[i + (int64_t)j * ldv];
}

void launch_extract_evd(const double *T, int64_t ldt, const double *V, int64_t ldv, int n, int vrows,
                        double *lam, double *Vout, int64_t ldvo, int *rank, cudaStream_t st)
{
    k_rank_desc<<<(n + 255) / 256, 256, 1024 * sizeof(double), st>>>(T, ldt, n, rank, lam);
    k_permute_cols<<<dim3((vrows + 255) / 256, n), 256, 0, st>>>(V, ldv, vrows, rank, Vout, ldvo);
    count_launch(2);
}

}  // namespace mpj
