// k_gemm.cu -- fp64 GEMM on the FP64 tensor pipe (DMMA) for sm_100a.
//
// sm_100a has no FP64 kind for tcgen05.mma (ptxas rejects ".kind::f64"), so
// the fp64 tensor path is the warp-level mma.sync.aligned.m8n8k4 f64
// instruction (SASS DMMA.8x8x4).  Used by Alg. 3 step 3 (T = Q^T A Q),
// CGS2 (step 2) and Alg. 5 step 3 (C = A Q).
//
// CTA tile 64 x 64 x 16, 4 warps (2 x 2), warp tile 32 x 32 = 4 x 4 DMMA
// fragments, 2-stage cp.async (LDGSTS) double buffer, padded shared layouts
// (2 wavefronts per 32-lane fragment load, the minimum for 8-byte lanes).
// Optional deterministic split-K for the tall-skinny products of CGS2.
#include "mpj_device.cuh"
#include "mpj_internal.h"

#include <algorithm>

namespace mpj {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int SKM = BM + 8;    // stride of a k-major tile  [BK][SKM]
constexpr int SMK = BK + 4;    // stride of an m-major tile [BM][SMK]
constexpr int TILE = (BK * SKM > BM * SMK) ? BK * SKM : BM * SMK;   // doubles per stage

__device__ __forceinline__ void cp_async8(double *dst, const double *src, bool pred)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(sz));
}
// two consecutive elements (16 bytes; src_bytes 8 or 0 zero-fill the rest)
__device__ __forceinline__ void cp_async16(double *dst, const double *src, int src_bytes)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Load the op(A) tile (rows i0.., k0..) into shared memory.
//   TA = false: A is m x k column-major -> k-major smem [kk][i]   (stride SKM)
//   TA = true : A is k x m column-major -> m-major smem [i][kk]   (stride SMK)
template <bool TA, bool V16>
__device__ __forceinline__ void load_a(double *s, const double *A, int64_t lda, int64_t m, int64_t k,
                                       int64_t i0, int64_t k0)
{
    if constexpr (V16) {   // 16-byte copies along the contiguous index (even lda, aligned A)
        #pragma unroll
        for (int e = threadIdx.x; e < BM * BK / 2; e += 128) {
            if (!TA) {
                const int kk = e / (BM / 2), ii = 2 * (e - kk * (BM / 2));
                const int64_t gi = i0 + ii, gk = k0 + kk;
                const int bytes = gk < k ? (gi + 1 < m ? 16 : (gi < m ? 8 : 0)) : 0;
                cp_async16(s + kk * SKM + ii, bytes ? A + gi + gk * lda : A, bytes);
            } else {
                const int ii = e / (BK / 2), kk = 2 * (e - ii * (BK / 2));
                const int64_t gi = i0 + ii, gk = k0 + kk;
                const int bytes = gi < m ? (gk + 1 < k ? 16 : (gk < k ? 8 : 0)) : 0;
                cp_async16(s + ii * SMK + kk, bytes ? A + gk + gi * lda : A, bytes);
            }
        }
        return;
    }
    #pragma unroll
    for (int e = threadIdx.x; e < BM * BK; e += 128) {
        if (!TA) {
            const int kk = e / BM, ii = e - kk * BM;
            const int64_t gi = i0 + ii, gk = k0 + kk;
            const bool ok = gi < m && gk < k;
            cp_async8(s + kk * SKM + ii, ok ? A + gi + gk * lda : A, ok);
        } else {
            const int ii = e / BK, kk = e - ii * BK;
            const int64_t gi = i0 + ii, gk = k0 + kk;
            const bool ok = gi < m && gk < k;
            cp_async8(s + ii * SMK + kk, ok ? A + gk + gi * lda : A, ok);
        }
    }
}

// op(B) tile (k0.., j0..): TB = false: B is k x n -> n-major smem [j][kk];
// TB = true: B is n x k -> k-major smem [kk][j].
template <bool TB, bool V16>
__device__ __forceinline__ void load_b(double *s, const double *B, int64_t ldb, int64_t n, int64_t k,
                                       int64_t j0, int64_t k0)
{
    if constexpr (V16) {
        #pragma unroll
        for (int e = threadIdx.x; e < BN * BK / 2; e += 128) {
            if (!TB) {
                const int jj = e / (BK / 2), kk = 2 * (e - jj * (BK / 2));
                const int64_t gj = j0 + jj, gk = k0 + kk;
                const int bytes = gj < n ? (gk + 1 < k ? 16 : (gk < k ? 8 : 0)) : 0;
                cp_async16(s + jj * SMK + kk, bytes ? B + gk + gj * ldb : B, bytes);
            } else {
                const int kk = e / (BN / 2), jj = 2 * (e - kk * (BN / 2));
                const int64_t gj = j0 + jj, gk = k0 + kk;
                const int bytes = gk < k ? (gj + 1 < n ? 16 : (gj < n ? 8 : 0)) : 0;
                cp_async16(s + kk * SKM + jj, bytes ? B + gj + gk * ldb : B, bytes);
            }
        }
        return;
    }
    #pragma unroll
    for (int e = threadIdx.x; e < BN * BK; e += 128) {
        if (!TB) {
            const int jj = e / BK, kk = e - jj * BK;
            const int64_t gj = j0 + jj, gk = k0 + kk;
            const bool ok = gj < n && gk < k;
            cp_async8(s + jj * SMK + kk, ok ? B + gk + gj * ldb : B, ok);
        } else {
            const int kk = e / BN, jj = e - kk * BN;
            const int64_t gj = j0 + jj, gk = k0 + kk;
            const bool ok = gj < n && gk < k;
            cp_async8(s + kk * SKM + jj, ok ? B + gj + gk * ldb : B, ok);
        }
    }
}

// split == 1: C = alpha acc + beta C.  split > 1: partial[z] = acc (m x n, ld m).
template <bool TA, bool TB, bool V16>
__global__ void __launch_bounds__(128) k_dgemm(int64_t m, int64_t n, int64_t k, double alpha,
                                               const double *__restrict__ A, int64_t lda,
                                               const double *__restrict__ B, int64_t ldb, double beta,
                                               double *__restrict__ C, int64_t ldc, int kchunk,
                                               double *__restrict__ partial, int upper_only,
                                               const int *__restrict__ skip)
{
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL): wait for the producer
    if (skip && *skip) return;                       // a conditional product (device-side decision)
    if (upper_only && (int64_t)blockIdx.x * BM >= ((int64_t)blockIdx.y + 1) * BN) return;   // strictly lower tile
    __shared__ __align__(16) double sA[2][TILE];
    __shared__ __align__(16) double sB[2][TILE];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tig = lane & 3;
    const int wm = warp >> 1, wn = warp & 1;
    const int64_t i0 = (int64_t)blockIdx.x * BM, j0 = (int64_t)blockIdx.y * BN;
    const int64_t kb = (int64_t)blockIdx.z * kchunk;
    const int64_t ke = min(k, kb + kchunk);

    // C of the epilogue (beta != 0) into L2 now: its loads come after the
    // k-loop, and for the short-K updates (the back-transformation's rank-128
    // Y -= V W, K = 128) their HBM latency was the largest stall (ncu: long
    // scoreboard 5.9 per issue, 52% tensor active)
    if (beta != 0.0 && !partial) {
        const int64_t gj = j0 + (threadIdx.x >> 1), gi = i0 + (threadIdx.x & 1) * 32;
        if (gj < n && gi < m) {
            const double *pc = C + gi + gj * ldc;
            asm volatile("prefetch.global.L2 [%0];\n" ::"l"(pc));
            if (gi + 16 < m) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(pc + 16));
        }
    }
    double acc[4][4][2];
    #pragma unroll
    for (int a = 0; a < 4; ++a)
        #pragma unroll
        for (int b = 0; b < 4; ++b) { acc[a][b][0] = 0.0; acc[a][b][1] = 0.0; }

    const int nk = (int)((ke - kb + BK - 1) / BK);
    if (nk > 0) {
        load_a<TA, V16>(sA[0], A, lda, m, ke, i0, kb);
        load_b<TB, V16>(sB[0], B, ldb, n, ke, j0, kb);
    }
    cp_commit();
    for (int it = 0; it < nk; ++it) {
        const int cur = it & 1;
        if (it + 1 < nk) {
            load_a<TA, V16>(sA[cur ^ 1], A, lda, m, ke, i0, kb + (int64_t)(it + 1) * BK);
            load_b<TB, V16>(sB[cur ^ 1], B, ldb, n, ke, j0, kb + (int64_t)(it + 1) * BK);
        }
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        const double *a_s = sA[cur], *b_s = sB[cur];
        #pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
            double af[4], bf[4];
            #pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                const int r = wm * 32 + mi * 8 + g, c = ks * 4 + tig;
                af[mi] = TA ? a_s[r * SMK + c] : a_s[c * SKM + r];
            }
            #pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                const int col = wn * 32 + ni * 8 + g, kr = ks * 4 + tig;
                bf[ni] = TB ? b_s[kr * SKM + col] : b_s[col * SMK + kr];
            }
            #pragma unroll
            for (int mi = 0; mi < 4; ++mi)
                #pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
        __syncthreads();
    }

    #pragma unroll
    for (int mi = 0; mi < 4; ++mi)
        #pragma unroll
        for (int ni = 0; ni < 4; ++ni)
            #pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int64_t gi = i0 + wm * 32 + mi * 8 + g;
                const int64_t gj = j0 + wn * 32 + ni * 8 + 2 * tig + e;
                if (gi < m && gj < n) {
                    if (partial) {
                        partial[(int64_t)blockIdx.z * m * n + gi + gj * m] = acc[mi][ni][e];
                    } else {
                        double v = alpha * acc[mi][ni][e];
                        if (beta != 0.0) v = __fma_rn(beta, C[gi + gj * ldc], v);
                        C[gi + gj * ldc] = v;
                    }
                }
            }
}

__global__ void k_splitk_reduce(int64_t m, int64_t n, int splits, const double *__restrict__ partial,
                                double alpha, double beta, double *__restrict__ C, int64_t ldc,
                                const int *__restrict__ skip)
{
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL)
    if (skip && *skip) return;
    const int64_t total = m * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * total + e];   // fixed order
        const int64_t j = e / m, i = e - j * m;
        double v = alpha * s;
        if (beta != 0.0) v = __fma_rn(beta, C[i + j * ldc], v);
        C[i + j * ldc] = v;
    }
}

// launch with programmatic stream serialisation: the kernel may be scheduled
// while its predecessor drains (the chains of small products in CGS and the
// back-transformation); it waits (griddepcontrol.wait) before touching data
template <typename... KA, typename... A>
static void launch_pdl_g(void (*k)(KA...), dim3 grid, dim3 block, cudaStream_t st, A... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, args...);
}

}  // namespace

void launch_dgemm(bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha, const double *A,
                  int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
                  cudaStream_t st, double *scratch, size_t scratch_elems, bool upper_only, const int *skip,
                  int min_splits)
{
    if (m <= 0 || n <= 0) return;
    const int64_t gm = (m + BM - 1) / BM, gn = (n + BN - 1) / BN;
    int splits = 1;
    const int64_t tiles = gm * gn;
    if (tiles < 148 && k >= 1024 && scratch) {
        splits = (int)std::min<int64_t>((296 + tiles - 1) / tiles, k / 256);
        while (splits > 1 && (size_t)splits * m * n > scratch_elems) --splits;
    }
    if (min_splits > splits && scratch && k >= 64 * min_splits) {    // caller's hint (shapes it measured)
        splits = min_splits;
        while (splits > 1 && (size_t)splits * m * n > scratch_elems) --splits;
    }
    int kchunk = (int)(((k + splits - 1) / splits + BK - 1) / BK * BK);
    if (kchunk <= 0) kchunk = BK;
    dim3 grd((unsigned)gm, (unsigned)gn, (unsigned)splits);
    double *part = splits > 1 ? scratch : nullptr;
    // 16-byte operand copies when every column start is 16-byte aligned
    const bool v16 = lda % 2 == 0 && ldb % 2 == 0 && ((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0;
#define GO(a, b, v) launch_pdl_g(k_dgemm<a, b, v>, grd, dim3(128), st, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, \
                                 kchunk, part, upper_only ? 1 : 0, skip)
#define GO2(a, b) do { if (v16) GO(a, b, true); else GO(a, b, false); } while (0)
    if (!ta && !tb) GO2(false, false);
    else if (ta && !tb) GO2(true, false);
    else if (!ta && tb) GO2(false, true);
    else GO2(true, true);
#undef GO2
#undef GO
    count_launch();
    if (splits > 1) {
        launch_pdl_g(k_splitk_reduce, dim3(592), dim3(256), st, m, n, splits, (const double *)part, alpha, beta, C,
                     ldc, skip);
        count_launch();
    }
}

}  // namespace mpj
