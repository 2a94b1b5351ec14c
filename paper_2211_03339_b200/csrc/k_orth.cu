// k_orth.cu -- Alg. 3 step 2: Q = orth(Z) in fp64.
//
// Reading R10: the paper's MGS (Lemma 2.1) is realised
// as left-looking blocked classical Gram-Schmidt with reorthogonalisation
// (CGS2), which matches MGS's orthogonality contract (it reaches O(omega)
// for any kappa(Z) << 1/omega, and Z is orthogonal to O(upsilon)).
//   for each panel X = Z(:, p0:p0+w):
//     twice:  R = Q(:, :p0)^T X ;  X = X - Q(:, :p0) R     (fp64 DMMA GEMMs)
//     inside the panel, column by column (k_panel_cgs2, one cooperative
//     launch): twice r = X(:, :j)^T x_j, x_j -= X(:, :j) r; then
//     x_j /= ||x_j||.  Dot products: per-CTA warp-shuffle reductions over a
//     row slab, then a fixed-order sum of the per-CTA partials (deterministic).
#include <cooperative_groups.h>

#include "mpj_device.cuh"
#include "mpj_internal.h"

#include <algorithm>

namespace mpj {

namespace {
constexpr int kPanel = 64;
constexpr int kOrthThreads = 256;

struct GridBar {
    unsigned *count;
    unsigned *gen;
};

__device__ __forceinline__ void grid_sync(GridBar gb, unsigned nblocks)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *vgen = gb.gen;
        const unsigned g0 = *vgen;
        __threadfence();
        const unsigned arrived = atomicAdd(gb.count, 1u);
        if (arrived == nblocks - 1) {
            atomicExch(gb.count, 0u);
            __threadfence();
            atomicAdd(gb.gen, 1u);
        } else {
            while (*vgen == g0) { __nanosleep(32); }
        }
        __threadfence();
    }
    __syncthreads();
}

// X: m x w panel (ld ldx), orthonormalised in place.  part: 2 x G x kPanel
// doubles (double-buffered partials); fail: set to 1 on a zero column.
__global__ void __launch_bounds__(kOrthThreads) k_panel_cgs2(double *__restrict__ X, int64_t ldx,
                                                             int64_t m, int w, double *part,
                                                             GridBar gb, int *fail)
{
    __shared__ double coef[kPanel];
    const unsigned G = gridDim.x;
    const int64_t rows_per = (m + G - 1) / G;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = min(m, r0 + rows_per);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int step = 0;
    for (int j = 0; j < w; ++j) {
        double *xj = X + (int64_t)j * ldx;
        for (int pass = (j == 0 ? 2 : 0); pass < 3; ++pass) {   // 0,1: projections; 2: norm
            const int nd = (pass < 2) ? j : 1;
            double *pbuf = part + (size_t)(step & 1) * G * kPanel;
            // per-CTA partial dot products: warp -> column i, lanes -> rows
            for (int i = warp; i < nd; i += kOrthThreads / 32) {
                const double *xi = (pass < 2) ? X + (int64_t)i * ldx : xj;
                double a = 0.0;
                for (int64_t r = r0 + lane; r < r1; r += 32) a = __fma_rn(xi[r], xj[r], a);
                #pragma unroll
                for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                if (lane == 0) pbuf[(size_t)blockIdx.x * kPanel + i] = a;
            }
            grid_sync(gb, G);
            if (threadIdx.x < nd) {
                double sum = 0.0;
                for (unsigned c = 0; c < G; ++c) sum += __ldcg(pbuf + (size_t)c * kPanel + threadIdx.x);
                coef[threadIdx.x] = sum;
            }
            __syncthreads();
            ++step;
            if (pass < 2) {
                for (int64_t r = r0 + threadIdx.x; r < r1; r += kOrthThreads) {
                    double x = xj[r];
                    for (int i = 0; i < nd; ++i) x = __fma_rn(-coef[i], X[r + (int64_t)i * ldx], x);
                    xj[r] = x;
                }
            } else {
                const double nrm = sqrt(coef[0]);
                if (!(nrm > 0.0)) {
                    if (blockIdx.x == 0 && threadIdx.x == 0) *fail = 1;
                } else {
                    for (int64_t r = r0 + threadIdx.x; r < r1; r += kOrthThreads) xj[r] = xj[r] / nrm;
                }
            }
            __syncthreads();
        }
    }
}
}  // namespace

size_t orth_workspace(int64_t n)
{
    // R (n x 64) + split-K scratch + partials + barrier words + fail flag
    return ((size_t)n * kPanel + dgemm_scratch_elems(n, kPanel) + 2 * 1024 * kPanel + 64) * sizeof(double);
}

size_t dgemm_scratch_elems(int64_t m, int64_t n)
{
    (void)m; (void)n;
    return (size_t)300 * 64 * 64;
}

mpj_status orth_cgs2(const double *Z, int64_t ldz, double *Q, int64_t ldq, int64_t m, int64_t n,
                     void *ws, cudaStream_t st)
{
    double *R = (double *)ws;
    double *scratch = R + (size_t)n * kPanel;
    const size_t scratch_elems = dgemm_scratch_elems(n, kPanel);
    double *part = scratch + scratch_elems;
    unsigned *bar = (unsigned *)(part + 2 * 1024 * kPanel);
    int *fail = (int *)(bar + 4);

    int dev = 0, nsm = 0;
    MPJ_CK(cudaGetDevice(&dev));
    MPJ_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    int per_sm = 0;
    MPJ_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_panel_cgs2, kOrthThreads, 0));
    int G = (int)std::min<int64_t>((int64_t)nsm * std::max(per_sm, 1), (m + 31) / 32);
    G = std::max(1, std::min(G, 1024));

    MPJ_CK(cudaMemsetAsync(bar, 0, 4 * sizeof(unsigned) + sizeof(int), st));
    if (Q != Z || ldq != ldz) launch_copy_pad<double, double>(Z, ldz, (int)m, (int)n, Q, ldq, (int)m, (int)n, st);

    for (int64_t p0 = 0; p0 < n; p0 += kPanel) {
        const int w = (int)std::min<int64_t>(kPanel, n - p0);
        double *X = Q + p0 * ldq;
        if (p0 > 0) {
            for (int rep = 0; rep < 2; ++rep) {
                launch_dgemm(true, false, p0, w, m, 1.0, Q, ldq, X, ldq, 0.0, R, p0, st, scratch,
                             scratch_elems);
                launch_dgemm(false, false, m, w, p0, -1.0, Q, ldq, R, p0, 1.0, X, ldq, st, scratch,
                             scratch_elems);
            }
        }
        GridBar gb{bar, bar + 1};
        int64_t ldx = ldq;
        void *args[] = {&X, &ldx, (void *)&m, (void *)&w, &part, &gb, &fail};
        MPJ_CK(cudaLaunchCooperativeKernel((void *)k_panel_cgs2, dim3(G), dim3(kOrthThreads), args, 0, st));
        count_launch();
    }
    int h_fail = 0;
    MPJ_CK(cudaMemcpyAsync(&h_fail, fail, sizeof(int), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaStreamSynchronize(st));
    if (h_fail) {
        set_error("orth: zero column during Gram-Schmidt (rank deficient Z)");
        return MPJ_ERR_RANKDEF;
    }
    return MPJ_OK;
}

}  // namespace mpj
