// k_tridiag.cu -- Alg. 3 step 1 as the paper states it ("[Z,~] =
// eig(A)  Symmetric QR factorization in low precision upsilon"; the paper ran
// LAPACK SSYEV / cusolverDnSsyevd there), reading R12' of
// DESIGN.md.  Three stages, all on the GPU:
//
//  1. Householder tridiagonalisation T = Q^T fl32(A) Q in binary32 (the
//     "low precision" of the step), blocked as LAPACK's ssytrd/slatrd with
//     64-column panels: one cooperative persistent kernel per panel.  Per
//     column j: (A) the column is corrected by the panel's earlier reflectors
//     and its tail norm reduced; (B) the reflector v is formed on the fly and
//     the symmetric product A22 v is taken from the LOWER triangle only (each
//     64 x 64 tile read once, used for y_I += A_IJ v_J and y_J += A_IJ^T v_I;
//     deterministic partial vectors instead of atomics), together with the
//     panel dot products and v^T A22 v; (C) every CTA finishes w = tau(A22 v -
//     V W^T v - W V^T v) - (tau/2)(w^T v) v for its rows.  Two grid barriers
//     per column.  After the panel: A22 -= V W^T + W V^T on the lower tiles
//     (rank-128 update).  Reflectors are stored below the subdiagonal as in
//     LAPACK (H = I - tau v v^T, v(0) = 1, beta = -sign(alpha) ||x||).
//  2. Eigen-decomposition of the tridiagonal in binary64: the matrix is split
//     where |e_i| <= omega sqrt(|d_i d_{i+1}|); each block's eigenvalues by
//     bisection on Sturm counts (one thread per eigenvalue), each eigenvector
//     by one twisted-factorisation solve (T - lambda I) x = gamma_r e_r with r
//     = argmin |gamma_r| (the inverse-iteration step of Dhillon & Parlett's
//     MRRR, exact for the computed lambda).  This replaces the QR iteration
//     of the paper's library (and of the oracle): the same eigenvectors (up to
//     sign) by a method with one independent thread per eigenpair.
//  3. Back-transformation Z = H_0 ... H_{n-3} Y in binary64 with compact WY
//     panels (I - V T V^T, LAPACK slarft) on the DMMA GEMM, then Z rounded to
//     binary32 with its columns in descending eigenvalue order.
#include "mpj_device.cuh"
#include "mpj_internal.h"

#include <algorithm>
#include <cmath>

namespace mpj {

namespace {

constexpr int TB = 64;       // tile = panel width
constexpr int NTH = 256;     // threads per CTA (8 warps)
constexpr int RED = 2 * TB + 4;   // per-CTA partial slots: norm, quad, 2 x TB dots

struct SytrdArgs {
    float *A;            // n x n, ld (lower triangle is the live matrix)
    int64_t ld;
    int n, nt;           // size, tiles per dimension (ceil(n / 64))
    float *V, *W;        // panel vectors, ldp x TB each (rows >= n are zero)
    int64_t ldp;
    float *acol;         // 2 x ldp: the corrected current column (double-buffered)
    float *d, *e, *tau;
    float *Prow, *Pcol;  // partial vectors, (nt (nt + 1) / 2) x TB each
    float *red;          // G x RED per-CTA partials
    unsigned *bar;       // grid barrier (count, generation)
    int k0, ncols;       // panel start column and its number of reflector columns
};

// ---- grid barrier (all CTAs co-resident: cooperative launch) ---------------
__device__ __forceinline__ void grid_sync(unsigned *bar)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// sum of v over the CTA (all threads call; result in every thread)
__device__ __forceinline__ float cta_sum_f(float v, float *sh)
{
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    float r = 0.f;
    #pragma unroll
    for (int i = 0; i < NTH / 32; ++i) r += sh[i];
    __syncthreads();
    return r;
}

// lower-triangle tile list of the trailing tiles T0..nt-1, row-major
__device__ __forceinline__ void tile_of(int f, int T0, int &I, int &J)
{
    int r = (int)((sqrtf(8.0f * (float)f + 1.0f) - 1.0f) * 0.5f);
    while (r * (r + 1) / 2 > f) --r;
    while ((r + 1) * (r + 2) / 2 <= f) ++r;
    I = T0 + r;
    J = T0 + (f - r * (r + 1) / 2);
}
__device__ __forceinline__ int flat_of(int I, int J, int T0) { return (I - T0) * (I - T0 + 1) / 2 + (J - T0); }

// y_i of the symmetric product (after barrier 2): fixed-order sum of the
// partial vectors of row i's tile row (one per chunk segment: the tile list is
// cut into chunks of L tiles, a segment starts at J = T0 or at a chunk start)
// and of its tile column (one per tile, the diagonal tile's strict lower part
// included)
__device__ __forceinline__ float y_of(const SytrdArgs &a, int i, int T0, int L)
{
    const int I = i >> 6, r = i & 63;
    float y = 0.f;
    for (int J = T0; J <= I; ++J) {
        const int f = flat_of(I, J, T0);
        if (J == T0 || f % L == 0) y += a.Prow[(size_t)f * TB + r];
    }
    for (int K = I; K < a.nt; ++K) y += a.Pcol[(size_t)flat_of(K, I, T0) * TB + r];
    return y;
}

// v_i of column j's reflector (v_{j+1} = 1, v_i = a_i scal below, 0 above)
__device__ __forceinline__ float v_of(const float *acol, int i, int j, float scal)
{
    return i <= j ? 0.f : (i == j + 1 ? 1.f : acol[i] * scal);
}

__global__ void __launch_bounds__(NTH, 2) k_sytrd_panel(SytrdArgs a)
{
    __shared__ float sh[NTH / 32];
    __shared__ float dots[2 * TB];    // v^T V(:, t), v^T W(:, t) (reduced)
    __shared__ float rowbuf[NTH / 32][TB];
    __shared__ float wq[NTH / 32];
    __shared__ float vj[TB], wj[TB];  // row j of the panel's V and W (t < jj)
    __shared__ float wnext;           // row j+1 of the column just finished (recomputed)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    const int n = a.n;
    const int64_t ld = a.ld, ldp = a.ldp;
    float *myred = a.red + (size_t)cta * RED;

    for (int jj = 0; jj < a.ncols; ++jj) {
        const int j = a.k0 + jj;
        float *acol = a.acol + (size_t)(jj & 1) * ldp;
        // ------------------------------------------------------------ phase A
        // a_i = A(i, j) - sum_{t < jj} V(i,t) W(j,t) + W(i,t) V(j,t), rows i >= j.
        // Row j of column jj-1 (V = 1, W = wnext) was recomputed by this CTA in
        // phase C; rows of earlier columns are at least one barrier old.
        if (tid < jj) {
            const bool last = tid == jj - 1;
            vj[tid] = last ? 1.0f : a.V[j + (size_t)tid * ldp];
            wj[tid] = last ? wnext : a.W[j + (size_t)tid * ldp];
        }
        __syncthreads();
        float part = 0.f;
        if (tid < TB) {
            for (int I = cta; I * TB < n; I += G) {
                const int i = I * TB + tid;
                if (i < j || i >= n) continue;
                float x = a.A[i + (size_t)j * ld];
                for (int t = 0; t < jj; ++t) {
                    x = __fmaf_rn(-a.V[i + (size_t)t * ldp], wj[t], x);
                    x = __fmaf_rn(-a.W[i + (size_t)t * ldp], vj[t], x);
                }
                acol[i] = x;
                if (i >= j + 2) part = __fmaf_rn(x, x, part);
            }
        }
        part = cta_sum_f(part, sh);
        if (tid == 0) myred[0] = part;
        grid_sync(a.bar);
        // ------------------------------------------------------------ phase B
        float tau, scal;
        {
            float s = 0.f;
            for (int c = 0; c < G; ++c) s += a.red[(size_t)c * RED];    // fixed order: same in every CTA
            const float alpha = (j + 1 < n) ? acol[j + 1] : 0.f;
            float beta;
            if (s == 0.f) {
                beta = alpha; tau = 0.f; scal = 0.f;     // H = I
            } else {
                const float nrm = sqrtf(__fmaf_rn(alpha, alpha, s));
                beta = alpha >= 0.f ? -nrm : nrm;
                tau = (beta - alpha) / beta;
                scal = 1.0f / (alpha - beta);
            }
            if (cta == 0 && tid == 0) {
                a.d[j] = acol[j];
                a.e[j] = beta;
                a.tau[j] = tau;
            }
        }
        // y = A22 v over the lower tiles of A22 (rows / columns >= j+1)
        const int T0 = (j + 1) >> 6;
        const int mt = a.nt - T0;
        const int total = mt * (mt + 1) / 2;
        const int L = (total + G - 1) / G;
        const int f0 = cta * L, f1 = min(total, f0 + L);
        float q = 0.f;                         // this lane's share of v^T A22 v
        float yr0 = 0.f, yr1 = 0.f;            // row partials of the current tile row (rows 2 lane, 2 lane + 1)
        if (f0 < f1) {
            int I, J;
            tile_of(f0, T0, I, J);
            int curI = I, segf = f0;
            for (int f = f0; f <= f1; ++f) {
                if (f == f1 || I != curI) {
                    // combine the 8 warps' row partials of tile row curI into Prow[segf]
                    rowbuf[warp][2 * lane] = yr0;
                    rowbuf[warp][2 * lane + 1] = yr1;
                    __syncthreads();
                    if (tid < TB) {
                        float y = 0.f;
                        #pragma unroll
                        for (int w = 0; w < NTH / 32; ++w) y += rowbuf[w][tid];
                        a.Prow[(size_t)segf * TB + tid] = y;
                    }
                    __syncthreads();
                    yr0 = yr1 = 0.f;
                    if (f == f1) break;
                    curI = I; segf = f;
                }
                // this warp: columns c = 8 warp + u (u < 8) of tile (I, J); lane: rows 2 lane, 2 lane + 1
                const int r0 = I * TB + 2 * lane;
                const int cb = J * TB + 8 * warp;
                const float vi0 = v_of(acol, r0, j, scal), vi1 = v_of(acol, r0 + 1, j, scal);
                float2 x[8];
                #pragma unroll
                for (int u = 0; u < 8; ++u) x[u] = *reinterpret_cast<const float2 *>(a.A + r0 + (size_t)(cb + u) * ld);
                float cz[8];
                #pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int c = cb + u;
                    const float vc = v_of(acol, c, j, scal);
                    float x0 = x[u].x, x1 = x[u].y;
                    if (I == J) {                 // diagonal tile: the lower triangle r >= c only
                        const float y0 = r0 >= c ? x0 : 0.f, y1 = r0 + 1 >= c ? x1 : 0.f;
                        yr0 = __fmaf_rn(y0, vc, yr0);
                        yr1 = __fmaf_rn(y1, vc, yr1);
                        if (r0 == c) q = __fmaf_rn(y0 * vc, vc, q);          // A_cc v_c^2
                        if (r0 + 1 == c) q = __fmaf_rn(y1 * vc, vc, q);
                        x0 = r0 > c ? x0 : 0.f;                              // strict lower part transposed
                        x1 = r0 + 1 > c ? x1 : 0.f;
                    } else {
                        yr0 = __fmaf_rn(x0, vc, yr0);
                        yr1 = __fmaf_rn(x1, vc, yr1);
                    }
                    cz[u] = __fmaf_rn(x1, vi1, x0 * vi0);
                }
                // the 8 column sums over the warp's 32 lanes (transpose-reduce: 9 shuffles)
                {
                    const bool h4 = lane & 16;
                    #pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float got = __shfl_xor_sync(0xffffffffu, h4 ? cz[u] : cz[u + 4], 16);
                        cz[u] = (h4 ? cz[u + 4] : cz[u]) + got;
                    }
                    const bool h3 = lane & 8;
                    #pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const float got = __shfl_xor_sync(0xffffffffu, h3 ? cz[u] : cz[u + 2], 8);
                        cz[u] = (h3 ? cz[u + 2] : cz[u]) + got;
                    }
                    const bool h2 = lane & 4;
                    const float got = __shfl_xor_sync(0xffffffffu, h2 ? cz[0] : cz[1], 4);
                    cz[0] = (h2 ? cz[1] : cz[0]) + got;
                    cz[0] += __shfl_xor_sync(0xffffffffu, cz[0], 2);
                    cz[0] += __shfl_xor_sync(0xffffffffu, cz[0], 1);
                }
                if ((lane & 3) == 0) {
                    const int u = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
                    const float vc = v_of(acol, cb + u, j, scal);
                    q = __fmaf_rn(2.0f * cz[0], vc, q);   // A_IJ and its mirror A_JI (strict lower part if I == J)
                    a.Pcol[(size_t)f * TB + 8 * warp + u] = cz[0];
                }
                if (++J > I) { ++I; J = T0; }
            }
        }
        // v^T A22 v of this CTA
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
        if (lane == 0) wq[warp] = q;
        __syncthreads();
        if (tid == 0) {
            float qs = 0.f;
            #pragma unroll
            for (int w = 0; w < NTH / 32; ++w) qs += wq[w];
            myred[1] = qs;
        }
        // panel dot products v^T V(:, t), v^T W(:, t) (t < jj) over this CTA's rows
        for (int t = warp; t < 2 * jj; t += NTH / 32) {
            const float *col = (t < jj ? a.V + (size_t)t * ldp : a.W + (size_t)(t - jj) * ldp);
            float acc = 0.f;
            for (int I = cta; I * TB < n; I += G)
                for (int r = lane; r < TB; r += 32) {
                    const int i = I * TB + r;
                    if (i >= j + 1 && i < n) acc = __fmaf_rn(col[i], v_of(acol, i, j, scal), acc);
                }
            #pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) myred[2 + t] = acc;
        }
        grid_sync(a.bar);
        // ------------------------------------------------------------ phase C
        // the dots and v^T A22 v (fixed order: identical in every CTA)
        for (int t = tid; t < 2 * jj; t += NTH) {
            float s = 0.f;
            for (int c = 0; c < G; ++c) s += a.red[(size_t)c * RED + 2 + t];
            dots[t] = s;
        }
        if (tid == 0) {
            float s = 0.f;
            for (int c = 0; c < G; ++c) s += a.red[(size_t)c * RED + 1];
            wq[0] = s;
        }
        __syncthreads();
        // v^T p = tau (v^T A22 v - 2 sum_t (v^T V_t)(v^T W_t)); alpha' = -(tau/2) v^T p
        float vtp = wq[0];
        for (int t = 0; t < jj; ++t) vtp = __fmaf_rn(-2.0f * dots[t], dots[jj + t], vtp);
        vtp *= tau;
        const float alph = -0.5f * tau * vtp;
        // w_i = tau (y_i - V(i,:) (W^T v) - W(i,:) (V^T v)) + alpha' v_i  (rows i >= j+1)
        auto w_at = [&](int i) {
            float y = y_of(a, i, T0, L);
            for (int t = 0; t < jj; ++t) {
                y = __fmaf_rn(-a.V[i + (size_t)t * ldp], dots[jj + t], y);
                y = __fmaf_rn(-a.W[i + (size_t)t * ldp], dots[t], y);
            }
            return __fmaf_rn(alph, v_of(acol, i, j, scal), tau * y);
        };
        if (tid < TB) {
            for (int I = cta; I * TB < n; I += G) {
                const int i = I * TB + tid;
                if (i < j + 1 || i >= n) continue;
                const float vi = v_of(acol, i, j, scal);
                a.W[i + (size_t)jj * ldp] = w_at(i);
                a.V[i + (size_t)jj * ldp] = vi;
                if (i >= j + 2) a.A[i + (size_t)j * ld] = vi;     // reflector storage (LAPACK layout)
            }
        }
        if (tid == 0 && j + 1 < n) wnext = w_at(j + 1);         // row j+1, for the next column's phase A
        __syncthreads();
    }
    // ------------------------------------------------------------ trailing update
    // A(s0:, s0:) -= V W^T + W V^T on the lower tiles (s0 = first row / column
    // after the panel)
    grid_sync(a.bar);
    const int s0 = a.k0 + a.ncols;
    if (s0 >= n) return;
    const int T1 = s0 >> 6;
    const int mt = a.nt - T1;
    const int total = mt * (mt + 1) / 2;
    extern __shared__ __align__(16) float smem[];
    float *sVI = smem, *sWI = sVI + TB * TB, *sVJ = sWI + TB * TB, *sWJ = sVJ + TB * TB;   // [t][r]
    const int tr = (tid & 15) * 4, tc = (tid >> 4) * 4;
    const int nk = a.ncols;
    for (int f = cta; f < total; f += G) {
        int I, J;
        tile_of(f, T1, I, J);
        __syncthreads();
        for (int e = tid; e < TB * TB; e += NTH) {
            const int r = e & 63, t = e >> 6;
            const bool okt = t < nk;
            sVI[t * TB + r] = okt ? a.V[I * TB + r + (size_t)t * ldp] : 0.f;
            sWI[t * TB + r] = okt ? a.W[I * TB + r + (size_t)t * ldp] : 0.f;
            sVJ[t * TB + r] = okt ? a.V[J * TB + r + (size_t)t * ldp] : 0.f;
            sWJ[t * TB + r] = okt ? a.W[J * TB + r + (size_t)t * ldp] : 0.f;
        }
        __syncthreads();
        float acc[4][4];
        #pragma unroll
        for (int x = 0; x < 4; ++x)
            #pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = 0.f;
        for (int t = 0; t < nk; ++t) {
            const float4 vi = *reinterpret_cast<const float4 *>(sVI + t * TB + tr);
            const float4 wi = *reinterpret_cast<const float4 *>(sWI + t * TB + tr);
            const float4 vc = *reinterpret_cast<const float4 *>(sVJ + t * TB + tc);
            const float4 wc = *reinterpret_cast<const float4 *>(sWJ + t * TB + tc);
            const float avi[4] = {vi.x, vi.y, vi.z, vi.w}, awi[4] = {wi.x, wi.y, wi.z, wi.w};
            const float avj[4] = {vc.x, vc.y, vc.z, vc.w}, awj[4] = {wc.x, wc.y, wc.z, wc.w};
            #pragma unroll
            for (int x = 0; x < 4; ++x)
                #pragma unroll
                for (int y = 0; y < 4; ++y) {
                    acc[x][y] = __fmaf_rn(avi[x], awj[y], acc[x][y]);
                    acc[x][y] = __fmaf_rn(awi[x], avj[y], acc[x][y]);
                }
        }
        #pragma unroll
        for (int y = 0; y < 4; ++y) {
            const int c = J * TB + tc + y;
            #pragma unroll
            for (int x = 0; x < 4; ++x) {
                const int r = I * TB + tr + x;
                if (r >= s0 && c >= s0 && r < n && c < n) a.A[r + (size_t)c * ld] -= acc[x][y];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// 2. the tridiagonal (d, e) in binary64
// ---------------------------------------------------------------------------
constexpr double kOmega = 1.1102230246251565e-16;

// d64, e2 (e_i^2, 0 where the matrix splits), bstart / bend (inclusive) of the
// unreduced block of each row, pivmin.  One CTA.
__global__ void __launch_bounds__(1024) k_tri_prep(const float *__restrict__ d, const float *__restrict__ e, int n,
                                                   double *d64, double *e64, double *e2, int *bstart, int *bend,
                                                   double *pivmin)
{
    __shared__ int sc[1024];
    __shared__ double smax[1024];
    const int tid = threadIdx.x, nth = blockDim.x;
    const int per = (n + nth - 1) / nth;
    const int i0 = tid * per, i1 = min(n, i0 + per);
    double emax = 0.0;
    for (int i = i0; i < i1; ++i) {
        d64[i] = (double)d[i];
        if (i + 1 < n) {
            const double ei = (double)e[i];
            const bool split = fabs(ei) <= kOmega * sqrt(fabs((double)d[i]) * fabs((double)d[i + 1]));
            e64[i] = split ? 0.0 : ei;
            e2[i] = split ? 0.0 : ei * ei;
            emax = fmax(emax, e2[i]);
        } else {
            e64[i] = 0.0;
            e2[i] = 0.0;
        }
    }
    __syncthreads();   // e2 of the neighbouring chunk is read below
    // block starts: inclusive max-scan of "row i starts a block" positions
    int last = -1;
    for (int i = i0; i < i1; ++i) if (i == 0 || e2[i - 1] == 0.0) last = i;
    sc[tid] = last;
    smax[tid] = emax;
    __syncthreads();
    for (int o = 1; o < nth; o <<= 1) {
        const int v = tid >= o ? sc[tid - o] : -1;
        const double m = tid >= o ? smax[tid - o] : 0.0;
        __syncthreads();
        sc[tid] = max(sc[tid], v);
        smax[tid] = fmax(smax[tid], m);
        __syncthreads();
    }
    int cur = tid > 0 ? sc[tid - 1] : -1;
    for (int i = i0; i < i1; ++i) {
        if (i == 0 || e2[i - 1] == 0.0) cur = i;
        bstart[i] = cur;
    }
    if (tid == nth - 1) pivmin[0] = 2.2250738585072014e-308 * fmax(1.0, smax[tid]);
    __syncthreads();
    // block ends: the same scan from the right
    int first = 1 << 30;
    for (int i = i1 - 1; i >= i0; --i) if (i == n - 1 || e2[i] == 0.0) first = i;
    sc[tid] = first;
    __syncthreads();
    for (int o = 1; o < nth; o <<= 1) {
        const int v = tid + o < nth ? sc[tid + o] : (1 << 30);
        __syncthreads();
        sc[tid] = min(sc[tid], v);
        __syncthreads();
    }
    cur = tid + 1 < nth ? sc[tid + 1] : (1 << 30);
    for (int i = i1 - 1; i >= i0; --i) {
        if (i == n - 1 || e2[i] == 0.0) cur = i;
        bend[i] = cur;
    }
}

// number of eigenvalues < x of the unreduced block [s, e] (Sturm count)
__device__ __forceinline__ int sturm_count(const double *__restrict__ d, const double *__restrict__ e2, int s, int e,
                                           double x, double pivmin)
{
    double q = d[s] - x;
    if (fabs(q) <= pivmin) q = -pivmin;
    int cnt = q < 0.0;
    for (int i = s + 1; i <= e; ++i) {
        q = (d[i] - x) - __ddiv_rn(e2[i - 1], q);
        if (fabs(q) <= pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

// thread t: the (t - bstart)-th smallest eigenvalue of its block, by bisection
__global__ void k_tri_bisect(const double *__restrict__ d, const double *__restrict__ e64,
                             const double *__restrict__ e2, const int *__restrict__ bstart,
                             const int *__restrict__ bend, const double *__restrict__ pivmin_p, int n,
                             double *lam)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int s = bstart[t], e = bend[t], k = t - s;
    const double pivmin = pivmin_p[0];
    if (s == e) { lam[t] = d[s]; return; }
    double lo = 1e308, hi = -1e308;
    for (int i = s; i <= e; ++i) {
        const double r = (i > s ? fabs(e64[i - 1]) : 0.0) + (i < e ? fabs(e64[i]) : 0.0);
        lo = fmin(lo, d[i] - r);
        hi = fmax(hi, d[i] + r);
    }
    const double pad = 2.0 * kOmega * fmax(fabs(lo), fabs(hi)) + pivmin;
    lo -= pad;
    hi += pad;
    for (int it = 0; it < 80; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        if (sturm_count(d, e2, s, e, mid, pivmin) > k) hi = mid;
        else lo = mid;
    }
    lam[t] = 0.5 * (lo + hi);
}

// thread t: eigenvector of lam[t] on its block by the twisted factorisation
// T - lam I = N_r Delta_r N_r^T (forward D+, backward D-), r = argmin |gamma_r|,
// x_r = 1: x_i = -(e_i / D+_i) x_{i+1} above r, x_{i+1} = -(e_i / D-_{i+1}) x_i
// below.  Column t of Y (ld ldy, zero outside the block) gets x / ||x||.
__global__ void k_tri_twisted(const double *__restrict__ d, const double *__restrict__ e64,
                              const double *__restrict__ e2, const int *__restrict__ bstart,
                              const int *__restrict__ bend, const double *__restrict__ pivmin_p,
                              const double *__restrict__ lam, int n, double *Dp, double *Dm, double *Y,
                              int64_t ldy)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int s = bstart[t], e = bend[t];
    double *y = Y + (size_t)t * ldy;
    if (s == e) { y[s] = 1.0; return; }
    const double pivmin = pivmin_p[0], l = lam[t];
    auto guard = [&](double q) { return fabs(q) < pivmin ? (q < 0.0 ? -pivmin : pivmin) : q; };
    // forward
    double q = guard(d[s] - l);
    Dp[(size_t)s * n + t] = q;
    for (int i = s + 1; i <= e; ++i) {
        q = guard((d[i] - l) - __ddiv_rn(e2[i - 1], q));
        Dp[(size_t)i * n + t] = q;
    }
    // backward, with gamma_i = D+_i + D-_i - (d_i - lam)
    q = guard(d[e] - l);
    Dm[(size_t)e * n + t] = q;
    int r = e;
    double gbest = fabs(Dp[(size_t)e * n + t] + q - (d[e] - l));
    for (int i = e - 1; i >= s; --i) {
        q = guard((d[i] - l) - __ddiv_rn(e2[i], q));
        Dm[(size_t)i * n + t] = q;
        const double g = fabs(Dp[(size_t)i * n + t] + q - (d[i] - l));
        if (g < gbest) { gbest = g; r = i; }
    }
    // solve
    double nrm = 1.0, x = 1.0;
    y[r] = 1.0;
    for (int i = r - 1; i >= s; --i) {
        x = -__ddiv_rn(e64[i], Dp[(size_t)i * n + t]) * x;
        y[i] = x;
        nrm = __fma_rn(x, x, nrm);
    }
    x = 1.0;
    for (int i = r; i < e; ++i) {
        x = -__ddiv_rn(e64[i], Dm[(size_t)(i + 1) * n + t]) * x;
        y[i + 1] = x;
        nrm = __fma_rn(x, x, nrm);
    }
    const double inv = 1.0 / sqrt(nrm);
    for (int i = s; i <= e; ++i) y[i] *= inv;
}

// rank of lam[t] in descending order (ties by index: stable)
__global__ void k_rank_lam(const double *__restrict__ lam, int n, int *rank)
{
    __shared__ double sl[1024];
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const double lt = t < n ? lam[t] : 0.0;
    int r = 0;
    for (int b0 = 0; b0 < n; b0 += 1024) {
        __syncthreads();
        for (int u = threadIdx.x; u < 1024; u += blockDim.x) sl[u] = b0 + u < n ? lam[b0 + u] : 0.0;
        __syncthreads();
        const int m = min(1024, n - b0);
        for (int u = 0; u < m; ++u) {
            const double lu = sl[u];
            r += (lu > lt) || (lu == lt && b0 + u < t);
        }
    }
    if (t < n) rank[t] = r;
}

// ---------------------------------------------------------------------------
// 3. back-transformation
// ---------------------------------------------------------------------------
// Vp (rows r0 = k0+1 .. n-1, ldv) of the reflectors j = k0 .. k0+nr-1 (column t
// = j - k0): 0 above row j+1, 1 at j+1, the stored v below; zero for t >= nr.
__global__ void k_build_vp(const float *__restrict__ A, int64_t lda, int n, int k0, int nr, double *Vp, int64_t ldv)
{
    const int t = blockIdx.y;
    const int r0 = k0 + 1;
    const int j = k0 + t;
    for (int i = r0 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double v = 0.0;
        if (t < nr) v = i < j + 1 ? 0.0 : (i == j + 1 ? 1.0 : (double)A[i + (size_t)j * lda]);
        Vp[(i - r0) + (size_t)t * ldv] = v;
    }
}

// Tp (64 x 64, ld 64) of H_k0 ... H_{k0+nr-1} = I - Vp Tp Vp^T (LAPACK dlarft,
// forward, columnwise) from the Gram matrix G = Vp^T Vp (ld 64).  One CTA.
__global__ void k_build_tp(const double *__restrict__ G, const float *__restrict__ tau, int k0, int nr, double *Tp)
{
    __shared__ double T[TB * TB];
    __shared__ double z[TB];
    const int tid = threadIdx.x;
    for (int e = tid; e < TB * TB; e += blockDim.x) T[e] = 0.0;
    __syncthreads();
    for (int t = 0; t < nr; ++t) {
        const double ta = (double)tau[k0 + t];
        // z = -tau_t Vp(:, 0:t)^T v_t = -tau_t G(0:t, t)
        if (tid < t) z[tid] = -ta * G[tid + t * TB];
        __syncthreads();
        // T(0:t, t) = T(0:t, 0:t) z
        if (tid < t) {
            double acc = 0.0;
            for (int u = tid; u < t; ++u) acc = __fma_rn(T[tid + u * TB], z[u], acc);
            T[tid + t * TB] = acc;
        }
        if (tid == 0) T[t + t * TB] = ta;
        __syncthreads();
    }
    for (int e = tid; e < TB * TB; e += blockDim.x) Tp[e] = T[e];
}

// V32(:, rank[t]) = fl32(Z(:, t))
__global__ void k_round_perm(const double *__restrict__ Z, int64_t ldz, int n, const int *__restrict__ rank,
                             float *Z32, int64_t ld32)
{
    const int t = blockIdx.y;
    const int rt = rank[t];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        Z32[i + (size_t)rt * ld32] = (float)Z[i + (size_t)t * ldz];
}

// Y(:, rank[t]) = Yb(:, t), lam_out[rank[t]] = lam[t]
__global__ void k_perm_cols(const double *__restrict__ Yb, int64_t ldb, int n, const int *__restrict__ rank,
                            const double *__restrict__ lam, double *Y, int64_t ldy, double *lam_out)
{
    const int t = blockIdx.y;
    const int rt = rank[t];
    if (blockIdx.x == 0 && threadIdx.x == 0) lam_out[rt] = lam[t];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        Y[i + (size_t)rt * ldy] = Yb[i + (size_t)t * ldb];
}

// tail of the reduction: the last 2 x 2 block after the last panel
__global__ void k_tri_tail(const float *__restrict__ A, int64_t lda, int n, float *d, float *e, float *tau)
{
    if (threadIdx.x != 0) return;
    const int j0 = n >= 2 ? n - 2 : 0;
    for (int j = j0; j < n; ++j) { d[j] = A[j + (size_t)j * lda]; tau[j] = 0.f; }
    if (n >= 2) e[n - 2] = A[(n - 1) + (size_t)(n - 2) * lda];
}

int coop_ctas()
{
    static int g = 0;
    if (!g) {
        int dev = 0, sms = 148, occ = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const size_t smem = 4 * TB * TB * sizeof(float);
        cudaFuncSetAttribute(k_sytrd_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sytrd_panel, NTH, smem);
        g = sms * std::max(1, std::min(occ, 2));
    }
    return g;
}

}  // namespace

// ---------------------------------------------------------------------------
// workspace and driver
// ---------------------------------------------------------------------------
struct SymqrWs {
    float *V, *W, *acol, *d, *e, *tau, *Prow, *Pcol, *red;
    unsigned *bar;
    double *d64, *e64, *e2, *lam, *piv, *Vp, *Gm, *Tp, *W1, *W2, *skw;
    int *bstart, *bend, *rank;
    size_t skw_elems;
};

static size_t carve_symqr(char *base, int64_t np, SymqrWs &w)
{
    size_t off = 0;
    auto take = [&](size_t bytes) -> void * {
        off = (off + 255) & ~(size_t)255;
        void *p = base ? base + off : nullptr;
        off += bytes;
        return p;
    };
    const int64_t nt = (np + TB - 1) / TB;
    const size_t ntiles = (size_t)nt * (nt + 1) / 2;
    const int G = 2 * 160;   // upper bound on the cooperative grid
    w.V = (float *)take(np * TB * 4);
    w.W = (float *)take(np * TB * 4);
    w.acol = (float *)take(2 * np * 4);
    w.d = (float *)take(np * 4);
    w.e = (float *)take(np * 4);
    w.tau = (float *)take(np * 4);
    w.Prow = (float *)take(ntiles * TB * 4);
    w.Pcol = (float *)take(ntiles * TB * 4);
    w.red = (float *)take((size_t)G * RED * 4);
    w.bar = (unsigned *)take(64);
    w.d64 = (double *)take(np * 8);
    w.e64 = (double *)take(np * 8);
    w.e2 = (double *)take(np * 8);
    w.lam = (double *)take(np * 8);
    w.piv = (double *)take(64);
    w.bstart = (int *)take(np * 4);
    w.bend = (int *)take(np * 4);
    w.rank = (int *)take(np * 4);
    w.Vp = (double *)take(np * TB * 8);
    w.Gm = (double *)take(TB * TB * 8);
    w.Tp = (double *)take(TB * TB * 8);
    w.W1 = (double *)take(np * TB * 8);
    w.W2 = (double *)take(np * TB * 8);
    w.skw_elems = (size_t)8 * TB * np;
    w.skw = (double *)take(w.skw_elems * 8);
    return off + 256;
}

size_t symqr_workspace(int64_t np)
{
    SymqrWs w;
    return carve_symqr(nullptr, np, w);
}

// 1. binary32 tridiagonalisation of A32 (n x n, lda; overwritten by the
// reflectors): d, e, tau in the workspace
static mpj_status sytrd_run(float *A32, int64_t lda, int n, SymqrWs &w, int64_t np, cudaStream_t st)
{
    const int nt = (int)(np / TB);
    const int G = coop_ctas();
    const size_t smem = 4 * TB * TB * sizeof(float);
    MPJ_CK(cudaMemsetAsync(w.bar, 0, 64, st));
    MPJ_CK(cudaMemsetAsync(w.acol, 0, 2 * np * 4, st));
    MPJ_CK(cudaMemsetAsync(w.d, 0, np * 4, st));
    MPJ_CK(cudaMemsetAsync(w.e, 0, np * 4, st));
    MPJ_CK(cudaMemsetAsync(w.tau, 0, np * 4, st));
    const int ncolumns = n - 2;    // reflector columns 0 .. n-3
    SytrdArgs a;
    a.A = A32; a.ld = lda; a.n = n; a.nt = nt; a.V = w.V; a.W = w.W; a.ldp = np; a.acol = w.acol;
    a.d = w.d; a.e = w.e; a.tau = w.tau; a.Prow = w.Prow; a.Pcol = w.Pcol; a.red = w.red; a.bar = w.bar;
    for (int k0 = 0; k0 < ncolumns; k0 += TB) {
        a.k0 = k0;
        a.ncols = std::min(TB, ncolumns - k0);
        MPJ_CK(cudaMemsetAsync(w.V, 0, np * TB * 4, st));
        MPJ_CK(cudaMemsetAsync(w.W, 0, np * TB * 4, st));
        void *args[] = {&a};
        MPJ_CK(cudaLaunchCooperativeKernel((const void *)k_sytrd_panel, dim3(G), dim3(NTH), args, smem, st));
        count_launch();
    }
    k_tri_tail<<<1, 32, 0, st>>>(A32, lda, n, w.d, w.e, w.tau);
    count_launch();
    return MPJ_OK;
}

// 2. eigenpairs of the tridiagonal (w.d, w.e): w.lam (block order), w.rank
// (descending rank), Y (n x n, ldy) the unit eigenvectors in block order
static mpj_status tri_eig_run(int n, SymqrWs &w, double *Y, int64_t ldy, double *Dp, double *Dm, cudaStream_t st)
{
    k_tri_prep<<<1, 1024, 0, st>>>(w.d, w.e, n, w.d64, w.e64, w.e2, w.bstart, w.bend, w.piv);
    k_tri_bisect<<<(n + 127) / 128, 128, 0, st>>>(w.d64, w.e64, w.e2, w.bstart, w.bend, w.piv, n, w.lam);
    MPJ_CK(cudaMemset2DAsync(Y, ldy * 8, 0, (size_t)n * 8, n, st));
    k_tri_twisted<<<(n + 127) / 128, 128, 0, st>>>(w.d64, w.e64, w.e2, w.bstart, w.bend, w.piv, w.lam, n, Dp, Dm, Y,
                                                    ldy);
    k_rank_lam<<<(n + 255) / 256, 256, 0, st>>>(w.lam, n, w.rank);
    count_launch(4);
    return MPJ_OK;
}

// 3. Y <- H_0 ... H_{n-3} Y (panels from the last to the first)
static mpj_status backtransform_run(const float *A32, int64_t lda, int n, SymqrWs &w, int64_t np, double *Y,
                                    int64_t ldy, cudaStream_t st)
{
    const int ncolumns = n - 2;
    for (int k0 = ((ncolumns - 1) / TB) * TB; ncolumns > 0 && k0 >= 0; k0 -= TB) {
        const int nr = std::min(TB, ncolumns - k0);
        const int r0 = k0 + 1, m = n - r0;
        k_build_vp<<<dim3((m + 255) / 256 > 32 ? 32 : (m + 255) / 256, TB), 256, 0, st>>>(A32, lda, n, k0, nr, w.Vp,
                                                                                          np);
        count_launch();
        launch_dgemm(true, false, TB, TB, m, 1.0, w.Vp, np, w.Vp, np, 0.0, w.Gm, TB, st, w.skw, w.skw_elems);
        k_build_tp<<<1, TB, 0, st>>>(w.Gm, w.tau, k0, nr, w.Tp);
        count_launch();
        launch_dgemm(true, false, TB, n, m, 1.0, w.Vp, np, Y + r0, ldy, 0.0, w.W1, TB, st, w.skw, w.skw_elems);
        launch_dgemm(false, false, TB, n, TB, 1.0, w.Tp, TB, w.W1, TB, 0.0, w.W2, TB, st);
        launch_dgemm(false, false, m, n, TB, -1.0, w.Vp, np, w.W2, TB, 1.0, Y + r0, ldy, st);
    }
    MPJ_CK(cudaGetLastError());
    return MPJ_OK;
}

static int64_t pad64(int64_t n) { return ((n + TB - 1) / TB) * TB; }

// Alg. 3 step 1 by "symmetric QR" (reading R12'): A32 (n x n, ld lda, binary32,
// symmetric; overwritten by the reduction) -> Z32 (n x n, ld ldz, columns in
// descending eigenvalue order).  Scratch: Y (fp64, ld ldy, >= n columns; holds
// Z in fp64, block order, on return), Dp, Dm (fp64, >= n x n each).
mpj_status low_evd_symqr(float *A32, int64_t lda, int n, float *Z32, int64_t ldz, double *Y, int64_t ldy,
                         double *Dp, double *Dm, void *ws, cudaStream_t st)
{
    if (n < 1) return MPJ_OK;
    const int64_t np = pad64(n);
    SymqrWs w;
    carve_symqr((char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255), np, w);
    MPJ_TRY(sytrd_run(A32, lda, n, w, np, st));
    MPJ_TRY(tri_eig_run(n, w, Y, ldy, Dp, Dm, st));
    MPJ_TRY(backtransform_run(A32, lda, n, w, np, Y, ldy, st));
    k_round_perm<<<dim3((n + 255) / 256 > 32 ? 32 : (n + 255) / 256, n), 256, 0, st>>>(Y, ldy, n, w.rank, Z32, ldz);
    count_launch();
    MPJ_CK(cudaGetLastError());
    return MPJ_OK;
}

// the stages alone, for the stage-level parity tests (C ABI below)
mpj_status sytrd_stage(float *A32, int64_t lda, int n, float *d, float *e, float *tau, cudaStream_t st)
{
    const int64_t np = pad64(n);
    void *ws = nullptr;
    MPJ_CK(cudaMallocAsync(&ws, symqr_workspace(np), st));
    SymqrWs w;
    carve_symqr((char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255), np, w);
    mpj_status s = sytrd_run(A32, lda, n, w, np, st);
    if (s == MPJ_OK) {
        MPJ_CK(cudaMemcpyAsync(d, w.d, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
        if (n > 1) MPJ_CK(cudaMemcpyAsync(e, w.e, (size_t)(n - 1) * 4, cudaMemcpyDeviceToDevice, st));
        MPJ_CK(cudaMemcpyAsync(tau, w.tau, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    }
    cudaFreeAsync(ws, st);
    return s;
}

mpj_status tridiag_eig_stage(const float *d, const float *e, int n, double *lam, double *Y, int64_t ldy,
                             cudaStream_t st)
{
    const int64_t np = pad64(n);
    void *ws = nullptr;
    double *scr = nullptr;
    MPJ_CK(cudaMallocAsync(&ws, symqr_workspace(np), st));
    MPJ_CK(cudaMallocAsync(&scr, (size_t)3 * n * n * sizeof(double), st));
    SymqrWs w;
    carve_symqr((char *)(((uintptr_t)ws + 255) & ~(uintptr_t)255), np, w);
    MPJ_CK(cudaMemcpyAsync(w.d, d, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    if (n > 1) MPJ_CK(cudaMemcpyAsync(w.e, e, (size_t)(n - 1) * 4, cudaMemcpyDeviceToDevice, st));
    double *Yb = scr, *Dp = scr + (size_t)n * n, *Dm = Dp + (size_t)n * n;
    mpj_status s = tri_eig_run(n, w, Yb, n, Dp, Dm, st);
    if (s == MPJ_OK) {
        k_perm_cols<<<dim3((n + 255) / 256 > 32 ? 32 : (n + 255) / 256, n), 256, 0, st>>>(Yb, n, n, w.rank, w.lam,
                                                                                          Y, ldy, lam);
        count_launch();
    }
    cudaFreeAsync(scr, st);
    cudaFreeAsync(ws, st);
    MPJ_CK(cudaGetLastError());
    return s;
}

}  // namespace mpj

extern "C" {

mpj_status mpjacobi_sytrd(float *A, int64_t n, int64_t lda, float *d, float *e, float *tau, void *stream)
{
    mpj::set_error("");
    if (n < 1 || lda < n || !A || !d || !tau || (n > 1 && !e) || n > (1 << 20)) {
        mpj::set_error("mpjacobi_sytrd: invalid argument");
        return MPJ_ERR_INVALID;
    }
    if (lda % 2) {   // the panel kernel reads float2 pairs of rows
        mpj::set_error("mpjacobi_sytrd: lda must be even");
        return MPJ_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    mpj_status s = mpj::sytrd_stage(A, lda, (int)n, d, e, tau, st);
    if (s == MPJ_OK && cudaStreamSynchronize(st) != cudaSuccess) {
        mpj::set_error("mpjacobi_sytrd: CUDA error");
        return MPJ_ERR_CUDA;
    }
    return s;
}

mpj_status mpjacobi_tridiag_eig(const float *d, const float *e, int64_t n, double *lam, double *Y, int64_t ldy,
                                void *stream)
{
    mpj::set_error("");
    if (n < 1 || ldy < n || !d || !lam || !Y || (n > 1 && !e) || n > (1 << 16)) {
        mpj::set_error("mpjacobi_tridiag_eig: invalid argument");
        return MPJ_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    mpj_status s = mpj::tridiag_eig_stage(d, e, (int)n, lam, Y, ldy, st);
    if (s == MPJ_OK && cudaStreamSynchronize(st) != cudaSuccess) {
        mpj::set_error("mpjacobi_tridiag_eig: CUDA error");
        return MPJ_ERR_CUDA;
    }
    return s;
}

}  // extern "C"
