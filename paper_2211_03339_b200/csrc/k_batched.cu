// k_batched.cu -- batched Alg. 3 for many small matrices, one
// matrix per CTA, everything in shared memory (SURVEY §8(a) row a11,
// BASELINE config 3: 4096 x n = 64).
//
// Per CTA (n <= 64, padded to 64 with zero rows/columns, reading R2):
//   a0  As = (A + A^T)/2, ||As||_F
//   a1  the binary32 eigendecomposition Z of fl32(As): by default symmetric
//       QR (reading R12': k_batched_symqr below); with
//       low_solver = MPJ_LOW_JACOBI fp32 sweeps with V32 = I (reading R12):
//       the ordering for n_p = 64, b = 32 is one block round (31 intra + 32
//       cross rounds, R1), run by inner_rounds_b<> (U in registers)
//   a2  Q = CGS2(fp64(Z)) (reading R10), column by column in shared memory,
//       dot products by warp-shuffle reductions
//   a3  T = Q^T As Q on the FP64 tensor pipe (two 64^3 DMMA tile products),
//       symmetrised (R11)
//   a4-a8 fp64 sweeps on T with V = Q, stop test ||off(T)||_F <= eps ||As||_F
//       (inner_rounds_pipe: the next round's parameters computed by one warp
//       while the other seven apply the current round out of place)
//   a10 lambda = diag(T) stable-descending, V's columns alike.
// a1 runs as its own kernel (k_batched_symqr: 49 KB of shared memory -> 4
// CTAs per SM; k_batched_low: T32 and V32 only, 35 KB -> 5 CTAs per SM); the
// rest (a0, a2-a10) in k_batched_evd: two
// 64 x 68 fp64 panels (70 KB; As is re-formed from A for a3) -> 3 CTAs per SM.
#include "mpj_block.cuh"
#include "mpj_device.cuh"
#include "mpj_internal.h"

#include <algorithm>
#include <map>
#include <mutex>

namespace mpj {
namespace {

using namespace blk;

struct BatchedArgs {
    const double *A;
    int n;
    float *Z;                 // fp32 stage output: V32 per matrix (64 x 64, ld 64)
    double *lam, *V;
    int *sweeps, *sweeps_low, *flag;
    const int2 *lsched;
    double eps, nu, eps_low, nu_low;
    int max_sweeps, max_sweeps_low, rule;
};

// sum over the CTA of v (all threads call); result broadcast to every thread
__device__ __forceinline__ double cta_sum(double v, double *red)
{
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double r = 0.0;
    #pragma unroll
    for (int i = 0; i < NT / 32; ++i) r += red[i];
    return r;
}

template <typename R, int LD = Lay<R>::LD>
__device__ __forceinline__ double sq_norm(const R *M, bool offdiag, double *red)
{
    double acc = 0.0;
    for (int e = threadIdx.x; e < TW * TW; e += NT) {
        const int i = e & (TW - 1), j = e >> 6;
        if (offdiag && i == j) continue;
        const double x = (double)M[i + j * LD];
        acc = __fma_rn(x, x, acc);
    }
    return cta_sum(acc, red);
}

// a1 as its own kernel: the fp32 stage needs only T32 and V32 (35 KB of
// shared memory -> 6 matrices per SM instead of the 2 of the fp64 kernel); it
// is ~80% of a matrix's inner rounds, which are latency bound, so concurrency
// is what speeds it up.  Writes V32 (and the low sweep count).
__global__ void __launch_bounds__(NT, 5) k_batched_low(BatchedArgs a)
{
    constexpr int LF = LayK<float>::LD;      // odd: conflict-free mirrored stores in the rounds
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *T32 = (float *)smem_raw, *V32 = T32 + TW * LF;
    __shared__ double red[NT / 32];
    __shared__ InnerSharedB sh;
    __shared__ InnerParams<float> pf;
    const int n = a.n, tid = threadIdx.x;
    const size_t mat = blockIdx.x;
    const double *Ag = a.A + mat * (size_t)n * n;
    const int2 bp = make_int2(0, 1);
    // T32 = fl32((A + A^T) / 2) (the fp64 symmetrisation of a0, then rounded)
    for (int e = tid; e < TW * TW; e += NT) {
        const int i = e & (TW - 1), j = e >> 6;
        const double x = (i < n && j < n) ? (Ag[i + (size_t)j * n] + Ag[j + (size_t)i * n]) * 0.5 : 0.0;
        T32[i + j * LF] = (float)x;
        V32[i + j * LF] = (i == j && i < n) ? 1.0f : 0.0f;
    }
    __syncthreads();
    const double nA32 = sqrt(sq_norm<float, LF>(T32, false, red));
    const double tol_low = a.eps_low * nA32;
    int swl = 0;
    for (; isfinite(nA32);) {               // non-finite input: flagged by k_batched_evd
        const double off = sqrt(sq_norm<float, LF>(T32, true, red));
        if (off <= tol_low || swl >= a.max_sweeps_low) break;
        ++swl;
        inner_rounds_b<float, LF>(T32, V32, true, a.lsched, (float)a.nu_low, a.rule, sh, pf);
    }
    float *Zg = a.Z + mat * (size_t)n * n;
    for (int e = tid; e < TW * TW; e += NT) {
        const int i = e & (TW - 1), j = e >> 6;
        if (i < n && j < n) Zg[i + j * n] = V32[i + j * LF];
    }
    if (tid == 0 && a.sweeps_low) a.sweeps_low[mat] = swl;
}

// ---------------------------------------------------------------------------
// a1 by symmetric QR in low precision (reading R12'), one matrix per
// CTA -- the single-matrix path's three stages (k_tridiag.cu) collapsed into
// shared memory for n <= 64:
//   S  binary32 Householder tridiagonalisation (LAPACK ssytd2, lower: H =
//      I - tau v v^T, v(0) = 1, beta = -sign(alpha) ||x||), 3 barriers per
//      column: reflector (warp 0); p = tau A22 v (4 threads per row) with the
//      partial sums of p^T v; A22 -= v w^T + w v^T, w = p - (tau/2)(p^T v) v
//      formed inline;
//   T  the tridiagonal (d, e) in binary64: splits where |e_i| <= omega
//      sqrt(|d_i d_{i+1}|), each eigenvalue by multisection on its unreduced
//      block (Sturm counts at 2 points per round, one lane each) to 2 omega
//      of max(|lambda|, Gershgorin bound), its eigenvector by the twisted
//      factorisation N_r D_r N_r^T (r = argmin |gamma_r|, x_r = 1), two
//      lanes per eigenvalue; divisions as reciprocal seed + two Newton steps
//      (rcp_nr);
//   B  Z = H_0 ... H_{n-3} X in binary64, each 4-thread group holding one
//      column of X in registers (no barrier per reflector), rounded to
//      binary32, columns in descending eigenvalue order.
// Shared memory: A (64 x 65 fp32) + X (64 x 64 fp64, row-major x_i^(t)) =
// 49 KB -> 4 CTAs per SM.
// ---------------------------------------------------------------------------
#ifndef MPJ_BATCHED_MS
#define MPJ_BATCHED_MS 2   // lanes per eigenvalue in the batched multisection (A/B builds)
#endif
constexpr int LAQ = 65;
constexpr size_t kSymqrSmem = (size_t)TW * LAQ * sizeof(float) + (size_t)TW * TW * sizeof(double);

// 1 / q to about one ulp: the MUFU reciprocal seed and two Newton steps
// (2^-23 -> 2^-46 -> rounding); q is never 0 or subnormal here (pivmin guard).
// Not correctly rounded -- the Sturm counts and twisted factorisations stay
// backward stable with a few-ulp relative perturbation of e_i^2 per step.
__device__ __forceinline__ double rcp_nr(double q)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double e = __fma_rn(-q, r, 1.0);
    r = __fma_rn(r, e, r);
    e = __fma_rn(-q, r, 1.0);
    return __fma_rn(r, e, r);
}

// number of eigenvalues < x of the unreduced block [s, e] (Sturm count)
__device__ __forceinline__ int sturm_cnt(const double *__restrict__ d, const double *__restrict__ e2, int s, int e,
                                         double x, double pivmin)
{
    double q = d[s] - x;
    if (fabs(q) <= pivmin) q = -pivmin;
    int cnt = q < 0.0;
    #pragma unroll 4
    for (int i = s + 1; i <= e; ++i) {
        q = __fma_rn(-e2[i - 1], rcp_nr(q), d[i] - x);
        if (fabs(q) <= pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

__global__ void __launch_bounds__(NT, 4) k_batched_symqr(BatchedArgs a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *X = (double *)smem_raw;                          // X[i * 64 + t]
    float *A = (float *)(X + TW * TW);                       // A[i + j * LAQ]
    __shared__ float tauv[TW], vv[TW], pp[TW];
    __shared__ float red[NT / 32];
    __shared__ double d64[TW], e64[TW], e2[TW], lam[TW], inrm[TW];
    __shared__ int bs[TW], be[TW], rnk[TW];
    __shared__ double pivmin_s;
    const int n = a.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t mat = blockIdx.x;
    const double *Ag = a.A + mat * (size_t)n * n;
    float *Zg = a.Z + mat * (size_t)n * n;

    // A = fl32((A + A^T) / 2), zero padded
    int nonfinite = 0;
    for (int e = tid; e < TW * TW; e += NT) {
        const int i = e & (TW - 1), j = e >> 6;
        double x = 0.0;
        if (i < n && j < n) {
            x = (Ag[i + (size_t)j * n] + Ag[j + (size_t)i * n]) * 0.5;
            nonfinite |= !isfinite(x);
        }
        A[i + j * LAQ] = (float)x;
    }
    if (__syncthreads_or(nonfinite)) {
        if (tid == 0) atomicOr(a.flag, 4);
        for (int e = tid; e < n * n; e += NT) Zg[e] = 0.f;
        return;
    }

    // S: tridiagonalisation
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1;
        if (warp == 0) {
            const float x0 = A[(k + 1) + k * LAQ];
            const float x1 = (1 + lane < m) ? A[(k + 1 + 1 + lane) + k * LAQ] : 0.f;
            const float x2 = (33 + lane < m) ? A[(k + 1 + 33 + lane) + k * LAQ] : 0.f;
            float s = __fmaf_rn(x2, x2, x1 * x1);
            #pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            float beta, t, scal;
            if (s == 0.f) { beta = x0; t = 0.f; scal = 0.f; }
            else {
                const float nrm = sqrtf(__fmaf_rn(x0, x0, s));
                beta = x0 >= 0.f ? -nrm : nrm;
                t = (beta - x0) / beta;
                scal = 1.0f / (x0 - beta);
            }
            if (1 + lane < m) { const float v = x1 * scal; vv[1 + lane] = v; A[(k + 2 + lane) + k * LAQ] = v; }
            if (33 + lane < m) { const float v = x2 * scal; vv[33 + lane] = v; A[(k + 34 + lane) + k * LAQ] = v; }
            if (lane == 0) { vv[0] = 1.f; tauv[k] = t; A[(k + 1) + k * LAQ] = beta; }
        }
        __syncthreads();
        const float t = tauv[k];
        // p = tau A22 v: row i of A22 by the 4 threads 4i .. 4i+3
        {
            const int i = tid >> 2, part = tid & 3;
            float acc = 0.f;
            if (i < m) {
                const float *row = A + (k + 1 + i);
                for (int j = part; j < m; j += 4) acc = __fmaf_rn(row[(k + 1 + j) * LAQ], vv[j], acc);
            }
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            const float p = t * acc;
            float pv = (part == 0 && i < m) ? p * vv[i] : 0.f;
            if (part == 0 && i < m) pp[i] = p;
            #pragma unroll
            for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
            if (lane == 0) red[warp] = pv;
        }
        __syncthreads();
        float pv = 0.f;
        #pragma unroll
        for (int w = 0; w < NT / 32; ++w) pv += red[w];
        const float K = 0.5f * t * pv;
        // A22 -= v w^T + w v^T
        for (int e = tid; e < m * TW; e += NT) {
            const int i = e & (TW - 1), j = e >> 6;
            if (i >= m) continue;
            const float vi = vv[i], vj = vv[j];
            const float wi = __fmaf_rn(-K, vi, pp[i]), wj = __fmaf_rn(-K, vj, pp[j]);
            float *x = A + (k + 1 + i) + (k + 1 + j) * LAQ;
            *x = __fmaf_rn(-wi, vj, __fmaf_rn(-vi, wj, *x));
        }
        __syncthreads();
    }

    // T: the tridiagonal in binary64
    if (tid < TW) {
        const int i = tid;
        double dd = 0.0, ee = 0.0, ee2 = 0.0;
        if (i < n) {
            dd = (double)A[i + i * LAQ];
            if (i + 1 < n) {
                const double ei = (double)A[(i + 1) + i * LAQ];
                const double di1 = (double)A[(i + 1) + (i + 1) * LAQ];
                const bool split = fabs(ei) <= 1.1102230246251565e-16 * sqrt(fabs(dd) * fabs(di1));
                ee = split ? 0.0 : ei;
                ee2 = split ? 0.0 : ei * ei;
            }
        }
        d64[i] = dd; e64[i] = ee; e2[i] = ee2;
        double mx = ee2;
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) inrm[warp] = mx;                          // scratch
    }
    __syncthreads();
    if (tid < n) {
        int s = tid, e = tid;
        while (s > 0 && e2[s - 1] != 0.0) --s;
        while (e < n - 1 && e2[e] != 0.0) ++e;
        bs[tid] = s; be[tid] = e;
    }
    if (tid == 0) pivmin_s = 2.2250738585072014e-308 * fmax(1.0, fmax(inrm[0], inrm[1]));
    __syncthreads();
    const double pivmin = pivmin_s;
    {
        // multisection: the MS lanes of eigenvalue t = tid / MS evaluate Sturm counts
        // at MS interior points of the interval, which shrinks (MS + 1)x per round,
        // until it is within 2 omega of max(|lo|, |hi|) or of the block's Gershgorin
        // bound (the Sturm count resolves nothing finer).  The other threads turn
        // the reflectors into explicit columns for B (v_{k+1} = 1, zeros above).
        constexpr int MS = MPJ_BATCHED_MS;
        const int t = tid / MS, l4 = tid % MS, base = lane & ~(MS - 1);
        const unsigned gmask = ((1u << MS) - 1) << base;
        const bool valid = t < n;
        if (t >= TW) {
            for (int e = tid - MS * TW; e < TW * TW; e += NT - MS * TW) {
                const int i = e & (TW - 1), k = e >> 6;
                if (k + 2 < n && i <= k + 1) A[i + k * LAQ] = (i == k + 1) ? 1.f : 0.f;
            }
        }
        const int s = valid ? bs[t] : 0, e = valid ? be[t] : 0, k = t - s;
        double lo = 1e308, hi = -1e308;
        for (int i = s + l4; i <= e; i += MS) {
            const double r = (i > s ? fabs(e64[i - 1]) : 0.0) + (i < e ? fabs(e64[i]) : 0.0);
            lo = fmin(lo, d64[i] - r);
            hi = fmax(hi, d64[i] + r);
        }
        #pragma unroll
        for (int o = 1; o < MS; o <<= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        const double gnorm = fmax(fabs(lo), fabs(hi));
        const double pad = 2.0 * 1.1102230246251565e-16 * gnorm + pivmin;
        lo -= pad; hi += pad;
        const double tabs = 2.0 * 1.1102230246251565e-16 * gnorm;
        if (valid && s < e) {
            for (int it = 0; it < 80; ++it) {
                if (hi - lo <= fmax(tabs, 2.0 * 1.1102230246251565e-16 * fmax(fabs(lo), fabs(hi)))) break;
                const double w = (hi - lo) * (1.0 / (MS + 1));
                double x = __fma_rn(w, (double)(l4 + 1), lo);
                x = fmin(fmax(x, lo), hi);
                const int c = sturm_cnt(d64, e2, s, e, x, pivmin);
                const unsigned ball = (__ballot_sync(gmask, c > k) & gmask) >> base;
                const int mh = ball ? __ffs(ball) - 1 : MS;      // first point with more than k below it
                const double xl = __shfl_sync(gmask, x, base + (mh > 0 ? mh - 1 : 0));
                const double xh = __shfl_sync(gmask, x, base + (mh < MS ? mh : MS - 1));
                lo = mh > 0 ? xl : lo;
                hi = mh < MS ? xh : hi;
            }
        }
        if (valid && l4 == 0) lam[t] = s < e ? 0.5 * (lo + hi) : d64[s];
    }
    __syncthreads();
    // twisted factorisations: lanes 2t (role 0) and 2t + 1 (role 1) for eigenvalue t;
    // warps 4..5 rank the eigenvalues meanwhile (descending, stable)
    if (tid < 2 * TW) {
        const int t = tid >> 1, role = tid & 1;
        const unsigned pmask = 3u << (lane & 30);
        const bool valid = t < n;
        const int s = valid ? bs[t] : 0, e = valid ? be[t] : 0;
        const double l = valid ? lam[t] : 0.0;
        auto guard = [&](double q) { return fabs(q) < pivmin ? (q < 0.0 ? -pivmin : pivmin) : q; };
        if (valid && s < e) {
            if (role == 0) {                                     // forward: D+_i -> X
                double q = guard(d64[s] - l);
                X[s * TW + t] = q;
                for (int i = s + 1; i <= e; ++i) {
                    q = guard(__fma_rn(-e2[i - 1], rcp_nr(q), d64[i] - l));
                    X[i * TW + t] = q;
                }
            }
        }
        __syncwarp(pmask);
        int r = s;
        if (valid && s < e && role == 1) {                       // backward: D-_i, gamma_i, argmin (ties: larger i)
            double q = guard(d64[e] - l);
            double gbest = fabs(X[e * TW + t] + q - (d64[e] - l));
            r = e;
            for (int i = e - 1; i >= s; --i) {
                q = guard(__fma_rn(-e2[i], rcp_nr(q), d64[i] - l));
                const double g = fabs(X[i * TW + t] + q - (d64[i] - l));
                if (g < gbest) { gbest = g; r = i; }
            }
        }
        r = __shfl_sync(pmask, r, (lane & 30) | 1);
        double nrm = 0.0;
        if (valid && s < e) {
            if (role == 0) {                                     // x_r = 1, upwards with D+
                double x = 1.0;
                nrm = 1.0;
                for (int i = r - 1; i >= s; --i) {
                    x = -(e64[i] * rcp_nr(X[i * TW + t])) * x;
                    X[i * TW + t] = x;
                    nrm = __fma_rn(x, x, nrm);
                }
            } else if (r < e) {                                  // D- again below r, then downwards
                double q = guard(d64[e] - l);
                X[e * TW + t] = q;
                for (int i = e - 1; i > r; --i) {
                    q = guard(__fma_rn(-e2[i], rcp_nr(q), d64[i] - l));
                    X[i * TW + t] = q;
                }
                double x = 1.0;
                for (int i = r; i < e; ++i) {
                    x = -(e64[i] * rcp_nr(X[(i + 1) * TW + t])) * x;
                    X[(i + 1) * TW + t] = x;
                    nrm = __fma_rn(x, x, nrm);
                }
            }
        }
        __syncwarp(pmask);
        const double nall = nrm + __shfl_xor_sync(pmask, nrm, 1);
        if (valid && role == 0) {
            X[r * TW + t] = 1.0;
            inrm[t] = s < e ? 1.0 / sqrt(nall) : 1.0;
        }
    } else if (tid < 3 * TW) {
        const int t = tid - 2 * TW;
        if (t < n) {
            const double lt = lam[t];
            int c = 0;
            for (int j = 0; j < n; ++j) {
                const double lj = lam[j];
                c += (lj > lt) || (lj == lt && j < t);
            }
            rnk[t] = c;
        }
    }
    __syncthreads();

    // B: Z = H_0 ... H_{n-3} X, column c by threads 4c .. 4c+3 (rows q + 4u)
    const int c = tid >> 2, q = tid & 3;
    double x[16];
    {
        const bool colv = c < n;
        const int s = colv ? bs[c] : 1, e = colv ? be[c] : 0;
        const double sc = colv ? inrm[c] : 0.0;
        #pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int i = q + 4 * u;
            x[u] = (i >= s && i <= e) ? X[i * TW + c] * sc : 0.0;
        }
    }
    for (int k = n - 3; k >= 0; --k) {
        const float tk = tauv[k];
        if (tk == 0.f) continue;
        const float *vcol = A + k * LAQ;                         // v (explicit: 1 at k + 1, 0 above)
        float v[16];
        double w0 = 0.0, w1 = 0.0;
        #pragma unroll
        for (int u = 0; u < 16; ++u) {
            v[u] = vcol[q + 4 * u];
            if (u & 1) w1 = __fma_rn((double)v[u], x[u], w1); else w0 = __fma_rn((double)v[u], x[u], w0);
        }
        double w = w0 + w1;
        w += __shfl_xor_sync(0xffffffffu, w, 1);
        w += __shfl_xor_sync(0xffffffffu, w, 2);
        const double f = (double)tk * w;
        #pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = __fma_rn(-f, (double)v[u], x[u]);
    }
    if (c < n) {
        const int col = rnk[c];
        #pragma unroll
        for (int u = 0; u < 16; ++u)
            if (q + 4 * u < n) Zg[(q + 4 * u) + col * n] = (float)x[u];
    }
    if (tid == 0 && a.sweeps_low) a.sweeps_low[mat] = 0;
}

__global__ void __launch_bounds__(NT, 3) k_batched_evd(BatchedArgs a)
{
    constexpr int LD = Lay<double>::LD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *RA = (double *)smem_raw;   // U (step 2), then As, W, T
    double *RB = RA + TW * LD;         // Z, then Q = V
    __shared__ double red[NT / 32];
    __shared__ double coef[TW];
    __shared__ WideParams<double> PP[2];
    __shared__ PipeMaps pm;
    __shared__ int rank_[TW];
    const int n = a.n, tid = threadIdx.x;
    const size_t mat = blockIdx.x;
    const double *Ag = a.A + mat * (size_t)n * n;
    // As = (A + A^T) / 2 (formed when needed, a3), ||As||_F, finiteness
    auto as_at = [&](int i, int j) { return (Ag[i + (size_t)j * n] + Ag[j + (size_t)i * n]) * 0.5; };
    double acc0 = 0.0;
    for (int e = tid; e < n * n; e += NT) {
        const double x = as_at(e % n, e / n);
        acc0 = __fma_rn(x, x, acc0);
    }
    const double normA = sqrt(cta_sum(acc0, red));
    if (!isfinite(normA)) {                  // NaN / Inf input: flagged, no sweeps
        if (tid == 0) atomicOr(a.flag, 4);
        return;
    }

    // a1 ran in k_batched_symqr / k_batched_low (or Z was given): n x n, ld n
    const float *Zg = a.Z + mat * (size_t)n * n;

    // a2: Q = the QR factor of Z (positive diag R; reading R10: the Q of MGS).
    // Z, step 1's binary32 eigenvectors, is orthogonal to O(upsilon): with
    // G = Z^T Z = I + E, ||E||_F <= 1e-4, R = chol(G) = I + U is the fixed point
    // of U = Phi(E - U^T U) (Phi: strict upper part + half the diagonal), and
    // R^{-1} = I - U + U^2 - U^3 + ...; two corrections and three inverse terms
    // leave O(||E||^4) <= 1e-16 -- Cholesky QR with the factor from 64^3 DMMA
    // tile products instead of a 64-step sequential factorisation (reading R10b).
    // Otherwise (a worse Z): CGS with the twice-is-enough check, column by column.
    const int warp = tid >> 5, lane = tid & 31;
    int bad = 0;
    for (int e = tid; e < TW * TW; e += NT) {
        const int i = e & (TW - 1), j = e >> 6;
        RB[i + j * LD] = (i < n && j < n) ? (double)Zg[i + j * n] : 0.0;
    }
    __syncthreads();
    bool series;
    {
        Acc<double> E;
        tile_mm<true>(RB, RB, E);                                // G = Z^T Z
        double ss = 0.0;
        E.each_ref([&](int i, int j, double &x) {
            x = (i < n && j < n) ? x - (i == j ? 1.0 : 0.0) : 0.0;
            ss = __fma_rn(x, x, ss);
        });
        const double nE = sqrt(cta_sum(ss, red));
        series = nE <= 1e-4;
        if (series) {
            auto phi = [&](int i, int j, double x) {
                RA[i + j * LD] = i < j ? x : (i == j ? 0.5 * x : 0.0);
            };
            E.each(phi);                                         // U0 = Phi(E)
            __syncthreads();
            for (int it = 0; it < 2; ++it) {                     // U <- Phi(E - U^T U)
                Acc<double> P;
                tile_mm<true>(RA, RA, P);
                __syncthreads();
                #pragma unroll
                for (int mi = 0; mi < 2; ++mi)
                    #pragma unroll
                    for (int ni = 0; ni < 4; ++ni)
                        #pragma unroll
                        for (int h = 0; h < 2; ++h) P.v[mi][ni][h] = E.v[mi][ni][h] - P.v[mi][ni][h];
                P.each(phi);
                __syncthreads();
            }
            // Q = Z - Z U + Z U^2 - Z U^3 (Horner on the left: Y_t = Y_{t-1} U in RB)
            Acc<double> S;
            S.each_ref([&](int i, int j, double &x) { x = RB[i + j * LD]; });
            for (int t = 1; t <= 3; ++t) {
                Acc<double> Y;
                tile_mm<false>(RB, RA, Y);
                __syncthreads();
                const double sg = (t & 1) ? -1.0 : 1.0;
                #pragma unroll
                for (int mi = 0; mi < 2; ++mi)
                    #pragma unroll
                    for (int ni = 0; ni < 4; ++ni)
                        #pragma unroll
                        for (int h = 0; h < 2; ++h) S.v[mi][ni][h] = __fma_rn(sg, Y.v[mi][ni][h], S.v[mi][ni][h]);
                if (t < 3) {
                    Y.each([&](int i, int j, double x) { RB[i + j * LD] = x; });
                    __syncthreads();
                }
            }
            S.each([&](int i, int j, double x) { RB[i + j * LD] = x; });
            __syncthreads();
        }
    }
    __shared__ int redo;
    for (int npass = 1; npass <= 2 && !series; ++npass) {
        if (npass > 1)
            for (int e = tid; e < TW * TW; e += NT) {
                const int i = e & (TW - 1), j = e >> 6;
                RB[i + j * LD] = (i < n && j < n) ? (double)Zg[i + j * n] : 0.0;
            }
        if (tid == 0) redo = 0;
        __syncthreads();
        for (int k = 0; k < n; ++k) {
            double *v = RB + k * LD;
            for (int pass = 0; pass < npass && k > 0; ++pass) {
                for (int j = warp; j < k; j += NT / 32) {
                    const double *qj = RB + j * LD;
                    double d = __fma_rn(qj[lane], v[lane], 0.0);
                    d = __fma_rn(qj[lane + 32], v[lane + 32], d);
                    #pragma unroll
                    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                    if (lane == 0) coef[j] = d;
                }
                __syncthreads();
                if (tid < TW) {
                    double x = v[tid];
                    for (int j = 0; j < k; ++j) x = __fma_rn(-coef[j], RB[tid + j * LD], x);
                    v[tid] = x;
                }
                __syncthreads();
            }
            double d = 0.0;
            if (tid < 32) {
                d = __fma_rn(v[lane], v[lane], 0.0);
                d = __fma_rn(v[lane + 32], v[lane + 32], d);
                #pragma unroll
                for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                if (lane == 0) coef[0] = sqrt(d);
            }
            __syncthreads();
            const double nrm = coef[0];
            if (!(nrm > 0.0)) bad = 1;
            else if (tid < TW) v[tid] = v[tid] / nrm;
            if (npass == 1 && tid == 0 && !(nrm >= 0.5)) redo = 1;
            __syncthreads();
        }
        if (!redo) break;
        bad = 0;
    }

    // a3: T = Q^T (As Q), symmetrised (As into RA, W = As Q over it)
    {
        for (int e = tid; e < TW * TW; e += NT) {
            const int i = e & (TW - 1), j = e >> 6;
            RA[i + j * LD] = (i < n && j < n) ? as_at(i, j) : 0.0;
        }
        __syncthreads();
        Acc<double> w;
        tile_mm<false>(RA, RB, w);       // W = As Q
        __syncthreads();
        w.each([&](int i, int j, double x) { RA[i + j * LD] = x; });
        __syncthreads();
        Acc<double> t;
        tile_mm<true>(RB, RA, t);        // T = Q^T W
        __syncthreads();
        t.each([&](int i, int j, double x) { RA[i + j * LD] = x; });
        __syncthreads();
        for (int e = tid; e < TW * TW; e += NT) {
            const int i = e & (TW - 1), j = e >> 6;
            if (i < j) {
                const double s = (RA[i + j * LD] + RA[j + i * LD]) * 0.5;
                RA[i + j * LD] = s;
                RA[j + i * LD] = s;
            }
        }
        __syncthreads();
    }

    // T and V to the odd leading dimension 65 for the rounds (the mirrored
    // column-stride stores of the pair tiles are then bank-conflict free; LD 68
    // serves the DMMA fragment loads above)
    constexpr int LR = LayK<double>::LD;
    {
        double ta[TW * TW / NT], tb[TW * TW / NT];
        #pragma unroll
        for (int u = 0; u < TW * TW / NT; ++u) {
            const int e = tid + NT * u, i = e & (TW - 1), j = e >> 6;
            ta[u] = RA[i + j * LD]; tb[u] = RB[i + j * LD];
        }
        __syncthreads();
        #pragma unroll
        for (int u = 0; u < TW * TW / NT; ++u) {
            const int e = tid + NT * u, i = e & (TW - 1), j = e >> 6;
            RA[i + j * LR] = ta[u]; RB[i + j * LR] = tb[u];
        }
        __syncthreads();
    }

    // a4-a8: fp64 sweeps
    const double tol = a.eps * normA;
    int sw = 0;
    bool conv = false;
    double *Tc = RA, *Vc = RB;               // the rounds swap the two buffers
    for (;;) {
        const double off = sqrt(sq_norm<double, LR>(Tc, true, red));
        if (off <= tol) { conv = true; break; }
        if (sw >= a.max_sweeps) break;
        ++sw;
        double *uo;
        Tc = inner_rounds_pipe<double>(Tc, Vc, a.lsched, a.nu, a.rule, PP, pm, &uo);
        Vc = uo;
    }

    // a10: extraction (stable descending rank)
    if (tid < n) {
        const double di = Tc[tid + tid * LR];
        int r = 0;
        for (int j = 0; j < n; ++j) {
            const double dj = Tc[j + j * LR];
            r += (dj > di) || (dj == di && j < tid);
        }
        rank_[tid] = r;
        a.lam[mat * n + r] = di;
    }
    __syncthreads();
    double *Vg = a.V + mat * (size_t)n * n;
    for (int e = tid; e < n * n; e += NT) {
        const int i = e % n, j = e / n;
        Vg[i + (size_t)rank_[j] * n] = Vc[i + j * LR];
    }
    if (tid == 0) {
        if (a.sweeps) a.sweeps[mat] = sw;
        if (!conv) atomicOr(a.flag, 1);
        if (bad) atomicOr(a.flag, 2);
    }
}

}  // namespace

mpj_status batched_evd(const double *A, int64_t n, int64_t batch, double *Lambda, double *V, int *sweeps,
                       int *sweeps_low, const float *Zin, float *Zout, cudaStream_t st, const mpj_config &cfg)
{
    // the 64-index intra-block schedule: read-only, uploaded once per device
    static std::mutex mu;
    static std::map<int, int2 *> sched_dev;
    int2 *lsched = nullptr;
    {
        int dev = 0;
        MPJ_CK(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(mu);
        auto it = sched_dev.find(dev);
        if (it == sched_dev.end()) {
            HostSchedule hs;
            build_schedule(64, 32, hs);
            int2 *d = nullptr;
            MPJ_CK(cudaMalloc(&d, hs.lsched.size() * sizeof(int2)));
            MPJ_CK(cudaMemcpy(d, hs.lsched.data(), hs.lsched.size() * sizeof(int2), cudaMemcpyHostToDevice));
            it = sched_dev.emplace(dev, d).first;
        }
        lsched = it->second;
    }
    constexpr int64_t kChunk = 16384;   // matrices per launch pair (Z scratch: 256 MB at most)
    struct Scratch {                    // freed on every exit
        cudaStream_t st; void *p = nullptr, *z = nullptr;
        ~Scratch() { if (p) cudaFreeAsync(p, st); if (z) cudaFreeAsync(z, st); }
    } sc{st};
    MPJ_CK(cudaMallocAsync(&sc.p, 256, st));
    int *flag = (int *)sc.p;
    float *Z = nullptr;
    if (!Zin && !Zout) {
        MPJ_CK(cudaMallocAsync(&sc.z, (size_t)std::min<int64_t>(batch, kChunk) * n * n * sizeof(float), st));
        Z = (float *)sc.z;
    }
    MPJ_CK(cudaMemsetAsync(flag, 0, sizeof(int), st));
    if (Zin && sweeps_low) MPJ_CK(cudaMemsetAsync(sweeps_low, 0, batch * sizeof(int), st));
    BatchedArgs a;
    a.A = A; a.n = (int)n; a.lam = Lambda; a.V = V; a.sweeps = sweeps; a.sweeps_low = sweeps_low;
    a.flag = flag; a.lsched = lsched; a.Z = Z;
    const double omega = 1.1102230246251565e-16, upsilon = 5.9604644775390625e-08;
    a.eps = cfg.eps_factor * omega; a.nu = cfg.nu_factor * omega;
    a.eps_low = eps_low_factor(cfg, n) * upsilon; a.nu_low = cfg.nu_low_factor * upsilon;
    a.max_sweeps = cfg.max_sweeps; a.max_sweeps_low = cfg.max_sweeps_low; a.rule = cfg.stop_rule;
    const int smem = 2 * TW * Lay<double>::LD * sizeof(double);
    const int smem_low = 2 * TW * LayK<float>::LD * sizeof(float);
    MPJ_CK(smem_optin((const void *)k_batched_evd, smem, NT, nullptr));
    MPJ_CK(smem_optin((const void *)k_batched_symqr, kSymqrSmem, NT, nullptr));
    const bool prof = prof_on();
    for (int64_t b0 = 0; b0 < batch; b0 += kChunk) {
        BatchedArgs ab = a;
        const int64_t nb = std::min<int64_t>(kChunk, batch - b0);
        ab.A = A + b0 * n * n; ab.lam = Lambda + b0 * n; ab.V = V + b0 * n * n;
        ab.sweeps = sweeps ? sweeps + b0 : nullptr;
        ab.sweeps_low = sweeps_low ? sweeps_low + b0 : nullptr;
        if (Zin) ab.Z = const_cast<float *>(Zin) + b0 * n * n;      // read only (k_batched_evd)
        else if (Zout) ab.Z = Zout + b0 * n * n;
        if (!Zin) {
            if (prof) prof_mark("batched_step1", st, true);
            if (cfg.low_solver == MPJ_LOW_JACOBI) k_batched_low<<<(unsigned)nb, NT, smem_low, st>>>(ab);
            else k_batched_symqr<<<(unsigned)nb, NT, kSymqrSmem, st>>>(ab);
            if (prof) prof_mark("batched_step1", st, false);
            count_launch();
        }
        if (prof) prof_mark("batched_evd_f64", st, true);
        k_batched_evd<<<(unsigned)nb, NT, smem, st>>>(ab);
        if (prof) prof_mark("batched_evd_f64", st, false);
        count_launch();
        MPJ_CK(cudaGetLastError());
    }
    int h_flag = 0;
    MPJ_CK(cudaMemcpyAsync(&h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaStreamSynchronize(st));
    if (h_flag & 4) { set_error("batched: non-finite entry in A"); return MPJ_ERR_NONFINITE; }
    if (h_flag & 2) { set_error("batched: rank-deficient Z in CGS2"); return MPJ_ERR_RANKDEF; }
    if (h_flag & 1) { set_error("batched: some matrix reached max_sweeps"); return MPJ_ERR_NOCONV; }
    return MPJ_OK;
}

}  // namespace mpj

extern "C" mpj_status mpjacobi_eig_batched_z(const double *A, int64_t n, int64_t batch, const float *Z_in,
                                             float *Z_out, double *Lambda, double *V, int *sweeps, int *sweeps_low,
                                             void *stream, const mpj_config *cfg_in)
{
    mpj::set_error("");
    if (n < 1 || n > 64 || batch < 1 || !A || !Lambda || !V) {
        mpj::set_error("mpjacobi_eig_batched: need 1 <= n <= 64, batch >= 1, non-NULL A/Lambda/V");
        return MPJ_ERR_INVALID;
    }
    mpj_config cfg;
    if (cfg_in) cfg = *cfg_in; else mpj_config_default_eig(&cfg);
    cudaStream_t st = (cudaStream_t)stream;
    mpj_status r = mpj::batched_evd(A, n, batch, Lambda, V, sweeps, sweeps_low, Z_in, Z_out, st, cfg);
    if (r == MPJ_OK && Z_in && Z_out)
        if (cudaMemcpyAsync(Z_out, Z_in, (size_t)batch * n * n * sizeof(float), cudaMemcpyDeviceToDevice, st) !=
            cudaSuccess) {
            mpj::set_error("mpjacobi_eig_batched_z: Z copy failed");
            return MPJ_ERR_CUDA;
        }
    return r;
}

extern "C" mpj_status mpjacobi_eig_batched(const double *A, int64_t n, int64_t batch, double *Lambda, double *V,
                                           int *sweeps, int *sweeps_low, void *stream, const mpj_config *cfg_in)
{
    return mpjacobi_eig_batched_z(A, n, batch, nullptr, nullptr, Lambda, V, sweeps, sweeps_low, stream, cfg_in);
}
