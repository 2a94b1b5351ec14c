// mpj_device.cuh -- device-side building blocks of the Jacobi hot path.
//
// Independent of oracle/ (no shared code); both follow the same paper text:
//   Lemma 3.1: mu = (a_qq - a_pp)/(2 a_pq),
//     t = 1/(mu + sqrt(1+mu^2)) (mu >= 0) | 1/(mu - sqrt(1+mu^2)) (mu < 0),
//     c = (1+t^2)^(-1/2), s = t c.
//   Threshold (Alg. 2/3 line 4): skip iff |a_pq| <= nu min(|a_pp|,|a_qq|)
//   (stop_rule 1: Remark 3.1, |a_pq| <= nu sqrt(a_pp a_qq)).
// Readings: R3 1+mu^2 = fma(mu,mu,1); R4 |mu| >= 2^26 (fp64) /
// 2^12 (fp32) uses t = 0.5/mu; R6 the Rutishauser tau-form of the update,
//   x' = x - s (y + tau x),  y' = y + s (x - tau y),  tau = s/(1+c),
// each as two explicit fused multiply-adds.  The library is compiled with
// -fmad=false so that no other contraction happens (bit-exact with the
// oracle's binary64/binary32 arithmetic).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mpj {

template <typename R> struct Prec;
template <> struct Prec<double> {
    static constexpr double mu_big = 67108864.0;  // 2^26
};
template <> struct Prec<float> {
    static constexpr float mu_big = 4096.0f;      // 2^12
};

__device__ __forceinline__ double fmaR(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fmaR(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double sqrtR(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ float sqrtR(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double divR(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float divR(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double absR(double a) { return fabs(a); }
__device__ __forceinline__ float absR(float a) { return fabsf(a); }
__device__ __forceinline__ double minR(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ float minR(float a, float b) { return fminf(a, b); }

// The threshold decision alone: 1 if the pair is skipped (rot_params and
// rot_params_fast take exactly this decision).
template <typename R>
__device__ __forceinline__ bool rot_skip(R app, R aqq, R apq, R nu, int rule)
{
    if (rule == 1) {
        R g = app * aqq;
        return (g > R(0)) ? (absR(apq) <= nu * sqrtR(g)) : (apq == R(0));
    }
    return absR(apq) <= nu * minR(absR(app), absR(aqq));
}

// Rotation parameters of Lemma 3.1 plus the threshold decision.
// Returns 1 if the pair rotates; on skip t = s = tau = 0 (identity update).
template <typename R>
__device__ __forceinline__ int rot_params(R app, R aqq, R apq, R nu, int rule, R &t, R &s, R &tau)
{
    // Branch-free form (no warp divergence on the K3 critical path).  It is
    // bit-identical to the literal reading: for mu < 0, 1/(mu - r) is exactly
    // -(1/(|mu| + r)) (the negation is exact), the sign follows "mu >= 0"
    // (so mu = -0 takes the + branch like the literal code), and for |mu| >=
    // 2^26 (2^12 fp32) 0.5/mu == sgn * (1/(2|mu|)) (2|mu| is exact and both
    // are the correctly rounded 1/(2 mu)).
    const bool skip = rot_skip<R>(app, aqq, apq, nu, rule);
    const R den = skip ? R(1) : R(2) * apq;
    const R mu = divR(aqq - app, den);
    const R amu = absR(mu);
    const R r = sqrtR(fmaR(mu, mu, R(1)));                    // inf for huge mu: not selected
    const R d = (amu < Prec<R>::mu_big) ? amu + r : R(2) * amu;
    const R sgn = (mu >= R(0)) ? R(1) : R(-1);
    const R tt = sgn * divR(R(1), d);
    const R c = divR(R(1), sqrtR(fmaR(tt, tt, R(1))));
    const R ss = tt * c;
    const R uu = divR(ss, R(1) + c);
    t = skip ? R(0) : tt;
    s = skip ? R(0) : ss;
    tau = skip ? R(0) : uu;
    return skip ? 0 : 1;
}

// The same rotation parameters with the divisions and square roots of the
// chain as MUFU seeds plus Newton steps (a few ulps, not correctly rounded):
// for K3's parameter warp, whose dependent divide / square-root chain is the
// latency of every inner round.  Changes the rotations at the rounding level
// only (the block variant is compared with the oracle to a tolerance); the
// scalar variant, the batched path and the SVD keep rot_params.
__device__ __forceinline__ double rcp_fast(double q)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double e = __fma_rn(-q, r, 1.0);
    r = __fma_rn(r, e, r);
    e = __fma_rn(-q, r, 1.0);
    return __fma_rn(r, e, r);
}
__device__ __forceinline__ double rsqrt_fast(double z)        // 1 / sqrt(z), z >= 1 here
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(z));
    double h = __fma_rn(-0.5 * z * y, y, 0.5);                 // y <- y (3/2 - z y^2 / 2), twice
    y = __fma_rn(y, h, y);
    h = __fma_rn(-0.5 * z * y, y, 0.5);
    return __fma_rn(y, h, y);
}
__device__ __forceinline__ float rcp_fast(float q) { return __frcp_rn(q); }
__device__ __forceinline__ float rsqrt_fast(float z) { return 1.0f / __fsqrt_rn(z); }

template <typename R>
__device__ __forceinline__ int rot_params_fast(R app, R aqq, R apq, R nu, int rule, R &t, R &s, R &tau)
{
    const bool skip = rot_skip<R>(app, aqq, apq, nu, rule);
    const R den = skip ? R(1) : R(2) * apq;
    const R mu = (aqq - app) * rcp_fast(den);
    const R amu = absR(mu);
    const R z = fmaR(mu, mu, R(1));
    const R r = z * rsqrt_fast(z);                               // sqrt(1 + mu^2)
    const R d = (amu < Prec<R>::mu_big) ? amu + r : R(2) * amu;
    const R sgn = (mu >= R(0)) ? R(1) : R(-1);
    const R tt = sgn * rcp_fast(d);
    const R c = rsqrt_fast(fmaR(tt, tt, R(1)));
    const R ss = tt * c;
    const R uu = ss * rcp_fast(R(1) + c);
    t = skip ? R(0) : tt;
    s = skip ? R(0) : ss;
    tau = skip ? R(0) : uu;
    return skip ? 0 : 1;
}

// J applied to an (x at index p, y at index q) pair: (x,y) <- (c x - s y, s x + c y).
template <typename R>
__device__ __forceinline__ void rot(R s, R tau, R &x, R &y)
{
    R x0 = x, y0 = y;
    x = fmaR(-s, fmaR(tau, x0, y0), x0);
    y = fmaR(s, fmaR(-tau, y0, x0), y0);
}

// ---------------------------------------------------------------------------
// Parallel ordering (reading R1): block merry-go-round with block size b.
// The host uploads
//   bsched[R * mb + k] = (top block, bottom block) of block pair k in block round R
//   lsched[s * (b/2) + j] = (top, bottom) local indices of intra round s (round 0 only)
// and pair (round r, slot k) is decoded here.  Pair orientation: p < q.
// ---------------------------------------------------------------------------
struct Sched {
    const int2 *bsched;   // (nb-1) x mb
    const int2 *lsched;   // (b-1) x (b/2), b > 1 only
    int b;                // block size (1 or even)
    int nb;               // n_p / b
    int np;               // padded order
};

__device__ __forceinline__ int2 pair_of(const Sched &S, int r, int k)
{
    const int b = S.b, mb = S.nb >> 1;
    int a, c;
    if (b > 1 && r < b - 1) {               // intra-block round r of block round 0
        const int kk = k / b, w = k - kk * b, hb = b >> 1;
        const int2 bp = S.bsched[kk];
        const int blk = (w < hb) ? bp.x : bp.y;
        const int2 lp = S.lsched[r * hb + (w < hb ? w : w - hb)];
        a = blk * b + lp.x; c = blk * b + lp.y;
    } else {
        const int rr = (b > 1) ? r - (b - 1) : r;
        const int R = rr / b, s = rr - R * b;
        const int kk = k / b, i = k - kk * b;
        const int2 bp = S.bsched[R * mb + kk];
        a = bp.x * b + i;
        int j = i + s; if (j >= b) j -= b;
        c = bp.y * b + j;
    }
    return a < c ? make_int2(a, c) : make_int2(c, a);
}

// Deterministic block reduction of a double (all threads of the block call it).
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *sh)
{
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = 0;
    if (threadIdx.x < 32) {
        r = (l < NT / 32) ? sh[l] : 0.0;
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    return r;  // valid in warp 0
}

}  // namespace mpj
