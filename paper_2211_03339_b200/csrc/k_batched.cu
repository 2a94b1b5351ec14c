// k_batched.cu -- batched Alg. 3 for many small matrices, one
// matrix per CTA, everything in shared memory (SURVEY §8(a) row a11,
// BASELINE config 3: 4096 x n = 64).
//
// Per CTA (n <= 64, padded to 64 with zero rows/columns, reading R2):
//   a0  As = (A + A^T)/2, ||As||_F
//   a1  fp32 sweeps on fl32(As) with V32 = I (reading R12): the ordering for
//       n_p = 64, b = 32 is one block round (31 intra + 32 cross rounds, R1),
//       run by inner_rounds_b<> (mpj_block.cuh: U in registers)
//   a2  Q = CGS2(fp64(V32)) (reading R10), column by column in shared memory,
//       dot products by warp-shuffle reductions
//   a3  T = Q^T As Q on the FP64 tensor pipe (two 64^3 DMMA tile products),
//       symmetrised (R11)
//   a4-a8 fp64 sweeps on T with V = Q, stop test ||off(T)||_F <= eps ||As||_F
//   a10 lambda = diag(T) stable-descending, V's columns alike.
// a1 runs as its own kernel (k_batched_low: T32 and V32 only, 35 KB of shared
// memory -> 6 CTAs per SM); the rest (a0, a2-a10) in k_batched_evd: three
// 64 x 68 fp64 panels (104 KB) -> 2 CTAs per SM.
#include "mpj_block.cuh"
#include "mpj_device.cuh"
#include "mpj_internal.h"

#include <algorithm>

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

template <typename R>
__device__ __forceinline__ double sq_norm(const R *M, bool offdiag, double *red)
{
    constexpr int LD = Lay<R>::LD;
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
    constexpr int LF = Lay<float>::LD;
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
    const double nA32 = sqrt(sq_norm<float>(T32, false, red));
    const double tol_low = a.eps_low * nA32;
    int swl = 0;
    for (;;) {
        const double off = sqrt(sq_norm<float>(T32, true, red));
        if (off <= tol_low || swl >= a.max_sweeps_low) break;
        ++swl;
        inner_rounds_b<float>(T32, V32, true, a.lsched, (float)a.nu_low, a.rule, sh, pf);
    }
    float *Zg = a.Z + mat * (size_t)TW * TW;
    for (int e = tid; e < TW * TW; e += NT) Zg[e] = V32[(e & (TW - 1)) + (e >> 6) * LF];
    if (tid == 0 && a.sweeps_low) a.sweeps_low[mat] = swl;
}

__global__ void __launch_bounds__(NT, 2) k_batched_evd(BatchedArgs a)
{
    constexpr int LD = Lay<double>::LD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *RA = (double *)smem_raw;   // As, later T
    double *RB = RA + TW * LD;         // A staging, later Q = V
    double *RC = RB + TW * LD;         // T32/V32, later W
    __shared__ double red[NT / 32];
    __shared__ double coef[TW];
    __shared__ InnerSharedB sh;
    __shared__ InnerParams<double> pd;
    __shared__ int rank_[TW];
    const int n = a.n, tid = threadIdx.x;
    const size_t mat = blockIdx.x;
    const double *Ag = a.A + mat * (size_t)n * n;
    const int2 bp = make_int2(0, 1);   // one block pair: local index == global index

    // a0
    for (int e = tid; e < TW * TW; e += NT) {
        const int i = e & (TW - 1), j = e >> 6;
        RB[i + j * LD] = (i < n && j < n) ? Ag[i + (size_t)j * n] : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < TW * TW; e += NT) {
        const int i = e & (TW - 1), j = e >> 6;
        RA[i + j * LD] = (RB[i + j * LD] + RB[j + i * LD]) * 0.5;
    }
    __syncthreads();
    const double normA = sqrt(sq_norm<double>(RA, false, red));

    // a1 ran in k_batched_low: Z = V32 of this matrix
    const float *Zg = a.Z + mat * (size_t)TW * TW;

    // a2: Q = CGS(Z), Z = fp64(V32) (real n x n block).  Z is the fp32
    // stage's V, orthogonal to O(upsilon) with unit columns: one projection
    // pass loses no significant part of a column (reading R10); if one does
    // (norm after the pass < 1/2, "twice is enough"), Q is redone with CGS2.
    const int warp = tid >> 5, lane = tid & 31;
    int bad = 0;
    __shared__ int redo;
    for (int npass = 1; npass <= 2; ++npass) {
        for (int e = tid; e < TW * TW; e += NT) {
            const int i = e & (TW - 1), j = e >> 6;
            RB[i + j * LD] = (i < n && j < n) ? (double)Zg[i + j * TW] : 0.0;
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

    // a3: T = Q^T (As Q), symmetrised
    {
        Acc<double> w;
        tile_mm<false>(RA, RB, w);       // W = As Q
        __syncthreads();
        w.each([&](int i, int j, double x) { RC[i + j * LD] = x; });
        __syncthreads();
        Acc<double> t;
        tile_mm<true>(RB, RC, t);        // T = Q^T W
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

    // a4-a8: fp64 sweeps
    const double tol = a.eps * normA;
    int sw = 0;
    bool conv = false;
    for (;;) {
        const double off = sqrt(sq_norm<double>(RA, true, red));
        if (off <= tol) { conv = true; break; }
        if (sw >= a.max_sweeps) break;
        ++sw;
        inner_rounds_b<double>(RA, RB, true, a.lsched, a.nu, a.rule, sh, pd);
    }

    // a10: extraction (stable descending rank)
    if (tid < n) {
        const double di = RA[tid + tid * LD];
        int r = 0;
        for (int j = 0; j < n; ++j) {
            const double dj = RA[j + j * LD];
            r += (dj > di) || (dj == di && j < tid);
        }
        rank_[tid] = r;
        a.lam[mat * n + r] = di;
    }
    __syncthreads();
    double *Vg = a.V + mat * (size_t)n * n;
    for (int e = tid; e < n * n; e += NT) {
        const int i = e % n, j = e / n;
        Vg[i + (size_t)rank_[j] * n] = RB[i + j * LD];
    }
    if (tid == 0) {
        if (a.sweeps) a.sweeps[mat] = sw;
        if (!conv) atomicOr(a.flag, 1);
        if (bad) atomicOr(a.flag, 2);
    }
}

}  // namespace

mpj_status batched_evd(const double *A, int64_t n, int64_t batch, double *Lambda, double *V, int *sweeps,
                       int *sweeps_low, cudaStream_t st, const mpj_config &cfg)
{
    HostSchedule hs;
    build_schedule(64, 32, hs);
    int2 *lsched = nullptr;
    int *flag = nullptr;
    float *Z = nullptr;
    MPJ_CK(cudaMallocAsync(&lsched, hs.lsched.size() * sizeof(int2) + 256, st));
    constexpr int64_t kChunk = 16384;   // matrices per launch pair (Z: 256 MB at most)
    MPJ_CK(cudaMallocAsync(&Z, (size_t)std::min<int64_t>(batch, kChunk) * TW * TW * sizeof(float), st));
    flag = (int *)(lsched + hs.lsched.size());
    MPJ_CK(cudaMemcpyAsync(lsched, hs.lsched.data(), hs.lsched.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    MPJ_CK(cudaMemsetAsync(flag, 0, sizeof(int), st));
    BatchedArgs a;
    a.A = A; a.n = (int)n; a.lam = Lambda; a.V = V; a.sweeps = sweeps; a.sweeps_low = sweeps_low;
    a.flag = flag; a.lsched = lsched; a.Z = Z;
    const double omega = 1.1102230246251565e-16, upsilon = 5.9604644775390625e-08;
    a.eps = cfg.eps_factor * omega; a.nu = cfg.nu_factor * omega;
    a.eps_low = eps_low_factor(cfg, n) * upsilon; a.nu_low = cfg.nu_low_factor * upsilon;
    a.max_sweeps = cfg.max_sweeps; a.max_sweeps_low = cfg.max_sweeps_low; a.rule = cfg.stop_rule;
    const int smem = 3 * TW * Lay<double>::LD * sizeof(double);
    const int smem_low = 2 * TW * Lay<float>::LD * sizeof(float);
    MPJ_CK(cudaFuncSetAttribute(k_batched_evd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const bool prof = prof_on();
    if (prof) prof_mark("batched_evd", st, true);
    for (int64_t b0 = 0; b0 < batch; b0 += kChunk) {
        BatchedArgs ab = a;
        const int64_t nb = std::min<int64_t>(kChunk, batch - b0);
        ab.A = A + b0 * n * n; ab.lam = Lambda + b0 * n; ab.V = V + b0 * n * n;
        ab.sweeps = sweeps ? sweeps + b0 : nullptr;
        ab.sweeps_low = sweeps_low ? sweeps_low + b0 : nullptr;
        k_batched_low<<<(unsigned)nb, NT, smem_low, st>>>(ab);
        k_batched_evd<<<(unsigned)nb, NT, smem, st>>>(ab);
        count_launch(2);
    }
    if (prof) prof_mark("batched_evd", st, false);
    int h_flag = 0;
    MPJ_CK(cudaMemcpyAsync(&h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaStreamSynchronize(st));
    cudaFreeAsync(lsched, st);
    cudaFreeAsync(Z, st);
    if (h_flag & 2) { set_error("batched: rank-deficient Z in CGS2"); return MPJ_ERR_RANKDEF; }
    if (h_flag & 1) { set_error("batched: some matrix reached max_sweeps"); return MPJ_ERR_NOCONV; }
    return MPJ_OK;
}

}  // namespace mpj

extern "C" mpj_status mpjacobi_eig_batched(const double *A, int64_t n, int64_t batch, double *Lambda, double *V,
                                           int *sweeps, int *sweeps_low, void *stream, const mpj_config *cfg_in)
{
    mpj::set_error("");
    if (n < 1 || n > 64 || batch < 1 || !A || !Lambda || !V) {
        mpj::set_error("mpjacobi_eig_batched: need 1 <= n <= 64, batch >= 1, non-NULL A/Lambda/V");
        return MPJ_ERR_INVALID;
    }
    mpj_config cfg;
    if (cfg_in) cfg = *cfg_in; else mpj_config_default_eig(&cfg);
    cudaStream_t st = (cudaStream_t)stream;
    return mpj::batched_evd(A, n, batch, Lambda, V, sweeps, sweeps_low, st, cfg);
}
