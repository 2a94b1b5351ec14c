// mpj_block.cuh -- 64 x 64 shared-memory building blocks shared by the block
// variant (k_block.cu) and the batched one-matrix-per-CTA path (k_batched.cu):
// the inner rounds of a block pair (Lemma 3.1, threshold P:194,
// ordering reading R1) and 64 x 64 x 64 tile products on the FP64 tensor pipe
// (mma.sync m8n8k4 -> DMMA) / FP32 FFMA.
#pragma once
#include "mpj_device.cuh"

namespace mpj {
namespace blk {

constexpr int BW = 32;   // b
constexpr int TW = 64;   // 2b
constexpr int NT = 256;  // threads per CTA

template <typename R> struct Lay;
template <> struct Lay<double> { static constexpr int LD = 68; };   // 2 wavefronts / DMMA frag
template <> struct Lay<float> { static constexpr int LD = 65; };    // conflict-free SIMT tiles

// global index of local index li (0..63) of block pair (I, J)
__device__ __forceinline__ int gidx(int2 bp, int li) { return li < BW ? bp.x * BW + li : bp.y * BW + (li - BW); }

// ---------------------------------------------------------------------------
// The rounds of one block pair on its 64 x 64 diagonal block D (shared memory,
// column-major, leading dimension LD), accumulating U <- U J (U may be NULL).
// Local index li <-> global index gidx(bp, li).  Rounds: if `intra`, the b-1
// merry-go-round rounds inside each half first (block round 0, reading R1),
// then the b cyclic-shift cross rounds.  Same Lemma 3.1 arithmetic and the
// same canonical tile order as the scalar kernels (k_rounds.cu).  Must be
// called by all NT threads of the CTA.  Returns the number of rotations
// (valid in thread 0).
// ---------------------------------------------------------------------------
struct InnerShared {
    int lp[BW], lq[BW], gp[BW];
    unsigned nrot;
};
template <typename R> struct InnerParams {
    R t[BW], s[BW], u[BW];
};

template <typename R>
__device__ __forceinline__ unsigned inner_rounds(R *D, R *U, int2 bp, bool intra, const int2 *__restrict__ lsched,
                                                 R nu, int rule, InnerShared &sh, InnerParams<R> &pr)
{
    constexpr int LD = Lay<R>::LD;
    const int tid = threadIdx.x;
    if (tid == 0) sh.nrot = 0;
    __syncthreads();
    const int nrounds = intra ? (BW - 1) + BW : BW;
    for (int s = 0; s < nrounds; ++s) {
        if (tid < BW) {
            int a, c;
            if (intra && s < BW - 1) {        // intra-block rounds (block round 0 only)
                const int hb = BW / 2, w = tid;
                const int2 lp = lsched[s * hb + (w < hb ? w : w - hb)];
                const int off = (w < hb) ? 0 : BW;
                a = off + lp.x; c = off + lp.y;
            } else {
                const int sc = intra ? s - (BW - 1) : s;
                a = tid;
                int j = tid + sc; if (j >= BW) j -= BW;
                c = BW + j;
            }
            const int ga = gidx(bp, a), gc = gidx(bp, c);
            const int lp = ga < gc ? a : c, lq = ga < gc ? c : a;
            R t, sn, u;
            const int did = rot_params<R>(D[lp + lp * LD], D[lq + lq * LD], D[lp + lq * LD], nu, rule, t, sn, u);
            sh.lp[tid] = lp; sh.lq[tid] = lq; sh.gp[tid] = ga < gc ? ga : gc;
            pr.t[tid] = t; pr.s[tid] = sn; pr.u[tid] = u;
            const unsigned bal = __ballot_sync(0xffffffffu, did);
            if (tid == 0) sh.nrot += __popc(bal);
        }
        __syncthreads();
        // D <- J^T D J on the 32 x 32 pair tiles (same canonical order as k_round_apply)
        for (int e = tid; e < BW * BW; e += NT) {
            const int kk = e & (BW - 1), ll = e >> 5;
            const int pk = sh.lp[kk], qk = sh.lq[kk];
            if (kk == ll) {
                const R apq = D[pk + qk * LD], t = pr.t[kk];
                D[pk + pk * LD] = fmaR(-t, apq, D[pk + pk * LD]);
                D[qk + qk * LD] = fmaR(t, apq, D[qk + qk * LD]);
                D[pk + qk * LD] = R(0);
                D[qk + pk * LD] = R(0);
                continue;
            }
            const int pl = sh.lp[ll], ql = sh.lq[ll];
            R x11 = D[pk + pl * LD], x21 = D[qk + pl * LD], x12 = D[pk + ql * LD], x22 = D[qk + ql * LD];
            const R sk = pr.s[kk], uk = pr.u[kk], sl = pr.s[ll], ul = pr.u[ll];
            if (sh.gp[kk] < sh.gp[ll]) {
                rot<R>(sk, uk, x11, x21); rot<R>(sk, uk, x12, x22);
                rot<R>(sl, ul, x11, x12); rot<R>(sl, ul, x21, x22);
            } else {
                rot<R>(sl, ul, x11, x12); rot<R>(sl, ul, x21, x22);
                rot<R>(sk, uk, x11, x21); rot<R>(sk, uk, x12, x22);
            }
            D[pk + pl * LD] = x11; D[qk + pl * LD] = x21; D[pk + ql * LD] = x12; D[qk + ql * LD] = x22;
        }
        // U <- U J (columns lp, lq)
        if (U) {
            for (int e = tid; e < BW * TW; e += NT) {
                const int r = e & (TW - 1), kk = e >> 6;
                const R sn = pr.s[kk];
                if (sn != R(0)) {
                    const int pk = sh.lp[kk], qk = sh.lq[kk];
                    R x = U[r + pk * LD], y = U[r + qk * LD];
                    rot<R>(sn, pr.u[kk], x, y);
                    U[r + pk * LD] = x; U[r + qk * LD] = y;
                }
            }
        }
        __syncthreads();
    }
    return sh.nrot;
}

// ---------------------------------------------------------------------------
// 64 x 64 x 64 tile products in shared memory.
//   C = op(A) * B  with A, B, C column-major (leading dimension LD);
//   TRANS_A: op(A) = A^T.
// fp64: 8 warps, warp w owns rows 8w..8w+7 (8 fragments of 8 x 8 along n),
// mma.sync m8n8k4 (DMMA).  fp32: 4 x 4 register tiles per thread (FFMA).
// Results are returned in registers (acc) -- callers store them.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <bool TRANS_A>
__device__ __forceinline__ void tile_mm_acc(const double *A, const double *B, double (&acc)[8][2])
{
    constexpr int LD = Lay<double>::LD;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
    const int row = warp * 8 + g;
    #pragma unroll 4
    for (int ks = 0; ks < TW / 4; ++ks) {
        const int kk = ks * 4 + tig;
        const double a = TRANS_A ? A[kk + row * LD] : A[row + kk * LD];
        #pragma unroll
        for (int f = 0; f < 8; ++f) {
            const double b = B[kk + (f * 8 + g) * LD];
            dmma884(acc[f][0], acc[f][1], a, b);
        }
    }
}
template <bool TRANS_A>
__device__ __forceinline__ void tile_mm(const double *A, const double *B, double (&acc)[8][2])
{
    #pragma unroll
    for (int f = 0; f < 8; ++f) { acc[f][0] = 0.0; acc[f][1] = 0.0; }
    tile_mm_acc<TRANS_A>(A, B, acc);
}
// element (i, j) of the accumulator fragment f, slot e
__device__ __forceinline__ int acc_row() { return (threadIdx.x >> 5) * 8 + ((threadIdx.x & 31) >> 2); }
__device__ __forceinline__ int acc_col(int f, int e) { return f * 8 + 2 * (threadIdx.x & 3) + e; }

template <bool TRANS_A>
__device__ __forceinline__ void tile_mm(const float *A, const float *B, float (&acc)[4][4])
{
    constexpr int LD = Lay<float>::LD;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    #pragma unroll
    for (int u = 0; u < 4; ++u)
        #pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.f;
    #pragma unroll 4
    for (int kk = 0; kk < TW; ++kk) {
        float a[4], b[4];
        #pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = ty + 16 * u;
            a[u] = TRANS_A ? A[kk + i * LD] : A[i + kk * LD];
        }
        #pragma unroll
        for (int v = 0; v < 4; ++v) b[v] = B[kk + (tx + 16 * v) * LD];
        #pragma unroll
        for (int u = 0; u < 4; ++u)
            #pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = __fmaf_rn(a[u], b[v], acc[u][v]);
    }
}

template <typename R> struct Acc;
template <> struct Acc<double> {
    double v[8][2];
    template <typename F> __device__ __forceinline__ void each(F f)
    {
        const int r = acc_row();
        #pragma unroll
        for (int q = 0; q < 8; ++q) { f(r, acc_col(q, 0), v[q][0]); f(r, acc_col(q, 1), v[q][1]); }
    }
};
template <> struct Acc<float> {
    float v[4][4];
    template <typename F> __device__ __forceinline__ void each(F f)
    {
        const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
        #pragma unroll
        for (int u = 0; u < 4; ++u)
            #pragma unroll
            for (int w = 0; w < 4; ++w) f(ty + 16 * u, tx + 16 * w, v[u][w]);
    }
};

// load a 64 x 64 tile whose rows are the block-pair rows (rp) and columns given by colmap
template <typename R>
__device__ __forceinline__ void load_tile(R *dst, const R *__restrict__ src, int64_t ld, int2 rp, int2 cp)
{
    constexpr int LD = Lay<R>::LD;
    for (int e = threadIdx.x; e < TW * TW; e += NT) {
        const int li = e & (TW - 1), lj = e >> 6;
        dst[li + lj * LD] = src[gidx(rp, li) + (int64_t)gidx(cp, lj) * ld];
    }
}
template <typename R>
__device__ __forceinline__ void load_u(R *dst, const R *__restrict__ Uk)
{
    constexpr int LD = Lay<R>::LD;
    for (int e = threadIdx.x; e < TW * TW; e += NT) {
        const int li = e & (TW - 1), lj = e >> 6;
        dst[li + lj * LD] = Uk[li + lj * TW];
    }
}

}  // namespace blk
}  // namespace mpj
