// k_block.cu -- block variant of the parallel-ordered Jacobi sweep (b = 32).
//
// The ordering (reading R1) groups the n_p - 1 rounds of a sweep into nb - 1
// block rounds.  In block round R, block pair k = (I, J) (merry-go-round on
// blocks) owns the 2b = 64 indices I*32.. and J*32.., and the b (or
// 2b-1 in R = 0) rounds of the block round only pair indices inside their own
// block pair.  Their rotation parameters depend only on the 64 x 64 diagonal
// block of the pair, so (exact arithmetic) the block round equals
//   K3 (k_block_solve): for each block pair, run its inner rounds on the
//       64 x 64 diagonal block in shared memory (same Lemma 3.1 arithmetic,
//       same canonical tile order as the scalar kernels) and accumulate the
//       product of its rotations U_k = J_1 J_2 ... (64 x 64);
//   K4 (k_block_apply): T(P_a, P_c) <- U_a^T T(P_a, P_c) U_c for every pair
//       of block pairs a < c (mirrored into (c, a)), and
//       V(:, P_c) <- V(:, P_c) U_c -- dense 64 x 64 x 64 products on the FP64
//       tensor pipe (mma.sync m8n8k4 -> DMMA) for fp64, FFMA for fp32.
// Diagonal blocks come from K3 directly.  Per block round and n_p = 8192 this
// is 8.5e9 + 8.6e9 flop (T upper tiles + V) on 1.8 GB of HBM traffic.
#include "mpj_device.cuh"
#include "mpj_internal.h"

namespace mpj {

namespace {

constexpr int BW = 32;   // b
constexpr int TW = 64;   // 2b
constexpr int NT = 256;  // threads per CTA

template <typename R> struct Lay;
template <> struct Lay<double> { static constexpr int LD = 68; };   // 2 wavefronts / DMMA frag
template <> struct Lay<float> { static constexpr int LD = 65; };    // conflict-free SIMT tiles

// global index of local index li (0..63) of block pair (I, J)
__device__ __forceinline__ int gidx(int2 bp, int li) { return li < BW ? bp.x * BW + li : bp.y * BW + (li - BW); }

// ---------------------------------------------------------------------------
// K3: inner solver.  One CTA per block pair.
// ---------------------------------------------------------------------------
template <typename R>
__global__ void __launch_bounds__(NT) k_block_solve(R *__restrict__ T, int64_t ldt, Sched S, int Rb, R nu,
                                                    int rule, R *__restrict__ Ubuf,
                                                    unsigned long long *__restrict__ cnt)
{
    constexpr int LD = Lay<R>::LD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R *D = (R *)smem_raw;          // 64 x LD, column-major
    R *U = D + TW * LD;            // 64 x LD
    __shared__ R st_[BW], ss_[BW], su_[BW];
    __shared__ int lp_[BW], lq_[BW], gp_[BW];
    __shared__ unsigned nrot;

    const int k = blockIdx.x;
    const int mb = S.nb >> 1;
    const int2 bp = S.bsched[Rb * mb + k];
    const int tid = threadIdx.x;

    // load the diagonal block and U = I
    for (int e = tid; e < TW * TW; e += NT) {
        const int li = e & (TW - 1), lj = e >> 6;
        D[li + lj * LD] = T[gidx(bp, li) + (int64_t)gidx(bp, lj) * ldt];
        U[li + lj * LD] = (li == lj) ? R(1) : R(0);
    }
    if (tid == 0) nrot = 0;
    __syncthreads();

    const int nrounds = (Rb == 0) ? (BW - 1) + BW : BW;
    for (int s = 0; s < nrounds; ++s) {
        if (tid < BW) {
            int a, c;
            if (Rb == 0 && s < BW - 1) {        // intra-block rounds (block round 0 only)
                const int hb = BW / 2, w = tid;
                const int2 lp = S.lsched[s * hb + (w < hb ? w : w - hb)];
                const int off = (w < hb) ? 0 : BW;
                a = off + lp.x; c = off + lp.y;
            } else {
                const int sc = (Rb == 0) ? s - (BW - 1) : s;
                a = tid;
                int j = tid + sc; if (j >= BW) j -= BW;
                c = BW + j;
            }
            const int ga = gidx(bp, a), gc = gidx(bp, c);
            const int lp = ga < gc ? a : c, lq = ga < gc ? c : a;
            R t, sn, u;
            const int did = rot_params<R>(D[lp + lp * LD], D[lq + lq * LD], D[lp + lq * LD], nu, rule, t, sn, u);
            lp_[tid] = lp; lq_[tid] = lq; gp_[tid] = ga < gc ? ga : gc;
            st_[tid] = t; ss_[tid] = sn; su_[tid] = u;
            const unsigned bal = __ballot_sync(0xffffffffu, did);
            if (tid == 0) nrot += __popc(bal);
        }
        __syncthreads();
        // D <- J^T D J on the 32 x 32 pair tiles (same canonical order as k_round_apply)
        for (int e = tid; e < BW * BW; e += NT) {
            const int kk = e & (BW - 1), ll = e >> 5;
            const int pk = lp_[kk], qk = lq_[kk];
            if (kk == ll) {
                const R apq = D[pk + qk * LD], t = st_[kk];
                D[pk + pk * LD] = fmaR(-t, apq, D[pk + pk * LD]);
                D[qk + qk * LD] = fmaR(t, apq, D[qk + qk * LD]);
                D[pk + qk * LD] = R(0);
                D[qk + pk * LD] = R(0);
                continue;
            }
            const int pl = lp_[ll], ql = lq_[ll];
            R x11 = D[pk + pl * LD], x21 = D[qk + pl * LD], x12 = D[pk + ql * LD], x22 = D[qk + ql * LD];
            const R sk = ss_[kk], uk = su_[kk], sl = ss_[ll], ul = su_[ll];
            if (gp_[kk] < gp_[ll]) {
                rot<R>(sk, uk, x11, x21); rot<R>(sk, uk, x12, x22);
                rot<R>(sl, ul, x11, x12); rot<R>(sl, ul, x21, x22);
            } else {
                rot<R>(sl, ul, x11, x12); rot<R>(sl, ul, x21, x22);
                rot<R>(sk, uk, x11, x21); rot<R>(sk, uk, x12, x22);
            }
            D[pk + pl * LD] = x11; D[qk + pl * LD] = x21; D[pk + ql * LD] = x12; D[qk + ql * LD] = x22;
        }
        // U <- U J (columns lp, lq)
        for (int e = tid; e < BW * TW; e += NT) {
            const int r = e & (TW - 1), kk = e >> 6;
            const R sn = ss_[kk];
            if (sn != R(0)) {
                const int pk = lp_[kk], qk = lq_[kk];
                R x = U[r + pk * LD], y = U[r + qk * LD];
                rot<R>(sn, su_[kk], x, y);
                U[r + pk * LD] = x; U[r + qk * LD] = y;
            }
        }
        __syncthreads();
    }
    // write back the diagonal block and U
    R *Uk = Ubuf + (size_t)k * TW * TW;
    for (int e = tid; e < TW * TW; e += NT) {
        const int li = e & (TW - 1), lj = e >> 6;
        T[gidx(bp, li) + (int64_t)gidx(bp, lj) * ldt] = D[li + lj * LD];
        Uk[li + lj * TW] = U[li + lj * LD];
    }
    if (tid == 0 && nrot) atomicAdd(cnt, (unsigned long long)nrot);
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
__device__ __forceinline__ void tile_mm(const double *A, const double *B, double (&acc)[8][2])
{
    constexpr int LD = Lay<double>::LD;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
    #pragma unroll
    for (int f = 0; f < 8; ++f) { acc[f][0] = 0.0; acc[f][1] = 0.0; }
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

// ---------------------------------------------------------------------------
// K4: apply.  blockIdx.x < ntT: T tile (a, c), a < c; else V tile.
// ---------------------------------------------------------------------------
template <typename R>
__global__ void __launch_bounds__(NT) k_block_apply(R *__restrict__ T, int64_t ldt, R *__restrict__ V,
                                                    int64_t ldv, int vrows, Sched S, int Rb,
                                                    const R *__restrict__ Ubuf, int ntT)
{
    constexpr int LD = Lay<R>::LD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R *X = (R *)smem_raw;
    R *Ua = X + TW * LD;
    R *Uc = Ua + TW * LD;
    const int mb = S.nb >> 1;
    const int2 *bsr = S.bsched + Rb * mb;
    int idx = blockIdx.x;
    if (idx < ntT) {
        // upper-triangular decode: idx -> (a, c), a < c
        int c = (int)((1.0 + sqrt(1.0 + 8.0 * idx)) * 0.5);
        while (c * (c - 1) / 2 > idx) --c;
        while ((c + 1) * c / 2 <= idx) ++c;
        const int a = idx - c * (c - 1) / 2;
        const int2 pa = bsr[a], pc = bsr[c];
        load_tile<R>(X, T, ldt, pa, pc);
        load_u<R>(Ua, Ubuf + (size_t)a * TW * TW);
        load_u<R>(Uc, Ubuf + (size_t)c * TW * TW);
        __syncthreads();
        Acc<R> y;
        tile_mm<true>(Ua, X, y.v);                 // Y = Ua^T X
        __syncthreads();
        y.each([&](int i, int j, R v) { X[i + j * LD] = v; });
        __syncthreads();
        Acc<R> w;
        tile_mm<false>(X, Uc, w.v);                // W = Y Uc
        __syncthreads();
        w.each([&](int i, int j, R v) { X[i + j * LD] = v; });
        __syncthreads();
        // store W into (a, c) and W^T into (c, a); both loops coalesced along rows
        for (int e = threadIdx.x; e < TW * TW; e += NT) {
            const int li = e & (TW - 1), lj = e >> 6;
            T[gidx(pa, li) + (int64_t)gidx(pc, lj) * ldt] = X[li + lj * LD];
            T[gidx(pc, li) + (int64_t)gidx(pa, lj) * ldt] = X[lj + li * LD];
        }
    } else {
        idx -= ntT;
        const int c = idx % mb, rt = idx / mb;
        const int2 pc = bsr[c];
        const int r0 = rt * TW;
        // X = V(r0:r0+64, P_c)
        for (int e = threadIdx.x; e < TW * TW; e += NT) {
            const int li = e & (TW - 1), lj = e >> 6;
            const int gi = r0 + li;
            X[li + lj * LD] = gi < vrows ? V[gi + (int64_t)gidx(pc, lj) * ldv] : R(0);
        }
        load_u<R>(Uc, Ubuf + (size_t)c * TW * TW);
        __syncthreads();
        Acc<R> w;
        tile_mm<false>(X, Uc, w.v);
        __syncthreads();
        w.each([&](int i, int j, R v) { X[i + j * LD] = v; });
        __syncthreads();
        for (int e = threadIdx.x; e < TW * TW; e += NT) {
            const int li = e & (TW - 1), lj = e >> 6;
            const int gi = r0 + li;
            if (gi < vrows) V[gi + (int64_t)gidx(pc, lj) * ldv] = X[li + lj * LD];
        }
    }
}

}  // namespace

template <typename R>
size_t block_scratch_bytes(int np, int b)
{
    (void)b;
    const int mb = np / (2 * BW);
    return (size_t)mb * TW * TW * sizeof(R);
}

template <typename R>
mpj_status block_sweep(R *T, int64_t ldt, R *V, int64_t ldv, int vrows, const DevSched &ds, R nu, int rule,
                       unsigned long long *cnt, void *scratch, cudaStream_t st)
{
    if (ds.b != BW) { set_error("block variant needs b = 32"); return MPJ_ERR_INVALID; }
    constexpr int LD = Lay<R>::LD;
    Sched S;
    S.bsched = ds.bsched; S.lsched = ds.lsched; S.b = ds.b; S.nb = ds.nb; S.np = ds.np;
    const int mb = ds.nb / 2;
    R *Ubuf = (R *)scratch;
    const size_t sm_solve = 2 * TW * LD * sizeof(R);
    const size_t sm_apply = 3 * TW * LD * sizeof(R);
    static bool attr_done[2] = {false, false};
    const int ti = sizeof(R) == 8 ? 0 : 1;
    if (!attr_done[ti]) {
        MPJ_CK(cudaFuncSetAttribute(k_block_solve<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_solve));
        MPJ_CK(cudaFuncSetAttribute(k_block_apply<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_apply));
        attr_done[ti] = true;
    }
    const int ntT = mb * (mb - 1) / 2;
    const int ntV = ((vrows + TW - 1) / TW) * mb;
    const char *nsolve = sizeof(R) == 8 ? "block_solve_f64" : "block_solve_f32";
    const char *napply = sizeof(R) == 8 ? "block_apply_f64" : "block_apply_f32";
    const bool prof = prof_on();
    for (int Rb = 0; Rb < ds.nb - 1; ++Rb) {
        if (prof) prof_mark(nsolve, st, true);
        k_block_solve<R><<<mb, NT, sm_solve, st>>>(T, ldt, S, Rb, nu, rule, Ubuf, cnt);
        if (prof) { prof_mark(nsolve, st, false); prof_mark(napply, st, true); }
        k_block_apply<R><<<ntT + ntV, NT, sm_apply, st>>>(T, ldt, V, ldv, vrows, S, Rb, Ubuf, ntT);
        if (prof) prof_mark(napply, st, false);
        count_launch(2);
    }
    return MPJ_OK;
}

template size_t block_scratch_bytes<double>(int, int);
template size_t block_scratch_bytes<float>(int, int);
template mpj_status block_sweep<double>(double *, int64_t, double *, int64_t, int, const DevSched &, double,
                                        int, unsigned long long *, void *, cudaStream_t);
template mpj_status block_sweep<float>(float *, int64_t, float *, int64_t, int, const DevSched &, float, int,
                                       unsigned long long *, void *, cudaStream_t);

}  // namespace mpj
