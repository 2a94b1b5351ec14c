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
#include "mpj_block.cuh"

namespace mpj {

namespace {

using namespace blk;

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
    __shared__ InnerShared sh;
    __shared__ InnerParams<R> pr;
    const int k = blockIdx.x;
    const int mb = S.nb >> 1;
    const int2 bp = S.bsched[Rb * mb + k];
    for (int e = threadIdx.x; e < TW * TW; e += NT) {
        const int li = e & (TW - 1), lj = e >> 6;
        D[li + lj * LD] = T[gidx(bp, li) + (int64_t)gidx(bp, lj) * ldt];
        U[li + lj * LD] = (li == lj) ? R(1) : R(0);
    }
    const unsigned nrot = inner_rounds<R>(D, U, bp, Rb == 0, S.lsched, nu, rule, sh, pr);
    R *Uk = Ubuf + (size_t)k * TW * TW;
    for (int e = threadIdx.x; e < TW * TW; e += NT) {
        const int li = e & (TW - 1), lj = e >> 6;
        T[gidx(bp, li) + (int64_t)gidx(bp, lj) * ldt] = D[li + lj * LD];
        Uk[li + lj * TW] = U[li + lj * LD];
    }
    if (threadIdx.x == 0 && nrot) atomicAdd(cnt, (unsigned long long)nrot);
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

// M(:, P_c) <- M(:, P_c) U_c for every block pair c of block round Rb (M has
// `rows` rows): the column update of the one-sided (SVD) block variant.
template <typename R>
void launch_block_apply_cols(R *M, int64_t ld, int rows, const DevSched &ds, int Rb, const R *Ubuf,
                             cudaStream_t st)
{
    constexpr int LD = Lay<R>::LD;
    Sched S;
    S.bsched = ds.bsched; S.lsched = ds.lsched; S.b = ds.b; S.nb = ds.nb; S.np = ds.np;
    const int mb = ds.nb / 2;
    const size_t sm_apply = 3 * TW * LD * sizeof(R);
    MPJ_CK_VOID(cudaFuncSetAttribute(k_block_apply<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_apply));
    const int ntV = ((rows + TW - 1) / TW) * mb;
    k_block_apply<R><<<ntV, NT, sm_apply, st>>>(nullptr, 0, M, ld, rows, S, Rb, Ubuf, 0);
    count_launch();
}
template void launch_block_apply_cols<double>(double *, int64_t, int, const DevSched &, int, const double *, cudaStream_t);
template void launch_block_apply_cols<float>(float *, int64_t, int, const DevSched &, int, const float *, cudaStream_t);

template size_t block_scratch_bytes<double>(int, int);
template size_t block_scratch_bytes<float>(int, int);
template mpj_status block_sweep<double>(double *, int64_t, double *, int64_t, int, const DevSched &, double,
                                        int, unsigned long long *, void *, cudaStream_t);
template mpj_status block_sweep<float>(float *, int64_t, float *, int64_t, int, const DevSched &, float, int,
                                       unsigned long long *, void *, cudaStream_t);

}  // namespace mpj
