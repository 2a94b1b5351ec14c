// k_mg.cu -- multi-GPU (column-block partitioned) Alg. 3, SURVEY §8(e).
//
// G ranks, one process (and GPU) each.  The mb = n_p/64 block-pair slots of
// the block merry-go-round (reading R1) are split into G contiguous ranges;
// rank g owns the 64 columns of each of its slots -- all n_p rows of those
// columns of T and V -- so the right rotations (columns) and the row mixes
// of its columns are local.  Per block round:
//   K3 (k_mg_solve)   inner rounds of the rank's block pairs (the 64 x 64
//                     diagonal blocks are local; they are symmetrised on load
//                     because the two triangles of T come from different
//                     ranks' tiles) -> U of each local slot
//   all-gather U      every rank needs every U_a for the left rotations of
//                     its columns (ncclAllGather, 32 KB per slot)
//   K4 (k_mg_apply)   T(P_a, P_c) <- U_a^T T(P_a, P_c) U_c for every slot a
//                     and own slot c (no mirror: (c, a) is another rank's),
//                     V(:, P_c) <- V(:, P_c) U_c  (DMMA / FFMA tiles)
//   exchange          the merry-go-round moves one block (32 columns of T and
//                     of V) across each rank boundary in each direction
//                     (ncclSend / ncclRecv, staged)
// Per sweep: ||off(T)||_F^2 partials all-reduced (8 bytes).
// Blocks keep a fixed physical position on their rank while they stay; the
// host plan (identical on every rank) tracks slot -> block -> position.
// Emulation: the same code runs G ranks in one process on one GPU with shared
// U buffers and device copies instead of NCCL (tests; no kernel waits on
// another).
#include <cmath>
#include <nccl.h>

#include "mpj_block.cuh"
#include "mpj_device.cuh"
#include "mpj_internal.h"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <vector>

namespace mpj {
namespace {

using namespace blk;

struct SlotInfo {
    int top, bot;     // global block ids (row indexing, orientation)
    int ptop, pbot;   // physical column bases (multiples of 32) in the rank's local T / V
};

__device__ __forceinline__ int pcol(const SlotInfo &s, int lj) { return lj < BW ? s.ptop + lj : s.pbot + lj - BW; }

template <typename R>
__global__ void __launch_bounds__(NTW) k_mg_solve(R *__restrict__ T, int64_t ldt, const SlotInfo *__restrict__ slots,
                                                  int slot0, const int2 *__restrict__ lsched, int intra, R nu,
                                                  int rule, R *__restrict__ Ubuf, unsigned long long *__restrict__ cnt)
{
    constexpr int LD = LayK<R>::LD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R *D0 = (R *)smem_raw;
    R *D1 = D0 + TW * LD;
    R *U = D1 + TW * LD;
    __shared__ unsigned nrot;
    __shared__ WideParams<R> P[2];
    const SlotInfo si = slots[blockIdx.x];
    const int2 bp = make_int2(si.top, si.bot);
    for (int e = threadIdx.x; e < TW * TW; e += NTW) {
        const int li = e & (TW - 1), lj = e >> 6;
        D0[li + lj * LD] = T[gidx(bp, li) + (int64_t)pcol(si, lj) * ldt];
        U[li + lj * LD] = (li == lj) ? R(1) : R(0);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < TW * TW; e += NTW) {      // symmetrise (rounding-level asymmetry)
        const int li = e & (TW - 1), lj = e >> 6;
        if (li < lj) {
            const R v = (D0[li + lj * LD] + D0[lj + li * LD]) * R(0.5);
            D1[li + lj * LD] = v;
            D1[lj + li * LD] = v;
        } else if (li == lj) {
            D1[li + lj * LD] = D0[li + lj * LD];
        }
    }
    __syncthreads();
    const R *D = inner_rounds_wide<R>(D1, D0, U, bp, intra != 0, lsched, nu, rule, P, &nrot);
    // slot stride: 64 x 64 fp64 words; an fp32 slot holds U and then U^T (the
    // k-major operand of the fp32 apply), so one all-gather carries both
    R *Uk = Ubuf + (size_t)(slot0 + blockIdx.x) * TW * TW * (8 / sizeof(R));
    for (int e = threadIdx.x; e < TW * TW; e += NTW) {
        const int li = e & (TW - 1), lj = e >> 6;
        T[gidx(bp, li) + (int64_t)pcol(si, lj) * ldt] = D[li + lj * LD];
        Uk[li + lj * TW] = U[li + lj * LD];
        if (sizeof(R) == 4) Uk[TW * TW + li + lj * TW] = U[lj + li * LD];
    }
    if (threadIdx.x == 0 && nrot) atomicAdd(cnt, (unsigned long long)nrot);
}

__device__ __forceinline__ void mg_cp16(void *dst, const void *src, int bytes)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}

// uid[s] = 1 iff the (all-gathered) rotation block of slot s is exactly I --
// no rotation happened there (a rotation with s = 0 is the identity too), so
// the tiles it multiplies are unchanged: exact to skip.  One CTA per slot.
template <typename R>
__global__ void __launch_bounds__(256) k_mg_uid(const R *__restrict__ Ubuf, int *__restrict__ uid,
                                                int *__restrict__ nid)
{
    const R *U = Ubuf + (size_t)blockIdx.x * TW * TW * (8 / sizeof(R));
    int ok = 1;
    for (int e = threadIdx.x; e < TW * TW; e += blockDim.x)
        ok &= (U[e] == ((e & (TW - 1)) == (e >> 6) ? R(1) : R(0)));
    ok = __syncthreads_and(ok);
    if (threadIdx.x == 0) {
        uid[blockIdx.x] = ok;
        if (ok) atomicAdd(nid, 1);
    }
}

struct MgApply {
    void *T, *V;
    int64_t ld;               // leading dimension of local T and V (= n_p)
    int vrows;                // n_p
    const SlotInfo *slots;    // local slots this round
    const int2 *gslots;       // global slot -> (top, bot) this round
    int slot0, mb, mbl;
    const void *Ubuf;
    const int *uid;           // per global slot: U exactly I
    const int *nid;           // number of such slots this round
    int ntT, ntV;
};

// item decode shared by the mg apply kernels: T tile (local slot cl, global
// slot a != own) or V tile (local slot cl, row tile r0)
__device__ __forceinline__ void mg_decode(const MgApply &p, int item, bool &ttile, int &cl, int &a, int &r0)
{
    ttile = item < p.ntT;
    a = 0;
    r0 = 0;
    if (ttile) {
        cl = item / (p.mb - 1);
        const int ai = item - cl * (p.mb - 1);
        a = ai < p.slot0 + cl ? ai : ai + 1;
    } else {
        const int idx = item - p.ntT;
        cl = idx % p.mbl;
        r0 = (idx / p.mbl) * TW;
    }
}

__device__ __forceinline__ bool mg_item_identity(const MgApply &p, int item)
{
    bool tt;
    int cl, a, r0;
    mg_decode(p, item, tt, cl, a, r0);
    const int cg = p.slot0 + cl;
    return p.uid[cg] && (!tt || p.uid[a]);
}

template <typename R>
__global__ void __launch_bounds__(NT) k_mg_apply(MgApply p)
{
    constexpr int LD = Lay<R>::LD, EPC = 16 / sizeof(R), CPC = TW / EPC;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R *x = (R *)smem_raw;
    R *ua = x + TW * LD;
    R *uc = ua + TW * LD;
    const R *Ub = (const R *)p.Ubuf;
    const int total = p.ntT + p.ntV;
    const bool skips = p.uid && *p.nid > 0;
    // this CTA's items blockIdx.x + k G; the second half of the grid walks them
    // backwards so the two CTAs of an SM do not load and store in lockstep
    const int G = gridDim.x;
    const int K = (int)blockIdx.x < total ? (total - 1 - (int)blockIdx.x) / G + 1 : 0;
    const bool rev = 2 * (int)blockIdx.x >= G;
    for (int kk = 0; kk < K; ++kk) {
        const int item = (int)blockIdx.x + (rev ? K - 1 - kk : kk) * G;
        if (skips && mg_item_identity(p, item)) continue;
        bool ttile;
        int cl, a, r0;
        mg_decode(p, item, ttile, cl, a, r0);
        const SlotInfo sc = p.slots[cl];
        const int cg = p.slot0 + cl;
        R *M = (R *)(ttile ? p.T : p.V);
        const int2 ra = ttile ? p.gslots[a] : make_int2(0, 0);
        for (int e = threadIdx.x; e < TW * CPC; e += NT) {
            const int lj = e / CPC, li = (e - lj * CPC) * EPC;
            const int64_t col = (int64_t)pcol(sc, lj) * p.ld;
            if (ttile) {
                mg_cp16(x + li + lj * LD, M + gidx(ra, li) + col, 16);
                mg_cp16(ua + li + lj * LD, Ub + (size_t)a * TW * TW * (8 / sizeof(R)) + li + lj * TW, 16);
            } else {
                const int rem = p.vrows - (r0 + li);
                const int bytes = rem >= EPC ? 16 : (rem > 0 ? rem * (int)sizeof(R) : 0);
                mg_cp16(x + li + lj * LD, M + (bytes ? (int64_t)(r0 + li) : 0) + col, bytes);
            }
            mg_cp16(uc + li + lj * LD, Ub + (size_t)cg * TW * TW * (8 / sizeof(R)) + li + lj * TW, 16);
        }
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();
        Acc<R> acc;
        // identity blocks (fp64): U_c = I -> W = U_a^T X only; U_a = I -> W = X U_c only
        const bool ic = skips && ttile && p.uid[cg];
        const bool ia = skips && ttile && p.uid[a];
        if (ttile && !ia) {
            tile_mm<true>(ua, x, acc);                  // Y = U_a^T X
            __syncthreads();
            acc.each([&](int i, int j, R v) { x[i + j * LD] = v; });
            __syncthreads();
        }
        if (!ic) tile_mm<false>(x, uc, acc);            // W = Y U_c  (or X U_c)
        __syncthreads();                                // shared memory free: store from registers
        if constexpr (sizeof(R) == 8) {
            acc.each2([&](int i, int j, R v0, R v1) {   // W(i, j), W(i, j + 1); j even, same 32-column block
                const int64_t col = (int64_t)pcol(sc, j) * p.ld;
                if (ttile) {
                    const int64_t gi = gidx(ra, i);
                    M[gi + col] = v0;
                    M[gi + col + p.ld] = v1;
                } else if (r0 + i < p.vrows) {
                    M[(r0 + i) + col] = v0;
                    M[(r0 + i) + col + p.ld] = v1;
                }
            });
            continue;
        }
        acc.each([&](int i, int j, R v) { x[i + j * LD] = v; });
        __syncthreads();
        for (int e = threadIdx.x; e < TW * CPC; e += NT) {
            const int lj = e / CPC, li = (e - lj * CPC) * EPC;
            const int64_t col = (int64_t)pcol(sc, lj) * p.ld;
            if (ttile) {
                *(int4 *)(M + gidx(ra, li) + col) = *(const int4 *)(x + li + lj * LD);
            } else if (r0 + li + EPC <= p.vrows) {
                *(int4 *)(M + (r0 + li) + col) = *(const int4 *)(x + li + lj * LD);
            } else {
                for (int q = 0; q < EPC && r0 + li + q < p.vrows; ++q) M[r0 + li + q + col] = x[li + q + lj * LD];
            }
        }
        __syncthreads();
    }
}

// fp64 apply of the partitioned sweep with two buffers per 256-thread group
// (three groups per SM), as k_block.cu's apply_x3_body: X / Y share one
// buffer, U_a and U_c the other (U_c's k-chunks stream into U_a's dead rows
// during Y = U_a^T X); k-chunked cp.async loads; results from the
// accumulators to global memory.
__device__ __forceinline__ void mg_wait_le(int n)
{
    switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;\n" ::); break;
    case 1: asm volatile("cp.async.wait_group 1;\n" ::); break;
    case 2: asm volatile("cp.async.wait_group 2;\n" ::); break;
    default: asm volatile("cp.async.wait_group 3;\n" ::); break;
    }
}

// GROUPED (the default launch): one CTA per SM of three 256-thread groups,
// each with its own buffers and named barrier, taking the SM's items from a
// shared-memory counter (k_block.cu, apply_x3_body: separate CTAs of one SM
// run at unequal speeds and finish far apart)
template <bool GROUPED>
__device__ __forceinline__ void mg_apply_x3_body(const MgApply &p, unsigned char *smem_raw)
{
    constexpr int LD = Lay<double>::LD, EPC = 2, CPC = TW / EPC;
    const int grp = GROUPED ? (int)(threadIdx.x >> 8) : 0;
    double *xb = (double *)smem_raw + (size_t)grp * 2 * TW * LD, *ub = xb + TW * LD;
    const double *Ub = (const double *)p.Ubuf;
    const int total = p.ntT + p.ntV;
    const bool skips = p.uid && *p.nid > 0;
    const int tid = GROUPED ? (int)(threadIdx.x & (NT - 1)) : (int)threadIdx.x;
    const int G = gridDim.x;
    const int K = (int)blockIdx.x < total ? (total - 1 - (int)blockIdx.x) / G + 1 : 0;
    const int phase = GROUPED ? 0 : (int)(3 * (int64_t)blockIdx.x / G);
    const int k0 = (phase * K) / 3;
    auto __syncthreads = [&]() {
        if constexpr (GROUPED) asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "r"(NT) : "memory");
        else ::__syncthreads();
    };
    int *s_ctr = (int *)(smem_raw + (size_t)3 * 2 * TW * LD * sizeof(double));
    int *s_nxt = s_ctr + 1 + 2 * grp;
    if constexpr (GROUPED) {
        if (threadIdx.x == 0) *s_ctr = 0;
        ::__syncthreads();
    }
    for (int kk = 0, it = 0;; ++kk, ++it) {
        if constexpr (GROUPED) {
            if (tid == 0) s_nxt[it & 1] = atomicAdd(s_ctr, 1);   // rewritten two barriers later
            __syncthreads();
            kk = s_nxt[it & 1];
        }
        if (kk >= K) break;
        int k = kk + k0;
        if (k >= K) k -= K;
        const int item = (int)blockIdx.x + k * G;
        if (skips && mg_item_identity(p, item)) continue;
        bool ttile;
        int cl, a, r0;
        mg_decode(p, item, ttile, cl, a, r0);
        const SlotInfo sc = p.slots[cl];
        const int cg = p.slot0 + cl;
        double *M = (double *)(ttile ? p.T : p.V);
        const double *Ucg = Ub + (size_t)cg * TW * TW;
        Acc<double> acc;
        if (ttile) {
            const int2 ra = p.gslots[a];
            const double *Uag = Ub + (size_t)a * TW * TW;
            const bool ia = skips && p.uid[a], ic = skips && p.uid[cg];
            if (!ia && !ic) {
                for (int ch = 0; ch < 4; ++ch) {                 // X and U_a rows 16ch.., 4 groups
                    for (int e = tid; e < TW * 8; e += NT) {
                        const int lj = e >> 3, li = 16 * ch + 2 * (e & 7);
                        mg_cp16(xb + li + lj * LD, M + gidx(ra, li) + (int64_t)pcol(sc, lj) * p.ld, 16);
                        mg_cp16(ub + li + lj * LD, Uag + li + lj * TW, 16);
                    }
                    asm volatile("cp.async.commit_group;\n" ::);
                }
                tile_mm_chunked<true>(ub, xb, acc, [&](int ch) {     // Y = U_a^T X
                    mg_wait_le(ch == 0 ? 3 : 2);
                    __syncthreads();
                    if (ch > 0) {                                    // U_c rows of chunk ch-1
                        for (int e = tid; e < TW * 8; e += NT) {
                            const int lj = e >> 3, li = 16 * (ch - 1) + 2 * (e & 7);
                            mg_cp16(ub + li + lj * LD, Ucg + li + lj * TW, 16);
                        }
                        asm volatile("cp.async.commit_group;\n" ::);
                    }
                });
                __syncthreads();
                for (int e = tid; e < TW * 8; e += NT) {
                    const int lj = e >> 3, li = 48 + 2 * (e & 7);
                    mg_cp16(ub + li + lj * LD, Ucg + li + lj * TW, 16);
                }
                asm volatile("cp.async.commit_group;\n" ::);
                acc.each([&](int i, int j, double v) { xb[i + j * LD] = v; });   // Y
                tile_mm_chunked<false>(xb, ub, acc, [&](int ch) { mg_wait_le(3 - ch); __syncthreads(); });
            } else {
                for (int e = tid; e < TW * CPC; e += NT) {
                    const int lj = e / CPC, li = (e - lj * CPC) * EPC;
                    mg_cp16(xb + li + lj * LD, M + gidx(ra, li) + (int64_t)pcol(sc, lj) * p.ld, 16);
                    mg_cp16(ub + li + lj * LD, (ia ? Ucg : Uag) + li + lj * TW, 16);
                }
                asm volatile("cp.async.commit_group;\n" ::);
                asm volatile("cp.async.wait_group 0;\n" ::);
                __syncthreads();
                if (ia) tile_mm<false>(xb, ub, acc);             // W = X U_c
                else tile_mm<true>(ub, xb, acc);                 // W = U_a^T X
            }
            __syncthreads();
            acc.each2([&](int i, int j, double v0, double v1) {
                const int64_t gi = gidx(ra, i), col = (int64_t)pcol(sc, j) * p.ld;
                M[gi + col] = v0;
                M[gi + col + p.ld] = v1;
            });
        } else {
            for (int ch = 0; ch < 4; ++ch) {
                for (int e = tid; e < 16 * CPC; e += NT) {       // X columns 16ch..
                    const int lj = 16 * ch + e / CPC, li = (e % CPC) * EPC;
                    const int rem = p.vrows - (r0 + li);
                    const int bytes = rem >= EPC ? 16 : (rem > 0 ? rem * 8 : 0);
                    mg_cp16(xb + li + lj * LD, M + (bytes ? (int64_t)(r0 + li) : 0) + (int64_t)pcol(sc, lj) * p.ld,
                            bytes);
                }
                for (int e = tid; e < TW * 8; e += NT) {         // U_c rows 16ch..
                    const int lj = e >> 3, li = 16 * ch + 2 * (e & 7);
                    mg_cp16(ub + li + lj * LD, Ucg + li + lj * TW, 16);
                }
                asm volatile("cp.async.commit_group;\n" ::);
            }
            tile_mm_chunked<false>(xb, ub, acc, [&](int ch) { mg_wait_le(3 - ch); __syncthreads(); });
            __syncthreads();
            acc.each2([&](int i, int j, double v0, double v1) {
                if (r0 + i < p.vrows) {
                    const int64_t col = (int64_t)pcol(sc, j) * p.ld;
                    M[(r0 + i) + col] = v0;
                    M[(r0 + i) + col + p.ld] = v1;
                }
            });
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
}

__global__ void __launch_bounds__(3 * NT, 1) k_mg_apply_f64g3(MgApply p)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    mg_apply_x3_body<true>(p, smem_raw);
}

// fp32 apply of the partitioned sweep: 128-thread CTAs with 8 x 4 FFMA tiles
// (4 CTAs/SM; k-major operands U^T from the slot's second half).  T tiles:
// Z = X U_c with X as stored (rows of slot a, own columns), then W = U_a^T Z
// from Z^T staged k-major (U_a = I: W = Z, U_a^T not loaded); V tiles: X U_c.
__device__ __forceinline__ void store_T84(const Acc84 &acc, float *CT, int tid)
{
    constexpr int LD = Lay<float>::LD;
    const int r = 4 * (tid & 7), c = 4 * (tid >> 3);
    #pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int row = r + (u & 3) + (u >> 2) * 32;
        *(float4 *)(CT + c + row * LD) = make_float4(acc.v[u][0], acc.v[u][1], acc.v[u][2], acc.v[u][3]);
    }
}

__global__ void __launch_bounds__(128) k_mg_apply_f32(MgApply p)
{
    constexpr int LD = Lay<float>::LD, EPC = 4, CPC = TW / EPC, NTH = 128;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *x = (float *)smem_raw, *uaT = x + TW * LD, *ucT = uaT + TW * LD;
    const float *Ub = (const float *)p.Ubuf;         // slot s: U at 8192 s, U^T at 8192 s + 4096
    const int total = p.ntT + p.ntV;
    const bool skips = p.uid && *p.nid > 0;
    const int tid = threadIdx.x;
    Acc84 acc;
    const int G = gridDim.x;
    const int K = (int)blockIdx.x < total ? (total - 1 - (int)blockIdx.x) / G + 1 : 0;
    const bool rev = (4 * (int)blockIdx.x / G) & 1;   // alternate directions among the CTAs of an SM
    for (int kk = 0; kk < K; ++kk) {
        const int item = (int)blockIdx.x + (rev ? K - 1 - kk : kk) * G;
        if (skips && mg_item_identity(p, item)) continue;
        bool ttile;
        int cl, a, r0;
        mg_decode(p, item, ttile, cl, a, r0);
        const SlotInfo sc = p.slots[cl];
        const int cg = p.slot0 + cl;
        float *M = (float *)(ttile ? p.T : p.V);
        const int2 ra = ttile ? p.gslots[a] : make_int2(0, 0);
        const bool two = ttile && !(skips && p.uid[a]);   // U_a^T Z needed
        for (int e = tid; e < TW * CPC; e += NTH) {
            const int lj = e / CPC, li = (e - lj * CPC) * EPC;
            const int64_t col = (int64_t)pcol(sc, lj) * p.ld;
            if (ttile) {
                mg_cp16(x + li + lj * LD, M + gidx(ra, li) + col, 16);
                if (two) mg_cp16(uaT + li + lj * LD, Ub + (size_t)a * 2 * TW * TW + TW * TW + li + lj * TW, 16);
            } else {
                const int rem = p.vrows - (r0 + li);
                const int bytes = rem >= EPC ? 16 : (rem > 0 ? rem * (int)sizeof(float) : 0);
                mg_cp16(x + li + lj * LD, M + (bytes ? (int64_t)(r0 + li) : 0) + col, bytes);
            }
            mg_cp16(ucT + li + lj * LD, Ub + (size_t)cg * 2 * TW * TW + TW * TW + li + lj * TW, 16);
        }
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();
        tile_op84_t(x, ucT, acc, tid);                      // Z = X U_c
        __syncthreads();
        if (two) {
            store_T84(acc, x, tid);                          // Z^T, k-major for the next product
            __syncthreads();
            tile_op84_t(uaT, x, acc, tid);                   // W = U_a^T Z
            __syncthreads();
        }
        // W from the accumulators: rows r..r+3 and r+32..r+35 (float4 each) of columns cc..cc+3
        const int r = 4 * (tid & 7), cc = 4 * (tid >> 3);
        #pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int64_t col = (int64_t)pcol(sc, cc + w) * p.ld;
            #pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float4 v = make_float4(acc.v[4 * h][w], acc.v[4 * h + 1][w], acc.v[4 * h + 2][w], acc.v[4 * h + 3][w]);
                const int li = r + 32 * h;
                if (ttile) {
                    *(float4 *)(M + gidx(ra, li) + col) = v;
                } else if (r0 + li + EPC <= p.vrows) {
                    *(float4 *)(M + (r0 + li) + col) = v;
                } else {
                    const float vv[4] = {v.x, v.y, v.z, v.w};
                    for (int q = 0; q < EPC && r0 + li + q < p.vrows; ++q) M[r0 + li + q + col] = vv[q];
                }
            }
        }
    }
}

// partial sums over the local columns of sum_{i != gcol(j)} T(i, j)^2 (offdiag) or all entries
template <typename R>
__global__ void __launch_bounds__(256) k_mg_norm(const R *__restrict__ T, int64_t ld, int rows, int ncl,
                                                 const int *__restrict__ colg, int offdiag, double *__restrict__ part)
{
    __shared__ double sh[32];
    double acc = 0.0;
    const int64_t total = (int64_t)rows * ncl;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e / rows), i = (int)(e - (int64_t)j * rows);
        if (offdiag && i == colg[j]) continue;
        const double v = (double)T[i + j * ld];
        acc = __fma_rn(v, v, acc);
    }
    const double s = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_mg_sum(const double *__restrict__ part, int n, double *__restrict__ out)
{
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
    const double s = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) out[0] = s;
}

// dst(:, j) = src(:, map[j]) (rows `rows`), converting type
template <typename Rs, typename Rd>
__global__ void k_gather_cols(const Rs *__restrict__ src, int64_t lds, const int *__restrict__ map, int rows,
                              Rd *__restrict__ dst, int64_t ldd)
{
    const int j = blockIdx.y;
    const int sj = map[j];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x)
        dst[i + (int64_t)j * ldd] = sj >= 0 ? (Rd)src[i + (int64_t)sj * lds] : Rd(0);
}

// identity columns: V(i, j) = (i == colg[j])
template <typename R>
__global__ void k_id_cols(R *__restrict__ V, int64_t ld, int rows, const int *__restrict__ colg, int nreal)
{
    const int j = blockIdx.y;
    const int g = colg[j];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x)
        V[i + (int64_t)j * ld] = (i == g && g < nreal) ? R(1) : R(0);
}

__global__ void k_diag_cols(const double *__restrict__ T, int64_t ld, int ncl, const int *__restrict__ colg,
                            double *__restrict__ d)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < ncl) d[j] = T[colg[j] + (int64_t)j * ld];
}

// ---------------------------------------------------------------------------
// host plan
// ---------------------------------------------------------------------------
struct Xfer {
    int src, sphys, dst, dphys;   // rank / physical block position
};

struct Plan {
    int G, np, nb, mb, mbl, n;
    std::vector<int> top, bot;                 // slot -> global block (current round)
    std::vector<std::vector<int>> phys;        // rank -> physical position -> global block
    // tables of one sweep
    std::vector<std::vector<SlotInfo>> slots;  // [round][rank * mbl + kl]
    std::vector<std::vector<int2>> gslots;     // [round][slot]
    std::vector<std::vector<Xfer>> xfers;      // [round]

    void init(int n_, int np_, int G_)
    {
        n = n_; np = np_; G = G_;
        nb = np / BW; mb = nb / 2; mbl = mb / G;
        top.resize(mb); bot.resize(mb);
        for (int k = 0; k < mb; ++k) { top[k] = 2 * k; bot[k] = 2 * k + 1; }
        phys.assign(G, std::vector<int>(2 * mbl));
        for (int g = 0; g < G; ++g)
            for (int p = 0; p < 2 * mbl; ++p) phys[g][p] = 2 * g * mbl + p;
    }
    int rank_of_slot(int k) const { return k / mbl; }
    int where(int g, int blk) const
    {
        for (int p = 0; p < 2 * mbl; ++p)
            if (phys[g][p] == blk) return p;
        return -1;
    }
    static void music(std::vector<int> &t, std::vector<int> &b)
    {
        const int m = (int)t.size();
        if (m < 2) return;
        std::vector<int> t2(m), b2(m);
        t2[0] = t[0]; t2[1] = b[0];
        for (int k = 2; k < m; ++k) t2[k] = t[k - 1];
        for (int k = 0; k < m - 1; ++k) b2[k] = b[k + 1];
        b2[m - 1] = t[m - 1];
        t.swap(t2); b.swap(b2);
    }
    // build the tables of one sweep (nb - 1 block rounds) from the current state,
    // advancing the state to the start of the next sweep
    void build_sweep()
    {
        slots.clear(); gslots.clear(); xfers.clear();
        for (int R = 0; R < nb - 1; ++R) {
            std::vector<SlotInfo> sl(G * mbl);
            std::vector<int2> gs(mb);
            for (int k = 0; k < mb; ++k) {
                gs[k] = make_int2(top[k], bot[k]);
                const int g = rank_of_slot(k), kl = k - g * mbl;
                SlotInfo s;
                s.top = top[k]; s.bot = bot[k];
                s.ptop = BW * where(g, top[k]);
                s.pbot = BW * where(g, bot[k]);
                sl[g * mbl + kl] = s;
            }
            slots.push_back(sl);
            gslots.push_back(gs);
            // advance the merry-go-round and work out the block moves between ranks
            std::vector<int> ot = top, ob = bot;
            music(top, bot);
            std::vector<std::vector<int>> after(G);
            for (int k = 0; k < mb; ++k) {
                after[rank_of_slot(k)].push_back(top[k]);
                after[rank_of_slot(k)].push_back(bot[k]);
            }
            std::vector<Xfer> xs;
            std::vector<std::vector<int>> freed(G);
            std::vector<std::vector<std::pair<int, int>>> arriving(G);   // (block, src rank)
            for (int g = 0; g < G; ++g) {
                for (int p = 0; p < 2 * mbl; ++p) {
                    const int blk = phys[g][p];
                    if (std::find(after[g].begin(), after[g].end(), blk) == after[g].end()) freed[g].push_back(p);
                }
                for (int blk : after[g]) {
                    if (where(g, blk) < 0) {
                        int src = -1;
                        for (int h = 0; h < G; ++h)
                            if (where(h, blk) >= 0) src = h;
                        arriving[g].push_back({blk, src});
                    }
                }
                std::sort(arriving[g].begin(), arriving[g].end());
            }
            for (int g = 0; g < G; ++g) {
                for (size_t i = 0; i < arriving[g].size(); ++i) {
                    const int blk = arriving[g][i].first, src = arriving[g][i].second;
                    xs.push_back(Xfer{src, where(src, blk), g, freed[g][i]});
                }
            }
            // commit the new physical maps
            std::vector<std::vector<int>> nphys = phys;
            for (const Xfer &x : xs) nphys[x.dst][x.dphys] = phys[x.src][x.sphys];
            phys.swap(nphys);
            xfers.push_back(xs);
        }
    }
    // local physical column -> global column (rank g), -1 never
    std::vector<int> colglob(int g) const
    {
        std::vector<int> c(BW * 2 * mbl);
        for (int p = 0; p < 2 * mbl; ++p)
            for (int i = 0; i < BW; ++i) c[p * BW + i] = phys[g][p] * BW + i;
        return c;
    }
};

// ---------------------------------------------------------------------------
// group of local ranks (1 with NCCL, G when emulating)
// ---------------------------------------------------------------------------
struct RankBufs {
    double *T = nullptr, *V = nullptr;
    float *T32 = nullptr, *V32 = nullptr;
    int *colg = nullptr;               // local column -> global column
    double *part = nullptr;            // norm partials (kRedBlocks) + result
    SlotInfo *slots = nullptr;         // [round][mbl] of the current sweep
    char *stage = nullptr;             // 2 blocks of T and V (fp64)
};

struct Group {
    int G = 1, nlocal = 1, me = 0;     // me: NCCL rank (nlocal == 1)
    ncclComm_t comm = nullptr;
    Plan plan;
    int n = 0, np = 0, ncl = 0;        // ncl: local columns
    std::vector<RankBufs> rk;
    void *Ubuf = nullptr;              // mb * 64 * 64 fp64 words (an fp32 slot: U, then U^T)
    int *uid = nullptr;                // mb identity flags + one count per round
    int2 *gslots = nullptr;            // [round][mb]
    int2 *lsched = nullptr;
    unsigned long long *cnt = nullptr;
    double *As = nullptr;              // symmetrised A (np x np), replicated
    double *h = nullptr;               // pinned host scalars
    cudaStream_t st = nullptr;
    int rank_of(int i) const { return nlocal == 1 ? me : i; }
};

static std::map<std::string, ncclComm_t> g_comms;
static std::mutex g_comms_mu;

mpj_status nccl_ck(ncclResult_t r, const char *what)
{
    if (r != ncclSuccess) {
        set_error(std::string(what) + ": " + ncclGetErrorString(r));
        return MPJ_ERR_NCCL;
    }
    return MPJ_OK;
}

template <typename R>
static mpj_status mg_norm(Group &g, bool offdiag, R **Ts, double &out)
{
    // partial per local rank, then sum over ranks
    double tot = 0.0;
    for (int i = 0; i < g.nlocal; ++i) {
        RankBufs &b = g.rk[i];
        k_mg_norm<R><<<kRedBlocks, 256, 0, g.st>>>(Ts[i], g.np, g.np, g.ncl, b.colg, offdiag ? 1 : 0, b.part);
        k_mg_sum<<<1, 256, 0, g.st>>>(b.part, kRedBlocks, b.part + kRedBlocks);
        count_launch(2);
        if (g.comm) {   // NCCL (one process per rank; also with a single rank)
            MPJ_TRY(nccl_ck(ncclAllReduce(b.part + kRedBlocks, b.part + kRedBlocks, 1, ncclDouble, ncclSum, g.comm, g.st),
                            "ncclAllReduce"));
        }
        MPJ_CK(cudaMemcpyAsync(g.h + i, b.part + kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost, g.st));
    }
    MPJ_CK(cudaStreamSynchronize(g.st));
    for (int i = 0; i < g.nlocal; ++i) tot += g.h[i];
    out = std::sqrt(tot);
    return MPJ_OK;
}

static void upload_colg(Group &g)
{
    for (int i = 0; i < g.nlocal; ++i) {
        std::vector<int> c = g.plan.colglob(g.rank_of(i));
        cudaMemcpyAsync(g.rk[i].colg, c.data(), c.size() * sizeof(int), cudaMemcpyHostToDevice, g.st);
    }
}

template <typename R>
static mpj_status mg_sweep(Group &g, R **Ts, R **Vs, R nu, int rule, bool first)
{
    Plan &P = g.plan;
    const int rounds = P.nb - 1;
    P.build_sweep();
    // upload this sweep's tables
    std::vector<int2> gs((size_t)rounds * P.mb);
    for (int r = 0; r < rounds; ++r) std::copy(P.gslots[r].begin(), P.gslots[r].end(), gs.begin() + (size_t)r * P.mb);
    MPJ_CK(cudaMemcpyAsync(g.gslots, gs.data(), gs.size() * sizeof(int2), cudaMemcpyHostToDevice, g.st));
    for (int i = 0; i < g.nlocal; ++i) {
        const int rr = g.rank_of(i);
        std::vector<SlotInfo> sl((size_t)rounds * P.mbl);
        for (int r = 0; r < rounds; ++r)
            std::copy(P.slots[r].begin() + rr * P.mbl, P.slots[r].begin() + (rr + 1) * P.mbl,
                      sl.begin() + (size_t)r * P.mbl);
        MPJ_CK(cudaMemcpyAsync(g.rk[i].slots, sl.data(), sl.size() * sizeof(SlotInfo), cudaMemcpyHostToDevice, g.st));
    }
    MPJ_CK(cudaStreamSynchronize(g.st));   // the host vectors above are about to die
    constexpr int LD = Lay<R>::LD;
    const size_t sm_solve = 3 * TW * LayK<R>::LD * sizeof(R), sm_apply = 3 * TW * LD * sizeof(R);
    const size_t sm_apply64g3 = 3 * 2 * TW * Lay<double>::LD * sizeof(double) + 8 * sizeof(int);
    MPJ_CK(smem_optin((const void *)k_mg_solve<R>, sm_solve, NTW, nullptr));
    MPJ_CK(smem_optin((const void *)k_mg_apply<R>, sm_apply, NT, nullptr));
    if (sizeof(R) == 4)
        MPJ_CK(smem_optin((const void *)k_mg_apply_f32, sm_apply, 128, nullptr));
    else
        MPJ_CK(smem_optin((const void *)k_mg_apply_f64g3, sm_apply64g3, 3 * NT, nullptr));
    int *nid = g.uid + P.mb;
    MPJ_CK(cudaMemsetAsync(nid, 0, (size_t)rounds * sizeof(int), g.st));
    int nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const size_t blk_bytes = (size_t)BW * g.np * sizeof(R);
    const bool prof = prof_on();
    const char *nsolve = sizeof(R) == 8 ? "mg_solve_f64" : "mg_solve_f32";
    const char *napply = sizeof(R) == 8 ? "mg_apply_f64" : "mg_apply_f32";
    for (int r = 0; r < rounds; ++r) {
        if (prof) prof_mark(nsolve, g.st, true);
        for (int i = 0; i < g.nlocal; ++i) {
            const int rr = g.rank_of(i);
            k_mg_solve<R><<<P.mbl, NTW, sm_solve, g.st>>>(Ts[i], g.np, g.rk[i].slots + (size_t)r * P.mbl, rr * P.mbl,
                                                          g.lsched, r == 0, nu, rule, (R *)g.Ubuf, g.cnt);
            count_launch();
        }
        if (prof) prof_mark(nsolve, g.st, false);
        if (g.comm) {   // NCCL (one process per rank; also with a single rank)
            const size_t per = (size_t)P.mbl * TW * TW * (8 / sizeof(R));   // fp32: U and U^T per slot
            R *U = (R *)g.Ubuf;
            MPJ_TRY(nccl_ck(ncclAllGather(U + g.me * per, U, per * sizeof(R), ncclChar, g.comm, g.st),
                            "ncclAllGather(U)"));
        }
        // identity rotation blocks (every rank sees the same all-gathered U)
        k_mg_uid<R><<<P.mb, 256, 0, g.st>>>((const R *)g.Ubuf, g.uid, nid + r);
        count_launch();
        if (prof) prof_mark(napply, g.st, true);
        // first sweep: (almost) no identity blocks -- its launches give the full-launch efficiency
        const std::string nfirst = std::string(napply) + ".sweep1";
        if (prof && first) prof_mark(nfirst.c_str(), g.st, true);
        for (int i = 0; i < g.nlocal; ++i) {
            const int rr = g.rank_of(i);
            MgApply ap;
            ap.T = Ts[i]; ap.V = Vs[i]; ap.ld = g.np; ap.vrows = g.np;
            ap.slots = g.rk[i].slots + (size_t)r * P.mbl;
            ap.gslots = g.gslots + (size_t)r * P.mb;
            ap.slot0 = rr * P.mbl; ap.mb = P.mb; ap.mbl = P.mbl; ap.Ubuf = g.Ubuf;
            ap.uid = g.uid; ap.nid = nid + r;
            ap.ntT = P.mbl * (P.mb - 1);
            ap.ntV = (g.np / TW) * P.mbl;
            if (sizeof(R) == 4) {
                const int grid = std::min(ap.ntT + ap.ntV, 4 * nsm);
                k_mg_apply_f32<<<grid, 128, sm_apply, g.st>>>(ap);
            } else {
                const int grid = std::min(ap.ntT + ap.ntV, nsm);
                k_mg_apply_f64g3<<<grid, 3 * NT, sm_apply64g3, g.st>>>(ap);
            }
            count_launch();
        }
        if (prof && first) prof_mark(nfirst.c_str(), g.st, false);
        if (prof) prof_mark(napply, g.st, false);
        // block moves across rank boundaries
        const std::vector<Xfer> &xs = P.xfers[r];
        if (xs.empty()) continue;
        if (g.nlocal == 1) {
            std::vector<Xfer> out, in;
            for (const Xfer &x : xs) {
                if (x.src == g.me) out.push_back(x);
                if (x.dst == g.me) in.push_back(x);
            }
            MPJ_TRY(nccl_ck(ncclGroupStart(), "ncclGroupStart"));
            for (const Xfer &x : out) {
                MPJ_TRY(nccl_ck(ncclSend(Ts[0] + (size_t)x.sphys * BW * g.np, blk_bytes, ncclChar, x.dst, g.comm, g.st),
                                "ncclSend(T)"));
                MPJ_TRY(nccl_ck(ncclSend(Vs[0] + (size_t)x.sphys * BW * g.np, blk_bytes, ncclChar, x.dst, g.comm, g.st),
                                "ncclSend(V)"));
            }
            for (size_t k = 0; k < in.size(); ++k) {
                MPJ_TRY(nccl_ck(ncclRecv(g.rk[0].stage + 2 * k * blk_bytes, blk_bytes, ncclChar, in[k].src, g.comm, g.st),
                                "ncclRecv(T)"));
                MPJ_TRY(nccl_ck(ncclRecv(g.rk[0].stage + (2 * k + 1) * blk_bytes, blk_bytes, ncclChar, in[k].src,
                                         g.comm, g.st),
                                "ncclRecv(V)"));
            }
            MPJ_TRY(nccl_ck(ncclGroupEnd(), "ncclGroupEnd"));
            for (size_t k = 0; k < in.size(); ++k) {
                MPJ_CK(cudaMemcpyAsync(Ts[0] + (size_t)in[k].dphys * BW * g.np, g.rk[0].stage + 2 * k * blk_bytes,
                                       blk_bytes, cudaMemcpyDeviceToDevice, g.st));
                MPJ_CK(cudaMemcpyAsync(Vs[0] + (size_t)in[k].dphys * BW * g.np,
                                       g.rk[0].stage + (2 * k + 1) * blk_bytes, blk_bytes, cudaMemcpyDeviceToDevice,
                                       g.st));
            }
        } else {
            // emulation: stage every moving block first, then place it
            std::vector<int> slot_of(xs.size());
            std::vector<int> used(g.nlocal, 0);
            for (size_t k = 0; k < xs.size(); ++k) {
                const Xfer &x = xs[k];
                slot_of[k] = used[x.dst]++;
                char *stg = g.rk[x.dst].stage + 2 * slot_of[k] * blk_bytes;
                MPJ_CK(cudaMemcpyAsync(stg, Ts[x.src] + (size_t)x.sphys * BW * g.np, blk_bytes, cudaMemcpyDeviceToDevice,
                                       g.st));
                MPJ_CK(cudaMemcpyAsync(stg + blk_bytes, Vs[x.src] + (size_t)x.sphys * BW * g.np, blk_bytes,
                                       cudaMemcpyDeviceToDevice, g.st));
            }
            for (size_t k = 0; k < xs.size(); ++k) {
                const Xfer &x = xs[k];
                char *stg = g.rk[x.dst].stage + 2 * slot_of[k] * blk_bytes;
                MPJ_CK(cudaMemcpyAsync(Ts[x.dst] + (size_t)x.dphys * BW * g.np, stg, blk_bytes, cudaMemcpyDeviceToDevice,
                                       g.st));
                MPJ_CK(cudaMemcpyAsync(Vs[x.dst] + (size_t)x.dphys * BW * g.np, stg + blk_bytes, blk_bytes,
                                       cudaMemcpyDeviceToDevice, g.st));
            }
        }
    }
    return MPJ_OK;
}

template <typename R>
static mpj_status mg_loop(Group &g, R **Ts, R **Vs, double tol, R nu, int rule, int max_sweeps, int &sweeps,
                          long long &rot, double *hist)
{
    MPJ_CK(cudaMemsetAsync(g.cnt, 0, sizeof(unsigned long long), g.st));
    sweeps = 0;
    mpj_status status = MPJ_ERR_NOCONV;
    for (;;) {
        upload_colg(g);
        double off = 0;
        MPJ_TRY(mg_norm<R>(g, true, Ts, off));
        if (hist && sweeps < 64) hist[sweeps] = off;
        if (!std::isfinite(off)) { set_error("non-finite off-norm"); return MPJ_ERR_NONFINITE; }
        if (off <= tol) { status = MPJ_OK; break; }
        if (sweeps >= max_sweeps) { status = MPJ_ERR_NOCONV; break; }
        ++sweeps;
        MPJ_TRY(mg_sweep<R>(g, Ts, Vs, nu, rule, sweeps == 1));
    }
    // rotation count: every rank's K3 adds its own slots -> sum over ranks
    unsigned long long c = 0;
    MPJ_CK(cudaMemcpyAsync(g.h, g.cnt, sizeof(c), cudaMemcpyDeviceToHost, g.st));
    MPJ_CK(cudaStreamSynchronize(g.st));
    std::memcpy(&c, g.h, sizeof(c));
    if (g.comm) {   // NCCL (one process per rank; also with a single rank)
        double v = (double)c;
        double *d = g.rk[0].part + kRedBlocks + 1;
        MPJ_CK(cudaMemcpyAsync(d, &v, sizeof(double), cudaMemcpyHostToDevice, g.st));
        MPJ_TRY(nccl_ck(ncclAllReduce(d, d, 1, ncclDouble, ncclSum, g.comm, g.st), "ncclAllReduce(cnt)"));
        MPJ_CK(cudaMemcpyAsync(g.h, d, sizeof(double), cudaMemcpyDeviceToHost, g.st));
        MPJ_CK(cudaStreamSynchronize(g.st));
        c = (unsigned long long)(g.h[0] + 0.5);
    }
    rot = (long long)c;
    return status;
}

}  // namespace

// the communicator of (unique id, rank, nranks), created once per process
mpj_status mg_comm(const void *nccl_id, int rank, int nranks, void **out)
{
    std::lock_guard<std::mutex> lk(g_comms_mu);
    std::string key((const char *)nccl_id, 128);
    key += std::to_string(rank) + "/" + std::to_string(nranks);
    auto it = g_comms.find(key);
    if (it == g_comms.end()) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        ncclComm_t c;
        MPJ_TRY(nccl_ck(ncclCommInitRank(&c, nranks, id, rank), "ncclCommInitRank"));
        it = g_comms.emplace(key, c).first;
    }
    *out = (void *)it->second;
    return MPJ_OK;
}


// local-columns gather of a full matrix: dst(:, j) = src(:, colg[j]) (colg on device)
template <typename Rs, typename Rd>
static void gather_cols(const Rs *src, int64_t lds, const int *colg, int rows, int ncols, Rd *dst, int64_t ldd,
                        cudaStream_t st)
{
    k_gather_cols<Rs, Rd><<<dim3((rows + 255) / 256 > 64 ? 64 : (rows + 255) / 256, ncols), 256, 0, st>>>(
        src, lds, colg, rows, dst, ldd);
    count_launch();
}

// all-gather the local column blocks of every rank into `all` (np x np,
// rank-major: rank h's ncl columns at h * ncl) -- NCCL or device copies
template <typename R>
static mpj_status mg_allgather_cols(Group &g, R **loc_bufs, R *all)
{
    const size_t loc = (size_t)g.np * g.ncl;
    if (g.comm) {   // NCCL (one process per rank; also with a single rank)
        MPJ_CK(cudaMemcpyAsync(all + (size_t)g.me * loc, loc_bufs[0], loc * sizeof(R), cudaMemcpyDeviceToDevice, g.st));
        MPJ_TRY(nccl_ck(ncclAllGather(all + (size_t)g.me * loc, all, loc * sizeof(R), ncclChar, g.comm, g.st),
                        "ncclAllGather(cols)"));
    } else {
        for (int i = 0; i < g.nlocal; ++i)
            MPJ_CK(cudaMemcpyAsync(all + (size_t)i * loc, loc_bufs[i], loc * sizeof(R), cudaMemcpyDeviceToDevice, g.st));
    }
    return MPJ_OK;
}

// global column -> column of the rank-major all-gathered buffer
static std::vector<int> global_to_gathered(const Group &g)
{
    std::vector<int> src(g.np, -1);
    for (int h = 0; h < g.G; ++h) {
        std::vector<int> cg = g.plan.colglob(h);
        for (int j = 0; j < g.ncl; ++j) src[cg[j]] = h * g.ncl + j;
    }
    return src;
}

mpj_status mg_eig(bool mixed, const double *A, int64_t n, int64_t lda, double *Lambda, double *V, int64_t ldv,
                  int *sweeps_out, const void *nccl_id, int rank, int nranks, int emulate, cudaStream_t user,
                  const mpj_config &cfg, mpj_report &rep, double *h_pin)
{
    const double omega = 1.1102230246251565e-16, upsilon = 5.9604644775390625e-08;
    Group g;
    g.st = user;
    g.h = h_pin;
    const bool use_nccl = nccl_id != nullptr;   // a one-rank communicator runs the same NCCL calls
    g.G = use_nccl ? nranks : std::max(1, emulate);
    g.nlocal = use_nccl ? 1 : g.G;
    g.me = use_nccl ? rank : 0;
    g.n = (int)n;
    g.np = padded_n(n, BW * g.G);
    g.plan.init((int)n, g.np, g.G);
    g.ncl = g.np / g.G;
    const int np = g.np, ncl = g.ncl, mb = g.plan.mb;
    rep.n_padded = np; rep.block_b = BW; rep.variant = MPJ_VARIANT_BLOCK;
    if (use_nccl) {
        void *c = nullptr;
        MPJ_TRY(mg_comm(nccl_id, rank, nranks, &c));
        g.comm = (ncclComm_t)c;
    }
    // stream-ordered allocations, released on every exit
    std::vector<void *> owned;
    struct Releaser {
        std::vector<void *> &v;
        cudaStream_t st;
        ~Releaser()
        {
            for (void *p : v) cudaFreeAsync(p, st);
            cudaStreamSynchronize(st);
        }
    } releaser{owned, g.st};
    bool oom = false;
    auto alloc = [&](size_t bytes) -> void * {
        void *p = nullptr;
        if (cudaMallocAsync(&p, bytes, g.st) != cudaSuccess) { oom = true; cudaGetLastError(); return nullptr; }
        owned.push_back(p);
        return p;
    };
    const size_t loc = (size_t)np * ncl;
    g.rk.resize(g.nlocal);
    for (auto &b : g.rk) {
        b.T = (double *)alloc(loc * 8); b.V = (double *)alloc(loc * 8);
        b.T32 = (float *)alloc(loc * 4); b.V32 = (float *)alloc(loc * 4);
        b.colg = (int *)alloc(ncl * sizeof(int));
        b.part = (double *)alloc((kRedBlocks + 8) * 8);
        b.slots = (SlotInfo *)alloc((size_t)g.plan.nb * g.plan.mbl * sizeof(SlotInfo));
        b.stage = (char *)alloc(4 * (size_t)BW * np * 8);
    }
    g.Ubuf = alloc((size_t)mb * TW * TW * 8);
    g.uid = (int *)alloc((size_t)(mb + g.plan.nb) * sizeof(int));
    g.gslots = (int2 *)alloc((size_t)g.plan.nb * mb * sizeof(int2));
    g.lsched = (int2 *)alloc((BW - 1) * (BW / 2) * sizeof(int2));
    g.cnt = (unsigned long long *)alloc(64);
    g.As = (double *)alloc((size_t)np * np * 8);
    double *full = (double *)alloc((size_t)np * np * 8);   // A staging, then Z / Q, then diag view
    double *gath = (double *)alloc((size_t)np * np * 8);   // rank-major all-gathered columns
    double *W = (double *)alloc(loc * 8);
    int *perm = (int *)alloc(np * sizeof(int));
    int *rankv = (int *)alloc(np * sizeof(int));
    double *lam = (double *)alloc(np * 8);
    void *orth_ws = alloc(orth_workspace(np));
    if (oom) { set_error("mg: out of device memory"); return MPJ_ERR_NOMEM; }
    HostSchedule hs;
    build_schedule(64, BW, hs);
    MPJ_CK(cudaMemcpyAsync(g.lsched, hs.lsched.data(), hs.lsched.size() * sizeof(int2), cudaMemcpyHostToDevice, g.st));

    // a0: A -> As (symmetrised, zero padded), ||A||_F (every rank holds A)
    MPJ_CK(cudaMemsetAsync(full, 0, (size_t)np * np * 8, g.st));
    MPJ_CK(cudaMemcpy2DAsync(full, np * 8, A, lda * 8, n * 8, n, cudaMemcpyDefault, g.st));
    launch_symmetrize(full, np, (int)n, g.As, np, np, g.st);
    double *red = g.rk[0].part;
    launch_norm<double>(g.As, np, np, np, false, red, red + kRedBlocks, g.st);
    MPJ_CK(cudaMemcpyAsync(g.h, red + kRedBlocks, 8, cudaMemcpyDeviceToHost, g.st));
    MPJ_CK(cudaStreamSynchronize(g.st));
    const double normA = g.h[0];
    rep.norm_a = normA;

    std::vector<double *> Ts(g.nlocal), Vs(g.nlocal);
    std::vector<float *> T32s(g.nlocal), V32s(g.nlocal);
    for (int i = 0; i < g.nlocal; ++i) {
        Ts[i] = g.rk[i].T; Vs[i] = g.rk[i].V; T32s[i] = g.rk[i].T32; V32s[i] = g.rk[i].V32;
    }
    upload_colg(g);
    const int gx = std::max(1, std::min(64, (np + 255) / 256));
    mpj_status s = MPJ_OK;
    if (mixed && cfg.low_solver != MPJ_LOW_JACOBI) {
        // a1 by symmetric QR in binary32 (reading R12'), the default:
        // every rank holds A, so every rank runs the single-GPU step 1 on it
        // (sequential per column; the same Z bits on every rank), then a2 / a3
        // exactly as below.  Scratch: A32, Z32, Y and D- here, D+ in `gath`.
        float *A32 = (float *)alloc((size_t)np * np * 4), *Z32 = (float *)alloc((size_t)np * np * 4);
        double *Y = (double *)alloc((size_t)np * np * 8), *Dm = (double *)alloc((size_t)np * np * 8);
        void *sws = alloc(symqr_workspace(np));
        if (oom) { set_error("mg: out of device memory (symmetric-QR step 1)"); return MPJ_ERR_NOMEM; }
        launch_copy_pad<double, float>(g.As, np, (int)n, (int)n, A32, np, (int)n, (int)n, g.st);
        const auto t0 = std::chrono::steady_clock::now();
        MPJ_TRY(low_evd_symqr(A32, np, (int)n, Z32, np, Y, np, gath, Dm, sws, g.st));
        launch_copy_pad<float, double>(Z32, np, (int)n, (int)n, full, np, np, np, g.st);
        MPJ_CK(cudaStreamSynchronize(g.st));
        rep.t_low = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        rep.sweeps_low = 0; rep.rotations_low = 0; rep.status_low = MPJ_OK;
        s = orth_cgs2(full, np, full, np, n, n, orth_ws, g.st);
        if (s != MPJ_OK) return s;
        for (int i = 0; i < g.nlocal; ++i) {
            gather_cols<double, double>(full, np, g.rk[i].colg, np, ncl, g.rk[i].V, np, g.st);
            launch_dgemm(false, false, np, ncl, np, 1.0, g.As, np, g.rk[i].V, np, 0.0, W, np, g.st);
            launch_dgemm(true, false, np, ncl, np, 1.0, full, np, W, np, 0.0, g.rk[i].T, np, g.st);
        }
        double off0 = 0;
        MPJ_TRY(mg_norm<double>(g, true, Ts.data(), off0));
        rep.off0 = off0;
    } else if (mixed) {
        // a1: fp32 stage on the column partition (reading R12)
        for (int i = 0; i < g.nlocal; ++i) {
            gather_cols<double, float>(g.As, np, g.rk[i].colg, np, ncl, g.rk[i].T32, np, g.st);
            k_id_cols<float><<<dim3(gx, ncl), 256, 0, g.st>>>(g.rk[i].V32, np, np, g.rk[i].colg, (int)n);
            count_launch();
        }
        launch_copy_pad<double, float>(g.As, np, np, np, (float *)full, np, np, np, g.st);
        launch_norm<float>((float *)full, np, np, np, false, red, red + kRedBlocks, g.st);
        MPJ_CK(cudaMemcpyAsync(g.h, red + kRedBlocks, 8, cudaMemcpyDeviceToHost, g.st));
        MPJ_CK(cudaStreamSynchronize(g.st));
        const double nA32 = g.h[0];
        int swl = 0;
        long long rotl = 0;
        mpj_status sl = mg_loop<float>(g, T32s.data(), V32s.data(), eps_low_factor(cfg, n) * upsilon * nA32,
                                       (float)(cfg.nu_low_factor * upsilon), cfg.stop_rule, cfg.max_sweeps_low, swl,
                                       rotl, rep.off_hist_low);
        if (sl != MPJ_OK && sl != MPJ_ERR_NOCONV) return sl;
        rep.sweeps_low = swl; rep.rotations_low = rotl; rep.status_low = sl;
        // a2: Z = the gathered fp32 V (fp64, global column order) -> Q = CGS2(Z) on every rank
        for (int i = 0; i < g.nlocal; ++i)
            launch_copy_pad<float, double>(g.rk[i].V32, np, np, ncl, (double *)g.rk[i].T, np, np, ncl, g.st);
        MPJ_TRY(mg_allgather_cols<double>(g, Ts.data(), gath));
        std::vector<int> src = global_to_gathered(g);
        MPJ_CK(cudaMemcpyAsync(perm, src.data(), np * sizeof(int), cudaMemcpyHostToDevice, g.st));
        k_gather_cols<double, double><<<dim3(gx, np), 256, 0, g.st>>>(gath, np, perm, np, full, np);
        count_launch();
        MPJ_CK(cudaStreamSynchronize(g.st));
        s = orth_cgs2(full, np, full, np, n, n, orth_ws, g.st);
        if (s != MPJ_OK) return s;
        // a3: local columns of T0 = Q^T A Q, V = Q(:, own)
        for (int i = 0; i < g.nlocal; ++i) {
            gather_cols<double, double>(full, np, g.rk[i].colg, np, ncl, g.rk[i].V, np, g.st);
            launch_dgemm(false, false, np, ncl, np, 1.0, g.As, np, g.rk[i].V, np, 0.0, W, np, g.st);
            launch_dgemm(true, false, np, ncl, np, 1.0, full, np, W, np, 0.0, g.rk[i].T, np, g.st);
        }
        double off0 = 0;
        MPJ_TRY(mg_norm<double>(g, true, Ts.data(), off0));
        rep.off0 = off0;
    } else {
        for (int i = 0; i < g.nlocal; ++i) {
            gather_cols<double, double>(g.As, np, g.rk[i].colg, np, ncl, g.rk[i].T, np, g.st);
            k_id_cols<double><<<dim3(gx, ncl), 256, 0, g.st>>>(g.rk[i].V, np, np, g.rk[i].colg, (int)n);
            count_launch();
        }
    }
    // a4-a8: fp64 sweeps
    {
        int sw = 0;
        long long rot = 0;
        s = mg_loop<double>(g, Ts.data(), Vs.data(), cfg.eps_factor * omega * normA, cfg.nu_factor * omega,
                            cfg.stop_rule, cfg.max_sweeps, sw, rot, rep.off_hist);
        rep.sweeps = sw; rep.rotations = rot; rep.status = s;
        if (sweeps_out) *sweeps_out = sw;
        if (s != MPJ_OK && s != MPJ_ERR_NOCONV) return s;
    }
    // a10: every rank gathers diag(T) and V, then sorts (stable, descending)
    upload_colg(g);
    std::vector<int> src = global_to_gathered(g);
    MPJ_CK(cudaMemcpyAsync(perm, src.data(), np * sizeof(int), cudaMemcpyHostToDevice, g.st));
    // the diagonal of each local T, stored as the first row of a scratch (ld 1 per column)
    for (int i = 0; i < g.nlocal; ++i) {
        k_diag_cols<<<(ncl + 255) / 256, 256, 0, g.st>>>(g.rk[i].T, np, ncl, g.rk[i].colg, (double *)g.rk[i].T32);
        count_launch();
    }
    {
        // all-gather the diagonals (ncl doubles per rank) through the column gather with np = 1 row
        std::vector<double *> dloc(g.nlocal);
        for (int i = 0; i < g.nlocal; ++i) dloc[i] = (double *)g.rk[i].T32;
        if (g.comm) {   // NCCL (one process per rank; also with a single rank)
            MPJ_TRY(nccl_ck(ncclAllGather(dloc[0], W, ncl, ncclDouble, g.comm, g.st), "ncclAllGather(diag)"));
        } else {
            for (int i = 0; i < g.nlocal; ++i)
                MPJ_CK(cudaMemcpyAsync(W + (size_t)i * ncl, dloc[i], ncl * 8, cudaMemcpyDeviceToDevice, g.st));
        }
    }
    MPJ_TRY(mg_allgather_cols<double>(g, Vs.data(), gath));
    // V in global column order -> As (no longer needed); diag in global order onto the diagonal of `full`
    k_gather_cols<double, double><<<dim3(gx, np), 256, 0, g.st>>>(gath, np, perm, np, g.As, np);
    k_gather_cols<double, double><<<dim3(1, np), 32, 0, g.st>>>(W, 1, perm, 1, full, np + 1);
    count_launch(2);
    cudaPointerAttributes at;
    const bool out_dev = cudaPointerGetAttributes(&at, V) == cudaSuccess && at.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    double *vout = out_dev ? V : gath;
    launch_extract_evd(full, np, g.As, np, (int)n, (int)n, lam, vout, out_dev ? ldv : n, rankv, g.st);
    MPJ_CK(cudaMemcpyAsync(Lambda, lam, n * 8, cudaMemcpyDefault, g.st));
    if (!out_dev) MPJ_CK(cudaMemcpy2DAsync(V, ldv * 8, vout, n * 8, n * 8, n, cudaMemcpyDeviceToHost, g.st));
    MPJ_CK(cudaStreamSynchronize(g.st));
    return s;
}

}  // namespace mpj

// Host-only view of the partition plan of one sweep (tests of the multi-rank
// bookkeeping without GPUs).  slots: rounds x mb x 4 ints (top, bot, ptop, pbot
// of global slot k, physical positions on rank k / mbl); xfers: rounds x
// (4 * nranks) x 4 ints (src, sphys, dst, dphys; physical positions in blocks
// of 32 columns); nxfer: rounds ints.
extern "C" mpj_status mpjacobi_mg_plan(int64_t n, int nranks, int *np_out, int *rounds_out, int *slots, int *xfers,
                                       int *nxfer)
{
    using namespace mpj;
    if (n < 1 || nranks < 1) { set_error("mpjacobi_mg_plan: invalid argument"); return MPJ_ERR_INVALID; }
    Plan P;
    const int np = padded_n(n, BW * nranks);
    P.init((int)n, np, nranks);
    if (np_out) *np_out = np;
    if (rounds_out) *rounds_out = P.nb - 1;
    if (!slots || !xfers || !nxfer) return MPJ_OK;
    P.build_sweep();
    const int maxx = 4 * nranks;
    for (int r = 0; r < P.nb - 1; ++r) {
        for (int k = 0; k < P.mb; ++k) {
            const SlotInfo &si = P.slots[r][k];   // index g * mbl + kl == global slot k
            int *o = slots + ((size_t)r * P.mb + k) * 4;
            o[0] = si.top; o[1] = si.bot; o[2] = si.ptop / BW; o[3] = si.pbot / BW;
        }
        const std::vector<Xfer> &xs = P.xfers[r];
        if ((int)xs.size() > maxx) { set_error("mpjacobi_mg_plan: too many transfers"); return MPJ_ERR_INVALID; }
        nxfer[r] = (int)xs.size();
        for (size_t i = 0; i < xs.size(); ++i) {
            int *o = xfers + ((size_t)r * maxx + i) * 4;
            o[0] = xs[i].src; o[1] = xs[i].sphys; o[2] = xs[i].dst; o[3] = xs[i].dphys;
        }
    }
    return MPJ_OK;
}

extern "C" mpj_status mpjacobi_nccl_unique_id(void *out, size_t bytes)
{
    if (!out || bytes < sizeof(ncclUniqueId)) {
        mpj::set_error("mpjacobi_nccl_unique_id: need a 128-byte buffer");
        return MPJ_ERR_INVALID;
    }
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) {
        mpj::set_error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
        return MPJ_ERR_NCCL;
    }
    std::memcpy(out, &id, sizeof(id));
    return MPJ_OK;
}
