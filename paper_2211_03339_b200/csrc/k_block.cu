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
#include <cuda.h>
#include <cudaTypedefs.h>
#include "mpj_internal.h"
#include "mpj_block.cuh"

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

namespace mpj {

namespace {

using namespace blk;

// ---------------------------------------------------------------------------
// K3: inner solver.  One CTA per block pair.
// ---------------------------------------------------------------------------
template <typename R, bool FASTP>
__global__ void __launch_bounds__(NTW) k_block_solve(R *__restrict__ T, int64_t ldt, Sched S, int Rb, R nu,
                                                     int rule, R *__restrict__ Ubuf,
                                                     unsigned long long *__restrict__ cnt,
                                                     int *__restrict__ uid, int *__restrict__ nid, int max_inner)
{
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL): wait for K4
    constexpr int LD = LayK<R>::LD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R *D0 = (R *)smem_raw;          // 64 x LD, column-major (double-buffered)
    R *D1 = D0 + TW * LD;
    R *U = D1 + TW * LD;            // 64 x LD
    __shared__ unsigned nrot;
    __shared__ WideParams<R> P[2];
    const int k = blockIdx.x;
    const int mb = S.nb >> 1;
    const int2 bp = S.bsched[Rb * mb + k];
    for (int e = threadIdx.x; e < TW * TW; e += NTW) {
        const int li = e & (TW - 1), lj = e >> 6;
        D0[li + lj * LD] = T[gidx(bp, li) + (int64_t)gidx(bp, lj) * ldt];
        U[li + lj * LD] = (li == lj) ? R(1) : R(0);
    }
    __syncthreads();
    // Block rounds in which no pair the inner rounds visit passes the rotation
    // test (at n = 8192, 521 of the 1275 block rounds of one EVD): every round
    // then only sets the visited a_pq to 0 (the skip branch) and U stays
    // I, so that is done directly -- the same T and U (up to the sign of a
    // zero) without the 32 / 63 dependent rounds.  Decided from the block as
    // loaded: with no rotation nothing else changes between rounds.
    __shared__ int any_rot;
    if (threadIdx.x == 0) any_rot = 0;
    __syncthreads();
    const bool all_pairs = Rb == 0 || max_inner > 0;       // intra-block rounds too
    const int npairs = all_pairs ? TW * (TW - 1) / 2 : BW * BW;
    auto pair_of_e = [&](int e, int &p, int &q) {
        if (all_pairs) {
            q = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)e)) * 0.5f);
            while (q * (q - 1) / 2 > e) --q;
            while ((q + 1) * q / 2 <= e) ++q;
            p = e - q * (q - 1) / 2;
        } else {
            p = e & (BW - 1); q = BW + (e >> 5);
        }
    };
    for (int e = threadIdx.x; e < npairs; e += NTW) {
        int p, q;
        pair_of_e(e, p, q);
        if (!rot_skip<R>(D0[p + p * LD], D0[q + q * LD], D0[p + q * LD], nu, rule)) any_rot = 1;
    }
    __syncthreads();
    const R *D = D0;
    if (any_rot) {
        // FASTP: the parameter warp's divide / square-root chain with MUFU seeds + Newton (reading R28)
        D = inner_rounds_wide<R, FASTP>(D0, D1, U, bp, Rb == 0, S.lsched, nu, rule, P, &nrot, max_inner);
    } else {
        for (int e = threadIdx.x; e < npairs; e += NTW) {
            int p, q;
            pair_of_e(e, p, q);
            D0[p + q * LD] = R(0);
            D0[q + p * LD] = R(0);
        }
        if (threadIdx.x == 0) nrot = 0;
        __syncthreads();
    }
    R *Uk = Ubuf + (size_t)k * TW * TW;
    R *UkT = Ubuf + (size_t)mb * TW * TW + (size_t)k * TW * TW;   // U^T (fp32 apply operand)
    R *UkS = Ubuf + 2 * (size_t)mb * TW * TW + (size_t)k * TW * TW;   // U^T, split-half layout
    for (int e = threadIdx.x; e < TW * TW; e += NTW) {
        const int li = e & (TW - 1), lj = e >> 6;
        T[gidx(bp, li) + (int64_t)gidx(bp, lj) * ldt] = D[li + lj * LD];
        Uk[li + lj * TW] = U[li + lj * LD];
        if (sizeof(R) == 4) {
            UkT[li + lj * TW] = U[lj + li * LD];
            // split-half U^T for the TMA apply: element (i, k) of U^T = U(k, i)
            UkS[(li >> 5) * (BW * TW) + lj * BW + (li & 31)] = U[lj + li * LD];
        }
    }
    if (threadIdx.x == 0) {
        if (nrot) atomicAdd(cnt, (unsigned long long)nrot);
        uid[k] = nrot == 0;   // no rotation: U_k is exactly I (K4 may skip it)
        if (nrot == 0) atomicAdd(nid, 1);
    }
}

// ---------------------------------------------------------------------------
// K4: apply (persistent, cp.async double-buffered).
// Work items: [0, ntT) upper tiles (a, c), a < c, of T:  W = U_a^T X U_c,
// stored to (a, c) and W^T to (c, a);  [ntT, ntT + ntV) row tiles of M (= V,
// or C for the one-sided SVD):  M(r0:r0+64, P_c) <- M(r0:r0+64, P_c) U_c.
// CTA b handles items b, b + G, b + 2G, ...; the loads of item i+1 (X, U_a,
// U_c: 16-byte LDGSTS) are in flight while item i is multiplied.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp16(void *dst, const void *src, int src_bytes)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }
// wait until at most n cp.async groups are pending (n <= 4)
__device__ __forceinline__ void cp_wait_le(int n)
{
    switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;\n" ::); break;
    case 1: asm volatile("cp.async.wait_group 1;\n" ::); break;
    case 2: asm volatile("cp.async.wait_group 2;\n" ::); break;
    case 3: asm volatile("cp.async.wait_group 3;\n" ::); break;
    default: asm volatile("cp.async.wait_group 4;\n" ::); break;
    }
}

struct ApplyArgs {
    void *T; int64_t ldt;
    void *M; int64_t ldm; int mrows;
    Sched S; int Rb;
    const void *Ubuf;
    const int *uid;       // per block pair: U is exactly I (nullptr: never skip)
    const int *nid;       // number of such block pairs this block round
    int ntT, ntV;
    int *ctr;             // zeroed item counter of this launch (nullptr: per-SM item lists only)
};

__device__ __forceinline__ void decode_upper(int idx, int &a, int &c)
{
    c = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)idx)) * 0.5f);   // fp32 estimate, exact after the fix-ups
    while (c * (c - 1) / 2 > idx) --c;
    while ((c + 1) * c / 2 <= idx) ++c;
    a = idx - c * (c - 1) / 2;
}

// rotation block k of this block round is exactly I (no rotation in K3)
// (`skips` = p.uid && *p.nid > 0, read once per CTA)
__device__ __forceinline__ bool block_identity(const ApplyArgs &p, int k, bool skips)
{
    return skips && p.uid[k] != 0;
}

// issue the loads of work item `item` into stage buffers (X, Ua, Uc); fp64 T
// tiles with one identity block skip that block's load (see k_block_apply)
template <typename R, int NTH = NT, bool V2 = false>
__device__ __forceinline__ void issue_item(const ApplyArgs &p, int item, R *X, R *Ua, R *Uc, bool skips = false)
{
    constexpr int LD = Lay<R>::LD, EPC = 16 / sizeof(R), CPC = TW / EPC;   // elements / chunks per column
    const int mb = p.S.nb >> 1;
    const int2 *bsr = p.S.bsched + p.Rb * mb;
    const R *Ub = (const R *)p.Ubuf;
    // fp32 uses the k-major operands U^T (second half of Ubuf) and, for T
    // tiles, X^T = T(P_c, P_a) (T is exactly symmetric)
    const bool f32 = sizeof(R) == 4;
    const R *UbO = f32 ? Ub + (size_t)mb * TW * TW : Ub;
    if (item < p.ntT) {
        int a, c;
        decode_upper(item, a, c);
        const int2 pa = bsr[a], pc = bsr[c];
        const int2 rr = f32 ? pc : pa, cc = f32 ? pa : pc;
        const bool la = f32 || !block_identity(p, a, skips), lc = f32 || !block_identity(p, c, skips);
        const R *T = (const R *)p.T;
        for (int e = threadIdx.x; e < TW * CPC; e += NTH) {
            const int lj = e / CPC, li = (e - lj * CPC) * EPC;
            cp16(X + li + lj * LD, T + gidx(rr, li) + (int64_t)gidx(cc, lj) * p.ldt, 16);
            if (la) cp16(Ua + li + lj * LD, UbO + (size_t)a * TW * TW + li + lj * TW, 16);
            if (lc) cp16(Uc + li + lj * LD, UbO + (size_t)c * TW * TW + li + lj * TW, 16);
        }
    } else {
        // V2: super-item of two row tiles (rows r0.. into X, r0+64.. into the Ua buffer)
        const int idx = item - p.ntT, c = idx % mb, r0 = (idx / mb) * (V2 ? 2 : 1) * TW;
        const int2 pc = bsr[c];
        const R *M = (const R *)p.M;
        for (int e = threadIdx.x; e < TW * CPC; e += NTH) {
            const int lj = e / CPC, li = (e - lj * CPC) * EPC;
            #pragma unroll
            for (int h = 0; h < (V2 ? 2 : 1); ++h) {
                const int rem = p.mrows - (r0 + h * TW + li);
                const int bytes = rem >= EPC ? 16 : (rem > 0 ? rem * (int)sizeof(R) : 0);
                const R *src = M + (bytes ? (int64_t)(r0 + h * TW + li) : 0) + (int64_t)gidx(pc, lj) * p.ldm;
                cp16((h ? Ua : X) + li + lj * LD, src, bytes);
            }
            cp16(Uc + li + lj * LD, UbO + (size_t)c * TW * TW + li + lj * TW, 16);
        }
    }
}

// An item whose rotation blocks are all exactly I (no rotation in K3: U_a =
// U_c = I for a T tile, U_c = I for an M tile) leaves its tile unchanged and is
// skipped -- exact, and in the last fp64 sweeps nearly every item.
__device__ __forceinline__ bool item_identity(const ApplyArgs &p, int item, int mb)
{
    if (!p.uid) return false;
    if (item < p.ntT) {
        int a, c;
        decode_upper(item, a, c);
        return p.uid[a] && p.uid[c];
    }
    return p.uid[(item - p.ntT) % mb] != 0;
}

// STAGES = 2: one CTA per SM prefetches item i+1 while computing item i;
// STAGES = 1: two CTAs per SM overlap each other's loads and epilogues.
// One fp64 work item with k-chunked loads (one-stage path): a full T tile
// issues X and U_a in four row chunks (GEMM 1's k) and then U_c, V tiles issue
// X columns and U_c rows in four chunks; each product waits only for the chunk
// it is about to use, so the first k-steps overlap the rest of the loads.
// Results go from the accumulators straight to global memory.
template <bool V2, bool SKIP>
__device__ __forceinline__ void apply_item_f64(const ApplyArgs &p, int item, double *x, double *ua, double *uc, int mb,
                                               const int2 *bsr)
{
    constexpr int LD = Lay<double>::LD, EPC = 2, CPC = TW / EPC;
    constexpr bool skips = SKIP;
    const double *Ub = (const double *)p.Ubuf;
    const int tid = threadIdx.x;
    if (item < p.ntT) {
        int a, c;
        decode_upper(item, a, c);
        const int2 pa = bsr[a], pc = bsr[c];
        const bool ia = block_identity(p, a, skips), ic = block_identity(p, c, skips);
        const double *T = (const double *)p.T;
        const double *Uag = Ub + (size_t)a * TW * TW, *Ucg = Ub + (size_t)c * TW * TW;
        Acc<double> acc;
        if (!ia && !ic) {
            for (int ch = 0; ch < 4; ++ch) {
                for (int e = tid; e < TW * 8; e += NT) {     // 64 columns x 8 segments of 2 rows
                    const int lj = e >> 3, li = 16 * ch + 2 * (e & 7);
                    cp16(x + li + lj * LD, T + gidx(pa, li) + (int64_t)gidx(pc, lj) * p.ldt, 16);
                    cp16(ua + li + lj * LD, Uag + li + lj * TW, 16);
                }
                cp_commit();
            }
            for (int e = tid; e < TW * CPC; e += NT) {
                const int lj = e / CPC, li = (e - lj * CPC) * EPC;
                cp16(uc + li + lj * LD, Ucg + li + lj * TW, 16);
            }
            cp_commit();
            tile_mm_chunked<true>(ua, x, acc, [&](int ch) { cp_wait_le(4 - ch); __syncthreads(); });   // Y = Ua^T X
            __syncthreads();
            acc.each([&](int i, int j, double v) { x[i + j * LD] = v; });
            cp_wait0();
            __syncthreads();
            tile_mm<false>(x, uc, acc);                      // W = Y Uc
        } else {
            // one identity block: a single product, the identity is not loaded
            for (int e = tid; e < TW * CPC; e += NT) {
                const int lj = e / CPC, li = (e - lj * CPC) * EPC;
                cp16(x + li + lj * LD, T + gidx(pa, li) + (int64_t)gidx(pc, lj) * p.ldt, 16);
                if (!ia) cp16(ua + li + lj * LD, Uag + li + lj * TW, 16);
                if (!ic) cp16(uc + li + lj * LD, Ucg + li + lj * TW, 16);
            }
            cp_commit();
            cp_wait0();
            __syncthreads();
            if (ia) tile_mm<false>(x, uc, acc);              // W = X Uc
            else tile_mm<true>(ua, x, acc);                  // W = Ua^T X
        }
        __syncthreads();                                     // shared memory free: store from registers
        double *Tw = (double *)p.T;
        acc.each2([&](int i, int j, double v0, double v1) {  // W(i, j), W(i, j + 1); j even
            const int64_t gi = gidx(pa, i), gj = gidx(pc, j);
            Tw[gi + gj * p.ldt] = v0;
            Tw[gi + (gj + 1) * p.ldt] = v1;
            *(double2 *)(Tw + gj + gi * p.ldt) = make_double2(v0, v1);   // W^T(j .. j+1, i)
        });
        return;
    }
    constexpr int NH = V2 ? 2 : 1;                           // row tiles in the item
    const int idx = item - p.ntT, c = idx % mb, r0 = (idx / mb) * NH * TW;
    const int2 pc = bsr[c];
    const double *M = (const double *)p.M;
    const double *Ucg = Ub + (size_t)c * TW * TW;
    for (int ch = 0; ch < 4; ++ch) {
        for (int e = tid; e < 16 * CPC * NH; e += NT) {      // columns 16ch .. 16ch+15 of X (each row tile)
            const int h = e / (16 * CPC), r = e - h * 16 * CPC;
            const int lj = 16 * ch + r / CPC, li = (r % CPC) * EPC;
            const int row = r0 + h * TW + li, rem = p.mrows - row;
            const int bytes = rem >= EPC ? 16 : (rem > 0 ? rem * 8 : 0);
            cp16((h ? ua : x) + li + lj * LD, M + (bytes ? (int64_t)row : 0) + (int64_t)gidx(pc, lj) * p.ldm, bytes);
        }
        for (int e = tid; e < TW * 8; e += NT) {              // rows 16ch .. 16ch+15 of U_c
            const int lj = e >> 3, li = 16 * ch + 2 * (e & 7);
            cp16(uc + li + lj * LD, Ucg + li + lj * TW, 16);
        }
        cp_commit();
    }
    auto wait = [&](int ch) { cp_wait_le(3 - ch); __syncthreads(); };
    Acc<double> acc, acc2;
    if constexpr (V2) tile_mm2_chunked(x, ua, uc, acc, acc2, wait);   // W = X Uc for both row tiles
    else tile_mm_chunked<false>(x, uc, acc, wait);                     // W = X Uc
    __syncthreads();                                         // shared memory free: store from registers
    double *Mw = (double *)p.M;
    auto put = [&](int i, int j, double v0, double v1) {
        if (r0 + i < p.mrows) {
            const int64_t gj = gidx(pc, j);
            Mw[(int64_t)(r0 + i) + gj * p.ldm] = v0;
            Mw[(int64_t)(r0 + i) + (gj + 1) * p.ldm] = v1;
        }
    };
    acc.each2(put);
    if constexpr (V2) acc2.each2([&](int i, int j, double v0, double v1) { put(i + TW, j, v0, v1); });
}

// ---------------------------------------------------------------------------
// fp64 apply with two buffers per CTA (3 CTAs / 24 warps per SM): a T tile's
// U_a is needed only by Y = U_a^T X and U_c only by W = Y U_c, so they share
// one buffer -- after the barrier that starts chunk c+1 of the first product,
// U_a's rows of chunk c are dead and U_c's rows of chunk c stream into them.
// X / Y share the other buffer.  V tiles: X columns and U_c rows in four
// chunks.  Results go from the accumulators to global memory.  The three
// CTAs of an SM start at different thirds of their item lists.
// ---------------------------------------------------------------------------
// GROUPED: one CTA per SM of three 256-thread groups, each running this body
// on its own two buffers with its own named barrier; the groups take the
// SM's items (static across SMs) from a shared-memory counter, so they finish
// within one item of each other.  Three separate CTAs per SM (GROUPED =
// false) hold equal item lists but run at unequal speeds on the shared SM
// (per-CTA timestamps, tools/k4_trace.py: CTAs of one SM end up to 310 us
// apart in a 676 us launch; 0.76 of the CTA-slot time occupied).
template <bool SKIP, bool GROUPED = false>
__device__ __forceinline__ void apply_x3_body(const ApplyArgs &p, unsigned char *smem_raw)
{
    constexpr int LD = Lay<double>::LD, EPC = 2, CPC = TW / EPC;
    constexpr bool skips = SKIP;
    const int grp = GROUPED ? (int)(threadIdx.x >> 8) : 0;
    double *xb = (double *)smem_raw + (size_t)grp * 2 * TW * LD, *ub = xb + TW * LD;
    const int mb = p.S.nb >> 1;
    const int total = p.ntT + p.ntV;
    const int2 *bsr = p.S.bsched + p.Rb * mb;
    const double *Ub = (const double *)p.Ubuf;
    const int tid = GROUPED ? (int)(threadIdx.x & (NT - 1)) : (int)threadIdx.x;
    const int G = gridDim.x;
    // GROUPED with an item counter (block_sweep's launches): the groups of all
    // SMs take items from one global counter over the COMPACT list of this
    // block round's non-identity items (T tiles first, then V tiles), built by
    // every CTA at its start from the identity flags: L = non-identity blocks,
    // T items c-major -- c in L: every a < c; c not in L: the a < c in L --
    // with P = prefix counts to map a counter value to its tile.  No item is
    // skipped after it is claimed, so all groups of all SMs end within about
    // one item (static per-SM lists: up to 317 us apart within an SM, ~4%
    // across SMs; identity skips unevenly spread).  Otherwise (no counter, or
    // mb > 1024): the SM's static list (items b + kG) and a shared-memory counter.
    int *s_ctr = (int *)(smem_raw + (size_t)3 * 2 * TW * LD * sizeof(double));
    int *s_nxt = s_ctr + 1 + 2 * grp;
    int *sL = s_ctr + 8, *sP = sL + mb;           // compact lists (GROUPED with a counter)
    const bool gcomp = GROUPED && p.ctr != nullptr && mb <= 1024;
    int nTc = p.ntT, mL = mb;                    // no identity blocks: the identity map
    if (gcomp && skips) {
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            int base = 0, pbase = 0;
            for (int c0 = 0; c0 < mb; c0 += 32) {
                const int c = c0 + lane;
                const bool ni = c < mb && !(skips && p.uid[c]);
                const unsigned bal = __ballot_sync(0xffffffffu, ni);
                const int before = base + __popc(bal & ((1u << lane) - 1u));
                if (ni) sL[before] = c;
                const int cnt = c < mb ? (ni ? c : before) : 0;
                int x = cnt;                                  // inclusive scan of cnt over the warp
                #pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (c < mb) sP[c] = pbase + x - cnt;
                pbase += __shfl_sync(0xffffffffu, x, 31);
                base += __popc(bal);
            }
            if (lane == 0) { sP[mb] = p.ntT ? pbase : 0; s_ctr[7] = base; }   // column-only launches: no T tiles
        }
        ::__syncthreads();
        nTc = sP[mb];
        mL = s_ctr[7];
    }
    const int nrt = p.ntV / mb;                  // row tiles of M
    const int K = gcomp ? nTc + nrt * mL
                        : (int)blockIdx.x < total ? (total - 1 - (int)blockIdx.x) / G + 1 : 0;
    const int phase = GROUPED ? 0 : (int)(3 * (int64_t)blockIdx.x / G);      // 0, 1, 2: the CTAs of an SM
    const int k0 = (phase * K) / 3;
    auto __syncthreads = [&]() {
        if constexpr (GROUPED) asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "r"(NT) : "memory");
        else ::__syncthreads();
    };
    auto item_of = [&](int kk) {
        if (gcomp && !skips) return kk;
        if (gcomp) {
            if (kk < nTc) {                          // T tile: the largest c with P[c] <= kk
                int lo = 0, hi = mb - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (sP[mid] <= kk) lo = mid; else hi = mid - 1;
                }
                const int c = lo, o = kk - sP[c];
                const bool cn = !(skips && p.uid[c]);
                const int a = cn ? o : sL[o];
                return c * (c - 1) / 2 + a;
            }
            const int q = kk - nTc;                      // V tile
            return p.ntT + (q / mL) * mb + sL[q % mL];
        }
        int k = kk + k0;
        if (k >= K) k -= K;
        return (int)blockIdx.x + k * G;
    };
    auto next_kk = [&](int kk) {
        while (skips && kk < K && item_identity(p, item_of(kk), mb)) ++kk;
        return kk;
    };
    // per group, the next item index: two slots by iteration parity (a slot is
    // rewritten only two barriers later)
    auto fetch = [&]() {                        // the group leader claims the next non-identity item
        if (gcomp) return min(atomicAdd(p.ctr, 1), K);
        int kk;
        do { kk = atomicAdd(s_ctr, 1); } while (skips && kk < K && item_identity(p, item_of(kk), mb));
        return kk < K ? kk : K;
    };
    struct It {
        int item, a, c, r0;
        int2 pa, pc;
        bool isT, ia, ic;
        const double *Uag, *Ucg;
    };
    auto decode = [&](int item) {
        It s;
        s.item = item;
        s.isT = item < p.ntT;
        if (s.isT) {
            decode_upper(item, s.a, s.c);
            s.pa = bsr[s.a]; s.pc = bsr[s.c];
            s.ia = block_identity(p, s.a, skips); s.ic = block_identity(p, s.c, skips);
            s.Uag = Ub + (size_t)s.a * TW * TW;
            s.r0 = 0;
        } else {
            const int idx = item - p.ntT;
            s.c = idx % mb; s.a = 0; s.r0 = (idx / mb) * TW;
            s.pc = bsr[s.c]; s.pa = s.pc;
            s.ia = s.ic = false;
            s.Uag = nullptr;
        }
        s.Ucg = Ub + (size_t)s.c * TW * TW;
        return s;
    };
    // the loads that precede an item's first product (issued while the
    // previous item's results are being stored)
    auto issue = [&](const It &s) {
        if (s.isT) {
            const double *T = (const double *)p.T;
            if (!s.ia && !s.ic) {
                for (int ch = 0; ch < 4; ++ch) {                 // X and U_a rows, 4 groups
                    for (int e = tid; e < TW * 8; e += NT) {
                        const int lj = e >> 3, li = 16 * ch + 2 * (e & 7);
                        cp16(xb + li + lj * LD, T + gidx(s.pa, li) + (int64_t)gidx(s.pc, lj) * p.ldt, 16);
                        cp16(ub + li + lj * LD, s.Uag + li + lj * TW, 16);
                    }
                    cp_commit();
                }
            } else {
                for (int e = tid; e < TW * CPC; e += NT) {
                    const int lj = e / CPC, li = (e - lj * CPC) * EPC;
                    cp16(xb + li + lj * LD, T + gidx(s.pa, li) + (int64_t)gidx(s.pc, lj) * p.ldt, 16);
                    cp16(ub + li + lj * LD, (s.ia ? s.Ucg : s.Uag) + li + lj * TW, 16);
                }
                cp_commit();
            }
        } else {
            const double *M = (const double *)p.M;
            for (int ch = 0; ch < 4; ++ch) {
                for (int e = tid; e < 16 * CPC; e += NT) {       // X columns 16ch..
                    const int lj = 16 * ch + e / CPC, li = (e % CPC) * EPC;
                    const int rem = p.mrows - (s.r0 + li);
                    const int bytes = rem >= EPC ? 16 : (rem > 0 ? rem * 8 : 0);
                    cp16(xb + li + lj * LD, M + (bytes ? (int64_t)(s.r0 + li) : 0) + (int64_t)gidx(s.pc, lj) * p.ldm,
                         bytes);
                }
                for (int e = tid; e < TW * 8; e += NT) {         // U_c rows 16ch..
                    const int lj = e >> 3, li = 16 * ch + 2 * (e & 7);
                    cp16(ub + li + lj * LD, s.Ucg + li + lj * TW, 16);
                }
                cp_commit();
            }
        }
    };
    auto compute = [&](const It &s, Acc<double> &acc) {
        if (s.isT && !s.ia && !s.ic) {
            // Y = U_a^T X; after chunk c's barrier, U_c rows of chunk c-1 replace U_a's
            tile_mm_chunked<true>(ub, xb, acc, [&](int ch) {
                cp_wait_le(ch == 0 ? 3 : 2);
                __syncthreads();
                if (ch > 0) {
                    for (int e = tid; e < TW * 8; e += NT) {
                        const int lj = e >> 3, li = 16 * (ch - 1) + 2 * (e & 7);
                        cp16(ub + li + lj * LD, s.Ucg + li + lj * TW, 16);
                    }
                    cp_commit();
                }
            });
            __syncthreads();                                      // GEMM 1 done: X and U_a chunk 3 free
            for (int e = tid; e < TW * 8; e += NT) {
                const int lj = e >> 3, li = 48 + 2 * (e & 7);
                cp16(ub + li + lj * LD, s.Ucg + li + lj * TW, 16);
            }
            cp_commit();
            acc.each([&](int i, int j, double v) { xb[i + j * LD] = v; });   // Y
            // W = Y U_c, chunk c of U_c is group (3 - c) from the end
            tile_mm_chunked<false>(xb, ub, acc, [&](int ch) { cp_wait_le(3 - ch); __syncthreads(); });
        } else if (s.isT) {
            cp_wait0();
            __syncthreads();
            if (s.ia) tile_mm<false>(xb, ub, acc);               // W = X Uc
            else tile_mm<true>(ub, xb, acc);                     // W = Ua^T X
        } else {
            tile_mm_chunked<false>(xb, ub, acc, [&](int ch) { cp_wait_le(3 - ch); __syncthreads(); });
        }
    };
    auto store = [&](const It &s, const Acc<double> &acc) {
        if (s.isT) {
            double *Tw = (double *)p.T;
            acc.each2([&](int i, int j, double v0, double v1) {
                const int64_t gi = gidx(s.pa, i), gj = gidx(s.pc, j);
                Tw[gi + gj * p.ldt] = v0;
                Tw[gi + (gj + 1) * p.ldt] = v1;
                *(double2 *)(Tw + gj + gi * p.ldt) = make_double2(v0, v1);
            });
        } else {
            double *Mw = (double *)p.M;
            acc.each2([&](int i, int j, double v0, double v1) {
                if (s.r0 + i < p.mrows) {
                    const int64_t gj = gidx(s.pc, j);
                    Mw[(int64_t)(s.r0 + i) + gj * p.ldm] = v0;
                    Mw[(int64_t)(s.r0 + i) + (gj + 1) * p.ldm] = v1;
                }
            });
        }
    };
    int kk;
    if constexpr (GROUPED) {
        if (threadIdx.x == 0) *s_ctr = 0;
        ::__syncthreads();
        if (tid == 0) s_nxt[0] = fetch();
        __syncthreads();
        kk = s_nxt[0];
    } else {
        kk = next_kk(0);
    }
    It cur;
    if (kk < K) {
        cur = decode(item_of(kk));
        issue(cur);
    }
    for (int it = 1; kk < K; ++it) {
        if constexpr (GROUPED) {
            if (tid == 0) s_nxt[it & 1] = fetch();                // read after the barriers of compute
        }
        Acc<double> acc;
        compute(cur, acc);
        __syncthreads();                                         // shared memory free
        const int kn = GROUPED ? s_nxt[it & 1] : next_kk(kk + 1);
        It nxt = cur;
        if (kn < K) {
            nxt = decode(item_of(kn));
            issue(nxt);                                          // next item's loads in flight ...
        }
        store(cur, acc);                                         // ... while this one's results go out
        cur = nxt;
        kk = kn;
    }
    cp_wait0();
}

// per-CTA start / end timestamps and SM of the last fp64 apply launch, for
// tools/k4_trace.py (a build with -DMPJ_K4_TRACE only)
#ifdef MPJ_K4_TRACE
__device__ unsigned long long g_k4_trace[1024 * 3];
__device__ __forceinline__ void k4_trace(int ev)
{
    if (threadIdx.x == 0 && blockIdx.x < 1024) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_k4_trace[blockIdx.x * 3 + ev] = t;
        if (ev == 0) {
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            g_k4_trace[blockIdx.x * 3 + 2] = sm;
        }
    }
}
#define K4_TRACE(ev) k4_trace(ev)
#else
#define K4_TRACE(ev)
#endif

__global__ void __launch_bounds__(NT, 3) k_block_apply_f64x3(ApplyArgs p)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL): wait for K3
    K4_TRACE(0);
    if (p.uid && *p.nid > 0) apply_x3_body<true>(p, smem_raw);
    else apply_x3_body<false>(p, smem_raw);
    K4_TRACE(1);
}

__global__ void __launch_bounds__(3 * NT, 1) k_block_apply_f64g3(ApplyArgs p)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL): wait for K3
    K4_TRACE(0);
    if (p.uid && *p.nid > 0) apply_x3_body<true, true>(p, smem_raw);
    else apply_x3_body<false, true>(p, smem_raw);
    K4_TRACE(1);
}

// SKIP: this block round has identity blocks (skip / one-product logic); the
// kernel picks the instantiation once per CTA so that launches without
// identities run the plain loop (the checks cost 3% per full launch).
template <typename R, int STAGES, bool VONLY, bool SKIP>
__device__ __forceinline__ void apply_body(const ApplyArgs &p, unsigned char *smem_raw)
{
    constexpr int NB = VONLY ? 2 : 3;             // buffers per stage (V tiles: X, Uc)
    // fp64 V tiles as super-items of two row tiles (X in the X and Ua buffers):
    // each U_c fragment feeds both tiles' DMMAs, half the per-item overhead
    constexpr bool V2 = sizeof(R) == 8 && !VONLY;
    constexpr int LD = Lay<R>::LD, EPC = 16 / sizeof(R), CPC = TW / EPC;
    R *buf = (R *)smem_raw;                       // stage s: X, Ua, Uc at buf + (NB s + {0,1,2}) * TW * LD
    const int mb = p.S.nb >> 1;
    const int total = p.ntT + (V2 ? ((p.ntV / mb + 1) / 2) * mb : p.ntV);
    const int2 *bsr = p.S.bsched + p.Rb * mb;
    constexpr bool skips = SKIP;
    // this CTA's items: blockIdx.x + k G, k < K.  With one stage, the second half
    // of the grid (the other CTA on an SM) walks its list backwards, so the two
    // co-resident CTAs are out of phase and one computes while the other loads
    // or stores (in lockstep both load at once and the DMMA pipe idles)
    const int G = gridDim.x;
    const int K = (int)blockIdx.x < total ? (total - 1 - (int)blockIdx.x) / G + 1 : 0;
    const bool rev = STAGES == 1 && 2 * (int)blockIdx.x >= G;
    auto item_at = [&](int k) { return (int)blockIdx.x + (rev ? K - 1 - k : k) * G; };
    auto next_k = [&](int k) {
        while (skips && k < K && item_identity(p, item_at(k), mb)) ++k;
        return k;
    };
    int k = next_k(0);
    if (STAGES == 2) {
        if (k < K) issue_item<R, NT, V2>(p, item_at(k), buf, buf + TW * LD, buf + (NB - 1) * TW * LD, skips);
        cp_commit();
    }
    for (int it = 0; k < K; ++it, k = next_k(k + 1)) {
        const int item = item_at(k);
        const int s = STAGES == 2 ? (it & 1) : 0;
        if constexpr (sizeof(R) == 8 && STAGES == 1) {
            double *b64 = (double *)buf;   // X, Ua, Uc (column-only launches: X, Uc)
            apply_item_f64<V2, SKIP>(p, item, b64, b64 + TW * LD, b64 + (NB - 1) * TW * LD, mb, bsr);
            continue;
        }
        if (STAGES == 2) {
            const int kn = next_k(k + 1);
            R *nb = buf + (size_t)(NB * (s ^ 1)) * TW * LD;
            if (kn < K) issue_item<R, NT, V2>(p, item_at(kn), nb, nb + TW * LD, nb + (NB - 1) * TW * LD, skips);
            cp_commit();
            cp_wait1();
        } else {
            issue_item<R, NT, V2>(p, item, buf, buf + TW * LD, buf + (NB - 1) * TW * LD, skips);
            cp_commit();
            cp_wait0();
        }
        __syncthreads();
        R *x = buf + (size_t)(NB * s) * TW * LD, *ua = x + TW * LD, *uc = x + (NB - 1) * TW * LD;
        if (item < p.ntT) {
            int a, c;
            decode_upper(item, a, c);
            const int2 pa = bsr[a], pc = bsr[c];
            if constexpr (sizeof(R) == 4) {
                AccOP o;
                tile_op((const float *)ua, (const float *)x, o);   // Y = Ua^T X  (U_a^T, X^T k-major)
                __syncthreads();
                store_op(o, (float *)x, nullptr);                   // Y column-major (k-major for GEMM 2)
                __syncthreads();
                tile_op((const float *)x, (const float *)uc, o);   // W = Y Uc   (Y, U_c^T k-major)
                __syncthreads();
                store_op(o, (float *)x, (float *)ua);               // W and W^T
            } else {
                // one identity block: a single product (the identity's load was skipped)
                const bool ia = block_identity(p, a, skips), ic = block_identity(p, c, skips);
                Acc<R> acc;
                if (ia) {
                    tile_mm<false>(x, uc, acc);                      // W = X Uc
                } else if (ic) {
                    tile_mm<true>(ua, x, acc);                       // W = Ua^T X
                } else {
                    tile_mm<true>(ua, x, acc);                       // Y = Ua^T X
                    __syncthreads();
                    acc.each([&](int i, int j, R v) { x[i + j * LD] = v; });
                    __syncthreads();
                    tile_mm<false>(x, uc, acc);                      // W = Y Uc
                }
                // shared memory is free after this barrier: W and W^T go straight from
                // the accumulators to T while the next item's loads are issued
                __syncthreads();
                R *T = (R *)p.T;
                acc.each2([&](int i, int j, R v0, R v1) {    // W(i, j), W(i, j + 1); j even
                    const int64_t gi = gidx(pa, i), gj = gidx(pc, j);
                    T[gi + gj * p.ldt] = v0;
                    T[gi + (gj + 1) * p.ldt] = v1;
                    *(double2 *)(T + gj + gi * p.ldt) = make_double2(v0, v1);   // W^T(j .. j+1, i)
                });
                continue;
            }
            __syncthreads();
            R *T = (R *)p.T;
            for (int e = threadIdx.x; e < TW * CPC; e += NT) {
                const int lj = e / CPC, li = (e - lj * CPC) * EPC;
                *(int4 *)(T + gidx(pa, li) + (int64_t)gidx(pc, lj) * p.ldt) = *(const int4 *)(x + li + lj * LD);
                *(int4 *)(T + gidx(pc, li) + (int64_t)gidx(pa, lj) * p.ldt) = *(const int4 *)(ua + li + lj * LD);
            }
        } else {
            constexpr int NH = V2 ? 2 : 1;               // row tiles in this item
            const int idx = item - p.ntT, c = idx % mb, r0 = (idx / mb) * NH * TW;
            const int2 pc = bsr[c];
            if constexpr (sizeof(R) == 4) {
                AccOP o;
                tile_op((const float *)x, (const float *)uc, o);   // W = X Uc (X column-major, U_c^T)
                __syncthreads();
                store_op(o, (float *)x, nullptr);
            } else if constexpr (V2) {
                Acc<R> acc, acc2;
                tile_mm2(x, ua, uc, acc, acc2);                      // W = X Uc for both row tiles
                __syncthreads();                                     // shared memory free: store from registers
                R *M = (R *)p.M;
                auto put = [&](int i, int j, R v0, R v1) {
                    if (r0 + i < p.mrows) {
                        const int64_t gj = gidx(pc, j);
                        M[(int64_t)(r0 + i) + gj * p.ldm] = v0;
                        M[(int64_t)(r0 + i) + (gj + 1) * p.ldm] = v1;
                    }
                };
                acc.each2(put);
                acc2.each2([&](int i, int j, R v0, R v1) { put(i + TW, j, v0, v1); });
                continue;
            } else {
                Acc<R> acc;
                tile_mm<false>(x, uc, acc);                          // W = X Uc
                __syncthreads();                                     // shared memory free: store from registers
                R *M = (R *)p.M;
                acc.each2([&](int i, int j, R v0, R v1) {
                    if (r0 + i < p.mrows) {
                        const int64_t gj = gidx(pc, j);
                        M[(int64_t)(r0 + i) + gj * p.ldm] = v0;
                        M[(int64_t)(r0 + i) + (gj + 1) * p.ldm] = v1;
                    }
                });
                continue;
            }
            __syncthreads();
            R *M = (R *)p.M;
            for (int e = threadIdx.x; e < NH * TW * CPC; e += NT) {
                const int lj = e / (NH * CPC), lr = (e - lj * NH * CPC) * EPC;   // lr: row in the item
                const int h = lr >= TW, li = lr - h * TW;
                const R *srcw = (h ? ua : x) + li + lj * LD;
                R *dst = M + (int64_t)(r0 + lr) + (int64_t)gidx(pc, lj) * p.ldm;
                if (r0 + lr + EPC <= p.mrows) {
                    *(int4 *)dst = *(const int4 *)srcw;
                } else {
                    for (int q = 0; q < EPC && r0 + lr + q < p.mrows; ++q) dst[q] = srcw[q];
                }
            }
        }
        __syncthreads();
    }
    cp_wait0();
}

template <typename R, int STAGES, bool VONLY = false>
__global__ void __launch_bounds__(NT) k_block_apply(ApplyArgs p)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (p.uid && *p.nid > 0) apply_body<R, STAGES, VONLY, true>(p, smem_raw);
    else apply_body<R, STAGES, VONLY, false>(p, smem_raw);
}

// fp32 apply with 8 x 4 register tiles: 128 threads per 64 x 64 tile, thread
// (tx, ty) = (tid & 7, tid >> 3) owns rows 4tx..4tx+3, 32+4tx..32+4tx+3 (so
// that the 8 lanes' vectors are 128 contiguous bytes, conflict-free) and
// columns 4ty..4ty+3;
// 4 CTAs per SM.  Per k and warp: two 128-bit LDS of A (8 distinct vectors,
// one wavefront each) and one of B (4 distinct, one wavefront) feed 32 FFMA --
// half the shared-memory wavefronts per FFMA of the 4 x 4 tile (AccOP), whose
// K4 is bound by the shared-memory pipe (ncu: L1 85%, FMA 49%).
constexpr int NT128 = 128;

__device__ __forceinline__ void tile_op84(const float *A, const float *B, Acc84 &acc)
{
    tile_op84_t(A, B, acc, threadIdx.x);
}
__device__ __forceinline__ void store_op84(const Acc84 &acc, float *C, float *CT)
{
    store_op84_t(acc, C, CT, threadIdx.x);
}

__global__ void __launch_bounds__(NT128) k_block_apply_f32w(ApplyArgs p)
{
    constexpr int LD = Lay<float>::LD, EPC = 4, CPC = TW / EPC;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *x = (float *)smem_raw, *ua = x + TW * LD, *uc = ua + TW * LD;
    const int total = p.ntT + p.ntV;
    const int mb = p.S.nb >> 1;
    const int2 *bsr = p.S.bsched + p.Rb * mb;
    const bool skips = p.uid && *p.nid > 0;
    Acc84 acc;
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
        if (skips && item_identity(p, item, mb)) continue;
        issue_item<float, NT128>(p, item, x, ua, uc);
        cp_commit();
        cp_wait0();
        __syncthreads();
        if (item < p.ntT) {
            int a, c;
            decode_upper(item, a, c);
            const int2 pa = bsr[a], pc = bsr[c];
            tile_op84(ua, x, acc);                      // Y = U_a^T X  (U_a^T, X^T k-major)
            __syncthreads();
            store_op84(acc, x, nullptr);
            __syncthreads();
            tile_op84(x, uc, acc);                      // W = Y U_c
            __syncthreads();
            store_op84(acc, x, ua);                     // W and W^T
            __syncthreads();
            float *T = (float *)p.T;
            for (int e = threadIdx.x; e < TW * CPC; e += NT128) {
                const int lj = e / CPC, li = (e - lj * CPC) * EPC;
                *(int4 *)(T + gidx(pa, li) + (int64_t)gidx(pc, lj) * p.ldt) = *(const int4 *)(x + li + lj * LD);
                *(int4 *)(T + gidx(pc, li) + (int64_t)gidx(pa, lj) * p.ldt) = *(const int4 *)(ua + li + lj * LD);
            }
        } else {
            const int idx = item - p.ntT, c = idx % mb, r0 = (idx / mb) * TW;
            const int2 pc = bsr[c];
            tile_op84(x, uc, acc);                      // W = X U_c
            __syncthreads();
            store_op84(acc, x, nullptr);
            __syncthreads();
            float *M = (float *)p.M;
            for (int e = threadIdx.x; e < TW * CPC; e += NT128) {
                const int lj = e / CPC, li = (e - lj * CPC) * EPC;
                float *dst = M + (int64_t)(r0 + li) + (int64_t)gidx(pc, lj) * p.ldm;
                if (r0 + li + EPC <= p.mrows) {
                    *(int4 *)dst = *(const int4 *)(x + li + lj * LD);
                } else {
                    for (int q = 0; q < EPC && r0 + li + q < p.mrows; ++q) dst[q] = x[li + q + lj * LD];
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// fp32 apply, warp-specialised TMA pipeline: one persistent CTA per SM = 1
// producer warp + 2 consumer groups of 128 threads (8 x 4 FFMA tiles).  A
// ring of WS_NS stages, each one work item's operands (X, U_a^T, U_c^T; 16 KB
// each, "split-half" layout: element (i, k) at (i / 32) * 2048 + 32 k + i % 32,
// so every 32 x 32 box is a contiguous 4 KB chunk and the GEMM's 128-bit
// operand reads stay conflict-free).  The producer loads item j into stage
// j % WS_NS: X as four 32 x 32 tensor-TMA boxes (T or V tensor map; rows past
// the end of V are zero-filled) and each U^T block as one 16 KB bulk copy
// (K3 writes them in this layout), all completing on the stage's "full"
// mbarrier; consumer group j % 2 waits on it, multiplies, stores its tile with
// 128-bit thread stores and releases the stage on its "empty" mbarrier.  Six
// TMA requests per item (per-column bulk copies -- 256 per item -- made the
// first version of this kernel request-rate bound, 2.4x slower).
// ---------------------------------------------------------------------------
constexpr int WS_NS = 4;
constexpr int WS_CG = 128;                     // threads per consumer group
constexpr int WS_NT = 32 + 2 * WS_CG;
constexpr int SH_HALF = BW * TW;               // 2048 floats: one 32-row half of a 64 x 64 operand
constexpr int SH_TILE = 2 * SH_HALF;           // 4096 floats = 16 KB

__device__ __forceinline__ int sh_idx(int i, int k) { return (i >> 5) * SH_HALF + k * BW + (i & 31); }

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity)
{
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n"
                 " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_box(void *dst, const CUtensorMap *map, int row, int col, uint64_t *bar)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                 ::"r"(smem_u32(dst)), "l"(map), "r"(row), "r"(col), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void group_sync(int id) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(WS_CG) : "memory"); }

// C = A B^T-style k-major product of split-half operands, 4 x 8 per thread:
// quarter-warp Q = tid / 8 of the group owns rows 32 (Q % 2) + 4 (tid % 8) ..+3
// and columns 8 (Q / 2) ..+7.  128-bit shared loads are serviced per quarter
// warp: A (8 lanes, 128 contiguous bytes) costs one wavefront per quarter and
// B is a broadcast inside each quarter, so a k-step is ~6-8 wavefronts per
// warp for 32 FFMA (the 8 x 4 mapping of k_block_apply_f32w: ~10, which made
// that kernel shared-memory bound).
struct Acc48 {
    float v[4][8];
};

__device__ __forceinline__ void tile_op_sh(const float *A, const float *B, Acc48 &acc, int tid)
{
    const int q = tid >> 3, l8 = tid & 7;
    const float *Ar = A + (q & 1) * SH_HALF + 4 * l8;
    const int cb = 8 * (q >> 1);
    const float *Bc = B + (cb >> 5) * SH_HALF + (cb & 31);
    #pragma unroll
    for (int u = 0; u < 4; ++u)
        #pragma unroll
        for (int w = 0; w < 8; ++w) acc.v[u][w] = 0.f;
    // two register sets for consecutive k (set 0: even k, set 1: odd k); each set is
    // reloaded right after it is consumed, so no register rotation at the back edge
    // (the single-set pipelined form cost one MOV per ~4 FFMA2)
    auto step = [&](const float4 &a, const float4 &b0, const float4 &b1) {
        const float av[4] = {a.x, a.y, a.z, a.w}, bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        #pragma unroll
        for (int u = 0; u < 4; ++u)
            #pragma unroll
            for (int w = 0; w < 8; w += 2) ffma2(av[u], bv[w], bv[w + 1], acc.v[u][w], acc.v[u][w + 1]);
    };
    float4 a0 = *(const float4 *)Ar, p0 = *(const float4 *)Bc, q0 = *(const float4 *)(Bc + 4);
    #pragma unroll 2
    for (int k = 0; k < TW; k += 2) {
        const float4 a1 = *(const float4 *)(Ar + (k + 1) * BW), p1 = *(const float4 *)(Bc + (k + 1) * BW),
                     q1 = *(const float4 *)(Bc + 4 + (k + 1) * BW);
        step(a0, p0, q0);
        if (k + 2 < TW) {
            a0 = *(const float4 *)(Ar + (k + 2) * BW);
            p0 = *(const float4 *)(Bc + (k + 2) * BW);
            q0 = *(const float4 *)(Bc + 4 + (k + 2) * BW);
        }
        step(a1, p1, q1);
    }
}

// C (split-half) and C^T stores of an Acc48
__device__ __forceinline__ void store_op_sh(const Acc48 &acc, float *C, float *CT, int tid)
{
    const int q = tid >> 3, l8 = tid & 7;
    const int r = 32 * (q & 1) + 4 * l8, c = 8 * (q >> 1);
    #pragma unroll
    for (int w = 0; w < 8; ++w)
        *(float4 *)(C + sh_idx(r, c + w)) = make_float4(acc.v[0][w], acc.v[1][w], acc.v[2][w], acc.v[3][w]);
    if (CT) {
        #pragma unroll
        for (int u = 0; u < 4; ++u) {
            *(float4 *)(CT + sh_idx(c, r + u)) = make_float4(acc.v[u][0], acc.v[u][1], acc.v[u][2], acc.v[u][3]);
            *(float4 *)(CT + sh_idx(c + 4, r + u)) = make_float4(acc.v[u][4], acc.v[u][5], acc.v[u][6], acc.v[u][7]);
        }
    }
}

// V super-items: two row tiles of the same column block (128 x 64 of M, one
// U_c) in a "split-quarter" layout (element (i, k) at (i / 32) 2048 + 32 k +
// i % 32).  8 x 8 per thread: quarter-warp Q owns rows 32 (Q % 2) + 4 l8 ..+3
// and 32 (Q % 2 + 2) + 4 l8 ..+3 and columns 8 (Q / 2) ..+7: a k-step is ~12
// shared-memory wavefronts per warp for 64 FFMA (4 x 8 tiles: ~16).
struct Acc88 {
    float v[8][8];
};

__device__ __forceinline__ void tile_op_88(const float *A, const float *B, Acc88 &acc, int tid)
{
    const int q = tid >> 3, l8 = tid & 7;
    const float *A0 = A + (q & 1) * SH_HALF + 4 * l8, *A1 = A0 + 2 * SH_HALF;
    const int cb = 8 * (q >> 1);
    const float *Bc = B + (cb >> 5) * SH_HALF + (cb & 31);
    #pragma unroll
    for (int u = 0; u < 8; ++u)
        #pragma unroll
        for (int w = 0; w < 8; ++w) acc.v[u][w] = 0.f;
    // two register sets (even / odd k), as in tile_op_sh
    auto step = [&](const float4 &x0, const float4 &x1, const float4 &y0, const float4 &y1) {
        const float av[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        const float bv[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
        #pragma unroll
        for (int u = 0; u < 8; ++u)
            #pragma unroll
            for (int w = 0; w < 8; w += 2) ffma2(av[u], bv[w], bv[w + 1], acc.v[u][w], acc.v[u][w + 1]);
    };
    float4 a0 = *(const float4 *)A0, a1 = *(const float4 *)A1, b0 = *(const float4 *)Bc,
           b1 = *(const float4 *)(Bc + 4);
    #pragma unroll 1
    for (int k = 0; k < TW; k += 2) {
        const float4 c0 = *(const float4 *)(A0 + (k + 1) * BW), c1 = *(const float4 *)(A1 + (k + 1) * BW),
                     d0 = *(const float4 *)(Bc + (k + 1) * BW), d1 = *(const float4 *)(Bc + 4 + (k + 1) * BW);
        step(a0, a1, b0, b1);
        if (k + 2 < TW) {
            a0 = *(const float4 *)(A0 + (k + 2) * BW);
            a1 = *(const float4 *)(A1 + (k + 2) * BW);
            b0 = *(const float4 *)(Bc + (k + 2) * BW);
            b1 = *(const float4 *)(Bc + 4 + (k + 2) * BW);
        }
        step(c0, c1, d0, d1);
    }
}

template <bool SKIP>
__device__ __forceinline__ void apply_f32ws_body(const ApplyArgs &p, const CUtensorMap &tmT, const CUtensorMap &tmM,
                                                 unsigned char *smem_raw)
{
    constexpr int SBUF = 3 * SH_TILE;
    float *ring = (float *)smem_raw;
    uint64_t *full = (uint64_t *)(smem_raw + (size_t)WS_NS * SBUF * sizeof(float));
    uint64_t *empty = full + WS_NS;
    const int mb = p.S.nb >> 1;
    // M tiles are processed as super-items of two row tiles (same column block)
    const int nrt = p.ntV / mb;
    const int total = p.ntT + ((nrt + 1) / 2) * mb;
    const int2 *bsr = p.S.bsched + p.Rb * mb;
    constexpr bool skips = SKIP;
    auto advance = [&](int i) {
        while (skips && i < total && item_identity(p, i, mb)) i += gridDim.x;
        return i;
    };
    if (threadIdx.x == 0) {
        for (int st = 0; st < WS_NS; ++st) { mbar_init(full + st, 1); mbar_init(empty + st, 1); }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        // ------------------------------------------------------------- producer
        if (threadIdx.x != 0) return;
        const float *UbS = (const float *)p.Ubuf + 2 * (size_t)mb * TW * TW;   // split-half U^T
        int j = 0;
        for (int item = advance(blockIdx.x); item < total; item = advance(item + gridDim.x), ++j) {
            const int st = j % WS_NS;
            mbar_wait(empty + st, ((j / WS_NS) & 1) ^ 1);
            float *x = ring + (size_t)st * SBUF, *ua = x + SH_TILE, *uc = ua + SH_TILE;
            uint64_t *bar = full + st;
            if (item < p.ntT) {
                int a, c;
                decode_upper(item, a, c);
                const int2 pa = bsr[a], pc = bsr[c];
                // one identity block: one product, no load of that block; if U_a = I the
                // consumer computes X U_c and needs X = T(P_a, P_c) itself, else X^T = T(P_c, P_a)
                const bool ia = block_identity(p, a, skips), ic = block_identity(p, c, skips);
                mbar_arrive_tx(bar, (ia || ic ? 2 : 3) * SH_TILE * sizeof(float));
                const int2 br = ia ? pa : pc, bc = ia ? pc : pa;   // box rows / columns
                tma_box(x, &tmT, br.x * BW, bc.x * BW, bar);
                tma_box(x + SH_HALF, &tmT, br.y * BW, bc.x * BW, bar);
                tma_box(x + BW * BW, &tmT, br.x * BW, bc.y * BW, bar);
                tma_box(x + SH_HALF + BW * BW, &tmT, br.y * BW, bc.y * BW, bar);
                if (!ia) bulk_g2s(ua, UbS + (size_t)a * SH_TILE, SH_TILE * sizeof(float), bar);
                if (!ic) bulk_g2s(uc, UbS + (size_t)c * SH_TILE, SH_TILE * sizeof(float), bar);
            } else {
                // super-item: rows r0 .. r0 + 127 of M (X occupies the X and U_a slots)
                const int idx = item - p.ntT, c = idx % mb, r0 = (idx / mb) * 2 * TW;
                const int2 pc = bsr[c];
                const int nq = (r0 + TW < p.mrows) ? 4 : 2;      // a lone last row tile: its half only
                mbar_arrive_tx(bar, (nq * 2 * BW * BW + SH_TILE) * sizeof(float));   // partial rows zero-filled
                for (int qh = 0; qh < nq; ++qh) {
                    tma_box(x + qh * SH_HALF, &tmM, r0 + qh * BW, pc.x * BW, bar);
                    tma_box(x + qh * SH_HALF + BW * BW, &tmM, r0 + qh * BW, pc.y * BW, bar);
                }
                bulk_g2s(uc, UbS + (size_t)c * SH_TILE, SH_TILE * sizeof(float), bar);
            }
        }
        return;
    }
    // ----------------------------------------------------------------- consumers
    const int g = (warp - 1) / (WS_CG / 32);               // group 0 / 1
    const int gt = threadIdx.x - 32 - g * WS_CG;            // thread within the group
    const int bar_id = 1 + g;
    Acc48 acc;
    Acc88 acc8;
    int j = 0;
    for (int item = advance(blockIdx.x); item < total; item = advance(item + gridDim.x), ++j) {
        if ((j & 1) != g) continue;
        const int st = j % WS_NS;
        mbar_wait(full + st, (j / WS_NS) & 1);
        float *x = ring + (size_t)st * SBUF, *ua = x + SH_TILE, *uc = ua + SH_TILE;
        const bool ttile = item < p.ntT;
        int a = 0, c, r0 = 0;
        if (ttile) {
            decode_upper(item, a, c);
        } else {
            const int idx = item - p.ntT;
            c = idx % mb;
            r0 = (idx / mb) * 2 * TW;
        }
        const int2 pa = bsr[a], pc = bsr[c];
        if (ttile) {
            const bool ia = block_identity(p, a, skips), ic = block_identity(p, c, skips);
            if (ia) {
                tile_op_sh(x, uc, acc, gt);                  // W = X U_c   (x = X)
            } else if (ic) {
                tile_op_sh(ua, x, acc, gt);                  // W = U_a^T X (x = X^T)
            } else {
                tile_op_sh(ua, x, acc, gt);                  // Y = U_a^T X
                group_sync(bar_id);
                store_op_sh(acc, x, nullptr, gt);
                group_sync(bar_id);
                tile_op_sh(x, uc, acc, gt);                  // W = Y U_c
            }
        } else {
            tile_op_88(x, uc, acc8, gt);                     // W = X U_c (128 x 64)
        }
        // the stage is no longer read: release it (generic-proxy reads are ordered
        // before the async-proxy refill) and store the results from registers
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        group_sync(bar_id);
        if (gt == 0) mbar_arrive(empty + st);
        const int q = gt >> 3, l8 = gt & 7;
        if (ttile) {
            // Acc48: rows r..r+3 (one 32-row block), columns cc..cc+7
            const int r = 32 * (q & 1) + 4 * l8, cc = 8 * (q >> 1);
            float *T = (float *)p.T;
            const int64_t gr = gidx(pa, r), gcc = gidx(pc, cc);
            #pragma unroll
            for (int w = 0; w < 8; ++w)                      // W(r..r+3, cc+w)
                *(float4 *)(T + gr + (int64_t)gidx(pc, cc + w) * p.ldt) =
                    make_float4(acc.v[0][w], acc.v[1][w], acc.v[2][w], acc.v[3][w]);
            #pragma unroll
            for (int u = 0; u < 4; ++u) {                    // W^T(cc..cc+7, r+u)
                float *dst = T + gcc + (int64_t)(gr + u) * p.ldt;
                *(float4 *)dst = make_float4(acc.v[u][0], acc.v[u][1], acc.v[u][2], acc.v[u][3]);
                *(float4 *)(dst + 4) = make_float4(acc.v[u][4], acc.v[u][5], acc.v[u][6], acc.v[u][7]);
            }
        } else {
            // Acc88: rows r..r+3 and r+64..r+67, columns cc..cc+7
            const int r = 32 * (q & 1) + 4 * l8, cc = 8 * (q >> 1);
            float *M = (float *)p.M;
            #pragma unroll
            for (int w = 0; w < 8; ++w) {
                const int64_t col = (int64_t)gidx(pc, cc + w) * p.ldm;
                if (r0 + r < p.mrows)                        // mrows % 4 == 0 on this path
                    *(float4 *)(M + (r0 + r) + col) = make_float4(acc8.v[0][w], acc8.v[1][w], acc8.v[2][w], acc8.v[3][w]);
                if (r0 + r + TW < p.mrows)
                    *(float4 *)(M + (r0 + r + TW) + col) =
                        make_float4(acc8.v[4][w], acc8.v[5][w], acc8.v[6][w], acc8.v[7][w]);
            }
        }
    }
}

__global__ void __launch_bounds__(WS_NT, 1) k_block_apply_f32ws(ApplyArgs p, const __grid_constant__ CUtensorMap tmT,
                                                                const __grid_constant__ CUtensorMap tmM)
{
    extern __shared__ __align__(128) unsigned char smem_ws[];   // TMA boxes need 128-byte alignment
    asm volatile("griddepcontrol.wait;\n" ::: "memory");       // launched early (PDL): wait for K3
    if (p.uid && *p.nid > 0) apply_f32ws_body<true>(p, tmT, tmM, smem_ws);
    else apply_f32ws_body<false>(p, tmT, tmM, smem_ws);
}

}  // namespace

template <typename R>
size_t block_scratch_bytes(int np, int b)
{
    (void)b;
    const int mb = np / (2 * BW);
    // U, U^T, identity flags, identity counts and apply item counters per block round
    return (sizeof(R) == 4 ? 3 : 2) * (size_t)mb * TW * TW * sizeof(R) + (size_t)(mb + 2 * mb + 2 * mb) * sizeof(int);
}

static int sm_count()
{
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

static int apply_stages()
{
    static int s = 0;
    if (!s) {
        const char *e = getenv("MPJ_APPLY_STAGES");
        s = (e && atoi(e) == 2) ? 2 : 1;
    }
    return s;
}

template <typename R, int STAGES, bool VONLY = false>
static cudaError_t launch_apply_s(const ApplyArgs &p, cudaStream_t st)
{
    constexpr int LD = Lay<R>::LD;
    const size_t smem = (VONLY ? 2 : 3) * STAGES * TW * LD * sizeof(R);
    int per_sm = 1;
    cudaError_t e = smem_optin((const void *)k_block_apply<R, STAGES, VONLY>, smem, NT, &per_sm);
    if (e != cudaSuccess) return e;
    const int total = p.ntT + p.ntV;
    const int grid = std::max(1, std::min(total, sm_count() * per_sm));
    k_block_apply<R, STAGES, VONLY><<<grid, NT, smem, st>>>(p);
    count_launch();
    return cudaGetLastError();
}

// launch with programmatic stream serialisation: the kernel may start while
// the previous one drains; it waits (griddepcontrol.wait) before touching data
template <typename... KA, typename... A>
static cudaError_t launch_pdl(void (*k)(KA...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

// MPJ_F64_APPLY: "2cta" the two-stage kernel, "x3" three CTAs per SM with
// static item lists, default g3 (three groups in one CTA per SM sharing the
// SM's items)
static int f64_apply_kind()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MPJ_F64_APPLY");
        v = (e && std::string(e) == "2cta") ? 0 : (e && std::string(e) == "x3") ? 1 : 2;
    }
    return v;
}

static cudaError_t launch_apply_f64g3(const ApplyArgs &p, cudaStream_t st)
{
    const int mb = p.S.nb >> 1;
    // three groups' buffers, counters, the compact lists (L, P) of the item counter
    const size_t smem = 3 * 2 * TW * Lay<double>::LD * sizeof(double) +
                        (8 + 2 * (size_t)std::min(mb, 1024) + 1) * sizeof(int);   // compact lists only for mb <= 1024
    cudaError_t e = smem_optin((const void *)k_block_apply_f64g3, smem, 3 * NT, nullptr);
    if (e != cudaSuccess) return e;
    const int total = p.ntT + p.ntV;
    const int grid = std::max(1, std::min(total, sm_count()));
    count_launch();
    return launch_pdl(k_block_apply_f64g3, dim3(grid), dim3(3 * NT), smem, st, p);
}

static cudaError_t launch_apply_f64x3(const ApplyArgs &p, cudaStream_t st)
{
    const size_t smem = 2 * TW * Lay<double>::LD * sizeof(double);
    int per_sm = 1;
    cudaError_t e = smem_optin((const void *)k_block_apply_f64x3, smem, NT, &per_sm);
    if (e != cudaSuccess) return e;
    const int total = p.ntT + p.ntV;
    const int grid = std::max(1, std::min(total, sm_count() * per_sm));
    count_launch();
    return launch_pdl(k_block_apply_f64x3, dim3(grid), dim3(NT), smem, st, p);
}

static int fp32_apply_kind()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MPJ_FP32_APPLY");
        v = (e && std::string(e) == "4x4") ? 0 : (e && std::string(e) == "8x4") ? 1 : 2;
    }
    return v;
}

static cudaError_t launch_apply_f32w(const ApplyArgs &p, cudaStream_t st)
{
    const size_t smem = 3 * TW * Lay<float>::LD * sizeof(float);
    int per_sm = 1;
    cudaError_t e = smem_optin((const void *)k_block_apply_f32w, smem, NT128, &per_sm);
    if (e != cudaSuccess) return e;
    const int total = p.ntT + p.ntV;
    const int grid = std::max(1, std::min(total, sm_count() * per_sm));
    k_block_apply_f32w<<<grid, NT128, smem, st>>>(p);
    count_launch();
    return cudaGetLastError();
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)f;
    });
    return fn;
}

// 2-D fp32 tensor map of a column-major rows x cols matrix, 32 x 32 boxes
static bool make_map32(CUtensorMap &m, const void *base, int64_t rows, int64_t cols, int64_t ld)
{
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
    cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
    cuuint32_t box[2] = {BW, BW}, es[2] = {1, 1};
    return enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// false: the TMA kernel is unavailable for these operands (the caller falls
// back to the 8x4 kernel); a launch error is returned through *err
static bool launch_apply_f32ws(const ApplyArgs &p, cudaStream_t st, cudaError_t *err)
{
    CUtensorMap mT, mM;
    // column updates only (SVD): no T tiles, M's map stands in for T's
    const bool hasT = p.T != nullptr;
    if (!make_map32(mT, hasT ? p.T : p.M, hasT ? p.S.np : p.mrows, p.S.np, hasT ? p.ldt : p.ldm) ||
        !make_map32(mM, p.M, p.mrows, p.S.np, p.ldm))
        return false;
    const size_t smem = (size_t)WS_NS * 3 * SH_TILE * sizeof(float) + 2 * WS_NS * sizeof(uint64_t);
    if (smem_optin((const void *)k_block_apply_f32ws, smem, WS_NT, nullptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    const int total = p.ntT + p.ntV;
    const int grid = std::max(1, std::min(total, sm_count()));
    *err = launch_pdl(k_block_apply_f32ws, dim3(grid), dim3(WS_NT), smem, st, p, mT, mM);
    count_launch();
    return true;
}

template <typename R>
static cudaError_t launch_apply(const ApplyArgs &p, cudaStream_t st)
{
    cudaError_t e = cudaSuccess;
    if (sizeof(R) == 4 && fp32_apply_kind() == 2 && p.mrows % 4 == 0 && launch_apply_f32ws(p, st, &e)) return e;
    if (sizeof(R) == 4 && fp32_apply_kind() >= 1) return launch_apply_f32w(p, st);
    if (sizeof(R) == 8 && apply_stages() == 1 && f64_apply_kind() == 2)   // also column-only (SVD) launches
        return launch_apply_f64g3(p, st);
    if (sizeof(R) == 8 && apply_stages() == 1 && f64_apply_kind() == 1)
        return launch_apply_f64x3(p, st);
    if (apply_stages() == 2) return launch_apply_s<R, 2>(p, st);
    // column updates only (the SVD): two buffers per CTA, 3 CTAs/SM (an
    // EVD launch split into T-only and V-only kernels gained nothing)
    if (p.ntT == 0) return launch_apply_s<R, 1, true>(p, st);
    return launch_apply_s<R, 1>(p, st);
}

template <typename R>
mpj_status block_sweep(R *T, int64_t ldt, R *V, int64_t ldv, int vrows, const DevSched &ds, R nu, int rule,
                       unsigned long long *cnt, void *scratch, cudaStream_t st, bool first_sweep, int max_brounds,
                       int max_inner)
{
    if (ds.b != BW) { set_error("block variant needs b = 32"); return MPJ_ERR_INVALID; }
    Sched S;
    S.bsched = ds.bsched; S.lsched = ds.lsched; S.b = ds.b; S.nb = ds.nb; S.np = ds.np;
    const int mb = ds.nb / 2;
    R *Ubuf = (R *)scratch;
    int *uid = (int *)(Ubuf + (sizeof(R) == 4 ? 3 : 2) * (size_t)mb * TW * TW);
    int *nid = uid + mb;                         // nb - 1 <= 2 mb block rounds
    int *ctr = nid + 2 * mb;                     // the apply's item counter per block round
    MPJ_CK(cudaMemsetAsync(nid, 0, (size_t)4 * mb * sizeof(int), st));
    const size_t sm_solve = 3 * TW * LayK<R>::LD * sizeof(R);
    // fp64: the fast parameter chain (R28) unless MPJ_K3_IEEE=1 (A/B and its parity test)
    const char *ie = getenv("MPJ_K3_IEEE");
    const bool fastp = sizeof(R) == 8 && !(ie && ie[0] == '1');
    auto solve = fastp ? k_block_solve<R, sizeof(R) == 8> : k_block_solve<R, false>;
    MPJ_CK(smem_optin((const void *)solve, sm_solve, NTW, nullptr));
    ApplyArgs ap{};
    ap.T = T; ap.ldt = ldt; ap.M = V; ap.ldm = ldv; ap.mrows = vrows; ap.S = S; ap.Ubuf = Ubuf; ap.uid = uid;
    ap.ntT = mb * (mb - 1) / 2;
    ap.ntV = ((vrows + TW - 1) / TW) * mb;
    const char *nsolve = sizeof(R) == 8 ? "block_solve_f64" : "block_solve_f32";
    const char *napply = sizeof(R) == 8 ? "block_apply_f64" : "block_apply_f32";
    const bool prof = prof_on();
    const int nbr = max_brounds >= 0 ? std::min(max_brounds, ds.nb - 1) : ds.nb - 1;
    for (int Rb = 0; Rb < nbr; ++Rb) {
        if (prof) prof_mark(nsolve, st, true);
        MPJ_CK(launch_pdl(solve, dim3(mb), dim3(NTW), sm_solve, st, T, ldt, S, Rb, nu, rule, Ubuf, cnt, uid,
                          nid + Rb, max_inner));
        count_launch();
        if (prof) { prof_mark(nsolve, st, false); prof_mark(napply, st, true); }
        ap.Rb = Rb;
        ap.nid = nid + Rb;
        ap.ctr = ctr + Rb;
        // the first sweep's launches are also timed apart: they have (almost) no
        // identity blocks, so they give the full-launch efficiency
        const std::string nfirst = std::string(napply) + ".sweep1";
        if (prof && first_sweep) prof_mark(nfirst.c_str(), st, true);
        MPJ_CK(launch_apply<R>(ap, st));
        if (prof && first_sweep) prof_mark(nfirst.c_str(), st, false);
        if (prof) prof_mark(napply, st, false);
    }
    if (prof) {   // identity-skip statistics (for the algorithmic-flop count of the roofline)
        std::vector<int> h(ds.nb - 1);
        MPJ_CK(cudaMemcpyAsync(h.data(), nid, h.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
        MPJ_CK(cudaStreamSynchronize(st));
        long long ids = 0, skt = 0, skv = 0, half = 0;
        long long allid = 0;
        for (int c : h) {
            ids += c;
            allid += c == mb;
            skt += (long long)c * (c - 1) / 2;
            skv += (long long)c * ((vrows + TW - 1) / TW);
            if (sizeof(R) == 8 || fp32_apply_kind() == 2) half += (long long)c * (mb - c);   // one product
        }
        const std::string base(napply);
        prof_add(base + ".identity_blocks", ids);
        prof_add(base + ".all_identity_rounds", allid);   // block rounds in which no block pair rotated
        prof_add(base + ".items", (long long)(ds.nb - 1) * (ap.ntT + ap.ntV));
        prof_add(base + ".skipped_t", skt);
        prof_add(base + ".skipped_v", skv);
        prof_add(base + ".half_t", half);
        if (first_sweep) {
            prof_add(base + ".sweep1.skipped_t", skt);
            prof_add(base + ".sweep1.skipped_v", skv);
            prof_add(base + ".sweep1.half_t", half);
        }
    }
    return MPJ_OK;
}

// M(:, P_c) <- M(:, P_c) U_c for every block pair c of block round Rb (M has
// `rows` rows): the column update of the one-sided (SVD) block variant.
// uid / nid (optional): identity flags and count of this block round (skip).
template <typename R>
cudaError_t launch_block_apply_cols(R *M, int64_t ld, int rows, const DevSched &ds, int Rb, const R *Ubuf,
                             cudaStream_t st, const int *uid, const int *nid, int *ctr)
{
    Sched S;
    S.bsched = ds.bsched; S.lsched = ds.lsched; S.b = ds.b; S.nb = ds.nb; S.np = ds.np;
    ApplyArgs ap{};
    ap.T = nullptr; ap.ldt = 0; ap.M = M; ap.ldm = ld; ap.mrows = rows; ap.S = S; ap.Rb = Rb; ap.Ubuf = Ubuf; ap.uid = uid; ap.nid = nid;
    ap.ctr = ctr;                                // zeroed item counter (nullptr: per-SM item lists)
    ap.ntT = 0;
    ap.ntV = ((rows + TW - 1) / TW) * (ds.nb / 2);
    return launch_apply<R>(ap, st);
}
template cudaError_t launch_block_apply_cols<double>(double *, int64_t, int, const DevSched &, int, const double *,
                                              cudaStream_t, const int *, const int *, int *);
template cudaError_t launch_block_apply_cols<float>(float *, int64_t, int, const DevSched &, int, const float *,
                                             cudaStream_t, const int *, const int *, int *);

template size_t block_scratch_bytes<double>(int, int);
template size_t block_scratch_bytes<float>(int, int);
template mpj_status block_sweep<double>(double *, int64_t, double *, int64_t, int, const DevSched &, double,
                                        int, unsigned long long *, void *, cudaStream_t, bool, int, int);
template mpj_status block_sweep<float>(float *, int64_t, float *, int64_t, int, const DevSched &, float, int,
                                       unsigned long long *, void *, cudaStream_t, bool, int, int);

#ifdef MPJ_K4_TRACE
}  // namespace mpj
extern "C" int mpjacobi_debug_k4_trace(unsigned long long *out)
{
    return cudaMemcpyFromSymbol(out, mpj::g_k4_trace, sizeof(mpj::g_k4_trace)) == cudaSuccess ? 0 : 1;
}
namespace mpj {
#endif
}  // namespace mpj
