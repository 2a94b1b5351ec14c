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
#include <cuda.h>
#include <cudaTypedefs.h>
#include "mpj_internal.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>

namespace mpj {

namespace {

constexpr int TB = 64;       // tile = panel width
constexpr int NTH = 256;     // threads per CTA (8 warps)
constexpr int RSLOT = 2 * TB + 2;  // per-row-block partials: [0] tail norm^2, [1 + s] panel dots (s < 2 TB)
constexpr int NCACHE = 1;          // own row blocks whose panel V / W rows live in shared memory
constexpr int NSTAGE = 3;          // TMA ring of 64 x 64 A22 tiles for the symmetric product
// dynamic shared memory: [V/W cache of NCACHE row blocks | NSTAGE tile stages]
// during the column loop; the syr2k's four 64 x 64 operand tiles after it
constexpr size_t SYTRD_SMEM = (2 * NCACHE + NSTAGE) * TB * TB * sizeof(float) > 4 * TB * TB * sizeof(float)
                                  ? (2 * NCACHE + NSTAGE) * TB * TB * sizeof(float)
                                  : 4 * TB * TB * sizeof(float);

// phase timestamps for tools/sytrd_trace.py (a build with -DMPJ_SYTRD_TRACE only)
#ifdef MPJ_SYTRD_TRACE
__device__ unsigned long long g_sytrd_trace[64 * 12 * 320];   // [column % 64][event][cta]
__device__ int g_trace_k0 = 0;                                // the panel recorded
__device__ __forceinline__ void sytrd_trace(int k0, int jj, int ev)
{
    if (threadIdx.x == 0 && k0 == g_trace_k0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_sytrd_trace[((size_t)jj * 12 + ev) * 320 + blockIdx.x] = t;
    }
}
#define SYTRD_TRACE(jj, ev) sytrd_trace(a.k0, jj, ev)
#else
#define SYTRD_TRACE(jj, ev)
#endif

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mb_arrive_tx(uint64_t *b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t *b, unsigned parity)
{
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n"
                 " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 " @!p bra WAIT_%=;\n}\n" ::"r"(su32(b)), "r"(parity) : "memory");
}
// one 64 x 64 fp32 box of A (rows r, columns c; out-of-range parts zero-filled)
__device__ __forceinline__ void tma_tile(float *dst, const CUtensorMap *map, int r, int c, uint64_t *bar)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                 ::"r"(su32(dst)), "l"(map), "r"(r), "r"(c), "r"(su32(bar)) : "memory");
}

struct SytrdArgs {
    float *A;            // n x n, ld (lower triangle is the live matrix)
    int64_t ld;
    int n, nt;           // size, tiles per dimension (ceil(n / 64))
    float *V, *W;        // panel vectors, ldp x TB each (rows >= n are zero)
    int64_t ldp;
    float *acol;         // 2 x ldp: the corrected current column (double-buffered)
    float *d, *e, *tau;
    float *Prow, *Pcol;  // partial vectors of A22 v, (nt (nt + 1) / 2) x TB each
    float *rred;         // RSLOT x ntp partials per row block (slot-major; written by the owner CTA)
    int ntp;             // nt rounded up to a multiple of 4 (float4 reductions)
    float *qred;         // G partials of v^T A22 v (one per CTA)
    unsigned *bar;       // grid barrier (count, generation)
    int k0, ncols;       // panel start column and its number of reflector columns
};

// ---- grid barrier (all CTAs co-resident: cooperative launch) ---------------
// bar[0] counts arrivals since the launch (zeroed before it); barrier number
// e (0, 1, ...) is passed when it reaches (e + 1) gridDim.x.  Only thread 0
// of each CTA arrives (release) and polls (acquire).
__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned &epoch)
{
    __syncthreads();
    ++epoch;
    if (threadIdx.x == 0) {
        const unsigned target = epoch * gridDim.x;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while ((int)(v - target) < 0);
    }
    __syncthreads();
}

// butterfly sum over a warp: every lane gets the same value (a + b == b + a)
__device__ __forceinline__ float warp_sum(float v)
{
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// the 8 sums of c[0..7] over the warp's 32 lanes (transpose-reduce, 9 shuffles):
// the result lands in every lane whose bits (4, 3, 2) index the sum; returns
// it, and the index through u
__device__ __forceinline__ float warp_sum8(float (&c)[8], int &u)
{
    const int lane = threadIdx.x & 31;
    const bool h4 = lane & 16;
    #pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float got = __shfl_xor_sync(0xffffffffu, h4 ? c[k] : c[k + 4], 16);
        c[k] = (h4 ? c[k + 4] : c[k]) + got;
    }
    const bool h3 = lane & 8;
    #pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float got = __shfl_xor_sync(0xffffffffu, h3 ? c[k] : c[k + 2], 8);
        c[k] = (h3 ? c[k + 2] : c[k]) + got;
    }
    const bool h2 = lane & 4;
    const float got = __shfl_xor_sync(0xffffffffu, h2 ? c[0] : c[1], 4);
    float r = (h2 ? c[1] : c[0]) + got;
    r += __shfl_xor_sync(0xffffffffu, r, 2);
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    u = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    return r;
}

// sum of p[k * stride], k in [k0, k1), by one warp in a fixed order
__device__ __forceinline__ float warp_sum_list(const float *p, int stride, int k0, int k1)
{
    const int lane = threadIdx.x & 31;
    float s0 = 0.f, s1 = 0.f;
    int k = k0 + lane;
    for (; k + 32 < k1; k += 64) {
        s0 += p[(size_t)k * stride];
        s1 += p[(size_t)(k + 32) * stride];
    }
    if (k < k1) s0 += p[(size_t)k * stride];
    return warp_sum(s0 + s1);
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

// the transposed contributions A_KI^T v_K (K >= I) to output block I are
// stored contiguously: Pcol[(cofs(I) + K - I) * 64 + r]
__device__ __forceinline__ int cofs(int I, int T0, int nt)
{
    const int m = I - T0;
    return m * nt - (m * T0 + m * (m - 1) / 2);
}

// part g (of `parts`) of y_i, the symmetric product at row i = I*64 + r: a
// fixed-order sum over the partial vectors of tile row I (one per chunk
// segment: the row-major tile list is cut into chunks of L tiles; a segment
// starts at J = T0 or at a chunk start inside the row; part 0 takes these) and
// of tile column I (one per tile K >= I, the diagonal tile's strict lower part
// included; part g takes K - I = g mod parts)
__device__ __forceinline__ float y_part(const SytrdArgs &a, int I, int r, int T0, int L, int g, int parts)
{
    float y0 = 0.f, y1 = 0.f, y2 = 0.f;
    if (g == 0) {
        const int fa = flat_of(I, T0, T0), fb = flat_of(I, I, T0);
        y0 = a.Prow[(size_t)fa * TB + r];
        for (int f = (fa / L + 1) * L; f <= fb; f += L) y0 += a.Prow[(size_t)f * TB + r];
    }
    const float *pc = a.Pcol + (size_t)cofs(I, T0, a.nt) * TB + r;
    const int cnt = a.nt - I;
    int k = g;
    #pragma unroll 8
    for (; k + parts < cnt; k += 2 * parts) {
        y1 += pc[(size_t)k * TB];
        y2 += pc[(size_t)(k + parts) * TB];
    }
    if (k < cnt) y1 += pc[(size_t)k * TB];
    return y0 + (y1 + y2);
}

// v_i of column j's reflector (v_{j+1} = 1, v_i = a_i scal below, 0 above)
__device__ __forceinline__ float v_of(const float *acol, int i, int j, float scal)
{
    return i <= j ? 0.f : (i == j + 1 ? 1.f : acol[i] * scal);
}

__global__ void __launch_bounds__(NTH, 2) k_sytrd_panel(SytrdArgs a, const __grid_constant__ CUtensorMap tmA)
{
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t fullb[NSTAGE], emptyb[NSTAGE];
    __shared__ float dots[2 * TB];     // v^T V(:, t), v^T W(:, t) (reduced)
    __shared__ float rowbuf[NTH / 32][TB];
    __shared__ float wq[NTH / 32];
    __shared__ float vj[TB], wj[TB];   // row j of the panel's V and W (t < jj)
    __shared__ float bc[4];            // broadcast scalars: tail norm^2, v^T A22 v, row j+1 of w
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, grp = tid >> 6, r64 = tid & 63;
    const int G = gridDim.x, cta = blockIdx.x;
    const int n = a.n, nt = a.nt;
    const int64_t ld = a.ld, ldp = a.ldp;
    const int nown = cta < nt ? (nt - 1 - cta) / G + 1 : 0;    // own row blocks I = cta + q G
    // V / W rows of the first NCACHE own row blocks: cache[q] = {V[t][r], W[t][r]}
    auto cV = [&](int q) { return smem + (size_t)q * 2 * TB * TB; };
    auto cW = [&](int q) { return smem + (size_t)q * 2 * TB * TB + TB * TB; };
    for (int e = tid; e < NCACHE * 2 * TB * TB; e += NTH) smem[e] = 0.f;
    float *stage = smem + NCACHE * 2 * TB * TB;     // NSTAGE x 64 x 64 (column-major tiles)
    if (tid == 0) {
        for (int k = 0; k < NSTAGE; ++k) { mb_init(&fullb[k], 1); mb_init(&emptyb[k], NTH / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    unsigned it_issued = 0, it_used = 0;           // tiles through the ring (this CTA, whole kernel)
    unsigned epoch = 0;                             // grid barriers passed
    // symv tile producer state (thread 0): next tile to issue and the ring index
    // at which the current column's chunk ends
    int pI = 0, pJ = 0, pT0 = 0;
    unsigned it_end = 0;
    auto issue = [&]() {
        const unsigned k = it_issued % NSTAGE;
        if (it_issued >= NSTAGE) mb_wait(&emptyb[k], ((it_issued / NSTAGE) - 1) & 1);
        mb_arrive_tx(&fullb[k], TB * TB * sizeof(float));
        tma_tile(stage + (size_t)k * TB * TB, &tmA, pI * TB, pJ * TB, &fullb[k]);
        ++it_issued;
        if (++pJ > pI) { ++pI; pJ = pT0; }
    };
    // thread 0: start streaming the chunk of column jc's symmetric product
    // (A22 is the panel-start matrix: its tiles can be fetched before v is known)
    auto start_column = [&](int jc) {
        const int T0c = (jc + 1) >> 6, mtc = nt - T0c, totc = mtc * (mtc + 1) / 2;
        const int Lc = (totc + G - 1) / G, fa = cta * Lc, fb = min(totc, fa + Lc);
        it_end = it_issued + (fb > fa ? (unsigned)(fb - fa) : 0u);
        if (fb > fa) {
            tile_of(fa, T0c, pI, pJ);
            pT0 = T0c;
            while (it_issued < it_end && it_issued < it_used + NSTAGE) issue();
        }
    };
    float pv = 0.f, pw = 0.f;        // V(j, tid), W(j, tid) of the next column (prefetched, tid < jj)
    float anext = 0.f;               // A(i, j) of the next column at this thread's own row (group 0)
    float wnext = 0.f;
    __syncthreads();

    for (int jj = 0; jj < a.ncols; ++jj) {
        const int j = a.k0 + jj;
        float *acol = a.acol + (size_t)(jj & 1) * ldp;
        SYTRD_TRACE(jj, 0);
        // ------------------------------------------------------------ phase A
        // a_i = A(i, j) - sum_{t < jj} V(i,t) W(j,t) + W(i,t) V(j,t), rows i >= j.
        // Row j of column jj-1 (V = 1, W = wnext) was recomputed by this CTA in
        // phase C; rows of earlier columns are at least one barrier old.
        if (tid < jj) {
            const bool last = tid == jj - 1;
            vj[tid] = last ? 1.0f : pv;
            wj[tid] = last ? wnext : pw;
        }
        if (jj == 0 && tid == 0) start_column(j);
        __syncthreads();
        for (int q = grp; q < nown; q += NTH / 64) {
            const int I = cta + q * G, i = I * TB + r64;
            float x = 0.f, part = 0.f;
            if (i >= j && i < n) {
                x = (q == 0 && jj > 0) ? anext : a.A[i + (size_t)j * ld];                if (q < NCACHE) {
                    const float *sv = cV(q), *sw = cW(q);
                    #pragma unroll 8
                    for (int t = 0; t < jj; ++t) {
                        x = __fmaf_rn(-sv[t * TB + r64], wj[t], x);
                        x = __fmaf_rn(-sw[t * TB + r64], vj[t], x);
                    }
                } else {
                    for (int t = 0; t < jj; ++t) {
                        x = __fmaf_rn(-a.V[i + (size_t)t * ldp], wj[t], x);
                        x = __fmaf_rn(-a.W[i + (size_t)t * ldp], vj[t], x);
                    }
                }
                acol[i] = x;
                if (i >= j + 2) part = x * x;
            }
            SYTRD_TRACE(jj, 10);
            part = warp_sum(part);
            // the two warps of this group: combine in a fixed order
            if (lane == 0) rowbuf[warp][0] = part;
            __syncwarp();
            asm volatile("bar.sync %0, 64;" ::"r"(1 + grp));
            if (r64 == 0) a.rred[I] = rowbuf[2 * grp][0] + rowbuf[2 * grp + 1][0];
            asm volatile("bar.sync %0, 64;" ::"r"(1 + grp));
        }
        SYTRD_TRACE(jj, 1);
        grid_sync(a.bar, epoch);
        SYTRD_TRACE(jj, 2);
        // ------------------------------------------------------------ phase B
        if (warp == 0) {
            const float s = warp_sum_list(a.rred, 1, (j + 2) >> 6, nt);
            if (lane == 0) bc[0] = s;
        }
        __syncthreads();
        float tau, scal;
        {
            const float s = bc[0];
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
        // v at this thread's row of the first own row block (group 0), for phase C
        const float vown = (nown > 0 && tid < TB) ? v_of(acol, cta * TB + tid, j, scal) : 0.f;
        // y = A22 v over the lower tiles of A22 (rows / columns >= j+1)
        const int T0 = (j + 1) >> 6;
        const int mt = nt - T0;
        const int total = mt * (mt + 1) / 2;
        const int L = (total + G - 1) / G;
        const int f0 = cta * L, f1 = min(total, f0 + L);
        float qv = 0.f;                        // this lane's share of v^T A22 v
        float yr0 = 0.f, yr1 = 0.f;            // row partials of the current tile row (rows 2 lane, 2 lane + 1)
        if (f0 < f1) {
            // thread 0 started the chunk's TMA stream (start_column); it keeps NSTAGE ahead
            int I, J;
            tile_of(f0, T0, I, J);
            int curI = I, segf = f0;
            // raw acol values of the next tile (scaled / masked when consumed)
            float acn[8], ain0, ain1;
            auto loadv = [&](int Ii, int Jj) {
                const int r0 = Ii * TB + 2 * lane, cb = Jj * TB + 8 * warp;
                #pragma unroll
                for (int u = 0; u < 8; ++u) acn[u] = acol[cb + u];
                ain0 = acol[r0];
                ain1 = acol[r0 + 1];
            };
            auto vmask = [&](int i, float raw) { return i <= j ? 0.f : (i == j + 1 ? 1.f : raw * scal); };
            loadv(I, J);
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
                const int r0 = I * TB + 2 * lane;
                const int cb = J * TB + 8 * warp;
                float vcc[8];
                #pragma unroll
                for (int u = 0; u < 8; ++u) vcc[u] = vmask(cb + u, acn[u]);
                const float vi0 = vmask(r0, ain0), vi1 = vmask(r0 + 1, ain1);
                int In = I, Jn = J + 1;
                if (Jn > In) { ++In; Jn = T0; }
                if (f + 1 < f1) loadv(In, Jn);
                // this warp: columns 8 warp + u of the staged tile, lane rows 2 lane, 2 lane + 1
                const unsigned k = it_used % NSTAGE;
                mb_wait(&fullb[k], (it_used / NSTAGE) & 1);
                const float *tl = stage + (size_t)k * TB * TB;
                float2 x[8];
                #pragma unroll
                for (int u = 0; u < 8; ++u) x[u] = *reinterpret_cast<const float2 *>(tl + (8 * warp + u) * TB + 2 * lane);
                __syncwarp();
                if (lane == 0) mb_arrive(&emptyb[k]);
                ++it_used;
                if (tid == 0 && it_issued < it_end) issue();
                float cz[8];
                #pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int c = cb + u;
                    const float vc = vcc[u];
                    float x0 = x[u].x, x1 = x[u].y;
                    if (I == J) {                 // diagonal tile: the lower triangle r >= c only
                        const float y0 = r0 >= c ? x0 : 0.f, y1 = r0 + 1 >= c ? x1 : 0.f;
                        yr0 = __fmaf_rn(y0, vc, yr0);
                        yr1 = __fmaf_rn(y1, vc, yr1);
                        if (r0 == c) qv = __fmaf_rn(y0 * vc, vc, qv);        // A_cc v_c^2
                        if (r0 + 1 == c) qv = __fmaf_rn(y1 * vc, vc, qv);
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
                    float vc = vcc[0];
                    #pragma unroll
                    for (int q2 = 1; q2 < 8; ++q2) vc = (u == q2) ? vcc[q2] : vc;   // no local-memory indexing
                    qv = __fmaf_rn(2.0f * cz[0], vc, qv);   // A_IJ and its mirror (strict lower part if I == J)
                    a.Pcol[(size_t)(cofs(J, T0, nt) + I - J) * TB + 8 * warp + u] = cz[0];
                }
                I = In; J = Jn;
            }
        }
        SYTRD_TRACE(jj, 3);
        // v^T A22 v of this CTA
        qv = warp_sum(qv);
        if (lane == 0) wq[warp] = qv;
        __syncthreads();
        if (tid == 0) {
            float qs = 0.f;
            #pragma unroll
            for (int w = 0; w < NTH / 32; ++w) qs += wq[w];
            a.qred[cta] = qs;
        }
        // panel dot products v^T V(:, t), v^T W(:, t) (t < jj) over the own row blocks:
        // warp w takes batches of 8 consecutive slots (slot sl < jj: V(:, sl), else W(:, sl - jj))
        for (int q = 0; q < nown; ++q) {
            const int I = cta + q * G;
            const int i0 = I * TB + lane, i1 = i0 + 32;
            const float v0 = i0 < n ? v_of(acol, i0, j, scal) : 0.f;
            const float v1 = i1 < n ? v_of(acol, i1, j, scal) : 0.f;
            for (int b8 = warp * 8; b8 < 2 * jj; b8 += NTH / 32 * 8) {
                float c[8];
                #pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int sl = b8 + k;
                    float x0 = 0.f, x1 = 0.f;
                    if (sl < 2 * jj) {
                        const int t = sl < jj ? sl : sl - jj;
                        if (q < NCACHE) {
                            const float *cc = (sl < jj ? cV(q) : cW(q)) + t * TB;
                            x0 = cc[lane]; x1 = cc[lane + 32];
                        } else {
                            const float *cc = (sl < jj ? a.V : a.W) + (size_t)t * ldp;
                            x0 = cc[i0]; x1 = cc[i1];
                        }
                    }
                    c[k] = __fmaf_rn(x1, v1, x0 * v0);
                }
                int u;
                const float acc = warp_sum8(c, u);
                if ((lane & 3) == 0 && b8 + u < 2 * jj) a.rred[(size_t)(1 + b8 + u) * a.ntp + I] = acc;
            }
        }
        SYTRD_TRACE(jj, 4);
        grid_sync(a.bar, epoch);
        SYTRD_TRACE(jj, 5);
        // ------------------------------------------------------------ phase C
        // only CTAs owning rows >= j+1 have work here (and need the reduced
        // dots, v^T A22 v and row j+1 of w); the others only keep the symv's
        // tile stream going (start_column) -- no redundant partial-sum traffic
        const bool active = nown > 0 && (cta + (nown - 1) * G) * TB + TB - 1 >= j + 1;
        if (!active) {
            if (jj + 1 < a.ncols && tid == 0) start_column(j + 1);
            continue;
        }
        // C1: every partial sum this CTA needs, loads issued together: the dots
        // (thread (half, slot)), v^T A22 v (warp 7, extra), y of the first own
        // row block (thread group grp takes part grp of the tile-column list);
        // and the next column's inputs that are already final: its symv tiles
        // (thread 0), V / W at its row j+1 (t < jj), A(:, j+1) at the own rows
        if (jj + 1 < a.ncols) {
            if (tid == 0) start_column(j + 1);
            if (tid < jj) { pv = a.V[(j + 1) + (size_t)tid * ldp]; pw = a.W[(j + 1) + (size_t)tid * ldp]; }
            if (tid < TB && nown > 0 && cta * TB + tid < n) anext = a.A[cta * TB + tid + (size_t)(j + 1) * ld];
        }
        {
            const int sl = tid & 127, half = tid >> 7;
            float s = 0.f;
            if (sl < 2 * jj) {
                const float4 *p = reinterpret_cast<const float4 *>(a.rred + (size_t)(1 + sl) * a.ntp);
                const int nq = a.ntp >> 2;
                float s0 = 0.f, s1 = 0.f;
                #pragma unroll 8
                for (int q4 = half; q4 < nq; q4 += 2) {
                    const float4 v4 = p[q4];
                    s0 += v4.x + v4.y;
                    s1 += v4.z + v4.w;
                }
                s = s0 + s1;
            }
            SYTRD_TRACE(jj, 11);
            float yp = 0.f;
            const int I0 = cta;                          // first own row block (if any)
            const bool own0 = nown > 0 && (I0 + 1) * TB > j + 1;
            if (own0) yp = y_part(a, I0, r64, T0, L, grp, NTH / 64);
            if (warp == NTH / 32 - 1) {
                const float4 *p = reinterpret_cast<const float4 *>(a.qred);
                const int nq = (G + 3) >> 2;
                float s0 = 0.f, s1 = 0.f;
                #pragma unroll 4
                for (int q4 = lane; q4 < nq; q4 += 32) {
                    const float4 v4 = p[q4];
                    s0 += v4.x + v4.y;
                    s1 += v4.z + v4.w;
                }
                const float qs = warp_sum(s0 + s1);
                if (lane == 0) bc[1] = qs;
            }
            if (half == 1 && sl < 2 * jj) dots[sl] = s;
            if (own0) rowbuf[grp * 2][r64] = yp;
            __syncthreads();
            if (half == 0 && sl < 2 * jj) dots[sl] = s + dots[sl];
            __syncthreads();
        }
        SYTRD_TRACE(jj, 8);
        // C2: sum_t (v^T V_t)(v^T W_t) by warp 0, then v^T p = tau (v^T A22 v - 2 sum),
        // alpha' = -(tau/2) v^T p
        if (warp == 0) {
            float sp = 0.f;
            for (int t = lane; t < jj; t += 32) sp = __fmaf_rn(dots[t], dots[jj + t], sp);
            sp = warp_sum(sp);
            if (lane == 0) bc[3] = sp;
        }
        __syncthreads();
        SYTRD_TRACE(jj, 9);
        const float vtp = tau * __fmaf_rn(-2.0f, bc[3], bc[1]);
        const float alph = -0.5f * tau * vtp;
        // w_i = tau (y_i - V(i,:) (W^T v) - W(i,:) (V^T v)) + alpha' v_i  (rows i >= j+1)
        for (int q = 0; q < nown; ++q) {
            const int I = cta + q * G;
            if ((I + 1) * TB <= j + 1) continue;
            if (q > 0) {      // (only when the grid has fewer CTAs than row blocks)
                rowbuf[grp * 2][r64] = y_part(a, I, r64, T0, L, grp, NTH / 64);
                __syncthreads();
            }
            if (grp == 0) {
                const int i = I * TB + r64;
                float y = ((rowbuf[0][r64] + rowbuf[2][r64]) + rowbuf[4][r64]) + rowbuf[6][r64];
                if (i >= j + 1 && i < n) {
                    float y2 = 0.f;
                    if (q < NCACHE) {
                        const float *sv = cV(q), *sw = cW(q);
                        #pragma unroll 8
                        for (int t = 0; t < jj; ++t) {
                            y = __fmaf_rn(-sv[t * TB + r64], dots[jj + t], y);
                            y2 = __fmaf_rn(-sw[t * TB + r64], dots[t], y2);
                        }
                    } else {
                        for (int t = 0; t < jj; ++t) {
                            y = __fmaf_rn(-a.V[i + (size_t)t * ldp], dots[jj + t], y);
                            y2 = __fmaf_rn(-a.W[i + (size_t)t * ldp], dots[t], y2);
                        }
                    }
                    y += y2;
                    const float vi = q == 0 ? vown : v_of(acol, i, j, scal);
                    const float w = __fmaf_rn(alph, vi, tau * y);
                    a.W[i + (size_t)jj * ldp] = w;
                    a.V[i + (size_t)jj * ldp] = vi;
                    if (q < NCACHE) { cW(q)[jj * TB + r64] = w; cV(q)[jj * TB + r64] = vi; }
                    if (i >= j + 2) a.A[i + (size_t)j * ld] = vi;     // reflector storage (LAPACK layout)
                }
            }
            __syncthreads();
        }
        SYTRD_TRACE(jj, 7);
        // row j+1 of this column's w, for the next column's phase A (every CTA):
        // warps 0-3 split the partial vectors of y_{j+1} and the correction
        if (jj + 1 < a.ncols && j + 1 < n) {
            const int i = j + 1, I = i >> 6, r = i & 63;
            if (warp < 4) {
                const int t4 = tid;          // 0..127
                float y = 0.f;
                const int fa = flat_of(I, T0, T0), fb = flat_of(I, I, T0);
                if (t4 == 0) y = a.Prow[(size_t)fa * TB + r];
                for (int f = (fa / L + 1 + t4) * L; f <= fb; f += 128 * L) y += a.Prow[(size_t)f * TB + r];
                const float *pc = a.Pcol + (size_t)cofs(I, T0, nt) * TB + r;
                if (t4 < nt - I) y += pc[(size_t)t4 * TB];
                if (t4 + 128 < nt - I) y += pc[(size_t)(t4 + 128) * TB];
                for (int k = t4 + 256; k < nt - I; k += 128) y += pc[(size_t)k * TB];
                float corr = 0.f;
                if (t4 < jj) corr = __fmaf_rn(pv, dots[jj + t4], pw * dots[t4]);   // V, W(j+1, t4) (prefetched)
                y = warp_sum(y);
                corr = warp_sum(corr);
                if (lane == 0) { rowbuf[warp][0] = y; rowbuf[warp][1] = corr; }
            }
            __syncthreads();
            if (tid == 0) {
                const float y = (rowbuf[0][0] + rowbuf[1][0]) + (rowbuf[2][0] + rowbuf[3][0]);
                const float corr = (rowbuf[0][1] + rowbuf[1][1]) + (rowbuf[2][1] + rowbuf[3][1]);
                bc[2] = __fmaf_rn(alph, 1.0f, tau * (y - corr));
            }
            __syncthreads();
            wnext = bc[2];
        }
        __syncthreads();
        SYTRD_TRACE(jj, 6);
    }
    // ------------------------------------------------------------ trailing update
    // A(s0:, s0:) -= V W^T + W V^T on the lower tiles (s0 = first row / column
    // after the panel)
    grid_sync(a.bar, epoch);
    const int s0 = a.k0 + a.ncols;
    if (s0 >= n) return;
    const int T1 = s0 >> 6;
    const int mt = nt - T1;
    const int total = mt * (mt + 1) / 2;
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

// 1 / q to about one ulp: the MUFU reciprocal seed and two Newton steps
// (2^-23 -> 2^-46 -> rounding); q is never 0 or subnormal here (pivmin
// guard).  Not correctly rounded: the Sturm counts and the twisted
// factorisations stay backward stable (a few-ulp relative perturbation of
// e_i^2 per step), at about half the dependent latency of a rounded division.
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
__device__ __forceinline__ int sturm_count(const double *__restrict__ d, const double *__restrict__ e2, int s, int e,
                                           double x, double pivmin)
{
    double q = d[s] - x;
    if (fabs(q) <= pivmin) q = -pivmin;
    int cnt = q < 0.0;
    #pragma unroll 8
    for (int i = s + 1; i <= e; ++i) {      // unrolled: the d / e2 loads run ahead of the q chain
        q = __fma_rn(-e2[i - 1], rcp_nr(q), d[i] - x);
        if (fabs(q) <= pivmin) q = -pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

// eigenvalue t (the (t - bstart)-th smallest of its block) by multisection:
// the MSEC lanes of a group evaluate Sturm counts at MSEC interior points of
// the current interval, which shrinks (MSEC + 1)x per round, until it is
// within 2 omega of max(|lo|, |hi|) or of the block's Gershgorin bound (the
// Sturm count resolves nothing finer).  MSEC = 32 (5 bits per round, a warp
// per eigenvalue) for n <= 2048, where the n eigenvalues alone would not
// fill the GPU; 8 above.
template <int MSEC>
__global__ void __launch_bounds__(256) k_tri_bisect(const double *__restrict__ d, const double *__restrict__ e64,
                                                    const double *__restrict__ e2, const int *__restrict__ bstart,
                                                    const int *__restrict__ bend,
                                                    const double *__restrict__ pivmin_p, int n, double *lam)
{
    const int lane8 = threadIdx.x & (MSEC - 1);
    const int t = blockIdx.x * (blockDim.x / MSEC) + threadIdx.x / MSEC;
    const bool valid = t < n;
    const int tt = valid ? t : n - 1;
    const int s = bstart[tt], e = bend[tt], k = tt - s;
    const double pivmin = pivmin_p[0];
    const int base = threadIdx.x & 31 & ~(MSEC - 1);
    const unsigned gmask = (MSEC == 32 ? 0xffffffffu : ((1u << MSEC) - 1)) << base;
    double lo = 1e308, hi = -1e308;
    // Gershgorin interval of the block (split over the group's lanes)
    for (int i = s + lane8; i <= e; i += MSEC) {
        const double r = (i > s ? fabs(e64[i - 1]) : 0.0) + (i < e ? fabs(e64[i]) : 0.0);
        lo = fmin(lo, d[i] - r);
        hi = fmax(hi, d[i] + r);
    }
    #pragma unroll
    for (int o = MSEC / 2; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(gmask, lo, o));
        hi = fmax(hi, __shfl_xor_sync(gmask, hi, o));
    }
    const double gnorm = fmax(fabs(lo), fabs(hi));
    const double pad = 2.0 * kOmega * gnorm + pivmin;
    lo -= pad;
    hi += pad;
    if (s < e) {
        for (int round = 0; round < 80; ++round) {
            if (hi - lo <= 2.0 * kOmega * fmax(gnorm, fmax(fabs(lo), fabs(hi)))) break;
            const double w = (hi - lo) / (MSEC + 1);
            double x = lo + w * (lane8 + 1);
            if (!(x > lo)) x = lo;
            if (!(x < hi)) x = hi;
            const int c = sturm_count(d, e2, s, e, x, pivmin);
            // first point with more than k eigenvalues below it bounds from above
            const unsigned ball = __ballot_sync(gmask, c > k) & gmask;
            const int m_hi = ball ? __ffs(ball) - 1 - base : MSEC;       // index of that point (MSEC: hi)
            const double nlo = m_hi > 0 ? __shfl_sync(gmask, x, base + m_hi - 1) : lo;
            const double nhi = m_hi < MSEC ? __shfl_sync(gmask, x, base + m_hi) : hi;
            const bool done = !(nlo < nhi) || (nlo == lo && nhi == hi);
            lo = nlo;
            hi = nhi;
            if (done) break;
        }
    }
    if (valid && lane8 == 0) lam[t] = s < e ? 0.5 * (lo + hi) : d[s];
}

// thread t: eigenvector of lam[t] on its block by the twisted factorisation
// T - lam I = N_r Delta_r N_r^T (forward D+, backward D-), r = argmin |gamma_r|,
// x_r = 1: x_i = -(e_i / D+_i) x_{i+1} above r, x_{i+1} = -(e_i / D-_{i+1}) x_i
// below.  Column t of Y (ld ldy, zero outside the block) gets x / ||x||.
__global__ void k_tri_twisted(const double *__restrict__ d, const double *__restrict__ e64,
                              const double *__restrict__ e2, const int *__restrict__ bstart,
                              const int *__restrict__ bend, const double *__restrict__ pivmin_p,
                              const double *__restrict__ lam, int n, double *__restrict__ Dp,
                              double *__restrict__ Dm, double *__restrict__ inv_nrm)
{
    // two lanes per eigenvalue: role 0 runs the forward factorisation (D+) and
    // the solve above r, role 1 the backward one (D-) and the solve below r --
    // the two division chains run side by side
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int t = gt >> 1, role = gt & 1;
    const unsigned pmask = 3u << (threadIdx.x & 30);
    const bool valid = t < n;
    const int tt = valid ? t : n - 1;
    const int s = bstart[tt], e = bend[tt];
    // x is written row-major into Dp (x_i at Dp[i n + t], over D+_i once it is
    // consumed): consecutive eigenvalues write consecutive words
    if (s == e) {
        if (valid && role == 0) { Dp[(size_t)s * n + t] = 1.0; inv_nrm[t] = 1.0; }
        return;
    }
    const double pivmin = pivmin_p[0], l = lam[tt];
    auto guard = [&](double q) { return fabs(q) < pivmin ? (q < 0.0 ? -pivmin : pivmin) : q; };
    if (valid) {
        if (role == 0) {                                   // forward
            double q = guard(d[s] - l);
            Dp[(size_t)s * n + t] = q;
            #pragma unroll 8
            for (int i = s + 1; i <= e; ++i) {
                q = guard(__fma_rn(-e2[i - 1], rcp_nr(q), d[i] - l));
                Dp[(size_t)i * n + t] = q;
            }
        } else {                                           // backward
            double q = guard(d[e] - l);
            Dm[(size_t)e * n + t] = q;
            #pragma unroll 8
            for (int i = e - 1; i >= s; --i) {
                q = guard(__fma_rn(-e2[i], rcp_nr(q), d[i] - l));
                Dm[(size_t)i * n + t] = q;
            }
        }
    }
    __syncwarp(pmask);
    // r = argmin |gamma_i|, gamma_i = D+_i + D-_i - (d_i - lam) (ties: the larger i,
    // as a scan from e downwards); each lane scans half of [s, e]
    const int mid = (s + e + 1) >> 1;
    const int i0 = role == 0 ? s : mid, i1 = role == 0 ? mid - 1 : e;
    double gbest = 1e308;
    int r = -1;
    if (valid) {
        #pragma unroll 8
        for (int i = i1; i >= i0; --i) {
            const double g = fabs(Dp[(size_t)i * n + t] + Dm[(size_t)i * n + t] - (d[i] - l));
            if (g < gbest) { gbest = g; r = i; }
        }
    }
    const double go = __shfl_xor_sync(pmask, gbest, 1);
    const int ro = __shfl_xor_sync(pmask, r, 1);
    // role 1's half holds the larger indices: it wins ties
    const bool mine_hi = role == 1;
    if (go < gbest || (go == gbest && !mine_hi && ro >= 0)) { gbest = go; r = ro; }
    __syncwarp(pmask);
    double nrm = 0.0;
    if (valid) {
        // the divisors are loaded 8 at a time ahead of the x chain (the store of
        // x_i goes to the slot just read, so the compiler cannot hoist the loads;
        // one exposed L2 latency per 8 steps instead of one per step)
        constexpr int PF = 8;
        if (role == 0) {                                   // x_r = 1, then upwards
            double x = 1.0;
            nrm = 1.0;
            for (int i = r - 1; i >= s; i -= PF) {
                double dv[PF];
                #pragma unroll
                for (int u = 0; u < PF; ++u) dv[u] = (i - u >= s) ? Dp[(size_t)(i - u) * n + t] : 1.0;
                #pragma unroll
                for (int u = 0; u < PF; ++u)
                    if (i - u >= s) {
                        x = -(e64[i - u] * rcp_nr(dv[u])) * x;
                        Dp[(size_t)(i - u) * n + t] = x;
                        nrm = __fma_rn(x, x, nrm);
                    }
            }
        } else {                                           // downwards
            double x = 1.0;
            for (int i = r; i < e; i += PF) {
                double dv[PF];
                #pragma unroll
                for (int u = 0; u < PF; ++u) dv[u] = (i + u < e) ? Dm[(size_t)(i + u + 1) * n + t] : 1.0;
                #pragma unroll
                for (int u = 0; u < PF; ++u)
                    if (i + u < e) {
                        x = -(e64[i + u] * rcp_nr(dv[u])) * x;
                        Dp[(size_t)(i + u + 1) * n + t] = x;
                        nrm = __fma_rn(x, x, nrm);
                    }
            }
        }
    }
    __syncwarp(pmask);
    if (valid && role == 0) Dp[(size_t)r * n + t] = 1.0;
    const double nrm_all = nrm + __shfl_xor_sync(pmask, nrm, 1);
    if (valid && role == 0) inv_nrm[t] = 1.0 / sqrt(nrm_all);
}

// Y(i, t) = x_i^(t) / ||x^(t)|| inside eigenvector t's block, 0 outside: a
// 32 x 32 tiled transpose of the row-major X (= Dp) into column-major Y
__global__ void k_tri_transpose(const double *__restrict__ X, int n, const int *__restrict__ bstart,
                                const int *__restrict__ bend, const double *__restrict__ inv_nrm, double *Y,
                                int64_t ldy)
{
    __shared__ double tile[32][33];
    const int i0 = blockIdx.y * 32, t0 = blockIdx.x * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;            // 32 x 8
    for (int r = ty; r < 32; r += 8) {                        // read rows i0 + r, columns t0 + tx
        const int i = i0 + r, t = t0 + tx;
        double v = 0.0;
        if (i < n && t < n && i >= bstart[t] && i <= bend[t]) v = X[(size_t)i * n + t] * inv_nrm[t];
        tile[r][tx] = v;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {                        // write column t0 + r, rows i0 + tx
        const int t = t0 + r, i = i0 + tx;
        if (i < n && t < n) Y[i + (size_t)t * ldy] = tile[tx][r];
    }
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
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL)
    const int t = blockIdx.y;
    const int r0 = k0 + 1;
    const int j = k0 + t;
    for (int i = r0 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double v = 0.0;
        if (t < nr) v = i < j + 1 ? 0.0 : (i == j + 1 ? 1.0 : (double)A[i + (size_t)j * lda]);
        Vp[(i - r0) + (size_t)t * ldv] = v;
    }
}

// Tp (BT x BT, ld BT) of H_k0 ... H_{k0+nr-1} = I - Vp Tp Vp^T (LAPACK dlarft,
// forward, columnwise) from the Gram matrix G = Vp^T Vp (ld BT).  One CTA of
// 256 threads: column t is T(0:t, t) = -tau_t T(0:t, 0:t) G(0:t, t), the
// triangular product split over four thread groups per row.
constexpr int BT = 2 * TB;       // back-transformation block (two sytrd panels)
__global__ void __launch_bounds__(1024) k_build_tp(const double *__restrict__ G, const float *__restrict__ tau, int k0,
                                                  int nr, double *Tp)
{
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL)
    extern __shared__ double tsm[];          // T (BT x BT+1), z (BT), part (2 x BT), M (3 x 32 x 32)
    double *T = tsm, *z = T + BT * (BT + 1), *part = z + BT;
    const int tid = threadIdx.x, row = tid & (BT - 1), grp = tid >> 7;   // fallback: 2 groups x 128 rows
    const int nthr = blockDim.x;
    constexpr int LS = BT + 1, QB = 32;      // leading dimension, diagonal block size
    double *M = part + 2 * BT;
    __shared__ int zero_tau;
    if (tid == 0) zero_tau = 0;
    __syncthreads();
    if (tid < nr && tau[k0 + tid] == 0.f) zero_tau = 1;
    __syncthreads();
    if (!zero_tau) {
        // T = S^{-1}, S = diag(1 / tau) + strict upper part of G (the compact-WY
        // identity T^{-1} + T^{-T} = V^T V in its triangular form, Joffrain et
        // al. 2006; exact for any nonzero tau): the 32 x 32 diagonal blocks by
        // back substitution (thread per column), then the off-diagonal blocks
        // T_ij = -T_ii sum_{k=i+1..j} S_ik T_kj by block diagonals -- 2 barriers
        // per block diagonal instead of 3 per reflector.  One array: S's strict
        // upper part above the diagonal, T transposed on and below it.
        auto tinv = [&](int i) { return i < nr ? (double)tau[k0 + i] : 1.0; };   // padding: identity
        for (int e = tid; e < BT * LS; e += nthr) T[e] = 0.0;
        __syncthreads();
        for (int e = tid; e < BT * BT; e += nthr) {
            const int i = e & (BT - 1), j = e / BT;
            if (i < j && j < nr) T[i + j * LS] = G[i + j * BT];
        }
        __syncthreads();
        if (tid < BT) {                                         // T_bb: column t of its 32-block
            const int t = tid, b0 = (t / QB) * QB;
            T[t + t * LS] = tinv(t);
            for (int i = t - 1; i >= b0; --i) {
                double acc = 0.0;
                for (int u = i + 1; u <= t; ++u) acc = __fma_rn(T[i + u * LS], T[t + u * LS], acc);
                T[t + i * LS] = -tinv(i) * acc;
            }
        }
        __syncthreads();
        for (int dg = 1; dg < BT / QB; ++dg) {                  // block diagonal dg: blocks (bi, bi + dg)
            const int nb = BT / QB - dg;
            for (int e = tid; e < nb * QB * QB; e += nthr) {     // M = sum_{k=i+1..j} S_ik T_kj
                const int bi = e / (QB * QB), r = (e / QB) % QB, cc = e % QB;
                const int i0 = bi * QB, col = (bi + dg) * QB + cc;
                double acc = 0.0;
                for (int u = i0 + QB; u <= col; ++u) acc = __fma_rn(T[(i0 + r) + u * LS], T[col + u * LS], acc);
                M[(size_t)bi * QB * QB + r * QB + cc] = acc;     // row-major: lanes (cc) consecutive
            }
            __syncthreads();
            for (int e = tid; e < nb * QB * QB; e += nthr) {     // T_ij = -T_ii M
                const int bi = e / (QB * QB), r = (e / QB) % QB, cc = e % QB;
                const int i0 = bi * QB, col = (bi + dg) * QB + cc;
                double acc = 0.0;
                for (int u = r; u < QB; ++u)
                    acc = __fma_rn(T[(i0 + u) + (i0 + r) * LS], M[(size_t)bi * QB * QB + u * QB + cc], acc);
                T[col + (i0 + r) * LS] = -acc;
            }
            __syncthreads();
        }
        for (int e = tid; e < BT * BT; e += nthr) {
            const int i = e & (BT - 1), j = e / BT;
            Tp[e] = (i <= j && j < nr) ? T[j + i * LS] : 0.0;
        }
        return;
    }
    for (int e = tid; e < BT * (BT + 1); e += nthr) T[e] = 0.0;
    __syncthreads();
    // a zero tau (an identity reflector): LAPACK's column recurrence
    double gnext = (tid < BT && nr > 0) ? G[tid] : 0.0;        // G(tid, t), loaded one step ahead
    for (int t = 0; t < nr; ++t) {
        const double ta = (double)tau[k0 + t];
        const double gcur = gnext;
        if (tid < BT && t + 1 < nr) gnext = G[tid + (t + 1) * BT];
        if (tid < t) z[tid] = -ta * gcur;
        __syncthreads();
        // T(row, t) = sum_{u = row}^{t-1} T(row, u) z(u): group grp takes u = row + grp, +2, ...
        double acc = 0.0;
        if (row < t && grp < 2)
            for (int u = row + grp; u < t; u += 2) acc = __fma_rn(T[row + u * (BT + 1)], z[u], acc);
        if (grp < 2) part[grp * BT + row] = acc;
        __syncthreads();
        if (tid < t) T[tid + t * (BT + 1)] = part[tid] + part[BT + tid];
        if (tid == 0) T[t + t * (BT + 1)] = ta;
        __syncthreads();
    }
    for (int e = tid; e < BT * BT; e += nthr) Tp[e] = T[(e & (BT - 1)) + (e / BT) * (BT + 1)];
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

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder()
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

// co-resident CTAs of the cooperative panel kernel on the current device (its
// shared-memory opt-in is per device: set through smem_optin on every call)
int coop_ctas()
{
    static std::mutex mu;
    static std::map<int, int> per_dev;
    int dev = 0;
    cudaGetDevice(&dev);
    int occ = 1;
    if (smem_optin((const void *)k_sytrd_panel, SYTRD_SMEM, NTH, &occ) != cudaSuccess) occ = 1;
    std::lock_guard<std::mutex> lk(mu);
    auto it = per_dev.find(dev);
    if (it == per_dev.end()) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        int want = 2;
        if (const char *e = getenv("MPJ_SYTRD_OCC")) want = std::max(1, atoi(e));   // A/B: CTAs per SM
        it = per_dev.emplace(dev, sms * std::max(1, std::min(occ, want))).first;
    }
    return it->second;
}

}  // namespace

// ---------------------------------------------------------------------------
// workspace and driver
// ---------------------------------------------------------------------------
struct SymqrWs {
    float *V, *W, *acol, *d, *e, *tau, *Prow, *Pcol, *rred, *qred;
    unsigned *bar;
    double *d64, *e64, *e2, *lam, *piv, *Vp, *Gm, *Tp, *W1, *W2, *skw, *inrm;
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
    w.rred = (float *)take((size_t)RSLOT * ((nt + 3) / 4 * 4) * 4);
    w.qred = (float *)take((size_t)(G + 4) * 4);
    w.bar = (unsigned *)take(64);
    w.d64 = (double *)take(np * 8);
    w.e64 = (double *)take(np * 8);
    w.e2 = (double *)take(np * 8);
    w.lam = (double *)take(np * 8);
    w.inrm = (double *)take(np * 8);
    w.piv = (double *)take(64);
    w.bstart = (int *)take(np * 4);
    w.bend = (int *)take(np * 4);
    w.rank = (int *)take(np * 4);
    w.Vp = (double *)take(np * BT * 8);
    w.Gm = (double *)take(BT * BT * 8);
    w.Tp = (double *)take(BT * BT * 8);
    w.W1 = (double *)take(np * BT * 8);
    w.W2 = (double *)take(np * BT * 8);
    w.skw_elems = (size_t)8 * BT * np;
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
namespace {
// ---------------------------------------------------------------------------
// 1'. Small n (the whole lower triangle fits the distributed shared memory of
// one 16-CTA cluster, n <= ~1150): the unblocked reduction (LAPACK ssytd2,
// the same reflectors as above) with the matrix resident in shared memory for
// all n - 2 columns.  CTA c owns rows i = 16 r + c (lower part, packed); per
// column k:
//   publish x = A(k+1:, k) at the own rows and the partial ||x(1:)||^2;
//   cluster barrier; gather x and the 16 partials (DSMEM, fixed order) ->
//   beta, tau, v, identical in every CTA;
//   y = A22 v: own-row dots (16 lanes per row) and own-column sums of the
//   strict lower part (thread per column), summed into this CTA's partial y;
//   cluster barrier; y_j = sum of the 16 partials (fixed order), p = tau y,
//   w = p - (tau/2)(p^T v) v in every CTA; A22 -= v w^T + w v^T on the own rows.
// Two cluster barriers per column (~0.2 us each) instead of the panel
// kernel's two grid barriers and L2 round trips per column -- what bounds the
// panel kernel at n ~ 1000 (tools/sytrd_trace.py: ~13-18 us per column).
// ---------------------------------------------------------------------------
constexpr int SCL = 16;          // CTAs per cluster (non-portable size)
constexpr int SCNT = 1024;       // threads per CTA

__host__ __device__ __forceinline__ int sc_rows(int n, int c) { return c < n ? (n - c + SCL - 1) / SCL : 0; }
__host__ __device__ __forceinline__ int sc_rm(int n) { return ((n + SCL - 1) / SCL + 3) / 4 * 4; }   // rows, padded
__host__ __device__ __forceinline__ int sc_rowlen(int r, int c) { return (SCL * r + c + 1 + 3) & ~3; }
// shared memory (floats): the exchange buffers at the same offsets in every CTA,
// then the local vectors and the packed own rows
struct ScLay {
    int rm, np4;
    int xin, nin, pin, pfull, vv, ww, part4, roff, own;
    __host__ __device__ ScLay(int n)
    {
        rm = sc_rm(n); np4 = (n + 3) / 4 * 4;
        xin = 0; nin = xin + SCL * rm; pin = nin + SCL; pfull = pin + SCL * rm;
        vv = pfull + SCL * rm; ww = vv + np4; part4 = ww + np4; roff = part4 + 4 * np4;
        own = roff + rm + 4;
    }
};
static size_t sc_smem(int n)
{
    ScLay L(n);
    int64_t mx = 0;
    for (int c = 0; c < SCL; ++c) {
        int64_t o = 0;
        for (int r = 0; r < sc_rows(n, c); ++r) o += sc_rowlen(r, c);
        mx = std::max(mx, o);
    }
    return ((size_t)L.own + (size_t)mx) * 4;
}

__device__ __forceinline__ unsigned sc_map(const void *p, int rank)
{
    unsigned r;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void sc_st4(unsigned a, float4 v)
{
    asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void sc_st(unsigned a, float v)
{
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void sc_cluster_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

#ifdef MPJ_SYTRD_TRACE
#define SCT(ev) if (k >= g_trace_k0 && k < g_trace_k0 + 64 && threadIdx.x == 0) { unsigned long long t_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_sytrd_trace[((size_t)(k - g_trace_k0) * 12 + (ev)) * 320 + c] = t_; }
#else
#define SCT(ev)
#endif

// Exchange pattern per column (all remote traffic is 16-byte stores, pushed
// by the owner; every read is local): x and the norm partials of the own rows
// to every CTA; the partial y of every row to the row's owner; the owner's p
// to every CTA.  Three cluster barriers per column.
__global__ void __launch_bounds__(SCNT, 1) k_sytrd_cluster(float *A, int64_t ld, int n, float *dout, float *eout,
                                                           float *tout)
{
    extern __shared__ __align__(16) float smem[];
    __shared__ float red[2][SCNT / 32];
    unsigned crank;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    const int c = (int)crank, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int R = sc_rows(n, c);
    const ScLay L(n);
    const int RM = L.rm;
    float *xin = smem + L.xin, *nin = smem + L.nin, *pin = smem + L.pin, *pfull = smem + L.pfull;
    float *vv = smem + L.vv, *ww = smem + L.ww, *part4 = smem + L.part4;
    int *roff = (int *)(smem + L.roff);
    float *Aown = smem + L.own;
    if (tid == 0) {
        int o = 0;
        for (int r = 0; r <= R; ++r) { roff[r] = o; if (r < R) o += sc_rowlen(r, c); }
    }
    __syncthreads();
    // own rows of the lower triangle (only the lower triangle is current when this
    // runs on the trailing matrix of the panel kernel), zero padded
    for (int r = 0; r < R; ++r) {
        const int i = SCL * r + c, len = sc_rowlen(r, c);
        for (int j = tid; j < len; j += SCNT) Aown[roff[r] + j] = j <= i ? A[i + (size_t)j * ld] : 0.f;
    }
    __syncthreads();
    // push the x of column kx (own rows i >= kx+1) and the partial norm (i >= kx+2) to every CTA
    auto push_x = [&](int kx) {
        if (tid < SCL * (RM / 4)) {
            const int dst = tid / (RM / 4), r4 = tid % (RM / 4);
            float v[4];
            #pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int r = 4 * r4 + u, i = SCL * r + c;
                v[u] = (r < R && i >= kx + 1) ? Aown[roff[r] + kx] : 0.f;
            }
            sc_st4(sc_map(xin + c * RM + 4 * r4, dst), make_float4(v[0], v[1], v[2], v[3]));
        } else if (warp == SCNT / 32 - 1) {
            float sq = 0.f;
            for (int r = lane; r < R; r += 32) {
                const int i = SCL * r + c;
                if (i >= kx + 2) { const float x = Aown[roff[r] + kx]; sq = __fmaf_rn(x, x, sq); }
            }
            #pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
            if (lane < SCL) sc_st(sc_map(nin + c, lane), sq);
        }
    };
    int k = 0;
    push_x(0);
    int rb = 0;
    for (k = 0; k + 2 < n; ++k) {
        SCT(0);
        sc_cluster_sync();                                               // #1: x, norm partials
        SCT(1);
        float s = 0.f;
        #pragma unroll
        for (int q = 0; q < SCL; ++q) s += nin[q];
        const float alpha = xin[((k + 1) % SCL) * RM + (k + 1) / SCL];
        float beta, tau, scal;
        if (s == 0.f) { beta = alpha; tau = 0.f; scal = 0.f; }
        else {
            const float nrm = sqrtf(__fmaf_rn(alpha, alpha, s));
            beta = alpha >= 0.f ? -nrm : nrm;
            tau = (beta - alpha) / beta;
            scal = 1.0f / (alpha - beta);
        }
        for (int j = tid; j < L.np4; j += SCNT)
            vv[j] = (j <= k || j >= n) ? 0.f : (j == k + 1 ? 1.f : xin[(j % SCL) * RM + j / SCL] * scal);
        if (tid == 0) {
            if (c == k % SCL) dout[k] = Aown[roff[k / SCL] + k];
            if (c == 0) { eout[k] = beta; tout[k] = tau; }
        }
        __syncthreads();                                                 // v
        SCT(2);
        const float4 *vv4 = reinterpret_cast<const float4 *>(vv);
        const int j40 = (k + 1) >> 2, nj4 = L.np4 >> 2;
        // own-row dots y_i = sum_{k < j <= i} A_ij v_j: 16 lanes per row, float4 columns
        float rdot[2] = {0.f, 0.f};
        #pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = h * (SCNT / 16) + (tid >> 4), l16 = tid & 15;
            float acc = 0.f;
            if (r < R) {
                const int i = SCL * r + c;
                const float4 *row = reinterpret_cast<const float4 *>(Aown + roff[r]);
                for (int j4 = j40 + l16; 4 * j4 <= i; j4 += 16) {
                    const float4 a = row[j4], v = vv4[j4];         // v_j = 0 for j <= k; masked j > i
                    const int j = 4 * j4;
                    acc = __fmaf_rn(a.x, v.x, acc);
                    if (j + 1 <= i) acc = __fmaf_rn(a.y, v.y, acc);
                    if (j + 2 <= i) acc = __fmaf_rn(a.z, v.z, acc);
                    if (j + 3 <= i) acc = __fmaf_rn(a.w, v.w, acc);
                }
            }
            #pragma unroll
            for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            rdot[h] = acc;
        }
        // own-column sums of the strict lower part: 256 float4 column groups x 4 row groups
        {
            const int rg = tid >> 8, cg = tid & 255;
            for (int j4 = j40 + cg; j4 < nj4; j4 += 256) {
                const int j = 4 * j4;
                float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
                int r = (j + 1 - c + SCL - 1) / SCL;             // first own row i > j
                r += (rg - r % 4 + 4) % 4;                       // ... of this row group
                for (; r < R; r += 4) {
                    const int i = SCL * r + c;
                    const float4 a = reinterpret_cast<const float4 *>(Aown + roff[r])[j4];
                    const float vi = vv[i];
                    a0 = __fmaf_rn(a.x, vi, a0);
                    if (i > j + 1) a1 = __fmaf_rn(a.y, vi, a1);
                    if (i > j + 2) a2 = __fmaf_rn(a.z, vi, a2);
                    if (i > j + 3) a3 = __fmaf_rn(a.w, vi, a3);
                }
                reinterpret_cast<float4 *>(part4 + rg * L.np4)[j4] = make_float4(a0, a1, a2, a3);
            }
        }
        if ((tid & 15) == 0) {                                           // own-row dots next to the column sums
            #pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int r = h * (SCNT / 16) + (tid >> 4);
                if (r < R) ww[SCL * r + c] = rdot[h];                    // ww: scratch until w is formed
            }
        }
        __syncthreads();                                                 // part4, row dots
        SCT(3);
        // partial y of every row j >= k+1 to its owner: pin[c][r] of CTA j % 16
        if (tid < SCL * (RM / 4)) {
            const int dst = tid / (RM / 4), r4 = tid % (RM / 4);
            float v[4];
            #pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = SCL * (4 * r4 + u) + dst;
                float y = 0.f;
                if (j >= k + 1 && j < n) {
                    y = ((part4[j] + part4[L.np4 + j]) + part4[2 * L.np4 + j]) + part4[3 * L.np4 + j];
                    if (dst == c) y += ww[j];                            // own row: its row dot
                }
                v[u] = y;
            }
            sc_st4(sc_map(pin + c * RM + 4 * r4, dst), make_float4(v[0], v[1], v[2], v[3]));
        }
        SCT(4);
        sc_cluster_sync();                                               // #2: partial y at the owners
        SCT(5);
        // owner: p_i = tau sum_c pin[c][r] for the own rows, pushed to every CTA
        if (tid < SCL * (RM / 4)) {
            const int dst = tid / (RM / 4), r4 = tid % (RM / 4);
            float v[4];
            #pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int r = 4 * r4 + u;
                float y = 0.f;
                #pragma unroll
                for (int q = 0; q < SCL; ++q) y += pin[q * RM + r];
                v[u] = tau * y;
            }
            sc_st4(sc_map(pfull + c * RM + 4 * r4, dst), make_float4(v[0], v[1], v[2], v[3]));
        }
        sc_cluster_sync();                                               // #3: p everywhere
        SCT(6);
        float pvp = 0.f;
        for (int j = k + 1 + tid; j < n; j += SCNT) {
            const float p = pfull[(j % SCL) * RM + j / SCL];
            ww[j] = p;
            pvp = __fmaf_rn(p, vv[j], pvp);
        }
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) pvp += __shfl_xor_sync(0xffffffffu, pvp, o);
        if (lane == 0) red[rb][warp] = pvp;
        __syncthreads();                                                 // p, dot partials
        float pv = 0.f;
        #pragma unroll
        for (int w = 0; w < SCNT / 32; ++w) pv += red[rb][w];
        rb ^= 1;
        const float K = 0.5f * tau * pv;
        for (int j = tid; j < L.np4; j += SCNT) ww[j] = (j <= k || j >= n) ? 0.f : __fmaf_rn(-K, vv[j], ww[j]);
        __syncthreads();                                                 // w
        SCT(7);
        // A22 -= v w^T + w v^T on the own rows (elements k < j <= i)
        {
            const int rg = tid >> 8, cg = tid & 255;
            const float4 *ww4 = reinterpret_cast<const float4 *>(ww);
            for (int j4 = j40 + cg; j4 < nj4; j4 += 256) {
                const int j = 4 * j4;
                const float4 vj = vv4[j4], wj = ww4[j4];          // zero for j <= k and j >= n
                int r = (j - c + SCL - 1) / SCL;                  // first own row i >= j
                if (r < 0) r = 0;
                r += (rg - r % 4 + 4) % 4;
                for (; r < R; r += 4) {
                    const int i = SCL * r + c;
                    float4 *px = reinterpret_cast<float4 *>(Aown + roff[r]) + j4;
                    float4 a = *px;
                    const float vi = vv[i], wi = ww[i];
                    a.x = __fmaf_rn(-vi, wj.x, __fmaf_rn(-wi, vj.x, a.x));
                    if (j + 1 <= i) a.y = __fmaf_rn(-vi, wj.y, __fmaf_rn(-wi, vj.y, a.y));
                    if (j + 2 <= i) a.z = __fmaf_rn(-vi, wj.z, __fmaf_rn(-wi, vj.z, a.z));
                    if (j + 3 <= i) a.w = __fmaf_rn(-vi, wj.w, __fmaf_rn(-wi, vj.w, a.w));
                    *px = a;
                }
            }
        }
        __syncthreads();                                                 // updated rows
        SCT(8);
        if (tid < R) {                                                   // column k keeps the reflector
            const int i = SCL * tid + c;
            if (i >= k + 2) Aown[roff[tid] + k] = vv[i];
            else if (i == k + 1) Aown[roff[tid] + k] = beta;
        }
        if (k + 3 < n) push_x(k + 1);                                    // next column (reads column k+1 only)
        SCT(9);
    }
    __syncthreads();
    // tail: d(n-2), d(n-1), e(n-2); tau(n-2) = tau(n-1) = 0
    if (tid == 0) {
        for (int i = (n >= 2 ? n - 2 : 0); i < n; ++i)
            if (i % SCL == c) dout[i] = Aown[roff[i / SCL] + i];
        if (n >= 2 && (n - 1) % SCL == c) eout[n - 2] = Aown[roff[(n - 1) / SCL] + (n - 2)];
        if (c == 0) for (int i = (n >= 2 ? n - 2 : 0); i < n; ++i) tout[i] = 0.f;
    }
    // the reflectors back to A (below the subdiagonal, as the panel kernel leaves them)
    for (int r = 0; r < R; ++r) {
        const int i = SCL * r + c;
        for (int kk = tid; kk <= i; kk += SCNT) A[i + (size_t)kk * ld] = Aown[roff[r] + kk];
    }
    sc_cluster_sync();                                                   // no CTA exits while peers may store into it
}

}  // namespace

// the one-cluster reduction of the n x n symmetric matrix at A (lower triangle,
// ld lda) when it fits a cluster's shared memory: d, e, tau (n entries) and the
// reflectors below the subdiagonal.  false: not launched (does not fit, or
// MPJ_SYTRD_CLUSTER=0)
static bool sytrd_cluster_launch(float *A, int64_t lda, int n, float *d, float *e, float *tau, cudaStream_t st,
                                 mpj_status *err)
{
    *err = MPJ_OK;
    if (n < 3 || n > 1536) return false;
    const char *env = getenv("MPJ_SYTRD_CLUSTER");
    const size_t smem = sc_smem(n);
    if ((env && env[0] == '0') || smem > 227 * 1024 - 1024) return false;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(SCL); cfg.blockDim = dim3(SCNT); cfg.dynamicSmemBytes = smem; cfg.stream = st;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = SCL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    // whether a 16-CTA cluster with this much shared memory fits: asked once per
    // (device, size) -- the occupancy query costs more than a small n's whole kernel
    static std::mutex mu;
    static std::map<std::pair<int, size_t>, bool> fits;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto key = std::make_pair(dev, smem);
        auto it = fits.find(key);
        if (it == fits.end()) {
            bool ok = cudaFuncSetAttribute(k_sytrd_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                          cudaSuccess &&
                      smem_optin((const void *)k_sytrd_cluster, smem, SCNT, nullptr) == cudaSuccess;
            int ncl = 0;
            if (ok) ok = cudaOccupancyMaxActiveClusters(&ncl, k_sytrd_cluster, &cfg) == cudaSuccess && ncl > 0;
            cudaGetLastError();            // a refused size only selects the panel kernel
            it = fits.emplace(key, ok).first;
        }
        if (!it->second) return false;
    }
    if (smem_optin((const void *)k_sytrd_cluster, smem, SCNT, nullptr) != cudaSuccess) return false;
    const bool prof = prof_on();
    if (prof) prof_mark("symqr_sytrd", st, true);
    const cudaError_t ce = cudaLaunchKernelEx(&cfg, k_sytrd_cluster, A, lda, n, d, e, tau);
    if (prof) prof_mark("symqr_sytrd", st, false);
    count_launch();
    if (ce != cudaSuccess) {
        set_error(std::string("sytrd cluster launch: ") + cudaGetErrorString(ce));
        *err = MPJ_ERR_CUDA;
    }
    return true;
}

static mpj_status sytrd_run(float *A32, int64_t lda, int n, SymqrWs &w, int64_t np, cudaStream_t st)
{
    {
        MPJ_CK(cudaMemsetAsync(w.d, 0, np * 4, st));
        MPJ_CK(cudaMemsetAsync(w.e, 0, np * 4, st));
        MPJ_CK(cudaMemsetAsync(w.tau, 0, np * 4, st));
        mpj_status err;
        if (sytrd_cluster_launch(A32, lda, n, w.d, w.e, w.tau, st, &err)) return err;
    }
    const int nt = (int)(np / TB);
    // a grid sized to the work: small matrices pay per-column barrier and
    // reduction latency over every CTA, so they get ~8 tiles per CTA
    const int tiles0 = nt * (nt + 1) / 2;
    const int G = std::max(1, std::min(coop_ctas(), std::max(8, (tiles0 + 7) / 8)));
    const size_t smem = SYTRD_SMEM;
    MPJ_CK(cudaMemsetAsync(w.bar, 0, 64, st));
    MPJ_CK(cudaMemsetAsync(w.acol, 0, 2 * np * 4, st));
    MPJ_CK(cudaMemsetAsync(w.d, 0, np * 4, st));
    MPJ_CK(cudaMemsetAsync(w.e, 0, np * 4, st));
    MPJ_CK(cudaMemsetAsync(w.tau, 0, np * 4, st));
    const int ncolumns = n - 2;    // reflector columns 0 .. n-3
    SytrdArgs a;
    a.A = A32; a.ld = lda; a.n = n; a.nt = nt; a.V = w.V; a.W = w.W; a.ldp = np; a.acol = w.acol;
    a.d = w.d; a.e = w.e; a.tau = w.tau; a.Prow = w.Prow; a.Pcol = w.Pcol; a.rred = w.rred; a.qred = w.qred;
    a.ntp = (nt + 3) / 4 * 4;
    MPJ_CK(cudaMemsetAsync(w.rred, 0, (size_t)RSLOT * a.ntp * 4, st));
    MPJ_CK(cudaMemsetAsync(w.qred, 0, (size_t)(G + 4) * 4, st));
    a.bar = w.bar;
    CUtensorMap tm;
    if (ncolumns > 0) {
        auto enc = tmap_encoder();
        if (!enc) { set_error("sytrd: cuTensorMapEncodeTiled unavailable"); return MPJ_ERR_CUDA; }
        cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};      // out-of-range rows / columns read as 0
        cuuint64_t strides[1] = {(cuuint64_t)lda * sizeof(float)};
        cuuint32_t box[2] = {TB, TB}, es[2] = {1, 1};
        if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A32, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            set_error("sytrd: tensor map (lda must be a multiple of 4)");
            return MPJ_ERR_INVALID;
        }
    }
    // the trailing matrix goes to the one-cluster kernel once it fits (n - k0 <=
    // ~1150): its columns cost ~7 us instead of the panel kernel's ~20 us of
    // grid barriers and partial-sum reductions
    int handoff = -1;
    {
        const char *env = getenv("MPJ_SYTRD_CLUSTER");
        if (!(env && env[0] == '0'))
            for (int k0 = TB; k0 < ncolumns; k0 += TB)
                if (n - k0 <= 1152 && sc_smem(n - k0) <= 227 * 1024 - 1024) { handoff = k0; break; }
    }
    for (int k0 = 0; k0 < ncolumns; k0 += TB) {
        if (k0 == handoff) {
            mpj_status err;
            if (sytrd_cluster_launch(A32 + k0 + (size_t)k0 * lda, lda, n - k0, w.d + k0, w.e + k0, w.tau + k0, st,
                                     &err))
                return err;                // it also wrote the tail (d, e, tau of the last columns)
        }
        a.k0 = k0;
        a.ncols = std::min(TB, ncolumns - k0);
        MPJ_CK(cudaMemsetAsync(w.V, 0, np * TB * 4, st));
        MPJ_CK(cudaMemsetAsync(w.W, 0, np * TB * 4, st));
        MPJ_CK(cudaMemsetAsync(w.bar, 0, 64, st));     // the grid barrier's arrival counter
        void *args[] = {&a, &tm};
        const bool prof = prof_on();
        if (prof) prof_mark("symqr_sytrd", st, true);
        MPJ_CK(cudaLaunchCooperativeKernel((const void *)k_sytrd_panel, dim3(G), dim3(NTH), args, smem, st));
        if (prof) prof_mark("symqr_sytrd", st, false);
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
    if (n <= 2048)
        k_tri_bisect<32><<<(n + 256 / 32 - 1) / (256 / 32), 256, 0, st>>>(w.d64, w.e64, w.e2, w.bstart, w.bend, w.piv,
                                                                           n, w.lam);
    else
        k_tri_bisect<8><<<(n + 256 / 8 - 1) / (256 / 8), 256, 0, st>>>(w.d64, w.e64, w.e2, w.bstart, w.bend, w.piv, n,
                                                                     w.lam);
    k_tri_twisted<<<(2 * n + 127) / 128, 128, 0, st>>>(w.d64, w.e64, w.e2, w.bstart, w.bend, w.piv, w.lam, n, Dp,
                                                        Dm, w.inrm);
    k_tri_transpose<<<dim3((n + 31) / 32, (n + 31) / 32), dim3(32, 8), 0, st>>>(Dp, n, w.bstart, w.bend, w.inrm, Y,
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
    for (int k0 = ((ncolumns - 1) / BT) * BT; ncolumns > 0 && k0 >= 0; k0 -= BT) {
        const int nr = std::min(BT, ncolumns - k0);
        const int r0 = k0 + 1, m = n - r0;
        launch_pdl_k(k_build_vp, dim3((m + 255) / 256 > 32 ? 32 : (m + 255) / 256, BT), dim3(256), 0, st, A32, lda, n, k0,
                     nr, w.Vp, np);
        count_launch();
        launch_dgemm(true, false, BT, BT, m, 1.0, w.Vp, np, w.Vp, np, 0.0, w.Gm, BT, st, w.skw, w.skw_elems);
        const size_t tsm = ((size_t)BT * (BT + 1) + 3 * BT + 3 * 32 * 32) * sizeof(double);
        MPJ_CK(smem_optin((const void *)k_build_tp, tsm, 1024, nullptr));
        launch_pdl_k(k_build_tp, dim3(1), dim3(1024), tsm, st, (const double *)w.Gm, (const float *)w.tau, k0, nr, w.Tp);
        count_launch();
        // W1 = Vp^T Y: only 2 x n/64 output tiles with K = m -- split K 4 ways (n = 8192: 58.6 -> 56.3 ms
        // for the whole back-transformation; MPJ_BT_SPLITS overrides for A/B runs)
        static const int bt_splits = getenv("MPJ_BT_SPLITS") ? std::max(1, atoi(getenv("MPJ_BT_SPLITS"))) : 4;
        launch_dgemm(true, false, BT, n, m, 1.0, w.Vp, np, Y + r0, ldy, 0.0, w.W1, BT, st, w.skw, w.skw_elems, false,
                     nullptr, bt_splits);
        launch_dgemm(false, false, BT, n, BT, 1.0, w.Tp, BT, w.W1, BT, 0.0, w.W2, BT, st);
        launch_dgemm(false, false, m, n, BT, -1.0, w.Vp, np, w.W2, BT, 1.0, Y + r0, ldy, st);
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
    const bool prof = prof_on();
    MPJ_TRY(sytrd_run(A32, lda, n, w, np, st));
    if (prof) prof_mark("symqr_trieig", st, true);
    MPJ_TRY(tri_eig_run(n, w, Y, ldy, Dp, Dm, st));
    if (prof) { prof_mark("symqr_trieig", st, false); prof_mark("symqr_backtransform", st, true); }
    MPJ_TRY(backtransform_run(A32, lda, n, w, np, Y, ldy, st));
    if (prof) prof_mark("symqr_backtransform", st, false);
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

#ifdef MPJ_SYTRD_TRACE
// copy the last panel's phase timestamps (64 x 8 x 320 u64) to host memory
int mpjacobi_debug_sytrd_trace(unsigned long long *out)
{
    return cudaMemcpyFromSymbol(out, mpj::g_sytrd_trace, sizeof(mpj::g_sytrd_trace)) == cudaSuccess ? 0 : 1;
}
int mpjacobi_debug_sytrd_trace_panel(int k0)
{
    return cudaMemcpyToSymbol(mpj::g_trace_k0, &k0, sizeof(int)) == cudaSuccess ? 0 : 1;
}
#endif

mpj_status mpjacobi_sytrd(float *A, int64_t n, int64_t lda, float *d, float *e, float *tau, void *stream)
{
    mpj::set_error("");
    if (n < 1 || lda < n || !A || !d || !tau || (n > 1 && !e) || n > (1 << 20)) {
        mpj::set_error("mpjacobi_sytrd: invalid argument");
        return MPJ_ERR_INVALID;
    }
    if (lda % 4) {   // the panel kernel's TMA tensor map needs 16-byte column strides
        mpj::set_error("mpjacobi_sytrd: lda must be a multiple of 4");
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
