// k_svd.cu -- Alg. 5: mixed-precision one-sided Jacobi SVD.
//
// One-sided (Hestenes) Jacobi rotates column pairs of C so that c_p^T c_q = 0
// (Lemma 5.1): with alpha = c_p^T c_p, beta = c_q^T c_q,
// gamma = c_p^T c_q the rotation is Lemma 3.1's with (a_pp, a_qq, a_pq) =
// (alpha, beta, gamma), applied when |gamma| > nu sqrt(alpha beta) --
// i.e. rot_params with stop_rule 1 (Remark 3.1's test) and nu = omega.
//
// Block variant with the ordering of reading R1 (b = 32).  Per block round:
//   k_gram        G_a = C(:, P_a)^T C(:, P_a) for every block pair a
//                 (64 x 64 x m DMMA products, split over m, fp64 partials);
//                 in the fp64 stage's late sweeps k_colexp + k_gram_exact
//                 form G_a noise-free instead (reading R21, below)
//   k_svd_solve   inner rounds on G_a (two-sided on the Gram == one-sided on
//                 the columns in exact arithmetic) accumulating U_a
//   block_apply   C(:, P_a) <- C(:, P_a) U_a, V(:, P_a) <- V(:, P_a) U_a
// Stop test before each sweep: ||off(C^T C)||_F <= eps ||C^T C||_F (full Gram,
// DMMA GEMM), and after each sweep the early stop rotations/N < 2e-4 (P:678,
// reading R15).  Extraction: sigma_j = ||c_j|| sorted descending (stable,
// R16), u_j = c_j / sigma_j, V's columns alike.
#include "mpj_block.cuh"
#include "mpj_device.cuh"
#include "mpj_internal.h"

#include <nccl.h>

#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace mpj {
namespace {

using namespace blk;

__device__ __forceinline__ void g_cp16(void *dst, const void *src, int src_bytes)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(src_bytes));
}

// partial Gram of block pair a over rows [z*kc, min(m, (z+1)*kc)), fp64 partials.
// 64-row chunks double-buffered with cp.async (rows past r1 zero-filled).
// Only the upper triangle of G is read (k_svd_solve), so in fp64 the two warps
// of the lower-left 32 x 32 quadrant (rows 32.., columns ..31) skip it: 3/4 of
// the DMMA work.
// fp32 chunk Gram: acc[u][w] = sum_k X[k + i LD] X[k + j LD] for the thread's
// rows i = tx + 16u and columns j = ty + 16w, as two interleaved partial sums
// (even k, odd k; each k ascending) added at the end of the chunk.  The chunk is
// column-major (rows of C contiguous), so four consecutive k of one column are
// one 128-bit load, and the (even, odd) pairs of two such loads are adjacent
// register pairs: one packed fma.rn.f32x2 per two products (8 LDS.128 per 32
// FFMA2).  A warp spans 8 row indices tx and 4 column indices ty (gram_tx /
// gram_ty), so each load touches 8 or 4 float4 words 68 floats apart -- one
// shared-memory wavefront each (the 16 x 2 split cost ~3).
__device__ __forceinline__ int gram_tx() { return ((threadIdx.x >> 5) & 1) * 8 + (threadIdx.x & 7); }
__device__ __forceinline__ int gram_ty() { return (threadIdx.x >> 6) * 4 + ((threadIdx.x >> 3) & 3); }
__device__ __forceinline__ void ffma2v(float a0, float a1, float b0, float b1, float &c0, float &c1)
{
    unsigned long long aa, bb, cc, r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(aa) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b0), "f"(b1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "f"(c0), "f"(c1));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(aa), "l"(bb), "l"(cc));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(c0), "=f"(c1) : "l"(r));
}
__device__ __forceinline__ void gram_chunk_f32(const float *X, float (&acc)[4][4])
{
    constexpr int LD = Lay<float>::LD;
    const int tx = gram_tx(), ty = gram_ty();
    float se[4][4], so[4][4];
    #pragma unroll
    for (int u = 0; u < 4; ++u)
        #pragma unroll
        for (int w = 0; w < 4; ++w) se[u][w] = so[u][w] = 0.f;
    #pragma unroll 2
    for (int kk = 0; kk < TW; kk += 4) {
        float4 a[4], b[4];
        #pragma unroll
        for (int u = 0; u < 4; ++u) a[u] = *(const float4 *)(X + kk + (tx + 16 * u) * LD);
        #pragma unroll
        for (int w = 0; w < 4; ++w) b[w] = *(const float4 *)(X + kk + (ty + 16 * w) * LD);
        #pragma unroll
        for (int u = 0; u < 4; ++u)
            #pragma unroll
            for (int w = 0; w < 4; ++w) {
                ffma2v(a[u].x, a[u].y, b[w].x, b[w].y, se[u][w], so[u][w]);
                ffma2v(a[u].z, a[u].w, b[w].z, b[w].w, se[u][w], so[u][w]);
            }
    }
    #pragma unroll
    for (int u = 0; u < 4; ++u)
        #pragma unroll
        for (int w = 0; w < 4; ++w) acc[u][w] = se[u][w] + so[u][w];
}

template <typename R>
__global__ void __launch_bounds__(NT) k_gram(const R *__restrict__ C, int64_t ldc, int m, Sched S, int Rb, int kc,
                                             double *__restrict__ Gpart, int splits)
{
    constexpr int LD = Lay<R>::LD, EPC = 16 / sizeof(R), CPC = TW / EPC;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R *Xb = (R *)smem_raw;                         // two 64 x LD buffers
    const int a = blockIdx.x, z = blockIdx.y;
    const int mb = S.nb >> 1;
    const int2 bp = S.bsched[Rb * mb + a];
    const int r0 = z * kc, r1 = min(m, r0 + kc);
    const int warp = threadIdx.x >> 5;
    const bool lower_left = sizeof(R) == 8 && (warp == 4 || warp == 6);
    Acc<double> tot;
    tot.zero();
    // fp32 products are accumulated per 64-row chunk in fp32, then in fp64
    double totf[16];
    #pragma unroll
    for (int i = 0; i < 16; ++i) totf[i] = 0.0;
    auto issue = [&](int c0, R *X) {
        for (int e = threadIdx.x; e < TW * CPC; e += NT) {
            const int lj = e / CPC, li = (e - lj * CPC) * EPC;
            const int rem = r1 - (c0 + li);
            const int bytes = rem >= EPC ? 16 : (rem > 0 ? rem * (int)sizeof(R) : 0);
            const R *src = C + (bytes ? (int64_t)(c0 + li) : 0) + (int64_t)gidx(bp, lj) * ldc;
            g_cp16(X + li + lj * LD, src, bytes);
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    if (r0 < r1) issue(r0, Xb);
    for (int c0 = r0, it = 0; c0 < r1; c0 += TW, ++it) {
        R *X = Xb + (size_t)(it & 1) * TW * LD;
        if (c0 + TW < r1) {
            issue(c0 + TW, Xb + (size_t)((it + 1) & 1) * TW * LD);
            asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncthreads();
        if constexpr (sizeof(R) == 8) {
            if (!lower_left) tile_mm_acc<true>((const double *)X, (const double *)X, tot);
        } else {
            float part[4][4];
            gram_chunk_f32((const float *)X, part);
            #pragma unroll
            for (int u = 0; u < 4; ++u)
                #pragma unroll
                for (int w = 0; w < 4; ++w) totf[u * 4 + w] += (double)part[u][w];
        }
        __syncthreads();
    }
    double *G = Gpart + ((size_t)a * splits + z) * TW * TW;
    if constexpr (sizeof(R) == 8) {
        if (!lower_left) tot.each([&](int i, int j, double v) { G[i + j * TW] = v; });
    } else {
        const int tx = gram_tx(), ty = gram_ty();   // gram_chunk_f32's mapping: rows tx+16u, cols ty+16w
        #pragma unroll
        for (int u = 0; u < 4; ++u)
            #pragma unroll
            for (int w = 0; w < 4; ++w) G[(tx + 16 * u) + (ty + 16 * w) * TW] = totf[u * 4 + w];
    }
}

// ---------------------------------------------------------------------------
// Noise-free Gram blocks (reading R21).  The test |c_p^T c_q| > omega
// ||c_p|| ||c_q|| (nu = omega) sits at the rounding noise of a plain fp64
// dot product (~omega sum_i |c_ip c_iq|), so the fp64 stage forms its Gram
// blocks from a per-column fixed-point split whose leading product the DMMA
// pipe sums exactly:
//   c_ij = 2^(e_j - k) (h_ij + r_ij),  h integer, |h| <= 2^k, |r| <= 1/2 exact,
// with 2^e_j > max_i |c_ij| (k_colexp before a sweep's first round, then the
// bound k_svd_solve derives from each round's U) and k = (53 - log2 kc) / 2 for kc rows
// per split (k = 21 at kc = 2048).  Then
//   G_pq = 2^(e_p + e_q - 2k) (H^T H + M + M^T),  M = (H + R/2)^T R
// (M + M^T = H^T R + R^T H + R^T R).  H^T H is a sum of kc integers of
// magnitude <= 2^(2k): every partial sum is an integer <= 2^53, so DMMA forms
// it exactly in any order.  M is formed in fp64; its rounding is omega times
// sum |h r| ~ 2^-k sum |c_p c_q| (scaled), 2^-k below the plain product's
// noise.  (R^T R cannot be dropped: ~sqrt(m)/12 in these units, a few times
// omega ||c_p|| ||c_q|| at m = 16384.)  Across splits the partials are summed
// in double-double (k_svd_solve).  Net: the Gram entry carries about
// 2^-(53+k) sum |c_ip c_iq| of error where the plain DMMA sum carries 2^-53.
// ---------------------------------------------------------------------------
constexpr int KC_EXACT = 2048;   // rows per split of k_gram_exact (=> k = 21)

// e_j with max_i |C_ij| < 2^e_j (frexp exponent; 0 for a zero column)
__global__ void __launch_bounds__(256) k_colexp(const double *__restrict__ C, int64_t ldc, int m,
                                                int *__restrict__ ex)
{
    __shared__ double sh[8];
    const int j = blockIdx.x;
    double mx = 0.0;
    for (int i = threadIdx.x; i < m; i += 256) mx = fmax(mx, fabs(C[i + (int64_t)j * ldc]));
    #pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = sh[0];
        for (int w = 1; w < 8; ++w) v = fmax(v, sh[w]);
        int e = 0;
        if (v > 0.0) frexp(v, &e);
        ex[j] = e;
    }
}

// acc += (H + R/2)^T R over one 64-row chunk (tile_mm_acc<true>'s mapping)
__device__ __forceinline__ void gram_hr(const double *H, const double *R, Acc<double> &acc)
{
    constexpr int LD = Lay<double>::LD;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
    const int rb = (warp >> 1) * 16 + g, cb = (warp & 1) * 32 + g;
    #pragma unroll 4
    for (int ks = 0; ks < TW / 4; ++ks) {
        const int kk = ks * 4 + tig;
        double a[2], b[4];
        #pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
            const int o = kk + (rb + mi * 8) * LD;
            a[mi] = __fma_rn(0.5, R[o], H[o]);
        }
        #pragma unroll
        for (int ni = 0; ni < 4; ++ni) b[ni] = R[kk + (cb + ni * 8) * LD];
        #pragma unroll
        for (int mi = 0; mi < 2; ++mi)
            #pragma unroll
            for (int ni = 0; ni < 4; ++ni) dmma884(acc.v[mi][ni][0], acc.v[mi][ni][1], a[mi], b[ni]);
    }
}

// partials of block pair a over rows [z kc, min(m, (z+1) kc)):
// Gpart[a][z][0] = H^T H (upper quadrants only), Gpart[a][z][1] = M = (H + R/2)^T R.
// One raw chunk buffer (cp.async) + the split H, R in shared memory: 104 KB,
// two CTAs per SM; the next chunk streams in while this one is multiplied.
__global__ void __launch_bounds__(NT) k_gram_exact(const double *__restrict__ C, int64_t ldc, int m, Sched S,
                                                   int Rb, int kc, int kbits, const int *__restrict__ ex,
                                                   double *__restrict__ Gpart, int splits)
{
    constexpr int LD = Lay<double>::LD, CPC = TW / 2, TL = TW * LD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *Xr = (double *)smem_raw;     // raw chunk
    double *H = Xr + TL, *Rm = H + TL;
    __shared__ double fsc[TW];
    const int a = blockIdx.x, z = blockIdx.y;
    const int mb = S.nb >> 1;
    const int2 bp = S.bsched[Rb * mb + a];
    const int r0 = z * kc, r1 = min(m, r0 + kc);
    const int warp = threadIdx.x >> 5;
    const bool lower_left = warp == 4 || warp == 6;   // H^T H is symmetric: upper quadrants only
    if (threadIdx.x < TW) fsc[threadIdx.x] = ldexp(1.0, kbits - ex[gidx(bp, threadIdx.x)]);
    Acc<double> hh, hr;
    hh.zero();
    hr.zero();
    auto issue = [&](int c0) {
        for (int e = threadIdx.x; e < TW * CPC; e += NT) {
            const int lj = e / CPC, li = (e - lj * CPC) * 2;
            const int rem = r1 - (c0 + li);
            const int bytes = rem >= 2 ? 16 : (rem > 0 ? 8 : 0);
            const double *src = C + (bytes ? (int64_t)(c0 + li) : 0) + (int64_t)gidx(bp, lj) * ldc;
            g_cp16(Xr + li + lj * LD, src, bytes);
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    if (r0 < r1) issue(r0);
    for (int c0 = r0; c0 < r1; c0 += TW) {
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();   // chunk landed (fsc visible); the previous chunk's products are done
        for (int e = threadIdx.x; e < TW * TW; e += NT) {
            const int li = e & (TW - 1), lj = e >> 6, o = li + lj * LD;
            const double t = Xr[o] * fsc[lj];   // exact: power-of-two scale
            const double h = rint(t);
            H[o] = h;
            Rm[o] = t - h;                      // exact
        }
        __syncthreads();
        if (c0 + TW < r1) issue(c0 + TW);
        if (!lower_left) tile_mm_acc<true>(H, H, hh);
        gram_hr(H, Rm, hr);
    }
    double *G = Gpart + ((size_t)a * splits + z) * 2 * TW * TW;
    if (!lower_left) hh.each([&](int i, int j, double v) { G[i + j * TW] = v; });
    hr.each([&](int i, int j, double v) { G[TW * TW + i + j * TW] = v; });
}

// G_ij (i <= j, local indices) of block pair bp from the k_gram_exact partials:
// sum_z HH (double-double) + sum_z (M_ij + M_ji), scaled by 2^(e_i + e_j - 2k)
__device__ __forceinline__ double gram_exact_entry(const double *G, int splits, int i, int j, int2 bp,
                                                   const int *__restrict__ ex, int kbits)
{
    constexpr size_t T2 = (size_t)TW * TW;
    double hi = 0.0, lo = 0.0, c = 0.0;
    for (int z = 0; z < splits; ++z) {   // fixed order
        const double *Gz = G + (size_t)z * 2 * T2;
        const double x = Gz[i + j * TW];
        const double s = hi + x, bb = s - hi;
        lo += (hi - (s - bb)) + (x - bb);   // TwoSum error
        hi = s;
        c += Gz[T2 + i + j * TW] + Gz[T2 + j + i * TW];
    }
    return ldexp(hi + (lo + c), ex[gidx(bp, i)] + ex[gidx(bp, j)] - 2 * kbits);
}

template <typename R, bool EXACT = false>
__global__ void __launch_bounds__(NTW) k_svd_solve(const double *__restrict__ Gpart, int splits, Sched S, int Rb,
                                                   R nu, R *__restrict__ Ubuf, unsigned long long *__restrict__ cnt,
                                                   int *__restrict__ uid, int *__restrict__ nid,
                                                   int *__restrict__ ex = nullptr, int kbits = 0)
{
    constexpr int LD = LayK<R>::LD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R *D0 = (R *)smem_raw;
    R *D1 = D0 + TW * LD;
    R *U = D1 + TW * LD;
    __shared__ unsigned nrot;
    __shared__ WideParams<R> P[2];
    __shared__ double gnorm[EXACT ? TW : 1];   // ||c_k|| of the block pair's columns (EXACT)
    const int a = blockIdx.x;
    const int mb = S.nb >> 1;
    const int2 bp = S.bsched[Rb * mb + a];
    const double *G = Gpart + (size_t)a * splits * (EXACT ? 2 : 1) * TW * TW;
    for (int e = threadIdx.x; e < TW * TW; e += NTW) {
        const int li = e & (TW - 1), lj = e >> 6;
        // the Gram block, exactly symmetric: both triangles from the (li <= lj) partial sums
        const int i0 = li < lj ? li : lj, j0 = li < lj ? lj : li;
        double g = 0.0;
        if constexpr (EXACT) {
            g = gram_exact_entry(G, splits, i0, j0, bp, ex, kbits);
        } else {
            for (int z = 0; z < splits; ++z) g += G[(size_t)z * TW * TW + i0 + j0 * TW];   // fixed order
        }
        D0[li + lj * LD] = (R)g;
        U[li + lj * LD] = (li == lj) ? R(1) : R(0);
        if (EXACT && li == lj) gnorm[li] = sqrt(fmax(g, 0.0));
    }
    __syncthreads();
    // no visited pair passes the test on the block as loaded: nothing rotates in
    // any round (k_block.cu, reading R29), U = I -- skip the dependent rounds
    // (the Gram block itself is discarded)
    __shared__ int any_rot;
    if (threadIdx.x == 0) any_rot = 0;
    __syncthreads();
    const int npairs = Rb == 0 ? TW * (TW - 1) / 2 : BW * BW;
    for (int e = threadIdx.x; e < npairs; e += NTW) {
        int p, q;
        if (Rb == 0) {
            q = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)e)) * 0.5f);
            while (q * (q - 1) / 2 > e) --q;
            while ((q + 1) * q / 2 <= e) ++q;
            p = e - q * (q - 1) / 2;
        } else {
            p = e & (BW - 1); q = BW + (e >> 5);
        }
        if (!rot_skip<R>(D0[p + p * LD], D0[q + q * LD], D0[p + q * LD], nu, /*rule=*/1)) any_rot = 1;
    }
    __syncthreads();
    if (any_rot) {
        inner_rounds_wide<R>(D0, D1, U, bp, Rb == 0, S.lsched, nu, /*rule=*/1, P, &nrot);
    } else if (threadIdx.x == 0) {
        nrot = 0;
    }
    if constexpr (EXACT) {
        // exponents for the next round's k_gram_exact (replaces a k_colexp pass over C):
        // max_i |c'_ij| <= ||c'_j|| <= sum_k |U_kj| ||c_k|| for c'_j = C(:, P_a) U(:, j);
        // the 2^-20 margin covers the rounding of this sum and of the column apply.
        // Every column sits in exactly one block pair per round, so all of ex is renewed;
        // this CTA read its columns' ex above (before inner_rounds_wide's barriers).
        __syncthreads();
        const int j = threadIdx.x >> 4, part = threadIdx.x & 15;   // 16 threads per column
        double bnd = 0.0;
        #pragma unroll
        for (int k = part * 4; k < part * 4 + 4; ++k) bnd += fabs((double)U[k + j * LD]) * gnorm[k];
        #pragma unroll
        for (int o = 8; o; o >>= 1) bnd += __shfl_xor_sync(0xffffffffu, bnd, o);
        if (part == 0) {
            int e = 0;
            if (bnd > 0.0) frexp(bnd * (1.0 + 0x1p-20), &e);
            ex[gidx(bp, j)] = e;
        }
    }
    R *Ua = Ubuf + (size_t)a * TW * TW;
    R *UaT = Ubuf + (size_t)mb * TW * TW + (size_t)a * TW * TW;   // U^T: operand of the fp32 apply
    for (int e = threadIdx.x; e < TW * TW; e += NTW) {
        const int li = e & (TW - 1), lj = e >> 6;
        Ua[li + lj * TW] = U[li + lj * LD];
        if (sizeof(R) == 4) {
            UaT[li + lj * TW] = U[lj + li * LD];
            // split-half U^T (operand of the TMA fp32 apply, see k_block.cu)
            UaT[(size_t)mb * TW * TW + (li >> 5) * (BW * TW) + lj * BW + (li & 31)] = U[lj + li * LD];
        }
    }
    if (threadIdx.x == 0) {
        if (nrot) atomicAdd(cnt, (unsigned long long)nrot);
        uid[a] = nrot == 0;   // U_a exactly I: the column updates skip block pair a
        if (nrot == 0) atomicAdd(nid, 1);
    }
}

__global__ void __launch_bounds__(256) k_colnorm(const double *__restrict__ C, int64_t ldc, int m,
                                                 double *__restrict__ nrm)
{
    __shared__ double sh[32];
    const int j = blockIdx.x;
    double acc = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const double x = C[i + (int64_t)j * ldc];
        acc = __fma_rn(x, x, acc);
    }
    const double s = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) nrm[j] = sqrt(s);
}

// rank[j] = stable descending position of nrm[j]; sigma[rank] = nrm[j]
__global__ void k_rank_vec(const double *__restrict__ key, int n, int *__restrict__ rank, double *__restrict__ out,
                           double thresh, int *__restrict__ flag)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double d = key[j];
    int r = 0;
    for (int i = 0; i < n; ++i) {
        const double e = key[i];
        r += (e > d) || (e == d && i < j);
    }
    rank[j] = r;
    out[r] = d;
    if (!(d > thresh)) atomicOr(flag, 1);
}

// U(:, rank[j]) = C(:, j) / nrm[j];  V(:, rank[j]) = Vin(:, j)
__global__ void k_svd_extract(const double *__restrict__ C, int64_t ldc, int m, const double *__restrict__ Vin,
                              int64_t ldvi, int n, const int *__restrict__ rank, const double *__restrict__ nrm,
                              double *__restrict__ U, int64_t ldu, double *__restrict__ V, int64_t ldv)
{
    const int j = blockIdx.y;
    const int r = rank[j];
    const double s = nrm[j];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        U[i + (int64_t)r * ldu] = s > 0.0 ? C[i + (int64_t)j * ldc] / s : 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        V[i + (int64_t)r * ldv] = Vin[i + (int64_t)j * ldvi];
}

}  // namespace

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct SvdPlan {
    int64_t m, n;
    int64_t ldc;              // leading dimension of the internal m-row buffers (Ad, C, C32): m rounded up
                              // to 8 so that every column starts 16-byte aligned (cp.async, TMA strides)
    int np, mb;
    int splits[3], kc[3];
    int kbits;                // fixed-point bits of k_gram_exact's split (reading R21)     // k_gram row splits / rows per split, [0] fp32, [1] fp64, [2] k_gram_exact
    double *Ad, *C, *V, *G, *Gpart, *nrm, *red_part, *red_out, *sig;
    float *C32, *V32;
    int2 *bsched, *lsched;
    void *Ubuf;
    unsigned long long *cnt;
    int *uid;                 // mb identity flags + (nb - 1) per-round identity counts
    int *ctr;                 // 2 (nb - 1) item counters of the column updates (single-GPU sweeps)
    int *rank, *flag;
    int *ex;                  // per-column exponents of the exact Gram (k_colexp)
    void *orth_ws;
};

static void carve_svd(char *base, size_t &off, int64_t m, int64_t n, SvdPlan &p)
{
    auto take = [&](size_t bytes) -> void * {
        off = (off + 255) & ~(size_t)255;
        void *r = base ? (void *)(base + off) : nullptr;
        off += bytes;
        return r;
    };
    p.m = m; p.n = n;
    p.ldc = (m + 7) / 8 * 8;
    p.np = padded_n(n, BW);
    p.mb = p.np / TW;
    // k_gram grid (mb, s): choose s <= 16 to minimise waves x (64-row chunks per
    // CTA + 1 for the unhidden first load), with 148 SMs x the resident CTAs per
    // SM (fp32: 2, register bound; fp64: 3, shared-memory bound).  The old
    // s = ceil(296 / mb) put 320 fp32 CTAs in two waves, the second 24 CTAs long.
    const int chunks = (int)((m + TW - 1) / TW);
    for (int f = 0; f < 3; ++f) {
        const int slots = 148 * (f == 1 ? 3 : 2);
        // k_gram_exact: at most KC_EXACT rows per split (its exactness bound)
        const int smin = f == 2 ? (chunks + KC_EXACT / TW - 1) / (KC_EXACT / TW) : 1;
        int best = smin;
        long best_cost = -1;
        for (int s = smin; s <= std::max(smin, std::min(16, chunks)); ++s) {
            const long waves = ((long)p.mb * s + slots - 1) / slots;
            const long cost = waves * ((chunks + s - 1) / s + 1);
            if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = s; }
        }
        p.splits[f] = best;
        p.kc[f] = (int)(((m + best - 1) / best + TW - 1) / TW * TW);
    }
    int lg = 0;
    while ((1 << lg) < p.kc[2]) ++lg;
    p.kbits = (53 - lg) / 2;
    const size_t mnp = (size_t)p.ldc * p.np, nn = (size_t)p.np * p.np;
    p.Ad = (double *)take(mnp * 8);
    p.C = (double *)take(mnp * 8);
    p.V = (double *)take(nn * 8);
    p.G = (double *)take(nn * 8);
    p.C32 = (float *)take(mnp * 4);
    p.V32 = (float *)take(nn * 4);
    p.Gpart = (double *)take((size_t)p.mb * std::max({p.splits[0], p.splits[1], 2 * p.splits[2]}) * TW * TW * 8);
    p.Ubuf = take((size_t)p.mb * TW * TW * 12);   // fp64 U, or fp32 U, U^T and split-half U^T
    p.nrm = (double *)take(p.np * 8);
    p.sig = (double *)take(p.np * 8);
    p.red_part = (double *)take(kRedBlocks * 8);
    p.red_out = (double *)take(64);
    const int nb = p.np / BW;
    p.bsched = (int2 *)take((size_t)std::max(nb - 1, 1) * std::max(nb / 2, 1) * sizeof(int2));
    p.lsched = (int2 *)take((size_t)(BW - 1) * (BW / 2) * sizeof(int2));
    p.cnt = (unsigned long long *)take(64);
    p.uid = (int *)take((size_t)(p.mb + std::max(nb - 1, 1)) * sizeof(int));
    p.ctr = (int *)take((size_t)2 * std::max(nb - 1, 1) * sizeof(int));
    p.rank = (int *)take(p.np * 4);
    p.flag = (int *)take(64);
    p.ex = (int *)take(p.np * 4);
    p.orth_ws = take(orth_workspace(p.np));
}

// one block round Rb of the one-sided sweep on (C, V): Gram blocks of the
// block pairs of ds (ds.nb / 2 slots), their inner solves, the column updates.
// uid / nid: identity flags (ds.nb / 2) and this round's identity count.
template <typename R>
static mpj_status svd_block_round(SvdPlan &p, R *C, R *V, const DevSched &ds, int Rb, R nu, cudaStream_t st,
                                  bool exact, int *uid, int *nid, int *ctr2 = nullptr)
{
    exact = exact && sizeof(R) == 8;
    Sched S;
    S.bsched = ds.bsched; S.lsched = ds.lsched; S.b = ds.b; S.nb = ds.nb; S.np = ds.np;
    const int mb = ds.nb / 2;
    constexpr int LD = Lay<R>::LD;
    const size_t sm_x = 2 * TW * LD * sizeof(R), sm_du = 3 * TW * LayK<R>::LD * sizeof(R);
    MPJ_CK(smem_optin((const void *)k_gram<R>, sm_x, NT, nullptr));
    MPJ_CK(smem_optin((const void *)k_svd_solve<R>, sm_du, NTW, nullptr));
    const size_t sm_xx = 3 * TW * Lay<double>::LD * sizeof(double);
    if (exact) {
        MPJ_CK(smem_optin((const void *)k_gram_exact, sm_xx, NT, nullptr));
        MPJ_CK(smem_optin((const void *)k_svd_solve<double, true>, sm_du, NTW, nullptr));
    }
    const bool prof = prof_on();
    const char *ng = sizeof(R) == 8 ? "svd_gram_f64" : "svd_gram_f32";
    const char *ns = sizeof(R) == 8 ? "svd_solve_f64" : "svd_solve_f32";
    const char *na = sizeof(R) == 8 ? "svd_apply_f64" : "svd_apply_f32";
    const int splits = p.splits[sizeof(R) == 8], kc = p.kc[sizeof(R) == 8];
    if (exact) {
        if (prof) prof_mark("svd_gram_exact", st, true);
        // column exponents: measured before the sweep's first round, then carried
        // forward by k_svd_solve's bounds
        if (Rb == 0) k_colexp<<<p.np, 256, 0, st>>>((const double *)C, p.ldc, (int)p.m, p.ex);
        k_gram_exact<<<dim3(mb, p.splits[2]), NT, sm_xx, st>>>((const double *)C, p.ldc, (int)p.m, S, Rb, p.kc[2],
                                                               p.kbits, p.ex, p.Gpart, p.splits[2]);
        if (prof) { prof_mark("svd_gram_exact", st, false); prof_mark(ns, st, true); }
        k_svd_solve<double, true><<<mb, NTW, sm_du, st>>>(p.Gpart, p.splits[2], S, Rb, (double)nu, (double *)p.Ubuf,
                                                          p.cnt, uid, nid, p.ex, p.kbits);
        count_launch(Rb == 0 ? 3 : 2);
    } else {
        if (prof) prof_mark(ng, st, true);
        k_gram<R><<<dim3(mb, splits), NT, sm_x, st>>>(C, p.ldc, (int)p.m, S, Rb, kc, p.Gpart, splits);
        if (prof) { prof_mark(ng, st, false); prof_mark(ns, st, true); }
        k_svd_solve<R><<<mb, NTW, sm_du, st>>>(p.Gpart, splits, S, Rb, nu, (R *)p.Ubuf, p.cnt, uid, nid);
        count_launch(2);
    }
    if (prof) { prof_mark(ns, st, false); prof_mark(na, st, true); }
    MPJ_CK(launch_block_apply_cols<R>(C, p.ldc, (int)p.m, ds, Rb, (const R *)p.Ubuf, st, uid, nid, ctr2));
    MPJ_CK(launch_block_apply_cols<R>(V, p.np, p.np, ds, Rb, (const R *)p.Ubuf, st, uid, nid,
                                      ctr2 ? ctr2 + 1 : nullptr));
    if (prof) prof_mark(na, st, false);
    return MPJ_OK;
}

template <typename R>
static mpj_status svd_block_sweep(SvdPlan &p, R *C, R *V, const DevSched &ds, R nu, cudaStream_t st, bool exact)
{
    int *uid = p.uid, *nid = p.uid + p.mb;
    MPJ_CK(cudaMemsetAsync(nid, 0, (size_t)(ds.nb - 1) * sizeof(int), st));
    MPJ_CK(cudaMemsetAsync(p.ctr, 0, (size_t)2 * (ds.nb - 1) * sizeof(int), st));
    for (int Rb = 0; Rb < ds.nb - 1; ++Rb)
        MPJ_TRY(svd_block_round<R>(p, C, V, ds, Rb, nu, st, exact, uid, nid + Rb, p.ctr + 2 * Rb));
    return MPJ_OK;
}

// fp64-stage Gram policy (reading R21): by default every fp64 sweep forms its
// Gram blocks noise-free (k_gram_exact), so the rotate / skip test is the
// paper's, evaluated as the long-double oracle evaluates it.  A bound x
// (MPJ_SVD_GRAM=x) uses the plain DMMA Gram (k_gram, 2.6x cheaper) for sweeps
// that follow a sweep rotating >= x N pairs -- sweeps where nearly every pair
// rotates whatever the noise -- and noise-free blocks after.  Measured at
// 16384 x 4096: noise-free 9 fp64 sweeps, 2.36 s; x = 0.1: 9 sweeps, 2.02 s;
// plain (MPJ_SVD_GRAM=dmma): 11 sweeps, 2.10 s.  At the parity-test sizes the
// noise-free policy is within one sweep of the oracle everywhere (plain: up to
// three more), x = 0.1 within two.
static double svd_exact_below()
{
    const char *e = getenv("MPJ_SVD_GRAM");
    if (!e || !*e || !strcmp(e, "exact")) return 2.0;
    if (!strcmp(e, "dmma")) return -1.0;
    return atof(e);
}

struct SvdStage {
    int sweeps = 0;
    long long rotations = 0;
    double hist[64] = {0};
    long long rot_hist[64] = {0};   // rotations applied in sweep k+1
    int nhist = 0;
};

// the one-sided Jacobi loop on (C, V) in precision R; Cd: fp64 image buffer for
// the stop test (== C when R is double)
template <typename R>
static mpj_status svd_loop(SvdPlan &p, R *C, R *V, double *Cd, const DevSched &ds, double eps_rel, R nu,
                           double early, int max_sweeps, double *h_pin, cudaStream_t st, SvdStage &out)
{
    const double N = 0.5 * (double)p.n * (double)(p.n - 1);
    mpj_status status = MPJ_ERR_NOCONV;
    unsigned long long prev = 0;
    double ratio = 1.0;   // rotations / N of the previous sweep
    const double xb = svd_exact_below();
    MPJ_CK(cudaMemsetAsync(p.cnt, 0, sizeof(unsigned long long), st));
    for (;;) {
        if ((void *)Cd != (void *)C)
            launch_copy_pad<R, double>(C, p.ldc, (int)p.m, p.np, Cd, p.ldc, (int)p.m, p.np, st);
        // C^T C is symmetric: only its upper tiles are formed and read (half the flops)
        launch_dgemm(true, false, p.np, p.np, p.m, 1.0, Cd, p.ldc, Cd, p.ldc, 0.0, p.G, p.np, st, nullptr, 0,
                     true);
        launch_norm_sym_upper(p.G, p.np, p.np, true, p.red_part, p.red_out, st);
        launch_norm_sym_upper(p.G, p.np, p.np, false, p.red_part, p.red_out + 1, st);
        MPJ_CK(cudaMemcpyAsync(h_pin, p.red_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
        MPJ_CK(cudaStreamSynchronize(st));
        const double off = h_pin[0], tot = h_pin[1];
        if (out.sweeps < 64) { out.hist[out.sweeps] = off; out.nhist = out.sweeps + 1; }
        if (!std::isfinite(off)) { set_error("non-finite Gram"); return MPJ_ERR_NONFINITE; }
        if (off <= eps_rel * tot) { status = MPJ_OK; break; }
        if (out.sweeps >= max_sweeps) { status = MPJ_ERR_NOCONV; break; }
        ++out.sweeps;
        MPJ_TRY(svd_block_sweep<R>(p, C, V, ds, nu, st, ratio < xb));
        MPJ_CK(cudaMemcpyAsync(h_pin, p.cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        MPJ_CK(cudaStreamSynchronize(st));
        unsigned long long now = 0;
        std::memcpy(&now, h_pin, sizeof(now));
        const unsigned long long rs = now - prev;
        prev = now;
        out.rotations = (long long)now;
        if (out.sweeps <= 64) out.rot_hist[out.sweeps - 1] = (long long)rs;
        ratio = N > 0 ? (double)rs / N : 0.0;
        if (early > 0 && N > 0 && (double)rs / N < early) { status = MPJ_OK; break; }
    }
    return status;
}

size_t svd_workspace(int64_t m, int64_t n)
{
    size_t off = 0;
    SvdPlan p;
    carve_svd(nullptr, off, m, n, p);
    return off + 256;
}

mpj_status svd_run(const double *A, int64_t m, int64_t n, int64_t lda, double *Sigma, double *U, int64_t ldu,
                   double *V, int64_t ldv, int *sweeps, void *workspace, size_t ws_bytes, cudaStream_t st,
                   const mpj_config &cfg, mpj_report &r, double *h_pin, bool a_dev, bool out_dev,
                   const float *Zin, bool zin_dev, float *Zout, bool zout_dev, int64_t ldz)
{
    const double omega = 1.1102230246251565e-16, upsilon = 5.9604644775390625e-08;
    size_t off = 0;
    SvdPlan p;
    carve_svd(nullptr, off, m, n, p);
    // a library-owned workspace is released on every exit, error exits included
    struct OwnWs {
        void *p = nullptr;
        cudaStream_t st;
        ~OwnWs() { if (p) cudaFreeAsync(p, st); }
    } own;
    own.st = st;
    if (!workspace) {
        MPJ_CK(cudaMallocAsync(&own.p, off + 256, st));
        workspace = own.p;
    } else if (ws_bytes < off + 256) {
        set_error("workspace too small");
        return MPJ_ERR_NOMEM;
    }
    char *base = (char *)(((uintptr_t)workspace + 255) & ~(uintptr_t)255);
    off = 0;
    carve_svd(base, off, m, n, p);
    const int np = p.np;
    r.n_padded = np; r.block_b = BW; r.variant = MPJ_VARIANT_BLOCK;

    HostSchedule hs;
    build_schedule(n, BW, hs);
    MPJ_CK(cudaMemcpyAsync(p.bsched, hs.bsched.data(), hs.bsched.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    MPJ_CK(cudaMemcpyAsync(p.lsched, hs.lsched.data(), hs.lsched.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    DevSched ds;
    ds.bsched = p.bsched; ds.lsched = p.lsched; ds.b = BW; ds.nb = hs.nb; ds.np = np; ds.rounds = hs.rounds;

    // a0: stage A (zero-padded columns), ||A||_F, finiteness
    const int64_t ldc = p.ldc;
    MPJ_CK(cudaMemsetAsync(p.Ad, 0, (size_t)ldc * np * 8, st));
    MPJ_CK(cudaMemcpy2DAsync(p.Ad, ldc * 8, A, lda * 8, m * 8, n,
                             a_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    MPJ_CK(cudaMemsetAsync(p.flag, 0, sizeof(int), st));
    launch_check_finite(p.Ad, ldc, (int)m, (int)n, p.flag, st);
    launch_norm<double>(p.Ad, ldc, (int)m, np, false, p.red_part, p.red_out, st);
    MPJ_CK(cudaMemcpyAsync(h_pin, p.red_out, sizeof(double), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaMemcpyAsync(h_pin + 1, p.flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaStreamSynchronize(st));
    const double normA = h_pin[0];
    int bad = 0;
    std::memcpy(&bad, h_pin + 1, sizeof(int));
    r.norm_a = normA;
    auto fin = [&](mpj_status s) { return s; };
    if (bad) { set_error("input has NaN/Inf"); return fin(MPJ_ERR_NONFINITE); }

    // a1: fp32 one-sided Jacobi on fl32(A) from V = I (reading R12)
    {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        if (Zin) {   // the caller's Z replaces the low-precision stage
            MPJ_CK(cudaMemsetAsync(p.V32, 0, (size_t)np * np * 4, st));
            MPJ_CK(cudaMemcpy2DAsync(p.V32, np * 4, Zin, ldz * 4, n * 4, n,
                                     zin_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
            r.status_low = MPJ_OK;
        } else {
            launch_copy_pad<double, float>(p.Ad, ldc, (int)m, np, p.C32, ldc, (int)m, np, st);
            MPJ_CK(cudaMemsetAsync(p.V32, 0, (size_t)np * np * 4, st));
            launch_identity<float>(p.V32, np, (int)n, (int)n, st);
            SvdStage lo;
            mpj_status sl = svd_loop<float>(p, p.C32, p.V32, p.C, ds, eps_low_factor(cfg, n) * upsilon,
                                            (float)(cfg.nu_low_factor * upsilon), cfg.early_stop_ratio,
                                            cfg.max_sweeps_low, h_pin, st, lo);
            if (sl != MPJ_OK && sl != MPJ_ERR_NOCONV) return fin(sl);
            r.sweeps_low = lo.sweeps; r.rotations_low = lo.rotations; r.status_low = sl;
        }
        if (Zout)
            MPJ_CK(cudaMemcpy2DAsync(Zout, ldz * 4, p.V32, np * 4, n * 4, n,
                                     zout_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0; cudaEventElapsedTime(&ms, e0, e1); r.t_low = ms * 1e-3;
        // a2: Q = CGS2(fp64(V32)) into V
        cudaEventRecord(e0, st);
        launch_copy_pad<float, double>(p.V32, np, (int)n, (int)n, p.G, np, (int)n, (int)n, st);
        MPJ_CK(cudaMemsetAsync(p.V, 0, (size_t)np * np * 8, st));
        mpj_status so = orth_cgs2(p.G, np, p.V, np, n, n, p.orth_ws, st);
        if (so != MPJ_OK) return fin(so);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); r.t_orth = ms * 1e-3;
        // a3: C = A Q
        cudaEventRecord(e0, st);
        MPJ_CK(cudaMemsetAsync(p.C, 0, (size_t)ldc * np * 8, st));
        launch_dgemm(false, false, m, n, n, 1.0, p.Ad, ldc, p.V, np, 0.0, p.C, ldc, st);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); r.t_precond = ms * 1e-3;
        cudaEventDestroy(e0); cudaEventDestroy(e1);
    }
    // a4-a8 (one-sided): fp64 sweeps
    SvdStage hi;
    {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        mpj_status sh = svd_loop<double>(p, p.C, p.V, p.C, ds, cfg.eps_factor * omega, cfg.nu_factor * omega,
                                         cfg.early_stop_ratio, cfg.max_sweeps, h_pin, st, hi);
        r.sweeps = hi.sweeps; r.rotations = hi.rotations; r.status = sh;
        r.off0 = hi.hist[0];
        for (int k = 0; k < hi.nhist && k < 64; ++k) r.off_hist[k] = hi.hist[k];
        for (int k = 0; k < 64; ++k) r.rot_hist[k] = hi.rot_hist[k];
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0; cudaEventElapsedTime(&ms, e0, e1); r.t_jacobi = ms * 1e-3;
        cudaEventDestroy(e0); cudaEventDestroy(e1);
        if (sh != MPJ_OK && sh != MPJ_ERR_NOCONV) return fin(sh);
        if (sweeps) *sweeps = hi.sweeps;
    }
    // a10: extraction
    k_colnorm<<<(unsigned)n, 256, 0, st>>>(p.C, ldc, (int)m, p.nrm);
    MPJ_CK(cudaMemsetAsync(p.flag, 0, sizeof(int), st));
    k_rank_vec<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p.nrm, (int)n, p.rank, p.sig, (double)n * omega * normA,
                                                            p.flag);
    count_launch(2);
    double *Ud = out_dev ? U : p.Ad;          // A is no longer needed: reuse its buffer
    double *Vd = out_dev ? V : p.G;
    double *Sd = out_dev ? Sigma : p.sig;
    const int64_t lduo = out_dev ? ldu : m, ldvo = out_dev ? ldv : np;
    if (out_dev) MPJ_CK(cudaMemcpyAsync(Sigma, p.sig, n * 8, cudaMemcpyDeviceToDevice, st));
    k_svd_extract<<<dim3(std::max<int64_t>(1, std::min<int64_t>(64, (m + 255) / 256)), (unsigned)n), 256, 0, st>>>(
        p.C, ldc, (int)m, p.V, np, (int)n, p.rank, p.nrm, Ud, lduo, Vd, ldvo);
    count_launch();
    (void)Sd;
    if (!out_dev) {
        MPJ_CK(cudaMemcpyAsync(Sigma, p.sig, n * 8, cudaMemcpyDeviceToHost, st));
        MPJ_CK(cudaMemcpy2DAsync(U, ldu * 8, Ud, m * 8, m * 8, n, cudaMemcpyDeviceToHost, st));
        MPJ_CK(cudaMemcpy2DAsync(V, ldv * 8, Vd, np * 8, n * 8, n, cudaMemcpyDeviceToHost, st));
    }
    MPJ_CK(cudaMemcpyAsync(h_pin + 2, p.flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaStreamSynchronize(st));
    int rd = 0;
    std::memcpy(&rd, h_pin + 2, sizeof(int));
    mpj_status s = (mpj_status)r.status;
    if (s == MPJ_OK && rd) { set_error("rank deficient: some sigma_j <= n omega ||A||_F"); s = MPJ_ERR_RANKDEF; }
    return fin(s);
}

// ---------------------------------------------------------------------------
// Multi-GPU Alg. 5 (column partition, ring only):
// one-sided rotations touch only the two column blocks of a block pair, so
// rank g owns the block-pair slots [g mb/G, (g+1) mb/G) of every block round
// and runs the single-GPU round kernels (Gram blocks, inner solve, column
// updates of C and V) on them alone -- a compacted copy of the schedule with
// the same global block ids, so every slot computes exactly what the
// single-GPU run computes.  C (m x n_p) and V (n_p x n_p) are stored whole on
// every rank, in global column positions; a rank keeps its current blocks up
// to date.  After a block round the 32-column blocks whose slot moves to
// another rank are sent there (ncclSend / ncclRecv into the same columns: the
// ring of the merry-go-round); before each sweep every block is broadcast
// from its owner (the stop test's Gram ||off(C^T C)||_F needs all of C; V
// rides along), then the stop decision is every rank's, identically.
// Step 1 (fp32 one-sided Jacobi) runs the same way; steps 2 and 3 (Q =
// orth(Z), C = A Q) are replicated.  Emulation (emulate = G > 1, no NCCL):
// G rank copies inside this process, transfers as device copies -- no kernel
// waits on another.  Results are bit-identical to mpjacobi_svd's for every G
// when n is a multiple of 64 G (same padding).
// ---------------------------------------------------------------------------
mpj_status mg_comm(const void *nccl_id, int rank, int nranks, void **out);

// the partition's data movement, from the schedule alone: owner[R][blk] = the
// rank whose slot holds column block blk in block round R (slot k belongs to
// rank k / (mb / G)); moves[R] = the blocks whose owner changes from round R
// to R+1 (src -> dst).  Identical on every rank.
struct Mv { int blk, src, dst; };
static void svd_mg_plan(const HostSchedule &hs, int G, std::vector<std::vector<int>> &owner,
                        std::vector<std::vector<Mv>> &moves)
{
    const int nb = hs.nb, mb = nb / 2, mbl = mb / G, rounds = nb - 1;
    owner.assign(rounds, std::vector<int>(nb));
    for (int R = 0; R < rounds; ++R)
        for (int k = 0; k < mb; ++k) {
            const int2 bp = hs.bsched[(size_t)R * mb + k];
            owner[R][bp.x] = owner[R][bp.y] = k / mbl;
        }
    moves.assign(std::max(rounds - 1, 0), {});
    for (int R = 0; R + 1 < rounds; ++R)
        for (int b = 0; b < nb; ++b)
            if (owner[R][b] != owner[R + 1][b]) moves[R].push_back(Mv{b, owner[R][b], owner[R + 1][b]});
}

namespace {
mpj_status svd_nccl_ck(ncclResult_t r, const char *what)
{
    if (r != ncclSuccess) {
        set_error(std::string(what) + ": " + ncclGetErrorString(r));
        return MPJ_ERR_NCCL;
    }
    return MPJ_OK;
}
}  // namespace

mpj_status svd_mg_run(const double *A, int64_t m, int64_t n, int64_t lda, double *Sigma, double *U, int64_t ldu,
                      double *V, int64_t ldv, int *sweeps, const void *nccl_id, int rank, int nranks, int emulate,
                      cudaStream_t st, const mpj_config &cfg, mpj_report &r, double *h_pin)
{
    const double omega = 1.1102230246251565e-16, upsilon = 5.9604644775390625e-08;
    const bool use_nccl = nccl_id != nullptr;
    const int G = use_nccl ? nranks : std::max(1, emulate);
    const int nloc = use_nccl ? 1 : G;
    ncclComm_t comm = nullptr;
    if (use_nccl) {
        void *c = nullptr;
        MPJ_TRY(mg_comm(nccl_id, rank, nranks, &c));
        comm = (ncclComm_t)c;
    }
    const int np = padded_n(n, BW * G);                  // mb = np / 64 slots, a multiple of G
    HostSchedule hs;
    build_schedule(np, BW, hs);
    const int nb = hs.nb, mb = nb / 2, mbl = mb / G, rounds = nb - 1;
    // per local copy: a full single-GPU plan (buffers sized for np columns)
    size_t off = 0;
    SvdPlan probe;
    carve_svd(nullptr, off, m, np, probe);
    std::vector<void *> owned;
    struct Rel {
        std::vector<void *> &v; cudaStream_t st;
        ~Rel() { for (void *p : v) cudaFreeAsync(p, st); }
    } rel{owned, st};
    std::vector<SvdPlan> P(nloc);
    std::vector<DevSched> D(nloc);
    std::vector<int> grank(nloc);
    for (int c = 0; c < nloc; ++c) {
        void *w = nullptr;
        if (cudaMallocAsync(&w, off + 256, st) != cudaSuccess) {
            cudaGetLastError();
            set_error("svd_mg: out of device memory");
            return MPJ_ERR_NOMEM;
        }
        owned.push_back(w);
        char *base = (char *)(((uintptr_t)w + 255) & ~(uintptr_t)255);
        size_t o2 = 0;
        carve_svd(base, o2, m, np, P[c]);
        P[c].n = n;
        P[c].mb = mbl;
        grank[c] = use_nccl ? rank : c;
        std::vector<int2> cb((size_t)std::max(rounds, 1) * mbl);
        for (int R = 0; R < rounds; ++R)
            for (int a = 0; a < mbl; ++a) cb[(size_t)R * mbl + a] = hs.bsched[(size_t)R * mb + grank[c] * mbl + a];
        MPJ_CK(cudaMemcpyAsync(P[c].bsched, cb.data(), cb.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
        MPJ_CK(cudaMemcpyAsync(P[c].lsched, hs.lsched.data(), hs.lsched.size() * sizeof(int2), cudaMemcpyHostToDevice,
                               st));
        D[c].bsched = P[c].bsched; D[c].lsched = P[c].lsched; D[c].b = BW; D[c].nb = 2 * mbl; D[c].np = np;
        D[c].rounds = hs.rounds;
    }
    r.n_padded = np; r.block_b = BW; r.variant = MPJ_VARIANT_BLOCK;
    // block owners per round and the moves between consecutive rounds of a sweep
    std::vector<std::vector<int>> owner;
    std::vector<std::vector<Mv>> moves;
    svd_mg_plan(hs, G, owner, moves);
    const int64_t ldc = P[0].ldc;
    auto loc = [&](int g) { return use_nccl ? (g == rank ? 0 : -1) : g; };   // local copy of rank g
    // column block blk of the m-row matrix X (ld ldx) / of V (ld np), element size es
    auto blk_ptr = [&](void *X, int64_t ldx, size_t es, int blk) { return (char *)X + (size_t)blk * BW * ldx * es; };
    // move / broadcast helpers over the per-copy buffers Cs, Vs (element size es)
    auto transfer = [&](std::vector<void *> &Cs, std::vector<void *> &Vs, size_t es, const std::vector<Mv> &mv,
                        bool with_ex) -> mpj_status {
        if (mv.empty()) return MPJ_OK;
        const size_t cb = (size_t)BW * ldc * es, vb = (size_t)BW * np * es, eb = BW * sizeof(int);
        if (!use_nccl) {
            for (const Mv &x : mv) {
                MPJ_CK(cudaMemcpyAsync(blk_ptr(Cs[x.dst], ldc, es, x.blk), blk_ptr(Cs[x.src], ldc, es, x.blk), cb,
                                       cudaMemcpyDeviceToDevice, st));
                MPJ_CK(cudaMemcpyAsync(blk_ptr(Vs[x.dst], np, es, x.blk), blk_ptr(Vs[x.src], np, es, x.blk), vb,
                                       cudaMemcpyDeviceToDevice, st));
                if (with_ex)
                    MPJ_CK(cudaMemcpyAsync(P[x.dst].ex + (size_t)x.blk * BW, P[x.src].ex + (size_t)x.blk * BW, eb,
                                           cudaMemcpyDeviceToDevice, st));
            }
            return MPJ_OK;
        }
        MPJ_TRY(svd_nccl_ck(ncclGroupStart(), "ncclGroupStart"));
        for (const Mv &x : mv) {
            if (x.src == rank) {
                MPJ_TRY(svd_nccl_ck(ncclSend(blk_ptr(Cs[0], ldc, es, x.blk), cb, ncclChar, x.dst, comm, st), "ncclSend"));
                MPJ_TRY(svd_nccl_ck(ncclSend(blk_ptr(Vs[0], np, es, x.blk), vb, ncclChar, x.dst, comm, st), "ncclSend"));
                if (with_ex)
                    MPJ_TRY(svd_nccl_ck(ncclSend(P[0].ex + (size_t)x.blk * BW, eb, ncclChar, x.dst, comm, st), "ncclSend"));
            } else if (x.dst == rank) {
                MPJ_TRY(svd_nccl_ck(ncclRecv(blk_ptr(Cs[0], ldc, es, x.blk), cb, ncclChar, x.src, comm, st), "ncclRecv"));
                MPJ_TRY(svd_nccl_ck(ncclRecv(blk_ptr(Vs[0], np, es, x.blk), vb, ncclChar, x.src, comm, st), "ncclRecv"));
                if (with_ex)
                    MPJ_TRY(svd_nccl_ck(ncclRecv(P[0].ex + (size_t)x.blk * BW, eb, ncclChar, x.src, comm, st), "ncclRecv"));
            }
        }
        MPJ_TRY(svd_nccl_ck(ncclGroupEnd(), "ncclGroupEnd"));
        return MPJ_OK;
    };
    // every block from its owner (ownership of round Rlast) to every copy
    auto gather_all = [&](std::vector<void *> &Cs, std::vector<void *> &Vs, size_t es, int Rlast) -> mpj_status {
        const size_t cb = (size_t)BW * ldc * es, vb = (size_t)BW * np * es;
        if (!use_nccl) {
            for (int b = 0; b < nb; ++b) {
                const int o = owner[Rlast][b];
                for (int c = 0; c < nloc; ++c) {
                    if (c == o) continue;
                    MPJ_CK(cudaMemcpyAsync(blk_ptr(Cs[c], ldc, es, b), blk_ptr(Cs[o], ldc, es, b), cb,
                                           cudaMemcpyDeviceToDevice, st));
                    MPJ_CK(cudaMemcpyAsync(blk_ptr(Vs[c], np, es, b), blk_ptr(Vs[o], np, es, b), vb,
                                           cudaMemcpyDeviceToDevice, st));
                }
            }
            return MPJ_OK;
        }
        if (G == 1) return MPJ_OK;
        MPJ_TRY(svd_nccl_ck(ncclGroupStart(), "ncclGroupStart"));
        for (int b = 0; b < nb; ++b) {
            const int o = owner[Rlast][b];
            void *pc = blk_ptr(Cs[0], ldc, es, b), *pv = blk_ptr(Vs[0], np, es, b);
            MPJ_TRY(svd_nccl_ck(ncclBroadcast(pc, pc, cb, ncclChar, o, comm, st), "ncclBroadcast"));
            MPJ_TRY(svd_nccl_ck(ncclBroadcast(pv, pv, vb, ncclChar, o, comm, st), "ncclBroadcast"));
        }
        MPJ_TRY(svd_nccl_ck(ncclGroupEnd(), "ncclGroupEnd"));
        return MPJ_OK;
    };
    // total rotations so far (all ranks)
    auto total_rot = [&]() -> unsigned long long {
        unsigned long long tot = 0;
        if (!use_nccl) {
            for (int c = 0; c < nloc; ++c) {
                unsigned long long v = 0;
                cudaMemcpyAsync(h_pin, P[c].cnt, sizeof(v), cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                std::memcpy(&v, h_pin, sizeof(v));
                tot += v;
            }
            return tot;
        }
        unsigned long long *scr = (unsigned long long *)(P[0].red_out + 4);
        ncclAllReduce(P[0].cnt, scr, 1, ncclUint64, ncclSum, comm, st);
        cudaMemcpyAsync(h_pin, scr, sizeof(tot), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        std::memcpy(&tot, h_pin, sizeof(tot));
        return tot;
    };
    // the one-sided loop on every copy (R = float: step 1; double: the fp64 stage)
    auto loop = [&](auto tag, double eps_rel, double nu, double early, int max_sweeps, SvdStage &out) -> mpj_status {
        using R = decltype(tag);
        std::vector<void *> Cs(nloc), Vs(nloc);
        for (int c = 0; c < nloc; ++c) {
            Cs[c] = sizeof(R) == 8 ? (void *)P[c].C : (void *)P[c].C32;
            Vs[c] = sizeof(R) == 8 ? (void *)P[c].V : (void *)P[c].V32;
        }
        const double N = 0.5 * (double)n * (double)(n - 1);
        mpj_status status = MPJ_ERR_NOCONV;
        unsigned long long prev = 0;
        double ratio = 1.0;
        const double xb = svd_exact_below();
        for (int c = 0; c < nloc; ++c) MPJ_CK(cudaMemsetAsync(P[c].cnt, 0, sizeof(unsigned long long), st));
        for (;;) {
            if (out.sweeps > 0) MPJ_TRY(gather_all(Cs, Vs, sizeof(R), rounds - 1));
            // stop test on copy 0 (every copy holds the same C now)
            SvdPlan &p = P[0];
            if (sizeof(R) == 4) launch_copy_pad<float, double>((float *)Cs[0], ldc, (int)m, np, p.C, ldc, (int)m, np, st);
            launch_dgemm(true, false, np, np, m, 1.0, p.C, ldc, p.C, ldc, 0.0, p.G, np, st, nullptr, 0, true);
            launch_norm_sym_upper(p.G, np, np, true, p.red_part, p.red_out, st);
            launch_norm_sym_upper(p.G, np, np, false, p.red_part, p.red_out + 1, st);
            MPJ_CK(cudaMemcpyAsync(h_pin, p.red_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
            MPJ_CK(cudaStreamSynchronize(st));
            const double offv = h_pin[0], tot = h_pin[1];
            if (out.sweeps < 64) { out.hist[out.sweeps] = offv; out.nhist = out.sweeps + 1; }
            if (!std::isfinite(offv)) { set_error("non-finite Gram"); return MPJ_ERR_NONFINITE; }
            if (offv <= eps_rel * tot) { status = MPJ_OK; break; }
            if (out.sweeps >= max_sweeps) { status = MPJ_ERR_NOCONV; break; }
            ++out.sweeps;
            const bool exact = sizeof(R) == 8 && ratio < xb;
            for (int c = 0; c < nloc; ++c)
                MPJ_CK(cudaMemsetAsync(P[c].uid + mbl, 0, (size_t)rounds * sizeof(int), st));
            for (int R0 = 0; R0 < rounds; ++R0) {
                for (int c = 0; c < nloc; ++c)
                    MPJ_TRY(svd_block_round<R>(P[c], (R *)Cs[c], (R *)Vs[c], D[c], R0, (R)nu, st, exact, P[c].uid,
                                               P[c].uid + mbl + R0));
                if (R0 + 1 < rounds) MPJ_TRY(transfer(Cs, Vs, sizeof(R), moves[R0], exact));
            }
            const unsigned long long now = total_rot();
            const unsigned long long rs = now - prev;
            prev = now;
            out.rotations = (long long)now;
            if (out.sweeps <= 64) out.rot_hist[out.sweeps - 1] = (long long)rs;
            ratio = N > 0 ? (double)rs / N : 0.0;
            if (early > 0 && N > 0 && (double)rs / N < early) { status = MPJ_OK; break; }
        }
        MPJ_TRY(gather_all(Cs, Vs, sizeof(R), rounds - 1));
        return status;
    };
    (void)loc;

    // a0: A staged into every copy (zero padded), ||A||_F, finiteness
    for (int c = 0; c < nloc; ++c) {
        MPJ_CK(cudaMemsetAsync(P[c].Ad, 0, (size_t)ldc * np * 8, st));
        MPJ_CK(cudaMemcpy2DAsync(P[c].Ad, ldc * 8, A, lda * 8, m * 8, n, cudaMemcpyDefault, st));
    }
    MPJ_CK(cudaMemsetAsync(P[0].flag, 0, sizeof(int), st));
    launch_check_finite(P[0].Ad, ldc, (int)m, (int)n, P[0].flag, st);
    launch_norm<double>(P[0].Ad, ldc, (int)m, np, false, P[0].red_part, P[0].red_out, st);
    MPJ_CK(cudaMemcpyAsync(h_pin, P[0].red_out, sizeof(double), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaMemcpyAsync(h_pin + 1, P[0].flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaStreamSynchronize(st));
    const double normA = h_pin[0];
    int bad = 0;
    std::memcpy(&bad, h_pin + 1, sizeof(int));
    r.norm_a = normA;
    if (bad) { set_error("input has NaN/Inf"); return MPJ_ERR_NONFINITE; }
    // a1: fp32 one-sided Jacobi on fl32(A), partitioned
    for (int c = 0; c < nloc; ++c) {
        launch_copy_pad<double, float>(P[c].Ad, ldc, (int)m, np, P[c].C32, ldc, (int)m, np, st);
        MPJ_CK(cudaMemsetAsync(P[c].V32, 0, (size_t)np * np * 4, st));
        launch_identity<float>(P[c].V32, np, (int)n, (int)n, st);
    }
    {
        SvdStage lo;
        mpj_status sl = loop(float(0), eps_low_factor(cfg, n) * upsilon, cfg.nu_low_factor * upsilon,
                             cfg.early_stop_ratio, cfg.max_sweeps_low, lo);
        if (sl != MPJ_OK && sl != MPJ_ERR_NOCONV) return sl;
        r.sweeps_low = lo.sweeps; r.rotations_low = lo.rotations; r.status_low = sl;
    }
    // a2, a3 (replicated): Q = orth(fp64(V32)) into V, C = A Q
    for (int c = 0; c < nloc; ++c) {
        SvdPlan &p = P[c];
        launch_copy_pad<float, double>(p.V32, np, (int)n, (int)n, p.G, np, (int)n, (int)n, st);
        MPJ_CK(cudaMemsetAsync(p.V, 0, (size_t)np * np * 8, st));
        MPJ_TRY(orth_cgs2(p.G, np, p.V, np, n, n, p.orth_ws, st));
        MPJ_CK(cudaMemsetAsync(p.C, 0, (size_t)ldc * np * 8, st));
        launch_dgemm(false, false, m, n, n, 1.0, p.Ad, ldc, p.V, np, 0.0, p.C, ldc, st);
    }
    // fp64 sweeps, partitioned
    SvdStage hi;
    mpj_status sh = loop(double(0), cfg.eps_factor * omega, cfg.nu_factor * omega, cfg.early_stop_ratio,
                         cfg.max_sweeps, hi);
    r.sweeps = hi.sweeps; r.rotations = hi.rotations; r.status = sh;
    r.off0 = hi.hist[0];
    for (int k = 0; k < hi.nhist && k < 64; ++k) r.off_hist[k] = hi.hist[k];
    for (int k = 0; k < 64; ++k) r.rot_hist[k] = hi.rot_hist[k];
    if (sh != MPJ_OK && sh != MPJ_ERR_NOCONV) return sh;
    if (sweeps) *sweeps = hi.sweeps;
    // a10: extraction from copy 0 (every copy holds the same C and V)
    SvdPlan &p = P[0];
    k_colnorm<<<(unsigned)n, 256, 0, st>>>(p.C, ldc, (int)m, p.nrm);
    MPJ_CK(cudaMemsetAsync(p.flag, 0, sizeof(int), st));
    k_rank_vec<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p.nrm, (int)n, p.rank, p.sig, (double)n * omega * normA,
                                                            p.flag);
    count_launch(2);
    MPJ_CK(cudaMemcpyAsync(Sigma, p.sig, n * 8, cudaMemcpyDefault, st));
    k_svd_extract<<<dim3(std::max<int64_t>(1, std::min<int64_t>(64, (m + 255) / 256)), (unsigned)n), 256, 0, st>>>(
        p.C, ldc, (int)m, p.V, np, (int)n, p.rank, p.nrm, U, ldu, V, ldv);
    count_launch();
    MPJ_CK(cudaMemcpyAsync(h_pin + 2, p.flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    MPJ_CK(cudaStreamSynchronize(st));
    int rd = 0;
    std::memcpy(&rd, h_pin + 2, sizeof(int));
    mpj_status s2 = (mpj_status)r.status;
    if (s2 == MPJ_OK && rd) { set_error("rank deficient: some sigma_j <= n omega ||A||_F"); s2 = MPJ_ERR_RANKDEF; }
    return s2;
}

}  // namespace mpj

// Host-only view of mpjacobi_svd_mg's partition plan (gloo test of the data
// movement): the padded order, the rounds, the block pairs of each round
// (rounds x mb int pairs, slot k on rank k / (mb / nranks)) and the moves
// between consecutive rounds (per round up to 4 nranks triples (blk, src, dst)).
extern "C" mpj_status mpjacobi_svd_mg_plan(int64_t n, int nranks, int *np_out, int *rounds_out, int *pairs,
                                           int *moves, int *nmoves)
{
    using namespace mpj;
    set_error("");
    if (n < 1 || nranks < 1) { set_error("mpjacobi_svd_mg_plan: invalid argument"); return MPJ_ERR_INVALID; }
    const int np = padded_n(n, BW * nranks);
    HostSchedule hs;
    build_schedule(np, BW, hs);
    const int mb = hs.nb / 2, rounds = hs.nb - 1;
    if (np_out) *np_out = np;
    if (rounds_out) *rounds_out = rounds;
    std::vector<std::vector<int>> owner;
    std::vector<std::vector<Mv>> mv;
    svd_mg_plan(hs, nranks, owner, mv);
    if (pairs)
        for (int R = 0; R < rounds; ++R)
            for (int k = 0; k < mb; ++k) {
                pairs[2 * ((size_t)R * mb + k)] = hs.bsched[(size_t)R * mb + k].x;
                pairs[2 * ((size_t)R * mb + k) + 1] = hs.bsched[(size_t)R * mb + k].y;
            }
    const int maxm = 4 * nranks;
    for (int R = 0; R + 1 < rounds; ++R) {
        if ((int)mv[R].size() > maxm) { set_error("mpjacobi_svd_mg_plan: too many moves"); return MPJ_ERR_INVALID; }
        if (nmoves) nmoves[R] = (int)mv[R].size();
        if (moves)
            for (size_t i = 0; i < mv[R].size(); ++i) {
                int *t = moves + 3 * ((size_t)R * maxm + i);
                t[0] = mv[R][i].blk; t[1] = mv[R][i].src; t[2] = mv[R][i].dst;
            }
    }
    return MPJ_OK;
}
