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
template <> struct Lay<float> { static constexpr int LD = 68; };    // 16-byte aligned columns (cp.async)
// K3's private 64 x 64 buffers (D, U): an odd leading dimension makes the
// column-stride (mirror) accesses of the inner rounds conflict-free for 4- and
// 8-byte words (LD = 68 maps a 32-lane column-stride access to 4 or 8 bank
// groups: 8-way conflicts that made K3 shared-memory bound).
template <typename R> struct LayK { static constexpr int LD = 65; };

// c0 += a b0, c1 += a b1 as one packed fp32x2 FMA (SASS FFMA2 with a scalar
// operand): each lane is a round-to-nearest fused multiply-add, bit-identical
// to two __fmaf_rn, in half the issue slots.
__device__ __forceinline__ void ffma2(float a, float b0, float b1, float &c0, float &c1)
{
    unsigned long long aa, bb, cc, r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
    asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b0), "f"(b1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "f"(c0), "f"(c1));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(aa), "l"(bb), "l"(cc));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(c0), "=f"(c1) : "l"(r));
}


// global index of local index li (0..63) of block pair (I, J)
__device__ __forceinline__ int gidx(int2 bp, int li) { return li < BW ? bp.x * BW + li : bp.y * BW + (li - BW); }

// Rotation parameters of one round (pair k: t, s, tau).
template <typename R> struct InnerParams {
    R t[BW], s[BW], u[BW];
};

// ---------------------------------------------------------------------------
// The rounds of one block pair on its 64 x 64 block D for the batched path
// (one block pair bp = (0, 1), NT = 256 threads): if `intra`, the b-1
// merry-go-round rounds inside each half first (block round 0, reading R1),
// then the b cyclic-shift cross rounds, with U in registers.  Thread (warp w, lane k) holds rows w + 8 i (i = 0..7) of U
// at columns k (top half) and 32 + k (bottom half) at the start of a call.
// Intra rounds pair columns inside each half (lsched): the two columns of a
// pair sit in two lanes, each lane fetches its partner's value (shuffle) and
// computes its own side with the same fused multiply-adds as rot().  Cross
// round s pairs k with 32 + (k + s) mod 32: lane k holds that bottom column
// (the bottoms move one lane per round), so the rotation is lane-local; after
// the 32 cross rounds the layout is back to the start.  D is updated as in
// the shared-memory version did (same element arithmetic, bit-identical
// results); U's shared-memory traffic, half of a round's, goes away.
// ---------------------------------------------------------------------------
struct InnerSharedB {
    int lp[BW], lq[BW], gp[BW];
    int part_t[BW], part_b[BW];     // intra rounds: partner column (within the half) of lane k
    int pair_t[BW], pair_b[BW];     // ... its pair index (parameters)
    int isp_t[BW], isp_b[BW];       // ... whether lane k's column is the pair's p
    unsigned nrot;
};

template <typename R>
__device__ __forceinline__ void rot_side(R s, R tau, bool isp, R &mine, R other)
{
    // rot(): x' = x - s (y + tau x), y' = y + s (x - tau y) (p = x, q = y)
    mine = isp ? fmaR(-s, fmaR(tau, mine, other), mine) : fmaR(s, fmaR(-tau, mine, other), mine);
}

template <typename R, int LD = Lay<R>::LD>
__device__ __forceinline__ unsigned inner_rounds_b(R *D, R *U, bool intra, const int2 *__restrict__ lsched, R nu,
                                                   int rule, InnerSharedB &sh, InnerParams<R> &pr)
{
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    R ut[8], ub[8];
    #pragma unroll
    for (int i = 0; i < 8; ++i) {
        ut[i] = U[(w + 8 * i) + lane * LD];
        ub[i] = U[(w + 8 * i) + (BW + lane) * LD];
    }
    // static tile items of this thread: e = tid + NT u -> off-diagonal tile (k, l), k < l
    constexpr int NE = (BW + BW * (BW - 1) / 2 + NT - 1) / NT;
    int tk[NE], tl[NE];
    #pragma unroll
    for (int u = 0; u < NE; ++u) {
        const int wt = tid + NT * u - BW;
        int ll = 1, kk = 0;
        if (wt >= 0) {
            ll = (int)((1.0f + sqrtf(1.0f + 8.0f * wt)) * 0.5f);
            while (ll * (ll - 1) / 2 > wt) --ll;
            while ((ll + 1) * ll / 2 <= wt) ++ll;
            kk = wt - ll * (ll - 1) / 2;
        }
        tk[u] = kk;
        tl[u] = ll;
    }
    if (tid == 0) sh.nrot = 0;
    __syncthreads();
    const int nrounds = intra ? (BW - 1) + BW : BW;
    for (int s = 0; s < nrounds; ++s) {
        const bool in_intra = intra && s < BW - 1;
        if (tid < BW) {
            int a, c;
            if (in_intra) {
                const int hb = BW / 2;
                const int2 lp = lsched[s * hb + (tid < hb ? tid : tid - hb)];
                const int off = (tid < hb) ? 0 : BW;
                a = off + lp.x; c = off + lp.y;
            } else {
                const int sc = intra ? s - (BW - 1) : s;
                a = tid;
                int j = tid + sc; if (j >= BW) j -= BW;
                c = BW + j;
            }
            const int lp = a < c ? a : c, lq = a < c ? c : a;   // bp = (0, 1): local == global order
            R t, sn, u;
            const int did = rot_params<R>(D[lp + lp * LD], D[lq + lq * LD], D[lp + lq * LD], nu, rule, t, sn, u);
            sh.lp[tid] = lp; sh.lq[tid] = lq; sh.gp[tid] = lp;
            pr.t[tid] = t; pr.s[tid] = sn; pr.u[tid] = u;
            if (in_intra) {
                if (tid < BW / 2) {
                    sh.part_t[lp] = lq; sh.part_t[lq] = lp; sh.pair_t[lp] = tid; sh.pair_t[lq] = tid;
                    sh.isp_t[lp] = 1; sh.isp_t[lq] = 0;
                } else {
                    sh.part_b[lp - BW] = lq - BW; sh.part_b[lq - BW] = lp - BW;
                    sh.pair_b[lp - BW] = tid; sh.pair_b[lq - BW] = tid;
                    sh.isp_b[lp - BW] = 1; sh.isp_b[lq - BW] = 0;
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, did);
            if (tid == 0) sh.nrot += __popc(bal);
        }
        __syncthreads();
        // D <- J^T D J: the 32 diagonal and 496 upper pair tiles (k < l), each
        // also stored at its mirror (what the (l, k) tile computes, bit for bit).
        // Thread tid owns items e = tid + NT u (u < NE); their (k, l) were decoded
        // once before the rounds (tk / tl, tl < 0: diagonal tile tk)
        #pragma unroll
        for (int u = 0; u < NE; ++u) {
            const int e = tid + NT * u;
            if (e >= BW + BW * (BW - 1) / 2) break;
            if (e < BW) {
                const int pk = sh.lp[e], qk = sh.lq[e];
                const R apq = D[pk + qk * LD], t = pr.t[e];
                D[pk + pk * LD] = fmaR(-t, apq, D[pk + pk * LD]);
                D[qk + qk * LD] = fmaR(t, apq, D[qk + qk * LD]);
                D[pk + qk * LD] = R(0);
                D[qk + pk * LD] = R(0);
                continue;
            }
            const int kk = tk[u], ll = tl[u];
            const int pk = sh.lp[kk], qk = sh.lq[kk], pl = sh.lp[ll], ql = sh.lq[ll];
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
            D[pl + pk * LD] = x11; D[pl + qk * LD] = x21; D[ql + pk * LD] = x12; D[ql + qk * LD] = x22;
        }
        // U <- U J in registers
        if (U) {
            if (in_intra) {
                const int pt = sh.part_t[lane], pb = sh.part_b[lane];
                const int jt = sh.pair_t[lane], jb = sh.pair_b[lane];
                const bool it = sh.isp_t[lane] != 0, ib = sh.isp_b[lane] != 0;
                const R st = pr.s[jt], tt = pr.u[jt], sb = pr.s[jb], tb = pr.u[jb];
                #pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const R ot = __shfl_sync(0xffffffffu, ut[i], pt), ob = __shfl_sync(0xffffffffu, ub[i], pb);
                    if (st != R(0)) rot_side<R>(st, tt, it, ut[i], ot);
                    if (sb != R(0)) rot_side<R>(sb, tb, ib, ub[i], ob);
                }
            } else {
                const R sk = pr.s[lane], tk = pr.u[lane];
                #pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (sk != R(0)) rot<R>(sk, tk, ut[i], ub[i]);   // p = a_k (top), q = b_k
                    ub[i] = __shfl_sync(0xffffffffu, ub[i], (lane + 1) & 31);
                }
            }
        }
        __syncthreads();
    }
    #pragma unroll
    for (int i = 0; i < 8; ++i) {
        U[(w + 8 * i) + lane * LD] = ut[i];
        U[(w + 8 * i) + (BW + lane) * LD] = ub[i];
    }
    __syncthreads();
    return sh.nrot;
}

// ---------------------------------------------------------------------------
// Pipelined inner rounds (NTW = 1024 threads) for the block variant's K3.
// Warps 1..31 apply round s (496 off-diagonal 2x2 tiles computed once in the
// canonical order of reading R7 and mirrored, 32 diagonal tiles, U <- U J),
// reading Dc and writing Dn; meanwhile warp 0 computes the rotation
// parameters of round s+1: for each next pair (p', q') it recomputes from Dc,
// with the very same arithmetic, the three entries Lemma 3.1 needs after
// round s (two diagonal updates and one element of one 2x2 tile), then runs
// rot_params.  One barrier per round; the parameter latency (divides,
// square roots) is hidden under the update phase.  Results are identical to
// inner_rounds.
// ---------------------------------------------------------------------------
constexpr int NTW = 1024;

// timing hook for tools/k3_trace.cu (empty in the library)
#ifndef MPJ_K3_TRACE
#define MPJ_K3_TRACE(event, round)
#endif

template <typename R>
struct WideParams {
    R t[BW], s[BW], u[BW];
    int p[BW], q[BW], gp[BW];
    int pos[TW];            // local index -> pair of this round
};

// local pair (a, c) of `lane` in round s
__device__ __forceinline__ void round_pair(int s, int lane, bool intra, const int2 *__restrict__ lsched, int &a,
                                           int &c)
{
    if (intra && s < BW - 1) {
        const int hb = BW / 2;
        const int2 lp = lsched[s * hb + (lane < hb ? lane : lane - hb)];
        const int off = (lane < hb) ? 0 : BW;
        a = off + lp.x; c = off + lp.y;
    } else {
        const int sc = intra ? s - (BW - 1) : s;
        a = lane;
        int j = lane + sc; if (j >= BW) j -= BW;
        c = BW + j;
    }
}

// position of D(i, j): full storage, or (SYM) the upper triangle only
template <typename R, bool SYM>
__device__ __forceinline__ int didx(int i, int j)
{
    constexpr int LD = LayK<R>::LD;
    return (!SYM || i <= j) ? i + j * LD : j + i * LD;
}

// the canonical 2x2 tile (rows of pair k, columns of pair l) after the round
template <typename R, bool SYM = false>
__device__ __forceinline__ void tile_after(const R *Dc, const WideParams<R> &P, int k, int l, R &x11, R &x21,
                                           R &x12, R &x22)
{
    const int pk = P.p[k], qk = P.q[k], pl = P.p[l], ql = P.q[l];
    const R sk = P.s[k], uk = P.u[k], sl = P.s[l], ul = P.u[l];
    x11 = Dc[didx<R, SYM>(pk, pl)]; x21 = Dc[didx<R, SYM>(qk, pl)];
    x12 = Dc[didx<R, SYM>(pk, ql)]; x22 = Dc[didx<R, SYM>(qk, ql)];
    if (P.gp[k] < P.gp[l]) {
        rot<R>(sk, uk, x11, x21); rot<R>(sk, uk, x12, x22);
        rot<R>(sl, ul, x11, x12); rot<R>(sl, ul, x21, x22);
    } else {
        rot<R>(sl, ul, x11, x12); rot<R>(sl, ul, x21, x22);
        rot<R>(sk, uk, x11, x21); rot<R>(sk, uk, x12, x22);
    }
}

// diagonal entry of local index i after the round
template <typename R, bool SYM = false>
__device__ __forceinline__ R diag_after(const R *Dc, const WideParams<R> &P, int i)
{
    constexpr int LD = LayK<R>::LD;
    const int k = P.pos[i], pk = P.p[k], qk = P.q[k];
    const R apq = Dc[didx<R, SYM>(pk, qk)];
    return i == pk ? fmaR(-P.t[k], apq, Dc[pk + pk * LD]) : fmaR(P.t[k], apq, Dc[qk + qk * LD]);
}

// UREG (cross rounds only): U lives in registers instead of shared memory.
// Update warp w (1..31) holds rows 2(w-1), 2(w-1)+1 (warps 1, 2 also rows 62,
// 63) at columns a_k = k and b_k = 32 + (k + s) mod 32 in lane k; pair k of
// round s rotates exactly these two columns, and b_k(s+1) = b_{k+1}(s), so
// the bottoms move one lane per round (shuffle).  This removes U's loads,
// stores and index reads -- about half of a round's shared-memory traffic,
// which bounds the rounds (tools/k3_trace.cu: the parameter warp's dependent
// loads queue behind it).  Same arithmetic (rot on (U(r,p), U(r,q))).
template <typename R, bool FAST>
__device__ __forceinline__ int rot_params_sel(R app, R aqq, R apq, R nu, int rule, R &t, R &s, R &tau)
{
    if constexpr (FAST) return rot_params_fast<R>(app, aqq, apq, nu, rule, t, s, tau);
    else return rot_params<R>(app, aqq, apq, nu, rule, t, s, tau);
}

template <typename R, bool UREG, bool FASTP = false>
__device__ __forceinline__ R *smem_rounds_wide(R *D0, R *D1, R *U, int2 bp, bool intra, int nrounds,
                                               const int2 *__restrict__ lsched, R nu, int rule,
                                               WideParams<R> (&PP)[2], unsigned &cnt)
{
    constexpr int LD = LayK<R>::LD;
    // the parameter warp is the LAST warp: the SM's warp arbiter issues
    // highest-warp-id first, and this warp's dependent chain is the critical path
    const int tid = threadIdx.x, lane = tid & 31, warp = (NTW / 32 - 1) - (tid >> 5);
    R *Dc = D0, *Dn = D1;
    // static assignment of the update work to the other threads
    int tk = -1, tl = -1, ur[3] = {0, 0, 0}, uk[3] = {-1, -1, -1};
    if (warp > 0) {
        const int w = (warp - 1) * 32 + lane, NW = NTW - 32;
        if (w < BW * (BW - 1) / 2) {
            int l = (int)((1.0f + sqrtf(1.0f + 8.0f * w)) * 0.5f);
            while (l * (l - 1) / 2 > w) --l;
            while ((l + 1) * l / 2 <= w) ++l;
            tk = w - l * (l - 1) / 2; tl = l;
        } else if (w < BW * (BW - 1) / 2 + BW) {
            tk = w - BW * (BW - 1) / 2; tl = -1;
        }
        if (!UREG) {
            #pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int e = w + j * NW;
                if (e < BW * TW) { ur[j] = e & (TW - 1); uk[j] = e >> 6; }
            }
        }
    }
    // UREG: rows of U in registers (update warps only)
    const bool flip = bp.x > bp.y;          // cross pair k: p = b_k if the bottom block comes first
    const int nrow = (warp == 1 || warp == 2) ? 3 : (warp > 0 ? 2 : 0);
    const int urow[3] = {2 * (warp - 1), 2 * (warp - 1) + 1, 62 + (warp - 1)};
    R ua[3] = {R(0), R(0), R(0)}, ub[3] = {R(0), R(0), R(0)};
    if (UREG) {
        #pragma unroll
        for (int j = 0; j < 3; ++j)
            if (j < nrow) { ua[j] = U[urow[j] + lane * LD]; ub[j] = U[urow[j] + (BW + lane) * LD]; }
    }
    // cross rounds (UREG): pair k of cross round x is (k, 32 + (k + x) mod 32), so
    // its p / q, its position in the order of global p indices and the pair of
    // a local index are arithmetic -- no dependent shared-memory index loads
    // on the parameter warp's critical path
    auto xp = [&](int k, int x) { return flip ? BW + ((k + x) & 31) : k; };
    auto xq = [&](int k, int x) { return flip ? k : BW + ((k + x) & 31); };
    auto xkey = [&](int k, int x) { return flip ? ((k + x) & 31) : k; };
    auto xpos = [&](int i, int x) { return i < BW ? i : ((i - BW - x) & 31); };
    R ct = R(0), cs = R(0), cu = R(0);      // parameter warp: (t, s, tau) of pair `lane` this round
    // parameters of round 0
    if (warp == 0) {
        int a, c;
        round_pair(0, lane, intra, lsched, a, c);
        const int ga = gidx(bp, a), gc = gidx(bp, c);
        const int pk = ga < gc ? a : c, qk = ga < gc ? c : a;
        R t, sk, uk;
        const int did = rot_params_sel<R, FASTP>(Dc[pk + pk * LD], Dc[qk + qk * LD], Dc[didx<R, UREG>(pk, qk)], nu, rule, t,
                                      sk, uk);
        ct = t; cs = sk; cu = uk;
        cnt += did;
        WideParams<R> &P = PP[0];
        P.t[lane] = t; P.s[lane] = sk; P.u[lane] = uk;
        P.p[lane] = pk; P.q[lane] = qk; P.gp[lane] = ga < gc ? ga : gc;
        P.pos[pk] = lane; P.pos[qk] = lane;
    }
    __syncthreads();
    for (int s = 0; s < nrounds; ++s) {
        const WideParams<R> &P = PP[s & 1];
        if (UREG && warp == 0) {
            if (s + 1 < nrounds) {
                WideParams<R> &N = PP[(s + 1) & 1];
                const int pn = xp(lane, s + 1), qn = xq(lane, s + 1);
                // pairs of round s holding pn and qn, and their parameters (registers of lanes k, l)
                const int k = xpos(pn, s), l = xpos(qn, s);
                const int kk = k < l ? k : l, ll = k < l ? l : k;
                const R tk_ = __shfl_sync(0xffffffffu, ct, k), tl_ = __shfl_sync(0xffffffffu, ct, l);
                const R sk_ = __shfl_sync(0xffffffffu, cs, kk), uk_ = __shfl_sync(0xffffffffu, cu, kk);
                const R sl_ = __shfl_sync(0xffffffffu, cs, ll), ul_ = __shfl_sync(0xffffffffu, cu, ll);
                // D(pn, pn) and D(qn, qn) after round s (diagonal formula of their pairs)
                const int pk = xp(k, s), qk = xq(k, s), pl = xp(l, s), ql = xq(l, s);
                const R apq_k = Dc[didx<R, true>(pk, qk)], apq_l = Dc[didx<R, true>(pl, ql)];
                const R app = pn == pk ? fmaR(-tk_, apq_k, Dc[pk + pk * LD]) : fmaR(tk_, apq_k, Dc[qk + qk * LD]);
                const R aqq = qn == pl ? fmaR(-tl_, apq_l, Dc[pl + pl * LD]) : fmaR(tl_, apq_l, Dc[ql + ql * LD]);
                // D(pn, qn) after round s: entry of the canonical tile (kk, ll), as the update warps compute it
                const int pkk = xp(kk, s), qkk = xq(kk, s), pll = xp(ll, s), qll = xq(ll, s);
                R x11 = Dc[didx<R, true>(pkk, pll)], x21 = Dc[didx<R, true>(qkk, pll)];
                R x12 = Dc[didx<R, true>(pkk, qll)], x22 = Dc[didx<R, true>(qkk, qll)];
                if (xkey(kk, s) < xkey(ll, s)) {
                    rot<R>(sk_, uk_, x11, x21); rot<R>(sk_, uk_, x12, x22);
                    rot<R>(sl_, ul_, x11, x12); rot<R>(sl_, ul_, x21, x22);
                } else {
                    rot<R>(sl_, ul_, x11, x12); rot<R>(sl_, ul_, x21, x22);
                    rot<R>(sk_, uk_, x11, x21); rot<R>(sk_, uk_, x12, x22);
                }
                // rows of the tile belong to pair kk, columns to ll
                const int rn = k < l ? pn : qn, cn = k < l ? qn : pn;
                const R apq = (rn == pkk) ? (cn == pll ? x11 : x12) : (cn == pll ? x21 : x22);
                R t, sk, uk;
                const int did = rot_params_sel<R, FASTP>(app, aqq, apq, nu, rule, t, sk, uk);
                MPJ_K3_TRACE(0, s);
                cnt += did;
                N.t[lane] = t; N.s[lane] = sk; N.u[lane] = uk;
                ct = t; cs = sk; cu = uk;
            }
        } else if (warp == 0) {
            if (s + 1 < nrounds) {
                WideParams<R> &N = PP[(s + 1) & 1];
                int a, c;
                round_pair(s + 1, lane, intra, lsched, a, c);
                const int ga = gidx(bp, a), gc = gidx(bp, c);
                const int pn = ga < gc ? a : c, qn = ga < gc ? c : a;
                const R app = diag_after<R, UREG>(Dc, P, pn), aqq = diag_after<R, UREG>(Dc, P, qn);
                // (pn, qn) lies in the tile of pairs k = pos[pn], l = pos[qn] (k != l)
                const int k = P.pos[pn], l = P.pos[qn];
                R x11, x21, x12, x22, apq;
                if (k < l) {            // computed tile (k, l): rows of k, columns of l
                    tile_after<R, UREG>(Dc, P, k, l, x11, x21, x12, x22);
                    apq = (pn == P.p[k]) ? (qn == P.p[l] ? x11 : x12) : (qn == P.p[l] ? x21 : x22);
                } else {                // mirror of tile (l, k): entry (qn, pn)
                    tile_after<R, UREG>(Dc, P, l, k, x11, x21, x12, x22);
                    apq = (qn == P.p[l]) ? (pn == P.p[k] ? x11 : x12) : (pn == P.p[k] ? x21 : x22);
                }
                R t, sk, uk;
                const int did = rot_params_sel<R, FASTP>(app, aqq, apq, nu, rule, t, sk, uk);
                MPJ_K3_TRACE(0, s);
                cnt += did;
                N.t[lane] = t; N.s[lane] = sk; N.u[lane] = uk;
                N.p[lane] = pn; N.q[lane] = qn; N.gp[lane] = ga < gc ? ga : gc;
                N.pos[pn] = lane; N.pos[qn] = lane;
            }
        } else {
            // static work of this thread (computed before the loop): tile (tk, tl)
            // (tl < 0: diagonal tile tk; tk < 0: none) and U items (ur[j], uk[j])
            if (tk >= 0) {
                if (tl >= 0 && UREG) {
                    // cross round: arithmetic pairs, upper triangle only (mirrored at the end)
                    const int pk = xp(tk, s), qk = xq(tk, s), pl = xp(tl, s), ql = xq(tl, s);
                    const R sk = P.s[tk], uk = P.u[tk], sl = P.s[tl], ul = P.u[tl];
                    R x11 = Dc[didx<R, true>(pk, pl)], x21 = Dc[didx<R, true>(qk, pl)];
                    R x12 = Dc[didx<R, true>(pk, ql)], x22 = Dc[didx<R, true>(qk, ql)];
                    if (xkey(tk, s) < xkey(tl, s)) {
                        rot<R>(sk, uk, x11, x21); rot<R>(sk, uk, x12, x22);
                        rot<R>(sl, ul, x11, x12); rot<R>(sl, ul, x21, x22);
                    } else {
                        rot<R>(sl, ul, x11, x12); rot<R>(sl, ul, x21, x22);
                        rot<R>(sk, uk, x11, x21); rot<R>(sk, uk, x12, x22);
                    }
                    Dn[didx<R, true>(pk, pl)] = x11; Dn[didx<R, true>(qk, pl)] = x21;
                    Dn[didx<R, true>(pk, ql)] = x12; Dn[didx<R, true>(qk, ql)] = x22;
                } else if (tl >= 0) {
                    R x11, x21, x12, x22;
                    tile_after<R, UREG>(Dc, P, tk, tl, x11, x21, x12, x22);
                    const int pk = P.p[tk], qk = P.q[tk], pl = P.p[tl], ql = P.q[tl];
                    {
                        Dn[pk + pl * LD] = x11; Dn[qk + pl * LD] = x21; Dn[pk + ql * LD] = x12; Dn[qk + ql * LD] = x22;
                        Dn[pl + pk * LD] = x11; Dn[pl + qk * LD] = x21; Dn[ql + pk * LD] = x12; Dn[ql + qk * LD] = x22;
                    }
                } else {
                    const int pk = UREG ? xp(tk, s) : P.p[tk], qk = UREG ? xq(tk, s) : P.q[tk];
                    const R apq = Dc[didx<R, UREG>(pk, qk)], t = P.t[tk];
                    Dn[pk + pk * LD] = fmaR(-t, apq, Dc[pk + pk * LD]);
                    Dn[qk + qk * LD] = fmaR(t, apq, Dc[qk + qk * LD]);
                    Dn[didx<R, UREG>(pk, qk)] = R(0);
                    if (!UREG) Dn[qk + pk * LD] = R(0);
                }
            }
            if (UREG) {
                const R sk = P.s[lane];
                if (sk != R(0)) {
                    const R tk = P.u[lane];
                    #pragma unroll
                    for (int j = 0; j < 3; ++j)
                        if (j < nrow) {
                            if (!flip) rot<R>(sk, tk, ua[j], ub[j]);
                            else rot<R>(sk, tk, ub[j], ua[j]);
                        }
                }
                #pragma unroll
                for (int j = 0; j < 3; ++j) ub[j] = __shfl_sync(0xffffffffu, ub[j], (lane + 1) & 31);
            } else if (U) {
                #pragma unroll
                for (int j = 0; j < 3; ++j) {
                    if (uk[j] < 0) continue;
                    const R sk = P.s[uk[j]];
                    if (sk != R(0)) {
                        const int pk = P.p[uk[j]], qk = P.q[uk[j]];
                        R x = U[ur[j] + pk * LD], y = U[ur[j] + qk * LD];
                        rot<R>(sk, P.u[uk[j]], x, y);
                        U[ur[j] + pk * LD] = x; U[ur[j] + qk * LD] = y;
                    }
                }
            }
            MPJ_K3_TRACE(1, s);
        }
        __syncthreads();
        MPJ_K3_TRACE(2, s);
        R *tmp = Dc; Dc = Dn; Dn = tmp;
    }
    if (UREG) {                             // lower triangle of D from the upper one
        for (int e = tid; e < TW * TW; e += NTW) {
            const int i = e & (TW - 1), j = e >> 6;
            if (i > j) Dc[i + j * LD] = Dc[j + i * LD];
        }
    }
    if (UREG) {                             // back to shared memory (the shuffle after the last round is undone)
        #pragma unroll
        for (int j = 0; j < 3; ++j) {
            const R v = __shfl_sync(0xffffffffu, ub[j], (lane + 31) & 31);
            if (j < nrow) {
                U[urow[j] + lane * LD] = ua[j];
                U[urow[j] + (BW + ((lane + nrounds - 1) & 31)) * LD] = v;
            }
        }
        __syncthreads();
    }
    return Dc;
}

// ---------------------------------------------------------------------------
// One full sweep of the rounds of the single block pair bp = (0, 1) with NT =
// 256 threads, pipelined as smem_rounds_wide: warp 7 computes round s+1's
// parameters from D before round s (the after-round formulas diag_after /
// tile_after, the very arithmetic of the update) while warps 0-6 apply round s
// out of place (Dc -> Dn).  One barrier per round instead of two, and the
// parameter latency (divides, square roots) off the critical path.  U in
// registers exactly as inner_rounds_b (warp w: rows w + 8 i).  D0, D1 and U in
// LayK layout (LD 65); U may alias D1 (it is read into registers first and
// written back to the buffer that does not hold the final D).  Results are
// bit-identical to inner_rounds_b.  Returns the buffer holding the final D
// (*uout: the one holding U).
struct PipeMaps {      // bytes: three CTAs of the batched kernel share an SM's shared memory
    unsigned char part_t[2][BW], part_b[2][BW], pair_t[2][BW], pair_b[2][BW], isp_t[2][BW], isp_b[2][BW];
};

template <typename R>
__device__ __forceinline__ R *inner_rounds_pipe(R *D0, R *D1, const int2 *__restrict__ lsched, R nu, int rule,
                                                WideParams<R> (&PP)[2], PipeMaps &pm, R **uout)
{
    constexpr int LD = LayK<R>::LD;
    constexpr int NU = NT - 32;                          // update threads (warps 0-6)
    constexpr int NI = BW + BW * (BW - 1) / 2;           // tile items: 32 diagonal + 496 pair tiles
    constexpr int NE = (NI + NU - 1) / NU;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const bool pwarp = w == NT / 32 - 1;
    R *U = D1;
    R ut[8], ub[8];
    #pragma unroll
    for (int i = 0; i < 8; ++i) {
        ut[i] = U[(w + 8 * i) + lane * LD];
        ub[i] = U[(w + 8 * i) + (BW + lane) * LD];
    }
    int tk[NE], tl[NE];
    #pragma unroll
    for (int u = 0; u < NE; ++u) {
        const int wt = tid + NU * u - BW;
        int ll = -1, kk = 0;
        if (wt >= 0 && wt < BW * (BW - 1) / 2) {
            ll = (int)((1.0f + sqrtf(1.0f + 8.0f * wt)) * 0.5f);
            while (ll * (ll - 1) / 2 > wt) --ll;
            while ((ll + 1) * ll / 2 <= wt) ++ll;
            kk = wt - ll * (ll - 1) / 2;
        }
        tk[u] = kk; tl[u] = ll;
    }
    // parameters (and the intra-round partner maps) of round s into buffer b;
    // s = 0 from D itself, later from Dc after round s-1 (params P)
    auto params = [&](int s, int b, const R *Dc, const WideParams<R> *P) {
        const bool in_intra = s < BW - 1;
        int a, c;
        round_pair(s, lane, true, lsched, a, c);
        const int pn = a < c ? a : c, qn = a < c ? c : a;   // bp = (0, 1): local order == global order
        R app, aqq, apq;
        if (!P) {
            app = Dc[pn + pn * LD]; aqq = Dc[qn + qn * LD]; apq = Dc[didx<R, true>(pn, qn)];
        } else {
            app = diag_after<R, true>(Dc, *P, pn);
            aqq = diag_after<R, true>(Dc, *P, qn);
            const int k = P->pos[pn], l = P->pos[qn];
            R x11, x21, x12, x22;
            if (k < l) {
                tile_after<R, true>(Dc, *P, k, l, x11, x21, x12, x22);
                apq = (pn == P->p[k]) ? (qn == P->p[l] ? x11 : x12) : (qn == P->p[l] ? x21 : x22);
            } else {
                tile_after<R, true>(Dc, *P, l, k, x11, x21, x12, x22);
                apq = (qn == P->p[l]) ? (pn == P->p[k] ? x11 : x12) : (pn == P->p[k] ? x21 : x22);
            }
        }
        R t, sk, uk;
        rot_params<R>(app, aqq, apq, nu, rule, t, sk, uk);
        WideParams<R> &N = PP[b];
        N.t[lane] = t; N.s[lane] = sk; N.u[lane] = uk;
        N.p[lane] = pn; N.q[lane] = qn; N.gp[lane] = pn;
        N.pos[pn] = lane; N.pos[qn] = lane;
        if (in_intra) {
            if (lane < BW / 2) {
                pm.part_t[b][pn] = qn; pm.part_t[b][qn] = pn; pm.pair_t[b][pn] = lane; pm.pair_t[b][qn] = lane;
                pm.isp_t[b][pn] = 1; pm.isp_t[b][qn] = 0;
            } else {
                pm.part_b[b][pn - BW] = qn - BW; pm.part_b[b][qn - BW] = pn - BW;
                pm.pair_b[b][pn - BW] = lane; pm.pair_b[b][qn - BW] = lane;
                pm.isp_b[b][pn - BW] = 1; pm.isp_b[b][qn - BW] = 0;
            }
        }
    };
    __syncthreads();                                     // U in registers: D1 is free
    if (pwarp) params(0, 0, D0, nullptr);
    __syncthreads();
    constexpr int NR = (BW - 1) + BW;
    R *Dc = D0, *Dn = D1;
    for (int s = 0; s < NR; ++s) {
        const int b = s & 1;
        const WideParams<R> &P = PP[b];
        const bool in_intra = s < BW - 1;
        if (pwarp) {
            if (s + 1 < NR) params(s + 1, b ^ 1, Dc, &P);
        } else {
            #pragma unroll
            for (int u = 0; u < NE; ++u) {
                const int e = tid + NU * u;
                if (e >= NI) break;
                if (e < BW) {
                    const int pk = P.p[e], qk = P.q[e];
                    const R apq = Dc[didx<R, true>(pk, qk)], t = P.t[e];
                    Dn[pk + pk * LD] = fmaR(-t, apq, Dc[pk + pk * LD]);
                    Dn[qk + qk * LD] = fmaR(t, apq, Dc[qk + qk * LD]);
                    Dn[didx<R, true>(pk, qk)] = R(0);
                } else {
                    // upper triangle only during the sweep (mirrored once at its end):
                    // half the stores of the full-storage update, the same values
                    R x11, x21, x12, x22;
                    tile_after<R, true>(Dc, P, tk[u], tl[u], x11, x21, x12, x22);
                    const int pk = P.p[tk[u]], qk = P.q[tk[u]], pl = P.p[tl[u]], ql = P.q[tl[u]];
                    Dn[didx<R, true>(pk, pl)] = x11; Dn[didx<R, true>(qk, pl)] = x21;
                    Dn[didx<R, true>(pk, ql)] = x12; Dn[didx<R, true>(qk, ql)] = x22;
                }
            }
        }
        // U <- U J in registers (every warp: its rows)
        if (in_intra) {
            const int pt = pm.part_t[b][lane], pb = pm.part_b[b][lane];
            const int jt = pm.pair_t[b][lane], jb = pm.pair_b[b][lane];
            const bool it = pm.isp_t[b][lane] != 0, ib = pm.isp_b[b][lane] != 0;
            const R st = P.s[jt], tt = P.u[jt], sb = P.s[jb], tb = P.u[jb];
            #pragma unroll
            for (int i = 0; i < 8; ++i) {
                const R ot = __shfl_sync(0xffffffffu, ut[i], pt), ob = __shfl_sync(0xffffffffu, ub[i], pb);
                if (st != R(0)) rot_side<R>(st, tt, it, ut[i], ot);
                if (sb != R(0)) rot_side<R>(sb, tb, ib, ub[i], ob);
            }
        } else {
            const R sk = P.s[lane], tk2 = P.u[lane];
            #pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (sk != R(0)) rot<R>(sk, tk2, ut[i], ub[i]);   // p = a_k (top), q = b_k
                ub[i] = __shfl_sync(0xffffffffu, ub[i], (lane + 1) & 31);
            }
        }
        __syncthreads();
        R *tmp = Dc; Dc = Dn; Dn = tmp;
    }
    // U back into the buffer that does not hold D; D's lower triangle from its upper one
    #pragma unroll
    for (int i = 0; i < 8; ++i) {
        Dn[(w + 8 * i) + lane * LD] = ut[i];
        Dn[(w + 8 * i) + (BW + lane) * LD] = ub[i];
    }
    for (int e = tid; e < TW * TW; e += NT) {
        const int i = e & (TW - 1), j = e >> 6;
        if (i > j) Dc[i + j * LD] = Dc[j + i * LD];
    }
    __syncthreads();
    *uout = Dn;
    return Dc;
}

// K3's inner rounds: the intra-block rounds of block round 0 in shared memory
// (their pairs follow the local schedule), then the cross rounds with U in
// registers.
template <typename R, bool FASTP = false>
__device__ __forceinline__ R *inner_rounds_wide(R *D0, R *D1, R *U, int2 bp, bool intra,
                                                const int2 *__restrict__ lsched, R nu, int rule,
                                                WideParams<R> (&PP)[2], unsigned *nrot, int max_inner = 0)
{
    R *Dc = D0, *X = D1;
    if (threadIdx.x == 0) *nrot = 0;
    // max_inner > 0: classic block Jacobi (reading R26) -- full inner sweeps
    // (intra + cross rounds: every pair of the 2b indices) until one rotates
    // no pair; else one pass (intra rounds in block round 0, then cross rounds)
    const int nsweep = max_inner > 0 ? max_inner : 1;
    __shared__ unsigned sweep_rot;
    for (int it = 0; it < nsweep; ++it) {
        unsigned cnt = 0;
        if (intra || max_inner > 0) {
            Dc = smem_rounds_wide<R, false, FASTP>(Dc, X, U, bp, true, BW - 1, lsched, nu, rule, PP, cnt);
            X = (Dc == D0) ? D1 : D0;
        }
        Dc = smem_rounds_wide<R, true, FASTP>(Dc, X, U, bp, false, BW, lsched, nu, rule, PP, cnt);
        X = (Dc == D0) ? D1 : D0;
        // rotation count: per-thread counts of the diagonal threads and the parameter warp
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (threadIdx.x == 0) sweep_rot = 0;
        __syncthreads();
        if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&sweep_rot, cnt);
        __syncthreads();
        const unsigned sr = sweep_rot;
        if (threadIdx.x == 0) *nrot += sr;
        __syncthreads();
        if (sr == 0) break;
    }
    return Dc;
}

// ---------------------------------------------------------------------------
// 64 x 64 x 64 tile products in shared memory.
//   C = op(A) * B  with A, B column-major (leading dimension Lay<R>::LD);
//   TRANS_A: op(A) = A^T.  Results stay in registers (Acc<R>).
// fp64: 8 warps in a 4 x 2 grid, warp tile 16 x 32 = 2 x 4 fragments of
//   mma.sync m8n8k4 (DMMA): per k-step 2 A + 4 B fragment loads feed 8 DMMA;
//   every fragment load is 2 shared-memory wavefronts (the minimum for 32
//   8-byte lanes) with LD = 68.
// fp32: thread (tx, ty) owns rows tx + 16u, columns ty + 16v (4 x 4): A loads
//   are consecutive words, B loads are warp broadcasts -> conflict-free.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <typename R> struct Acc;
template <> struct Acc<double> {
    double v[2][4][2];
    __device__ __forceinline__ void zero()
    {
        #pragma unroll
        for (int a = 0; a < 2; ++a)
            #pragma unroll
            for (int b = 0; b < 4; ++b) { v[a][b][0] = 0.0; v[a][b][1] = 0.0; }
    }
    template <typename F> __device__ __forceinline__ void each(F f) const
    {
        const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31;
        const int r0 = (warp >> 1) * 16 + (lane >> 2), c0 = (warp & 1) * 32 + 2 * (lane & 3);
        #pragma unroll
        for (int mi = 0; mi < 2; ++mi)
            #pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                f(r0 + mi * 8, c0 + ni * 8, v[mi][ni][0]);
                f(r0 + mi * 8, c0 + ni * 8 + 1, v[mi][ni][1]);
            }
    }
    // as each, the entry by reference
    template <typename F> __device__ __forceinline__ void each_ref(F f)
    {
        const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31;
        const int r0 = (warp >> 1) * 16 + (lane >> 2), c0 = (warp & 1) * 32 + 2 * (lane & 3);
        #pragma unroll
        for (int mi = 0; mi < 2; ++mi)
            #pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                f(r0 + mi * 8, c0 + ni * 8, v[mi][ni][0]);
                f(r0 + mi * 8, c0 + ni * 8 + 1, v[mi][ni][1]);
            }
    }
    // (i, j) pairs with j, j+1 adjacent: f2(i, j, v_j, v_j+1)
    template <typename F> __device__ __forceinline__ void each2(F f) const
    {
        const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31;
        const int r0 = (warp >> 1) * 16 + (lane >> 2), c0 = (warp & 1) * 32 + 2 * (lane & 3);
        #pragma unroll
        for (int mi = 0; mi < 2; ++mi)
            #pragma unroll
            for (int ni = 0; ni < 4; ++ni) f(r0 + mi * 8, c0 + ni * 8, v[mi][ni][0], v[mi][ni][1]);
    }
};
template <> struct Acc<float> {
    float v[4][4];
    __device__ __forceinline__ void zero()
    {
        #pragma unroll
        for (int u = 0; u < 4; ++u)
            #pragma unroll
            for (int w = 0; w < 4; ++w) v[u][w] = 0.f;
    }
    template <typename F> __device__ __forceinline__ void each(F f) const
    {
        const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
        #pragma unroll
        for (int u = 0; u < 4; ++u)
            #pragma unroll
            for (int w = 0; w < 4; ++w) f(tx + 16 * u, ty + 16 * w, v[u][w]);
    }
};

template <bool TRANS_A>
__device__ __forceinline__ void tile_mm_acc(const double *A, const double *B, Acc<double> &acc)
{
    constexpr int LD = Lay<double>::LD;
    const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
    const int rb = (warp >> 1) * 16 + g, cb = (warp & 1) * 32 + g;
    #pragma unroll 4
    for (int ks = 0; ks < TW / 4; ++ks) {
        const int kk = ks * 4 + tig;
        double a[2], b[4];
        #pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
            const int row = rb + mi * 8;
            a[mi] = TRANS_A ? A[kk + row * LD] : A[row + kk * LD];
        }
        #pragma unroll
        for (int ni = 0; ni < 4; ++ni) b[ni] = B[kk + (cb + ni * 8) * LD];
        #pragma unroll
        for (int mi = 0; mi < 2; ++mi)
            #pragma unroll
            for (int ni = 0; ni < 4; ++ni) dmma884(acc.v[mi][ni][0], acc.v[mi][ni][1], a[mi], b[ni]);
    }
}

// C1 = A1 B, C2 = A2 B (fp64, A column-major): the same warp tile of two
// row tiles, every B fragment feeding both (16 DMMA per 8 fragment loads)
__device__ __forceinline__ void tile_mm2(const double *A1, const double *A2, const double *B, Acc<double> &c1,
                                         Acc<double> &c2)
{
    constexpr int LD = Lay<double>::LD;
    const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
    const int rb = (warp >> 1) * 16 + g, cb = (warp & 1) * 32 + g;
    c1.zero();
    c2.zero();
    #pragma unroll 2
    for (int ks = 0; ks < TW / 4; ++ks) {
        const int kk = ks * 4 + tig;
        double a1[2], a2[2], b[4];
        #pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
            a1[mi] = A1[rb + mi * 8 + kk * LD];
            a2[mi] = A2[rb + mi * 8 + kk * LD];
        }
        #pragma unroll
        for (int ni = 0; ni < 4; ++ni) b[ni] = B[kk + (cb + ni * 8) * LD];
        #pragma unroll
        for (int mi = 0; mi < 2; ++mi)
            #pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                dmma884(c1.v[mi][ni][0], c1.v[mi][ni][1], a1[mi], b[ni]);
                dmma884(c2.v[mi][ni][0], c2.v[mi][ni][1], a2[mi], b[ni]);
            }
    }
}

// k-chunked fp64 products: before the 4 k-steps of chunk c (k = 16c .. 16c+15)
// wait(c) runs (a cp.async group wait + barrier), so the product starts as soon
// as the first chunk of its operands has landed
template <bool TRANS_A, typename W>
__device__ __forceinline__ void tile_mm_chunked(const double *A, const double *B, Acc<double> &acc, W wait)
{
    constexpr int LD = Lay<double>::LD;
    const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
    const int rb = (warp >> 1) * 16 + g, cb = (warp & 1) * 32 + g;
    acc.zero();
    #pragma unroll 1
    for (int ch = 0; ch < 4; ++ch) {
        wait(ch);
        #pragma unroll
        for (int ks = 4 * ch; ks < 4 * ch + 4; ++ks) {
            const int kk = ks * 4 + tig;
            double a[2], b[4];
            #pragma unroll
            for (int mi = 0; mi < 2; ++mi) {
                const int row = rb + mi * 8;
                a[mi] = TRANS_A ? A[kk + row * LD] : A[row + kk * LD];
            }
            #pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[ni] = B[kk + (cb + ni * 8) * LD];
            #pragma unroll
            for (int mi = 0; mi < 2; ++mi)
                #pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma884(acc.v[mi][ni][0], acc.v[mi][ni][1], a[mi], b[ni]);
        }
    }
}

template <typename W>
__device__ __forceinline__ void tile_mm2_chunked(const double *A1, const double *A2, const double *B,
                                                 Acc<double> &c1, Acc<double> &c2, W wait)
{
    constexpr int LD = Lay<double>::LD;
    const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31, g = lane >> 2, tig = lane & 3;
    const int rb = (warp >> 1) * 16 + g, cb = (warp & 1) * 32 + g;
    c1.zero();
    c2.zero();
    #pragma unroll 1
    for (int ch = 0; ch < 4; ++ch) {
        wait(ch);
        #pragma unroll 2
        for (int ks = 4 * ch; ks < 4 * ch + 4; ++ks) {
            const int kk = ks * 4 + tig;
            double a1[2], a2[2], b[4];
            #pragma unroll
            for (int mi = 0; mi < 2; ++mi) {
                a1[mi] = A1[rb + mi * 8 + kk * LD];
                a2[mi] = A2[rb + mi * 8 + kk * LD];
            }
            #pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[ni] = B[kk + (cb + ni * 8) * LD];
            #pragma unroll
            for (int mi = 0; mi < 2; ++mi)
                #pragma unroll
                for (int ni = 0; ni < 4; ++ni) {
                    dmma884(c1.v[mi][ni][0], c1.v[mi][ni][1], a1[mi], b[ni]);
                    dmma884(c2.v[mi][ni][0], c2.v[mi][ni][1], a2[mi], b[ni]);
                }
        }
    }
}

template <bool TRANS_A>
__device__ __forceinline__ void tile_mm_acc(const float *A, const float *B, Acc<float> &acc)
{
    constexpr int LD = Lay<float>::LD;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    #pragma unroll 4
    for (int kk = 0; kk < TW; ++kk) {
        float a[4], b[4];
        #pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = tx + 16 * u;
            a[u] = TRANS_A ? A[kk + i * LD] : A[i + kk * LD];
        }
        #pragma unroll
        for (int w = 0; w < 4; ++w) b[w] = B[kk + (ty + 16 * w) * LD];
        // scalar FMAs: the operands come from scalar strided loads, pairing them
        // for FFMA2 costs register moves (measured slower in the SVD Gram)
        #pragma unroll
        for (int u = 0; u < 4; ++u)
            #pragma unroll
            for (int w = 0; w < 4; ++w) acc.v[u][w] = __fmaf_rn(a[u], b[w], acc.v[u][w]);
    }
}

// fp32 outer-product form for operands stored "k-major": C[i, j] = sum_k
// A[i + k LD] B[j + k LD].  Thread (tx, ty) = (tid & 15, tid >> 4) owns rows
// 4tx..4tx+3 and columns 4ty..4ty+3: one 128-bit LDS for each operand per k
// (A: 16 distinct contiguous vectors per warp, B: a broadcast) feeds 16 FFMA.
struct AccOP {
    float v[4][4];
    __device__ __forceinline__ int r0() const { return 4 * (threadIdx.x & 15); }
    __device__ __forceinline__ int c0() const { return 4 * (threadIdx.x >> 4); }
};
__device__ __forceinline__ void tile_op(const float *A, const float *B, AccOP &acc)
{
    constexpr int LD = 68;
    const int ra = 4 * (threadIdx.x & 15), cb = 4 * (threadIdx.x >> 4);
    #pragma unroll
    for (int u = 0; u < 4; ++u)
        #pragma unroll
        for (int w = 0; w < 4; ++w) acc.v[u][w] = 0.f;
    float4 a = *(const float4 *)(A + ra), b = *(const float4 *)(B + cb);
    #pragma unroll 8
    for (int k = 0; k < TW; ++k) {
        const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
        if (k + 1 < TW) {                         // register prefetch of the next k
            a = *(const float4 *)(A + ra + (k + 1) * LD);
            b = *(const float4 *)(B + cb + (k + 1) * LD);
        }
        #pragma unroll
        for (int u = 0; u < 4; ++u)
            #pragma unroll
            for (int w = 0; w < 4; w += 2) ffma2(av[u], bv[w], bv[w + 1], acc.v[u][w], acc.v[u][w + 1]);
    }
}
// C (column-major) and C^T (column-major) stores of an AccOP, 128-bit each
__device__ __forceinline__ void store_op(const AccOP &acc, float *C, float *CT)
{
    constexpr int LD = 68;
    const int r = acc.r0(), c = acc.c0();
    #pragma unroll
    for (int w = 0; w < 4; ++w)
        *(float4 *)(C + r + (c + w) * LD) = make_float4(acc.v[0][w], acc.v[1][w], acc.v[2][w], acc.v[3][w]);
    if (CT) {
        #pragma unroll
        for (int u = 0; u < 4; ++u)
            *(float4 *)(CT + c + (r + u) * LD) = make_float4(acc.v[u][0], acc.v[u][1], acc.v[u][2], acc.v[u][3]);
    }
}

// fp32 8 x 4 register tiles (128 threads per 64 x 64 tile): thread tid =
// (tx, ty) = (tid % 8, tid / 8) owns rows 4tx..4tx+3, 32+4tx..32+4tx+3 and
// columns 4ty..4ty+3; C = A B^T-style k-major product (A[i + k LD], B[j + k LD]).
struct Acc84 {
    float v[8][4];
};

__device__ __forceinline__ void tile_op84_t(const float *A, const float *B, Acc84 &acc, int tid)
{
    constexpr int LD = Lay<float>::LD;
    const int ra = 4 * (tid & 7), cb = 4 * (tid >> 3);
    #pragma unroll
    for (int u = 0; u < 8; ++u)
        #pragma unroll
        for (int w = 0; w < 4; ++w) acc.v[u][w] = 0.f;
    float4 a0 = *(const float4 *)(A + ra), a1 = *(const float4 *)(A + ra + 32), b = *(const float4 *)(B + cb);
    #pragma unroll 4
    for (int k = 0; k < TW; ++k) {
        const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w}, bv[4] = {b.x, b.y, b.z, b.w};
        if (k + 1 < TW) {                         // register prefetch of the next k
            a0 = *(const float4 *)(A + ra + (k + 1) * LD);
            a1 = *(const float4 *)(A + ra + 32 + (k + 1) * LD);
            b = *(const float4 *)(B + cb + (k + 1) * LD);
        }
        #pragma unroll
        for (int u = 0; u < 8; ++u)
            #pragma unroll
            for (int w = 0; w < 4; w += 2) ffma2(av[u], bv[w], bv[w + 1], acc.v[u][w], acc.v[u][w + 1]);
    }
}

__device__ __forceinline__ void store_op84_t(const Acc84 &acc, float *C, float *CT, int tid)
{
    constexpr int LD = Lay<float>::LD;
    const int r = 4 * (tid & 7), c = 4 * (tid >> 3);
    #pragma unroll
    for (int w = 0; w < 4; ++w) {
        *(float4 *)(C + r + (c + w) * LD) = make_float4(acc.v[0][w], acc.v[1][w], acc.v[2][w], acc.v[3][w]);
        *(float4 *)(C + r + 32 + (c + w) * LD) = make_float4(acc.v[4][w], acc.v[5][w], acc.v[6][w], acc.v[7][w]);
    }
    if (CT) {
        #pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int row = r + (u & 3) + (u >> 2) * 32;
            *(float4 *)(CT + c + row * LD) = make_float4(acc.v[u][0], acc.v[u][1], acc.v[u][2], acc.v[u][3]);
        }
    }
}

template <bool TRANS_A, typename R>
__device__ __forceinline__ void tile_mm(const R *A, const R *B, Acc<R> &acc)
{
    acc.zero();
    tile_mm_acc<TRANS_A>(A, B, acc);
}

}  // namespace blk
}  // namespace mpj
