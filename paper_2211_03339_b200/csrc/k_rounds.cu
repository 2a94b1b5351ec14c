// k_rounds.cu -- the scalar (one-round-at-a-time) Jacobi kernels.
//
// One round of the parallel ordering = n_p/2 disjoint rotations J_r
// (P:741).  Alg. 3 steps 7-8 for every pair of the round:
//   K1 (k_round_params): threshold test + Lemma 3.1 from T at the start of the
//      round -> (p, q, t, s, tau) per slot; counts applied rotations (JU).
//   K2 (k_round_apply):  T <- J_r^T T J_r on 2x2 tiles.  Tile (k, l) holds rows
//      {p_k, q_k} x columns {p_l, q_l}.  The canonical order (reading R7) is
//      "rotate rows by pair k, then columns by pair l" for the tile whose row
//      pair has the smaller p; the other tile of the symmetric couple is its
//      exact mirror.  Because T is exactly symmetric, each thread reads its own
//      tile, evaluates the canonical expression in (possibly transposed)
//      order and writes its own tile: no mirror writes, coalesced along k.
//      Diagonal tiles: t_pp - t a_pq, t_qq + t a_pq, pivot := 0.
//   K3 (k_round_apply_v): V <- V J_r, two columns per pair.
//   K2+K3 fused (k_round_apply_fused, the default): thread (row i, column
//      pair l) writes T'(i, {p_l, q_l}) (out of place: T' is the other buffer)
//      and V(i, {p_l, q_l}): a warp reads and writes 32 consecutive rows of
//      both columns of T and V (coalesced); the partner row of i (the other
//      index of i's pair k) is read from the same two columns (L1/L2 hits: the
//      columns stream through anyway).  The 2x2 tile (k, l) is evaluated by
//      both of its row threads with the canonical expression, each keeping its
//      own row: bit-identical to K2.
// Bytes per round (the HBM roofline of this variant): T and V are read and
// written once each: 4 * 8 * n_p^2 bytes (fp64).
#include "mpj_device.cuh"
#include "mpj_internal.h"

namespace mpj {

template <typename R>
__global__ void __launch_bounds__(256) k_round_params(const R *__restrict__ T, int64_t ldt, Sched S,
                                                      int r, R nu, int rule, int2 *__restrict__ pq,
                                                      R *__restrict__ tt, R *__restrict__ ss,
                                                      R *__restrict__ uu,
                                                      unsigned long long *__restrict__ cnt,
                                                      int *__restrict__ pos)
{
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL)
    const int h = S.np >> 1;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    int did = 0;
    if (k < h) {
        const int2 pr = pair_of(S, r, k);
        R t, s, u;
        did = rot_params<R>(T[pr.x + pr.x * ldt], T[pr.y + pr.y * ldt], T[pr.x + pr.y * ldt], nu,
                            rule, t, s, u);
        pq[k] = pr; tt[k] = t; ss[k] = s; uu[k] = u;
        if (pos) { pos[pr.x] = k; pos[pr.y] = k | (1 << 30); }   // row -> (slot, is q)
    }
    const int c = __syncthreads_count(did);
    if (threadIdx.x == 0 && c) atomicAdd(cnt, (unsigned long long)c);
}

template <typename R>
__global__ void __launch_bounds__(256) k_round_apply(R *__restrict__ T, int64_t ldt,
                                                     const int2 *__restrict__ pq,
                                                     const R *__restrict__ tt,
                                                     const R *__restrict__ ss,
                                                     const R *__restrict__ uu, int h)
{
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL)
    const int k = blockIdx.x * 32 + threadIdx.x;   // row pair (fast index -> coalesced)
    const int l = blockIdx.y * 8 + threadIdx.y;    // column pair
    if (k >= h || l >= h) return;
    const int2 a = pq[k];
    if (k == l) {
        const int p = a.x, q = a.y;
        const R apq = T[p + q * ldt], t = tt[k];
        T[p + p * ldt] = fmaR(-t, apq, T[p + p * ldt]);
        T[q + q * ldt] = fmaR(t, apq, T[q + q * ldt]);
        T[p + q * ldt] = R(0);
        T[q + p * ldt] = R(0);
        return;
    }
    const int2 c = pq[l];
    R *c0 = T + (int64_t)c.x * ldt, *c1 = T + (int64_t)c.y * ldt;
    R x11 = c0[a.x], x21 = c0[a.y], x12 = c1[a.x], x22 = c1[a.y];
    const R sk = ss[k], uk = uu[k], sl = ss[l], ul = uu[l];
    if (a.x < c.x) {          // canonical tile: rows by k, then columns by l
        rot<R>(sk, uk, x11, x21); rot<R>(sk, uk, x12, x22);
        rot<R>(sl, ul, x11, x12); rot<R>(sl, ul, x21, x22);
    } else {                  // mirror of the canonical tile (l, k)
        rot<R>(sl, ul, x11, x12); rot<R>(sl, ul, x21, x22);
        rot<R>(sk, uk, x11, x21); rot<R>(sk, uk, x12, x22);
    }
    c0[a.x] = x11; c0[a.y] = x21; c1[a.x] = x12; c1[a.y] = x22;
}

template <typename R>
__global__ void __launch_bounds__(256) k_round_apply_v(R *__restrict__ V, int64_t ldv, int vrows,
                                                       const int2 *__restrict__ pq,
                                                       const R *__restrict__ ss,
                                                       const R *__restrict__ uu)
{
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL)
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (i >= vrows) return;
    const int2 a = pq[k];
    const R s = ss[k];
    if (s == R(0)) return;   // skipped pair: identity (the tau-form is exact then)
    R *vp = V + (int64_t)a.x * ldv, *vq = V + (int64_t)a.y * ldv;
    R x = vp[i], y = vq[i];
    rot<R>(s, uu[k], x, y);
    vp[i] = x; vq[i] = y;
}

template <typename R>
__global__ void __launch_bounds__(256) k_round_apply_fused(const R *__restrict__ T, R *__restrict__ Tout,
                                                           int64_t ldt, R *__restrict__ V,
                                                           int64_t ldv, int vrows, int np,
                                                           const int2 *__restrict__ pq, const int *__restrict__ pos,
                                                           const R *__restrict__ tt, const R *__restrict__ ss,
                                                           const R *__restrict__ uu)
{
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // launched early (PDL)
    const int i = blockIdx.x * blockDim.x + threadIdx.x;   // row
    const int l = blockIdx.y;                              // column pair
    const int2 c = pq[l];
    const R sl = ss[l], ul = uu[l];
    // V <- V J_r on columns (p_l, q_l) (right rotation only)
    if (i < vrows && sl != R(0)) {
        R *vp = V + (int64_t)c.x * ldv, *vq = V + (int64_t)c.y * ldv;
        R x = vp[i], y = vq[i];
        rot<R>(sl, ul, x, y);
        vp[i] = x; vq[i] = y;
    }
    if (i >= np) return;
    const int ps = pos[i], k = ps & ((1 << 30) - 1);
    const bool isq = ps >> 30;
    const int2 a = pq[k];
    const R *c0 = T + (int64_t)c.x * ldt, *c1 = T + (int64_t)c.y * ldt;
    R *o0 = Tout + (int64_t)c.x * ldt, *o1 = Tout + (int64_t)c.y * ldt;
    if (k == l) {                      // diagonal tile: P:102, P:195 (pivot := 0)
        const R apq = c1[a.x], t = tt[k];
        if (!isq) { o0[a.x] = fmaR(-t, apq, c0[a.x]); o1[a.x] = R(0); }
        else { o1[a.y] = fmaR(t, apq, c1[a.y]); o0[a.y] = R(0); }
        return;
    }
    R x11 = c0[a.x], x21 = c0[a.y], x12 = c1[a.x], x22 = c1[a.y];
    const R sk = ss[k], uk = uu[k];
    if (a.x < c.x) {          // canonical tile: rows by k, then columns by l
        rot<R>(sk, uk, x11, x21); rot<R>(sk, uk, x12, x22);
        rot<R>(sl, ul, x11, x12); rot<R>(sl, ul, x21, x22);
    } else {                  // mirror of the canonical tile (l, k)
        rot<R>(sl, ul, x11, x12); rot<R>(sl, ul, x21, x22);
        rot<R>(sk, uk, x11, x21); rot<R>(sk, uk, x12, x22);
    }
    if (!isq) { o0[a.x] = x11; o1[a.x] = x12; }
    else { o0[a.y] = x21; o1[a.y] = x22; }
}

static inline Sched to_sched(const DevSched &d)
{
    Sched s;
    s.bsched = d.bsched; s.lsched = d.lsched; s.b = d.b; s.nb = d.nb; s.np = d.np;
    return s;
}

template <typename R>
void launch_round_params(const R *T, int64_t ldt, const DevSched &S, int r, R nu, int rule,
                         int2 *pq, R *t, R *s, R *u, unsigned long long *cnt, cudaStream_t st, int *pos)
{
    const int h = S.np / 2;
    launch_pdl_k(k_round_params<R>, dim3((h + 255) / 256), dim3(256), 0, st, T, ldt, to_sched(S), r, nu, rule, pq, t, s, u,
                 cnt, pos);
    count_launch();
}

template <typename R>
void launch_round_apply_fused_oop(const R *T, R *Tout, int64_t ldt, R *V, int64_t ldv, int vrows, int np,
                                  const int2 *pq, const int *pos, const R *t, const R *s, const R *u, cudaStream_t st)
{
    const int rows = vrows > np ? vrows : np;
    dim3 grd((rows + 255) / 256, np / 2);
    launch_pdl_k(k_round_apply_fused<R>, grd, dim3(256), 0, st, T, Tout, ldt, V, ldv, vrows, np, pq, pos, t, s, u);
    count_launch();
}

template <typename R>
void launch_round_apply(R *T, int64_t ldt, const int2 *pq, const R *t, const R *s, const R *u,
                        int h, cudaStream_t st)
{
    dim3 blk(32, 8), grd((h + 31) / 32, (h + 7) / 8);
    launch_pdl_k(k_round_apply<R>, grd, blk, 0, st, T, ldt, pq, t, s, u, h);
    count_launch();
}

template <typename R>
void launch_round_apply_v(R *V, int64_t ldv, int vrows, const int2 *pq, const R *s, const R *u,
                          int h, cudaStream_t st)
{
    dim3 grd((vrows + 255) / 256, h);
    launch_pdl_k(k_round_apply_v<R>, grd, dim3(256), 0, st, V, ldv, vrows, pq, s, u);
    count_launch();
}

#define INST(R)                                                                                  \
    template void launch_round_params<R>(const R *, int64_t, const DevSched &, int, R, int, int2 *, \
                                         R *, R *, R *, unsigned long long *, cudaStream_t, int *); \
    template void launch_round_apply_fused_oop<R>(const R *, R *, int64_t, R *, int64_t, int, int,  \
                                                  const int2 *, const int *, const R *, const R *,  \
                                                  const R *, cudaStream_t);                        \
    template void launch_round_apply<R>(R *, int64_t, const int2 *, const R *, const R *,         \
                                        const R *, int, cudaStream_t);                           \
    template void launch_round_apply_v<R>(R *, int64_t, int, const int2 *, const R *, const R *,  \
                                          int, cudaStream_t);
INST(double)
INST(float)
#undef INST

}  // namespace mpj
