/*
 * mpj_oracle.c -- plain, slow CPU oracle for the mixed-precision Jacobi method
 * of Zhang & Bai, arXiv 2211.03339 ("A mixed precision Jacobi method for the
 * symmetric eigenvalue problem").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this file.  It
 * shares no code, header, table or constant generator with the CUDA path in
 * paper_2211_03339_b200/csrc/, and it never imports or links it.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n (the LaTeX source).
 * Readings of the paper where it is silent or ambiguous are numbered R1..Rn
 * and listed in DESIGN.md section "Readings of the paper".
 *
 * Conventions: all matrices column-major, leading dimension = rows, indices
 * 0-based (the paper is 1-based).  Rotation arithmetic is IEEE binary64 (or
 * binary32 for the low-precision stage) with the explicit fma() calls written
 * below and NO other contraction (build with -ffp-contract=off).  Sums that
 * are reductions (dot products, norms, matrix products) are accumulated in
 * long double and rounded once, as BASELINE.json's north_star asks
 * ("long-double accumulation").
 *
 * Parity status of each exported function is stated in its comment; every
 * function here is pinned by a -m "not gpu" test in tests/test_oracle_*.py.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>

typedef long double ldbl;

#define IDX(i, j, ld) ((size_t)(i) + (size_t)(j) * (size_t)(ld))

/* ------------------------------------------------------------------------ */
/* Parallel ordering.                                                */
/*                                                                           */
/* The paper runs its GPU versions with "some non-overlapping order, e.g.,  */
/* the merry-go-round ordering (1,2),(3,4),...,(n-1,n),(1,4),...,(n-3,n-1), */
/* (1,6),...,(n,n-2)".  That is the Golub-Van Loan "music" round-    */
/* robin.  Reading R1: we use a one-parameter family of          */
/* round-robin orderings, "block merry-go-round with block size b":         */
/*   * n is padded to n_p = multiple of 2b with zero rows/columns (R2);      */
/*   * the nb = n_p/b blocks are paired by the merry-go-round on blocks,     */
/*     nb-1 block rounds;                                                    */
/*   * in block round 0, each block is first swept internally by b-1         */
/*     merry-go-round rounds on its own b indices;                          */
/*   * in every block round, block pair (I,J) then runs b "cross" rounds     */
/*     pairing I*b+i with J*b+((i+s) mod b), s = 0..b-1.                     */
/* Every round is a perfect matching of the n_p indices, there are n_p-1     */
/* rounds, and every pair (i,j), i<j, appears exactly once per sweep.  For   */
/* b = 1 this IS the paper's merry-go-round (tests/test_oracle_ordering.py   */
/* pins the prefix printed at P:741).                                        */
/* Within a pair, p = min, q = max (Lemma 3.1 is stated for i<j).      */
/* ------------------------------------------------------------------------ */

/* GVL music: top[0] fixed; new_top[1] = bot[0]; new_top[k] = top[k-1] (k>1);
 * new_bot[k] = bot[k+1] (k<m-1); new_bot[m-1] = top[m-1]. */
static void music(int *top, int *bot, int m)
{
    if (m < 2) return;
    int *nt = (int *)malloc(sizeof(int) * m), *nbt = (int *)malloc(sizeof(int) * m);
    for (int k = 0; k < m; ++k) {
        if (k == 0) nt[k] = top[0];
        else if (k == 1) nt[k] = bot[0];
        else nt[k] = top[k - 1];
        if (k == m - 1) nbt[k] = top[k];
        else nbt[k] = bot[k + 1];
    }
    memcpy(top, nt, sizeof(int) * m);
    memcpy(bot, nbt, sizeof(int) * m);
    free(nt); free(nbt);
}

int orc_padded_n(int n, int b)
{
    int w = 2 * b;
    return ((n + w - 1) / w) * w;
}

/* Write the whole schedule: round r, slot k -> (P[r*h+k], Q[r*h+k]),
 * h = n_p/2, r < n_p-1.  Returns n_p-1 (the number of rounds), or -1 if b is
 * not 1 and not even. */
int orc_schedule(int n, int b, int *P, int *Q)
{
    if (b < 1 || (b > 1 && (b & 1))) return -1;
    int np = orc_padded_n(n, b), nb = np / b, mb = nb / 2, h = np / 2;
    int *btop = (int *)malloc(sizeof(int) * mb), *bbot = (int *)malloc(sizeof(int) * mb);
    int *ltop = (int *)malloc(sizeof(int) * (b / 2 + 1)), *lbot = (int *)malloc(sizeof(int) * (b / 2 + 1));
    for (int k = 0; k < mb; ++k) { btop[k] = 2 * k; bbot[k] = 2 * k + 1; }
    int r = 0;
    for (int R = 0; R < nb - 1; ++R) {
        if (R == 0 && b > 1) {
            int lm = b / 2;
            for (int k = 0; k < lm; ++k) { ltop[k] = 2 * k; lbot[k] = 2 * k + 1; }
            for (int s = 0; s < b - 1; ++s) {
                int slot = 0;
                for (int k = 0; k < mb; ++k) {
                    int blk[2] = { btop[k], bbot[k] };
                    for (int e = 0; e < 2; ++e)
                        for (int j = 0; j < lm; ++j) {
                            int a = blk[e] * b + ltop[j], c = blk[e] * b + lbot[j];
                            P[(size_t)r * h + slot] = a < c ? a : c;
                            Q[(size_t)r * h + slot] = a < c ? c : a;
                            ++slot;
                        }
                }
                music(ltop, lbot, lm);
                ++r;
            }
        }
        for (int s = 0; s < b; ++s) {
            int slot = 0;
            for (int k = 0; k < mb; ++k)
                for (int i = 0; i < b; ++i) {
                    int a = btop[k] * b + i, c = bbot[k] * b + (i + s) % b;
                    P[(size_t)r * h + slot] = a < c ? a : c;
                    Q[(size_t)r * h + slot] = a < c ? c : a;
                    ++slot;
                }
            ++r;
        }
        music(btop, bbot, mb);
    }
    free(btop); free(bbot); free(ltop); free(lbot);
    return r;
}

/* ------------------------------------------------------------------------ */
/* Norms (P:39 notation; off(G) = G - diag(G)).                              */
/* Reading R9: off(T) is summed directly over i != j, never as               */
/* ||T||_F^2 - sum t_ii^2 (that form cancels).                               */
/* ------------------------------------------------------------------------ */
double orc_fro_f64(const double *A, int m, int n, int lda)
{
    ldbl s = 0;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < m; ++i) { ldbl x = A[IDX(i, j, lda)]; s += x * x; }
    return (double)sqrtl(s);
}

double orc_off_f64(const double *A, int n, int lda)
{
    ldbl s = 0;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i)
            if (i != j) { ldbl x = A[IDX(i, j, lda)]; s += x * x; }
    return (double)sqrtl(s);
}

double orc_fro_f32(const float *A, int m, int n, int lda)
{
    ldbl s = 0;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < m; ++i) { ldbl x = A[IDX(i, j, lda)]; s += x * x; }
    return (double)sqrtl(s);
}

double orc_off_f32(const float *A, int n, int lda)
{
    ldbl s = 0;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i)
            if (i != j) { ldbl x = A[IDX(i, j, lda)]; s += x * x; }
    return (double)sqrtl(s);
}

/* ------------------------------------------------------------------------ */
/* Lemma 3.1 and the threshold test of Alg. 2/3.   */
/* Instantiated for binary64 (ω = 2^-53) and binary32 (υ = 2^-24).     */
/*                                                                           */
/*   skip  iff |a_pq| <= nu * min(|a_pp|, |a_qq|)        (R5: the     */
/*         sqrt(a_pp a_qq) rule of Remark 3.1, is stop_rule = 1)      */
/*   mu = (a_qq - a_pp) / (2 a_pq)    */
/*   t  = 1/(mu + sqrt(1+mu^2)) if mu >= 0 else 1/(mu - sqrt(1+mu^2))        */
/*        (R3: 1+mu^2 formed as fma(mu,mu,1); R4: for |mu| >= MU_BIG the     */
/*         rotation uses t = 0.5/mu, the limit form, to avoid mu^2 overflow) */
/*   c  = (1+t^2)^(-1/2), s = t c   */
/*   tau = s/(1+c)   (Rutishauser form of the update, reading R6)            */
/*                                                                           */
/* Update of a pair of entries x (index p) and y (index q) by J:   */
/*   x' = c x - s y = x - s (y + tau x) = fma(-s, fma(tau, x, y), x)        */
/*   y' = s x + c y = y + s (x - tau y) = fma( s, fma(-tau, y, x), y)       */
/* ------------------------------------------------------------------------ */
#define DEFINE_PRECISION(SUF, REAL, FMA, SQRT, FABS, FMIN, MU_BIG)                     \
    static int rot_params_##SUF(REAL app, REAL aqq, REAL apq, REAL nu, int rule,       \
                                REAL *t_, REAL *s_, REAL *tau_)                        \
    {                                                                                  \
        int skip;                                                                      \
        if (rule == 1) {                                                               \
            REAL g = app * aqq;                                                        \
            skip = (g > (REAL)0) ? (FABS(apq) <= nu * SQRT(g)) : (apq == (REAL)0);      \
        } else {                                                                       \
            skip = FABS(apq) <= nu * FMIN(FABS(app), FABS(aqq));                       \
        }                                                                              \
        if (skip) { *t_ = 0; *s_ = 0; *tau_ = 0; return 0; }                           \
        REAL mu = (aqq - app) / ((REAL)2 * apq);                                       \
        REAL t;                                                                        \
        if (FABS(mu) < (REAL)(MU_BIG)) {                                               \
            REAL r = SQRT(FMA(mu, mu, (REAL)1));                                       \
            t = (mu >= (REAL)0) ? (REAL)1 / (mu + r) : (REAL)1 / (mu - r);              \
        } else {                                                                       \
            t = (REAL)0.5 / mu;                                                        \
        }                                                                              \
        REAL c = (REAL)1 / SQRT(FMA(t, t, (REAL)1));                                   \
        REAL s = t * c;                                                                \
        *t_ = t; *s_ = s; *tau_ = s / ((REAL)1 + c);                                   \
        return 1;                                                                      \
    }                                                                                  \
    static inline void rot_##SUF(REAL s, REAL tau, REAL *x, REAL *y)                   \
    {                                                                                  \
        REAL x0 = *x, y0 = *y;                                                         \
        *x = FMA(-s, FMA(tau, x0, y0), x0);                                            \
        *y = FMA(s, FMA(-tau, y0, x0), y0);                                            \
    }                                                                                  \
    /* One round of m disjoint pairs applied to padded T, V (n_p x n_p).            */ \
    /* All rotation parameters are taken from T at the start of the round (the      */ \
    /* pairs are disjoint, so this equals applying them one after another in exact   */ \
    /* arithmetic).  2x2 tile (rows of pair k, cols of pair l) with P[k] < P[l] is    */ \
    /* updated rows-then-columns and mirrored into (l,k) (reading R7); diagonal       */ \
    /* tiles use t_pp - t a_pq, t_qq + t a_pq and an exact zero pivot. */ \
    static long long round_##SUF(REAL *T, REAL *V, int np, int vrows, const int *P,    \
                                 const int *Q, int m, REAL nu, int rule,               \
                                 REAL *tt, REAL *ss, REAL *uu)                         \
    {                                                                                  \
        long long nrot = 0;                                                            \
        for (int k = 0; k < m; ++k) {                                                  \
            int p = P[k], q = Q[k];                                                    \
            nrot += rot_params_##SUF(T[IDX(p, p, np)], T[IDX(q, q, np)],               \
                                     T[IDX(p, q, np)], nu, rule, &tt[k], &ss[k], &uu[k]); \
        }                                                                              \
        _Pragma("omp parallel for schedule(dynamic, 4)")                               \
        for (int k = 0; k < m; ++k) {                                                  \
            int pk = P[k], qk = Q[k];                                                  \
            for (int l = 0; l < m; ++l) {                                              \
                int pl = P[l], ql = Q[l];                                              \
                if (!(pk < pl)) continue;                                              \
                REAL x11 = T[IDX(pk, pl, np)], x12 = T[IDX(pk, ql, np)];               \
                REAL x21 = T[IDX(qk, pl, np)], x22 = T[IDX(qk, ql, np)];               \
                rot_##SUF(ss[k], uu[k], &x11, &x21);                                   \
                rot_##SUF(ss[k], uu[k], &x12, &x22);                                   \
                rot_##SUF(ss[l], uu[l], &x11, &x12);                                   \
                rot_##SUF(ss[l], uu[l], &x21, &x22);                                   \
                T[IDX(pk, pl, np)] = x11; T[IDX(pk, ql, np)] = x12;                    \
                T[IDX(qk, pl, np)] = x21; T[IDX(qk, ql, np)] = x22;                    \
                T[IDX(pl, pk, np)] = x11; T[IDX(ql, pk, np)] = x12;                    \
                T[IDX(pl, qk, np)] = x21; T[IDX(ql, qk, np)] = x22;                    \
            }                                                                          \
        }                                                                              \
        for (int k = 0; k < m; ++k) {                                                  \
            int p = P[k], q = Q[k];                                                    \
            REAL apq = T[IDX(p, q, np)];                                               \
            T[IDX(p, p, np)] = FMA(-tt[k], apq, T[IDX(p, p, np)]);                      \
            T[IDX(q, q, np)] = FMA(tt[k], apq, T[IDX(q, q, np)]);                       \
            T[IDX(p, q, np)] = 0; T[IDX(q, p, np)] = 0;                                \
        }                                                                              \
        if (V) {                                                                       \
            _Pragma("omp parallel for schedule(static)")                               \
            for (int k = 0; k < m; ++k)                                                \
                for (int i = 0; i < vrows; ++i)                                        \
                    rot_##SUF(ss[k], uu[k], &V[IDX(i, P[k], vrows)], &V[IDX(i, Q[k], vrows)]); \
        }                                                                              \
        return nrot;                                                                   \
    }

DEFINE_PRECISION(f64, double, fma, sqrt, fabs, fmin, 67108864.0 /* 2^26 */)
DEFINE_PRECISION(f32, float, fmaf, sqrtf, fabsf, fminf, 4096.0f /* 2^12 */)

/* Exported single-rotation parameters (for the Lemma 3.1 pins). */
int orc_rotation_f64(double app, double aqq, double apq, double nu, int rule,
                     double *t, double *s, double *tau)
{
    return rot_params_f64(app, aqq, apq, nu, rule, t, s, tau);
}
int orc_rotation_f32(float app, float aqq, float apq, float nu, int rule,
                     float *t, float *s, float *tau)
{
    return rot_params_f32(app, aqq, apq, nu, rule, t, s, tau);
}

/* ------------------------------------------------------------------------ */
/* Alg. 2 / the loop of Alg. 3, steps 4-11, with the  */
/* parallel ordering above.  T and V are n x n (ld n), updated in place.     */
/* Stop test before every sweep (reading R8): ||off(T)||_F <= tol, where     */
/* the caller passes tol = eps * ||A||_F.  Returns 0 on convergence, */
/* 2 if max_sweeps sweeps ran without meeting the test (the last iterate is  */
/* kept).  off_hist[k] = ||off(T)||_F before sweep k (k <= sweeps), if given */
/* (first 64 values only).  max_rounds >= 0 truncates the run after  */
/* that many rounds in total (single-round parity tests); -1 = no limit.     */
/* ------------------------------------------------------------------------ */
#define DEFINE_JACOBI(SUF, REAL, OFF)                                                  \
    int orc_jacobi_evd_##SUF(REAL *T, REAL *V, int n, int b, double tol, double nu_d,  \
                             int rule, int max_sweeps, long long max_rounds,           \
                             int *sweeps_out, long long *rot_out, double *off_hist)   \
    {                                                                                  \
        int np = orc_padded_n(n, b), h = np / 2, nr = np - 1;                          \
        if (n < 1) return 1;                                                           \
        int *P = (int *)malloc(sizeof(int) * (size_t)nr * h);                          \
        int *Q = (int *)malloc(sizeof(int) * (size_t)nr * h);                          \
        if (orc_schedule(n, b, P, Q) != nr) { free(P); free(Q); return 1; }            \
        REAL *Tp = (REAL *)calloc((size_t)np * np, sizeof(REAL));                      \
        REAL *Vp = (REAL *)calloc((size_t)np * np, sizeof(REAL));                      \
        for (int j = 0; j < n; ++j)                                                    \
            for (int i = 0; i < n; ++i) {                                              \
                Tp[IDX(i, j, np)] = T[IDX(i, j, n)];                                   \
                Vp[IDX(i, j, np)] = V[IDX(i, j, n)];                                   \
            }                                                                          \
        REAL *tt = (REAL *)malloc(sizeof(REAL) * h), *ss = (REAL *)malloc(sizeof(REAL) * h); \
        REAL *uu = (REAL *)malloc(sizeof(REAL) * h);                                   \
        REAL nu = (REAL)nu_d;                                                          \
        int sweeps = 0, status = 2;                                                    \
        long long rot = 0, rounds_done = 0;                                            \
        for (;;) {                                                                     \
            double off = OFF(Tp, np, np);                                              \
            if (off_hist && sweeps < 64) off_hist[sweeps] = off;                       \
            if (off <= tol) { status = 0; break; }                                     \
            if (sweeps >= max_sweeps) { status = 2; break; }                           \
            if (max_rounds >= 0 && rounds_done >= max_rounds) { status = 0; break; }   \
            ++sweeps;                                                                  \
            for (int r = 0; r < nr; ++r) {                                             \
                if (max_rounds >= 0 && rounds_done >= max_rounds) break;               \
                rot += round_##SUF(Tp, Vp, np, np, P + (size_t)r * h, Q + (size_t)r * h, h, \
                                   nu, rule, tt, ss, uu);                              \
                ++rounds_done;                                                         \
            }                                                                          \
        }                                                                              \
        for (int j = 0; j < n; ++j)                                                    \
            for (int i = 0; i < n; ++i) {                                              \
                T[IDX(i, j, n)] = Tp[IDX(i, j, np)];                                   \
                V[IDX(i, j, n)] = Vp[IDX(i, j, np)];                                   \
            }                                                                          \
        if (sweeps_out) *sweeps_out = sweeps;                                          \
        if (rot_out) *rot_out = rot;                                                   \
        free(P); free(Q); free(Tp); free(Vp); free(tt); free(ss); free(uu);            \
        return status;                                                                 \
    }

DEFINE_JACOBI(f64, double, orc_off_f64)
DEFINE_JACOBI(f32, float, orc_off_f32)

/* ------------------------------------------------------------------------ */
/* Alg. 2 literally: row-cyclic order (1,2),(1,3),...,(n-1,n),   */
/* each rotation computed from the CURRENT T and applied at once.  Used     */
/* only for the paper-pattern tests (Table 1).  fp64.             */
/* ------------------------------------------------------------------------ */
int orc_jacobi_rowcyclic_f64(double *T, double *V, int n, double tol, double nu, int rule,
                             int max_sweeps, int *sweeps_out, long long *rot_out,
                             double *off_hist)
{
    int sweeps = 0, status = 2;
    long long rot = 0;
    for (;;) {
        double off = orc_off_f64(T, n, n);
        if (off_hist && sweeps < 64) off_hist[sweeps] = off;
        if (off <= tol) { status = 0; break; }
        if (sweeps >= max_sweeps) { status = 2; break; }
        ++sweeps;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                double t, s, tau;
                int doit = rot_params_f64(T[IDX(p, p, n)], T[IDX(q, q, n)], T[IDX(p, q, n)],
                                          nu, rule, &t, &s, &tau);
                double apq = T[IDX(p, q, n)];
                if (!doit) { T[IDX(p, q, n)] = 0; T[IDX(q, p, n)] = 0; continue; }
                ++rot;
                for (int k = 0; k < n; ++k) {
                    if (k == p || k == q) continue;
                    double x = T[IDX(p, k, n)], y = T[IDX(q, k, n)];
                    rot_f64(s, tau, &x, &y);
                    T[IDX(p, k, n)] = x; T[IDX(k, p, n)] = x;
                    T[IDX(q, k, n)] = y; T[IDX(k, q, n)] = y;
                }
                T[IDX(p, p, n)] = fma(-t, apq, T[IDX(p, p, n)]);
                T[IDX(q, q, n)] = fma(t, apq, T[IDX(q, q, n)]);
                T[IDX(p, q, n)] = 0; T[IDX(q, p, n)] = 0;
                if (V)
                    for (int i = 0; i < n; ++i) rot_f64(s, tau, &V[IDX(i, p, n)], &V[IDX(i, q, n)]);
            }
    }
    if (sweeps_out) *sweeps_out = sweeps;
    if (rot_out) *rot_out = rot;
    return status;
}

/* ------------------------------------------------------------------------ */
/* Modified Gram-Schmidt in fp64 (Alg. 3 step 2; Lemma 2.1). */
/* Left-looking column MGS (reading R10): for column k, v = z_k; for j < k:  */
/* r_jk = q_j^T v (current v), v = v - r_jk q_j; r_kk = ||v||; q_k = v/r_kk. */
/* Dot products and norms accumulate in long double.  Z is m x n (m >= n),   */
/* Q is m x n, R is n x n upper triangular (may be NULL).  Returns 3 if a    */
/* column norm is zero (rank deficient), else 0.                             */
/* ------------------------------------------------------------------------ */
int orc_mgs_f64(const double *Z, int m, int n, double *Q, double *R)
{
    if (R) memset(R, 0, sizeof(double) * (size_t)n * n);
    double *v = (double *)malloc(sizeof(double) * m);
    for (int k = 0; k < n; ++k) {
        for (int i = 0; i < m; ++i) v[i] = Z[IDX(i, k, m)];
        for (int j = 0; j < k; ++j) {
            ldbl acc = 0;
            for (int i = 0; i < m; ++i) acc += (ldbl)Q[IDX(i, j, m)] * (ldbl)v[i];
            double r = (double)acc;
            if (R) R[IDX(j, k, n)] = r;
            for (int i = 0; i < m; ++i) v[i] = v[i] - r * Q[IDX(i, j, m)];
        }
        ldbl nn = 0;
        for (int i = 0; i < m; ++i) nn += (ldbl)v[i] * (ldbl)v[i];
        double nrm = (double)sqrtl(nn);
        if (!(nrm > 0)) { free(v); return 3; }
        if (R) R[IDX(k, k, n)] = nrm;
        for (int i = 0; i < m; ++i) Q[IDX(i, k, m)] = v[i] / nrm;
    }
    free(v);
    return 0;
}

/* C (m x n) = op(A) * B with long double accumulation, rounded once.
 * transA = 0: A is m x k (lda = m); transA = 1: A is k x m (lda = k). */
void orc_gemm_f64(int transA, const double *A, const double *B, double *C, int m, int n, int k)
{
    _Pragma("omp parallel for schedule(static)")
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < m; ++i) {
            ldbl acc = 0;
            for (int l = 0; l < k; ++l) {
                ldbl a = transA ? A[IDX(l, i, k)] : A[IDX(i, l, m)];
                acc += a * (ldbl)B[IDX(l, j, k)];
            }
            C[IDX(i, j, m)] = (double)acc;
        }
}

/* Alg. 3 step 3: T = Q^T A Q formed as W = A Q, T = Q^T W (each    */
/* product accumulated in long double), then symmetrised T = (T + T^T)/2    */
/* (reading R11; the paper's T is symmetric by definition).                 */
void orc_qtaq_f64(const double *A, const double *Q, int n, double *T)
{
    double *W = (double *)malloc(sizeof(double) * (size_t)n * n);
    orc_gemm_f64(0, A, Q, W, n, n, n);
    orc_gemm_f64(1, Q, W, T, n, n, n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < j; ++i) {
            double a = (T[IDX(i, j, n)] + T[IDX(j, i, n)]) * 0.5;
            T[IDX(i, j, n)] = a; T[IDX(j, i, n)] = a;
        }
    free(W);
}

/* Stable sort of keys descending (eigenvalues "arranged in decreasing */
/* order"); perm[k] = original index of the k-th largest.  Insertion-merge   */
/* free: a plain stable merge sort.                                          */
static void msort_desc(const double *key, int *perm, int *tmp, int lo, int hi)
{
    if (hi - lo < 2) return;
    int mid = (lo + hi) / 2;
    msort_desc(key, perm, tmp, lo, mid);
    msort_desc(key, perm, tmp, mid, hi);
    int i = lo, j = mid, k = lo;
    while (i < mid && j < hi) {
        if (key[perm[j]] > key[perm[i]]) tmp[k++] = perm[j++];
        else tmp[k++] = perm[i++];
    }
    while (i < mid) tmp[k++] = perm[i++];
    while (j < hi) tmp[k++] = perm[j++];
    for (k = lo; k < hi; ++k) perm[k] = tmp[k];
}

void orc_sort_desc(const double *key, int n, int *perm)
{
    int *tmp = (int *)malloc(sizeof(int) * (n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) perm[i] = i;
    msort_desc(key, perm, tmp, 0, n);
    free(tmp);
}

/* ------------------------------------------------------------------------ */
/* Configuration shared by the drivers below (mirrors mpj_config in         */
/* include/mpjacobi.h, but defined independently here).                     */
/* ------------------------------------------------------------------------ */
typedef struct {
    double eps_factor;      /* eps = eps_factor * omega (0.1)              */
    double nu_factor;       /* nu = nu_factor * omega (20 eig, 1 svd)      */
    double eps_low_factor;  /* low stage eps = f * upsilon; <= 0: R12's rule       */
    double nu_low_factor;   /* low stage nu = nu_low_factor * upsilon (R12: 20/1)  */
    double early_stop;      /* svd: stop when sweep rotations / N < this (2e-4)    */
    int max_sweeps;         /* R13: 60                                             */
    int max_sweeps_low;     /* low stage cap (R13: 60)                             */
    int rule;               /* 0 = min rule, 1 = sqrt rule        */
    int b;                  /* ordering block size (R1)                           */
    int low_solver;         /* EVD step 1 (R12): 0/2 = symmetric QR (Householder    */
                            /* tridiagonalisation + implicit QR), 1 = fp32 */
                            /* parallel Jacobi                                     */
} orc_cfg;

typedef struct {
    int sweeps, sweeps_low, status, status_low;
    long long rotations, rotations_low;
    double normA, off0;     /* ||A||_F and ||off(Q^T A Q)||_F                      */
    double off_hist[64];
    double rot_hist[64];    /* svd: rotations applied in fp64 sweep k+1 (k < 64)   */
} orc_report;

#define OMEGA 1.1102230246251565e-16     /* 2^-53 */
#define UPSILON 5.9604644775390625e-08   /* 2^-24 */

/* Low-stage stop tolerance factor (reading R12): the fp32 stage's attainable
 * ||off(T32)||/||A||_F grows like sqrt(n) upsilon, so eps_low = max(10,
 * 1.25 sqrt(n)) upsilon (= 10 upsilon at n = 64) unless eps_low_factor > 0. */
static double orc_eps_low(const orc_cfg *cfg, int n)
{
    if (cfg->eps_low_factor > 0) return cfg->eps_low_factor;
    double f = 1.25 * sqrt((double)n);
    return f > 10.0 ? f : 10.0;
}

/* Extract (Alg. 3 output): lambda = diag(T) sorted descending       */
/* (stable), columns of V permuted alike.                                   */
static void extract_evd(const double *T, double *V, int n, double *lam)
{
    double *d = (double *)malloc(sizeof(double) * n);
    int *perm = (int *)malloc(sizeof(int) * n);
    double *Vs = (double *)malloc(sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i) d[i] = T[IDX(i, i, n)];
    orc_sort_desc(d, n, perm);
    for (int k = 0; k < n; ++k) {
        lam[k] = d[perm[k]];
        memcpy(Vs + (size_t)k * n, V + (size_t)perm[k] * n, sizeof(double) * n);
    }
    memcpy(V, Vs, sizeof(double) * (size_t)n * n);
    free(d); free(perm); free(Vs);
}

/* Low-precision stage of Alg. 3 (step 1), reading R12: the same     */
/* parallel-ordered Jacobi in binary32 on fl32(A) from V = I.  Returns the   */
/* fp32 eigenvector matrix Z (n x n).                                        */
int orc_low_evd(const double *A, int n, const orc_cfg *cfg, float *Z, orc_report *rep)
{
    float *T32 = (float *)malloc(sizeof(float) * (size_t)n * n);
    for (size_t i = 0; i < (size_t)n * n; ++i) T32[i] = (float)A[i];
    memset(Z, 0, sizeof(float) * (size_t)n * n);
    for (int i = 0; i < n; ++i) Z[IDX(i, i, n)] = 1.0f;
    double nA32 = orc_fro_f32(T32, n, n, n);
    int sw = 0; long long rot = 0;
    int st = orc_jacobi_evd_f32(T32, Z, n, cfg->b, orc_eps_low(cfg, n) * UPSILON * nA32,
                                cfg->nu_low_factor * UPSILON, cfg->rule, cfg->max_sweeps_low,
                                -1, &sw, &rot, NULL);
    if (rep) { rep->sweeps_low = sw; rep->rotations_low = rot; rep->status_low = st; }
    free(T32);
    return st;
}

/* ------------------------------------------------------------------------ */
/* Classic block Jacobi with full inner diagonalisation (SURVEY 8(f) row 4;  */
/* the parallel Jacobi context of P:27), reading R26: the indices are cut    */
/* into nb = n_p/b blocks of b; a block round pairs the blocks by the         */
/* merry-go-round on blocks; for every block pair (I, J) the 2b x 2b  */
/* submatrix S = T(P, P), P = block I u block J, is diagonalised by inner     */
/* Jacobi sweeps (the 2b - 1 rounds of the R1 ordering on 2b indices with     */
/* block size b, Lemma 3.1 with the same threshold nu) until an inner sweep  */
/* rotates no pair (or max_inner sweeps), accumulating U = J_1 J_2 ...; then */
/* T(P_a, P_c) <- U_a^T T(P_a, P_c) U_c for every two block pairs a != c      */
/* (the two products each accumulated in long double and rounded),            */
/* T(P_a, P_a) <- the diagonalised S_a, V(:, P_c) <- V(:, P_c) U_c.  A sweep */
/* is the nb - 1 block rounds; the stop test as Alg. 2.  off_hist    */
/* and the return value as orc_jacobi_evd.  rot counts inner rotations.       */
/* ------------------------------------------------------------------------ */
int orc_block_jacobi_evd_f64(double *T, double *V, int n, int b, double tol, double nu, int rule,
                             int max_sweeps, int max_inner, int *sweeps_out, long long *rot_out,
                             double *off_hist)
{
    if (n < 1 || b < 1 || (b > 1 && (b & 1))) return 1;
    const int np = orc_padded_n(n, b), nb = np / b, mb = nb / 2, w = 2 * b;
    double *Tp = (double *)calloc((size_t)np * np, sizeof(double));
    double *Vp = (double *)calloc((size_t)np * np, sizeof(double));
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            Tp[IDX(i, j, np)] = T[IDX(i, j, n)];
            Vp[IDX(i, j, np)] = V[IDX(i, j, n)];
        }
    int *btop = (int *)malloc(sizeof(int) * (mb > 0 ? mb : 1)), *bbot = (int *)malloc(sizeof(int) * (mb > 0 ? mb : 1));
    int *idx = (int *)malloc(sizeof(int) * (size_t)(mb > 0 ? mb : 1) * w);
    double *Us = (double *)malloc(sizeof(double) * (size_t)(mb > 0 ? mb : 1) * w * w);
    double *Ss = (double *)malloc(sizeof(double) * (size_t)(mb > 0 ? mb : 1) * w * w);
    double *Tn = (double *)malloc(sizeof(double) * (size_t)np * np);
    int sweeps = 0, status = 2;
    long long rot = 0;
    for (;;) {
        const double off = orc_off_f64(Tp, np, np);
        if (off_hist && sweeps < 64) off_hist[sweeps] = off;
        if (off <= tol) { status = 0; break; }
        if (sweeps >= max_sweeps) { status = 2; break; }
        ++sweeps;
        for (int k = 0; k < mb; ++k) { btop[k] = 2 * k; bbot[k] = 2 * k + 1; }
        for (int R = 0; R < nb - 1; ++R) {
            long long rr = 0;
            /* inner diagonalisation of every block pair's S (disjoint: independent) */
            _Pragma("omp parallel for reduction(+:rr) schedule(dynamic,1)")
            for (int k = 0; k < mb; ++k) {
                const int I = btop[k] < bbot[k] ? btop[k] : bbot[k], J = btop[k] < bbot[k] ? bbot[k] : btop[k];
                int *ix = idx + (size_t)k * w;
                for (int i = 0; i < b; ++i) { ix[i] = I * b + i; ix[b + i] = J * b + i; }
                double *S = Ss + (size_t)k * w * w, *U = Us + (size_t)k * w * w;
                for (int j = 0; j < w; ++j)
                    for (int i = 0; i < w; ++i) {
                        S[IDX(i, j, w)] = Tp[IDX(ix[i], ix[j], np)];
                        U[IDX(i, j, w)] = i == j ? 1.0 : 0.0;
                    }
                for (int it = 0; it < max_inner; ++it) {
                    int sw = 0;
                    long long r1 = 0;
                    orc_jacobi_evd_f64(S, U, w, b, 0.0, nu, rule, 1, -1, &sw, &r1, NULL);
                    rr += r1;
                    if (r1 == 0) break;
                }
            }
            rot += rr;
            /* T <- U^T T U by blocks (off-diagonal pairs), diagonal blocks from S */
            memcpy(Tn, Tp, sizeof(double) * (size_t)np * np);
            _Pragma("omp parallel for schedule(dynamic,1)")
            for (int a = 0; a < mb; ++a) {
                const int *ia = idx + (size_t)a * w;
                const double *Ua = Us + (size_t)a * w * w;
                double *Y = (double *)malloc(sizeof(double) * (size_t)w * w);
                for (int c = 0; c < mb; ++c) {
                    const int *ic = idx + (size_t)c * w;
                    if (c == a) {
                        const double *S = Ss + (size_t)a * w * w;
                        for (int j = 0; j < w; ++j)
                            for (int i = 0; i < w; ++i) Tn[IDX(ia[i], ia[j], np)] = S[IDX(i, j, w)];
                        continue;
                    }
                    const double *Uc = Us + (size_t)c * w * w;
                    for (int j = 0; j < w; ++j)          /* Y = U_a^T X */
                        for (int i = 0; i < w; ++i) {
                            ldbl acc = 0;
                            for (int l = 0; l < w; ++l) acc += (ldbl)Ua[IDX(l, i, w)] * (ldbl)Tp[IDX(ia[l], ic[j], np)];
                            Y[IDX(i, j, w)] = (double)acc;
                        }
                    for (int j = 0; j < w; ++j)          /* W = Y U_c */
                        for (int i = 0; i < w; ++i) {
                            ldbl acc = 0;
                            for (int l = 0; l < w; ++l) acc += (ldbl)Y[IDX(i, l, w)] * (ldbl)Uc[IDX(l, j, w)];
                            Tn[IDX(ia[i], ic[j], np)] = (double)acc;
                        }
                }
                free(Y);
            }
            memcpy(Tp, Tn, sizeof(double) * (size_t)np * np);
            /* V(:, P_c) <- V(:, P_c) U_c */
            _Pragma("omp parallel for schedule(static)")
            for (int r = 0; r < np; ++r) {
                double row[256];
                for (int c = 0; c < mb; ++c) {
                    const int *ic = idx + (size_t)c * w;
                    const double *Uc = Us + (size_t)c * w * w;
                    for (int j = 0; j < w; ++j) {
                        ldbl acc = 0;
                        for (int l = 0; l < w; ++l) acc += (ldbl)Vp[IDX(r, ic[l], np)] * (ldbl)Uc[IDX(l, j, w)];
                        row[j] = (double)acc;
                    }
                    for (int j = 0; j < w; ++j) Vp[IDX(r, ic[j], np)] = row[j];
                }
            }
            music(btop, bbot, mb);
        }
    }
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            T[IDX(i, j, n)] = Tp[IDX(i, j, np)];
            V[IDX(i, j, n)] = Vp[IDX(i, j, np)];
        }
    if (sweeps_out) *sweeps_out = sweeps;
    if (rot_out) *rot_out = rot;
    free(Tp); free(Vp); free(btop); free(bbot); free(idx); free(Us); free(Ss); free(Tn);
    return status;
}

/* ------------------------------------------------------------------------ */
/* Alg. 3 step 1 as the paper states it ("[Z,~] = eig(A)  Symmetric   */
/* QR factorization in low precision upsilon"; the paper ran LAPACK SSYEV /  */
/* cusolverDnSsyevd), reading R12': in binary32,               */
/*   1. Householder tridiagonalisation T = Q^T fl32(A) Q (Golub & Van Loan,  */
/*      Alg. 8.3.1), reflectors in the LAPACK convention                     */
/*        H = I - tau v v^T, v(0) = 1, beta = -sign(alpha) ||x||,             */
/*        tau = (beta - alpha) / beta, v(1:) = x(1:) / (alpha - beta)          */
/*      (H = I, tau = 0, when x(1:) = 0);                                    */
/*   2. Q = H_0 H_1 ... H_{n-3} formed explicitly (backward accumulation);   */
/*   3. the symmetric QR algorithm on T (GvL Alg. 8.3.3: implicit QR steps   */
/*      with the Wilkinson shift, Alg. 8.3.2, deflation when |t_{k+1,k}| <=  */
/*      upsilon (|t_kk| + |t_{k+1,k+1}|)), rotations accumulated Z = Q G ...; */
/*   4. eigenvalues diag(T) sorted descending (stable), Z's columns alike.   */
/* T is kept dense (plain and obviously the algorithm; O(n^3) per QR step    */
/* pass is fine at oracle sizes).  Element updates are binary32 values;     */
/* each dot product / multi-term update is accumulated in long double and    */
/* rounded once.                                                             */
/* ------------------------------------------------------------------------ */

/* LAPACK-convention Householder vector of x (length m >= 1): returns tau,    */
/* writes beta and v (v[0] = 1).                                             */
static float house_f32(const float *x, int m, float *v, float *beta_out)
{
    const float alpha = x[0];
    ldbl s = 0;
    for (int i = 1; i < m; ++i) s += (ldbl)x[i] * (ldbl)x[i];
    v[0] = 1.0f;
    if (s == 0) {
        for (int i = 1; i < m; ++i) v[i] = 0.0f;
        *beta_out = alpha;
        return 0.0f;
    }
    const float nrm = (float)sqrtl((ldbl)alpha * (ldbl)alpha + s);
    const float beta = alpha >= 0 ? -nrm : nrm;
    const float tau = (beta - alpha) / beta;
    const float scal = alpha - beta;
    for (int i = 1; i < m; ++i) v[i] = x[i] / scal;
    *beta_out = beta;
    return tau;
}

/* 1. In place on the n x n symmetric A (both triangles kept): on return      */
/* d[k] = T_kk, e[k] = T_{k+1,k}, A(k+2:n, k) = v_k(1:), tau[k] (k < n-2).    */
int orc_sytrd_f32(float *A, int n, float *d, float *e, float *tau)
{
    float *x = (float *)malloc(sizeof(float) * (n > 0 ? n : 1));
    float *v = (float *)malloc(sizeof(float) * (n > 0 ? n : 1));
    float *p = (float *)malloc(sizeof(float) * (n > 0 ? n : 1));
    float *w = (float *)malloc(sizeof(float) * (n > 0 ? n : 1));
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1;                    /* trailing size */
        for (int i = 0; i < m; ++i) x[i] = A[IDX(k + 1 + i, k, n)];
        float beta;
        const float t = house_f32(x, m, v, &beta);
        tau[k] = t;
        /* p = tau A22 v, K = tau/2 p^T v, w = p - K v */
        for (int i = 0; i < m; ++i) {
            ldbl acc = 0;
            for (int j = 0; j < m; ++j) acc += (ldbl)A[IDX(k + 1 + i, k + 1 + j, n)] * (ldbl)v[j];
            p[i] = (float)((ldbl)t * acc);
        }
        ldbl pv = 0;
        for (int i = 0; i < m; ++i) pv += (ldbl)p[i] * (ldbl)v[i];
        const float K = (float)((ldbl)t * pv / 2);
        for (int i = 0; i < m; ++i) w[i] = (float)((ldbl)p[i] - (ldbl)K * (ldbl)v[i]);
        /* A22 -= v w^T + w v^T */
        for (int j = 0; j < m; ++j)
            for (int i = 0; i < m; ++i) {
                float *a = &A[IDX(k + 1 + i, k + 1 + j, n)];
                *a = (float)((ldbl)*a - (ldbl)v[i] * (ldbl)w[j] - (ldbl)w[i] * (ldbl)v[j]);
            }
        A[IDX(k + 1, k, n)] = beta;
        A[IDX(k, k + 1, n)] = beta;
        for (int i = 1; i < m; ++i) { A[IDX(k + 1 + i, k, n)] = v[i]; A[IDX(k, k + 1 + i, n)] = 0.0f; }
    }
    for (int k = 0; k < n; ++k) d[k] = A[IDX(k, k, n)];
    for (int k = 0; k + 1 < n; ++k) e[k] = A[IDX(k + 1, k, n)];
    for (int k = n - 2; k < n; ++k) if (k >= 0) tau[k] = 0.0f;
    free(x); free(v); free(p); free(w);
    return 0;
}

/* 2. Q = H_0 ... H_{n-3} from orc_sytrd_f32's output (v_k below the first   */
/* subdiagonal of column k, tau).  Backward accumulation Q <- H_k Q.         */
void orc_orgtr_f32(const float *A, int n, const float *tau, float *Q)
{
    memset(Q, 0, sizeof(float) * (size_t)n * n);
    for (int i = 0; i < n; ++i) Q[IDX(i, i, n)] = 1.0f;
    float *v = (float *)malloc(sizeof(float) * (n > 0 ? n : 1));
    for (int k = n - 3; k >= 0; --k) {
        const int m = n - k - 1;
        v[0] = 1.0f;
        for (int i = 1; i < m; ++i) v[i] = A[IDX(k + 1 + i, k, n)];
        for (int j = 0; j < n; ++j) {
            ldbl acc = 0;
            for (int i = 0; i < m; ++i) acc += (ldbl)v[i] * (ldbl)Q[IDX(k + 1 + i, j, n)];
            const ldbl f = (ldbl)tau[k] * acc;
            for (int i = 0; i < m; ++i) {
                float *q = &Q[IDX(k + 1 + i, j, n)];
                *q = (float)((ldbl)*q - f * (ldbl)v[i]);
            }
        }
    }
    free(v);
}

/* GvL Alg. 5.1.3: c, s with [c s; -s c]^T [a; b] = [r; 0]. */
static void givens_f32(float a, float b, float *c, float *s)
{
    if (b == 0.0f) { *c = 1.0f; *s = 0.0f; return; }
    if (fabsf(b) > fabsf(a)) {
        const float t = -a / b;
        *s = 1.0f / sqrtf(fmaf(t, t, 1.0f));
        *c = *s * t;
    } else {
        const float t = -b / a;
        *c = 1.0f / sqrtf(fmaf(t, t, 1.0f));
        *s = *c * t;
    }
}

/* rows (i, k) of the dense T: [r_i; r_k] <- G^T [r_i; r_k]; columns alike */
static void rot_rows_f32(float *T, int n, int i, int k, float c, float s)
{
    for (int j = 0; j < n; ++j) {
        const float x = T[IDX(i, j, n)], y = T[IDX(k, j, n)];
        T[IDX(i, j, n)] = (float)((ldbl)c * x - (ldbl)s * y);
        T[IDX(k, j, n)] = (float)((ldbl)s * x + (ldbl)c * y);
    }
}
static void rot_cols_f32(float *M, int rows, int ld, int i, int k, float c, float s)
{
    for (int r = 0; r < rows; ++r) {
        const float x = M[IDX(r, i, ld)], y = M[IDX(r, k, ld)];
        M[IDX(r, i, ld)] = (float)((ldbl)c * x - (ldbl)s * y);
        M[IDX(r, k, ld)] = (float)((ldbl)s * x + (ldbl)c * y);
    }
}

/* 3. The symmetric QR algorithm (GvL Alg. 8.3.3) on the tridiagonal (d, e),  */
/* rotations accumulated into Z (n x n, in: Q, out: Q G_1 G_2 ...).  On      */
/* return d holds the eigenvalues (unsorted).  Returns the number of         */
/* implicit QR steps, or -1 if 30 n steps did not converge.                  */
int orc_tridiag_qr_f32(float *d, float *e, int n, float *Z)
{
    float *T = (float *)calloc((size_t)n * n, sizeof(float));
    for (int k = 0; k < n; ++k) T[IDX(k, k, n)] = d[k];
    for (int k = 0; k + 1 < n; ++k) { T[IDX(k + 1, k, n)] = e[k]; T[IDX(k, k + 1, n)] = e[k]; }
    int steps = 0;
    for (;;) {
        /* deflation (GvL 8.3.4 with tol = upsilon) */
        for (int k = 0; k + 1 < n; ++k)
            if (fabsf(T[IDX(k + 1, k, n)]) <= UPSILON * (fabsf(T[IDX(k, k, n)]) + fabsf(T[IDX(k + 1, k + 1, n)]))) {
                T[IDX(k + 1, k, n)] = 0.0f;
                T[IDX(k, k + 1, n)] = 0.0f;
            }
        /* largest trailing diagonal part, then the unreduced block above it */
        int m = n - 1;
        while (m > 0 && T[IDX(m, m - 1, n)] == 0.0f) --m;
        if (m == 0) break;
        int l = m - 1;
        while (l > 0 && T[IDX(l, l - 1, n)] != 0.0f) --l;
        if (++steps > 30 * n) { free(T); return -1; }
        /* one implicit QR step with Wilkinson shift on T(l:m, l:m) (GvL 8.3.2) */
        const float tmm = T[IDX(m, m, n)], tm1 = T[IDX(m - 1, m - 1, n)], em = T[IDX(m, m - 1, n)];
        const float dd = (tm1 - tmm) / 2.0f;
        const float sg = dd >= 0.0f ? 1.0f : -1.0f;
        const float mu = tmm - em * em / (dd + sg * sqrtf(fmaf(dd, dd, em * em)));
        float x = T[IDX(l, l, n)] - mu, z = T[IDX(l + 1, l, n)];
        for (int k = l; k < m; ++k) {
            float c, s;
            givens_f32(x, z, &c, &s);
            rot_rows_f32(T, n, k, k + 1, c, s);
            rot_cols_f32(T, n, n, k, k + 1, c, s);
            if (k > l) {            /* the bulge the rotation was chosen to annihilate */
                T[IDX(k + 1, k - 1, n)] = 0.0f;
                T[IDX(k - 1, k + 1, n)] = 0.0f;
            }
            rot_cols_f32(Z, n, n, k, k + 1, c, s);
            if (k + 1 < m) { x = T[IDX(k + 1, k, n)]; z = T[IDX(k + 2, k, n)]; }
        }
    }
    for (int k = 0; k < n; ++k) d[k] = T[IDX(k, k, n)];
    free(T);
    return steps;
}

/* Step 1 by symmetric QR (steps 1-4 above) on fl32(A): Z (n x n, columns in */
/* descending eigenvalue order), lam32 (n, may be NULL).  Returns 0, or 2 if */
/* the QR iteration did not converge.                                        */
int orc_low_evd_symqr(const double *A, int n, float *Z, float *lam32, orc_report *rep)
{
    size_t nn = (size_t)n * n;
    float *A32 = (float *)malloc(sizeof(float) * nn);
    for (size_t i = 0; i < nn; ++i) A32[i] = (float)A[i];
    float *d = (float *)malloc(sizeof(float) * n), *e = (float *)malloc(sizeof(float) * n);
    float *tau = (float *)malloc(sizeof(float) * n), *Q = (float *)malloc(sizeof(float) * nn);
    orc_sytrd_f32(A32, n, d, e, tau);
    orc_orgtr_f32(A32, n, tau, Q);
    const int steps = orc_tridiag_qr_f32(d, e, n, Q);
    double *key = (double *)malloc(sizeof(double) * n);
    int *perm = (int *)malloc(sizeof(int) * n);
    for (int k = 0; k < n; ++k) key[k] = d[k];
    orc_sort_desc(key, n, perm);
    for (int k = 0; k < n; ++k) {
        memcpy(Z + (size_t)k * n, Q + (size_t)perm[k] * n, sizeof(float) * n);
        if (lam32) lam32[k] = d[perm[k]];
    }
    if (rep) { rep->sweeps_low = 0; rep->rotations_low = steps; rep->status_low = steps < 0 ? 2 : 0; }
    free(A32); free(d); free(e); free(tau); free(Q); free(key); free(perm);
    return steps < 0 ? 2 : 0;
}

/* Alg. 3 end to end.  A: n x n (symmetrised internally, R14).   */
/* Outputs lam (n, descending), V (n x n).  If Zin != NULL it is used as the */
/* low-precision eigenvector matrix instead of the fp32 Jacobi stage (the    */
/* paper used LAPACK SSYEV there; tests pass scipy's ssyevd Z).       */
int orc_mp_evd(const double *Ain, int n, const orc_cfg *cfg, const float *Zin,
               double *lam, double *V, orc_report *rep)
{
    size_t nn = (size_t)n * n;
    double *A = (double *)malloc(sizeof(double) * nn);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) A[IDX(i, j, n)] = (Ain[IDX(i, j, n)] + Ain[IDX(j, i, n)]) * 0.5;
    double nA = orc_fro_f64(A, n, n, n);
    float *Z = (float *)malloc(sizeof(float) * nn);
    orc_report r0; memset(&r0, 0, sizeof(r0));
    if (Zin) memcpy(Z, Zin, sizeof(float) * nn);
    else if (cfg->low_solver == 1) orc_low_evd(A, n, cfg, Z, &r0);
    else orc_low_evd_symqr(A, n, Z, NULL, &r0);
    double *Zd = (double *)malloc(sizeof(double) * nn), *T = (double *)malloc(sizeof(double) * nn);
    for (size_t i = 0; i < nn; ++i) Zd[i] = (double)Z[i];
    int st = orc_mgs_f64(Zd, n, n, V, NULL);
    if (st) { free(A); free(Z); free(Zd); free(T); return st; }
    orc_qtaq_f64(A, V, n, T);
    r0.normA = nA;
    r0.off0 = orc_off_f64(T, n, n);
    int sw = 0; long long rot = 0;
    st = orc_jacobi_evd_f64(T, V, n, cfg->b, cfg->eps_factor * OMEGA * nA, cfg->nu_factor * OMEGA,
                            cfg->rule, cfg->max_sweeps, -1, &sw, &rot, r0.off_hist);
    r0.sweeps = sw; r0.rotations = rot; r0.status = st;
    extract_evd(T, V, n, lam);
    if (rep) *rep = r0;
    free(A); free(Z); free(Zd); free(T);
    return st;
}

/* Alg. 2 from T = A, P = I ("plain fp64 Jacobi"), same ordering. */
int orc_plain_evd(const double *Ain, int n, const orc_cfg *cfg, double *lam, double *V,
                  orc_report *rep)
{
    size_t nn = (size_t)n * n;
    double *T = (double *)malloc(sizeof(double) * nn);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) T[IDX(i, j, n)] = (Ain[IDX(i, j, n)] + Ain[IDX(j, i, n)]) * 0.5;
    memset(V, 0, sizeof(double) * nn);
    for (int i = 0; i < n; ++i) V[IDX(i, i, n)] = 1.0;
    orc_report r0; memset(&r0, 0, sizeof(r0));
    r0.normA = orc_fro_f64(T, n, n, n);
    r0.off0 = orc_off_f64(T, n, n);
    int sw = 0; long long rot = 0;
    int st = orc_jacobi_evd_f64(T, V, n, cfg->b, cfg->eps_factor * OMEGA * r0.normA,
                                cfg->nu_factor * OMEGA, cfg->rule, cfg->max_sweeps, -1, &sw,
                                &rot, r0.off_hist);
    r0.sweeps = sw; r0.rotations = rot; r0.status = st;
    extract_evd(T, V, n, lam);
    if (rep) *rep = r0;
    free(T);
    return st;
}

/* ------------------------------------------------------------------------ */
/* One-sided (Hestenes) Jacobi, Alg. 4 / Alg. 5 steps 4-13 (P:469-484,       */
/* P:499-508), Lemma 5.1.  Same ordering as above (the pairs of  */
/* a round are disjoint columns, so the round equals sequential application  */
/* exactly).  C is m x n, V is n x n.  alpha = c_p^T c_p, beta = c_q^T c_q,   */
/* gamma = c_p^T c_q (long double accumulation).  Rotate iff                */
/* |gamma| > nu sqrt(alpha beta); mu = (beta - alpha)/(2 gamma).     */
/* Stop before a sweep when ||off(C^T C)||_F <= tol_rel ||C^T C||_F, */
/* or after a sweep whose rotation count / N < early_stop (R15).      */
/* ------------------------------------------------------------------------ */
static void gram_norms(const double *C, int m, int n, double *off, double *tot)
{
    /* per-column partial sums (column j holds the i <= j part of row j of the
       Gram matrix), then a fixed-order sum: deterministic for any thread count */
    ldbl *po = (ldbl *)calloc((size_t)n, sizeof(ldbl)), *pt = (ldbl *)calloc((size_t)n, sizeof(ldbl));
    _Pragma("omp parallel for schedule(dynamic,4)")
    for (int j = 0; j < n; ++j)
        for (int i = 0; i <= j; ++i) {
            ldbl g = 0;
            for (int r = 0; r < m; ++r) g += (ldbl)C[IDX(r, i, m)] * (ldbl)C[IDX(r, j, m)];
            ldbl g2 = g * g;
            if (i == j) pt[j] += g2;
            else { po[j] += 2 * g2; pt[j] += 2 * g2; }
        }
    ldbl so = 0, st = 0;
    for (int j = 0; j < n; ++j) { so += po[j]; st += pt[j]; }
    free(po); free(pt);
    *off = (double)sqrtl(so);
    *tot = (double)sqrtl(st);
}

void orc_gram_offnorm(const double *C, int m, int n, double *off, double *tot)
{
    gram_norms(C, m, n, off, tot);
}

#define DEFINE_ONESIDED(SUF, REAL)                                                     \
    int orc_jacobi_svd_##SUF(REAL *C, REAL *V, int m, int n, int b, double eps_rel,    \
                             double nu_d, double early_stop, int max_sweeps,           \
                             int *sweeps_out, long long *rot_out, double *off_hist,   \
                             double *rot_hist)                                         \
    {                                                                                  \
        int np = orc_padded_n(n, b), h = np / 2, nr = np - 1;                          \
        int *P = (int *)malloc(sizeof(int) * (size_t)nr * h);                          \
        int *Q = (int *)malloc(sizeof(int) * (size_t)nr * h);                          \
        orc_schedule(n, b, P, Q);                                                      \
        double N = 0.5 * (double)n * (double)(n - 1);                                  \
        int sweeps = 0, status = 2;                                                    \
        long long rot = 0;                                                             \
        double *Cd = (double *)malloc(sizeof(double) * (size_t)m * n);                 \
        for (;;) {                                                                     \
            double off, tot;                                                           \
            for (size_t i = 0; i < (size_t)m * n; ++i) Cd[i] = (double)C[i];           \
            gram_norms(Cd, m, n, &off, &tot);                                          \
            if (off_hist && sweeps < 64) off_hist[sweeps] = tot > 0 ? off / tot : 0;   \
            if (off <= eps_rel * tot) { status = 0; break; }                           \
            if (sweeps >= max_sweeps) { status = 2; break; }                           \
            ++sweeps;                                                                  \
            long long rs = 0;                                                          \
            for (int r = 0; r < nr; ++r) {                                             \
                const int *Pr = P + (size_t)r * h, *Qr = Q + (size_t)r * h;            \
                _Pragma("omp parallel for reduction(+:rs) schedule(dynamic,1)")       \
                for (int k = 0; k < h; ++k) {                                          \
                    int p = Pr[k], q = Qr[k];                                          \
                    if (q >= n) continue; /* padded dummy column: zero, never rotated */ \
                    ldbl al = 0, be = 0, ga = 0;                                       \
                    for (int i = 0; i < m; ++i) {                                      \
                        ldbl x = C[IDX(i, p, m)], y = C[IDX(i, q, m)];                 \
                        al += x * x; be += y * y; ga += x * y;                         \
                    }                                                                  \
                    REAL a = (REAL)al, bb = (REAL)be, g = (REAL)ga;                    \
                    REAL nu = (REAL)nu_d;                                              \
                    if (!(fabsl((ldbl)g) > (ldbl)nu * sqrtl((ldbl)a * (ldbl)bb))) continue; \
                    REAL t, s, tau;                                                    \
                    /* Lemma 5.1 uses Lemma 3.1's formulas with a_ii=alpha, a_jj=beta, \
                       a_ij=gamma; the threshold was decided above (rule-free call). */ \
                    rot_params_##SUF(a, bb, g, (REAL)0, 0, &t, &s, &tau);              \
                    for (int i = 0; i < m; ++i) rot_##SUF(s, tau, &C[IDX(i, p, m)], &C[IDX(i, q, m)]); \
                    for (int i = 0; i < n; ++i) rot_##SUF(s, tau, &V[IDX(i, p, n)], &V[IDX(i, q, n)]); \
                    rs += 1;                                                           \
                }                                                                      \
            }                                                                          \
            rot += rs;                                                                 \
            if (rot_hist && sweeps <= 64) rot_hist[sweeps - 1] = (double)rs;           \
            if (early_stop > 0 && N > 0 && (double)rs / N < early_stop) {              \
                /* recompute the history entry for the final state */                  \
                status = 0;                                                            \
                break;                                                                 \
            }                                                                          \
        }                                                                              \
        if (sweeps_out) *sweeps_out = sweeps;                                          \
        if (rot_out) *rot_out = rot;                                                   \
        free(P); free(Q); free(Cd);                                                    \
        return status;                                                                 \
    }

DEFINE_ONESIDED(f64, double)
DEFINE_ONESIDED(f32, float)

/* Alg. 5 steps 14-16: reorder columns of [C; V] by ||c_j||    */
/* descending (stable, R16), sigma_j = ||c_j||, u_j = c_j / sigma_j.         */
/* Returns 3 if some sigma_j <= n * omega * ||A||_F (rank deficient, R17).   */
static int extract_svd(const double *C, const double *Vin, int m, int n, double normA,
                       double *sig, double *U, double *V)
{
    double *nr = (double *)malloc(sizeof(double) * n);
    int *perm = (int *)malloc(sizeof(int) * n);
    for (int j = 0; j < n; ++j) {
        ldbl s = 0;
        for (int i = 0; i < m; ++i) s += (ldbl)C[IDX(i, j, m)] * (ldbl)C[IDX(i, j, m)];
        nr[j] = (double)sqrtl(s);
    }
    orc_sort_desc(nr, n, perm);
    int st = 0;
    for (int k = 0; k < n; ++k) {
        int j = perm[k];
        sig[k] = nr[j];
        if (!(nr[j] > n * OMEGA * normA)) st = 3;
        for (int i = 0; i < m; ++i) U[IDX(i, k, m)] = nr[j] > 0 ? C[IDX(i, j, m)] / nr[j] : 0.0;
        memcpy(V + (size_t)k * n, Vin + (size_t)j * n, sizeof(double) * n);
    }
    free(nr); free(perm);
    return st;
}

/* Alg. 5 end to end.  A: m x n, m >= n.  Low-precision SVD     */
/* (step 1) = one-sided Jacobi in binary32 on fl32(A) from V = I (R12).      */
/* Zin (n x n fp32) may replace it.                                          */
int orc_mp_svd(const double *A, int m, int n, const orc_cfg *cfg, const float *Zin,
               double *sig, double *U, double *V, orc_report *rep)
{
    if (m < n) return 1;
    size_t mn = (size_t)m * n, nn = (size_t)n * n;
    orc_report r0; memset(&r0, 0, sizeof(r0));
    r0.normA = orc_fro_f64(A, m, n, m);
    float *Z = (float *)malloc(sizeof(float) * nn);
    if (Zin) memcpy(Z, Zin, sizeof(float) * nn);
    else {
        float *C32 = (float *)malloc(sizeof(float) * mn);
        for (size_t i = 0; i < mn; ++i) C32[i] = (float)A[i];
        memset(Z, 0, sizeof(float) * nn);
        for (int i = 0; i < n; ++i) Z[IDX(i, i, n)] = 1.0f;
        int sw = 0; long long rot = 0;
        r0.status_low = orc_jacobi_svd_f32(C32, Z, m, n, cfg->b, orc_eps_low(cfg, n) * UPSILON,
                                           cfg->nu_low_factor * UPSILON, cfg->early_stop,
                                           cfg->max_sweeps_low, &sw, &rot, NULL, NULL);
        r0.sweeps_low = sw; r0.rotations_low = rot;
        free(C32);
    }
    double *Zd = (double *)malloc(sizeof(double) * nn);
    double *Q = (double *)malloc(sizeof(double) * nn);
    double *C = (double *)malloc(sizeof(double) * mn);
    for (size_t i = 0; i < nn; ++i) Zd[i] = (double)Z[i];
    int st = orc_mgs_f64(Zd, n, n, Q, NULL);
    if (st) { free(Z); free(Zd); free(Q); free(C); return st; }
    orc_gemm_f64(0, A, Q, C, m, n, n);  /* C = A Q, V = Q */
    double off, tot;
    gram_norms(C, m, n, &off, &tot);
    r0.off0 = off;
    int sw = 0; long long rot = 0;
    st = orc_jacobi_svd_f64(C, Q, m, n, cfg->b, cfg->eps_factor * OMEGA, cfg->nu_factor * OMEGA,
                            cfg->early_stop, cfg->max_sweeps, &sw, &rot, r0.off_hist, r0.rot_hist);
    r0.sweeps = sw; r0.rotations = rot; r0.status = st;
    int st2 = extract_svd(C, Q, m, n, r0.normA, sig, U, V);
    if (rep) *rep = r0;
    free(Z); free(Zd); free(Q); free(C);
    return st ? st : st2;
}

/* Alg. 4 from C = A, V = I: the plain one-sided Jacobi SVD. */
int orc_plain_svd(const double *A, int m, int n, const orc_cfg *cfg, double *sig, double *U,
                  double *V, orc_report *rep)
{
    if (m < n) return 1;
    size_t mn = (size_t)m * n, nn = (size_t)n * n;
    orc_report r0; memset(&r0, 0, sizeof(r0));
    r0.normA = orc_fro_f64(A, m, n, m);
    double *C = (double *)malloc(sizeof(double) * mn), *W = (double *)calloc(nn, sizeof(double));
    memcpy(C, A, sizeof(double) * mn);
    for (int i = 0; i < n; ++i) W[IDX(i, i, n)] = 1.0;
    double off, tot;
    gram_norms(C, m, n, &off, &tot);
    r0.off0 = off;
    int sw = 0; long long rot = 0;
    int st = orc_jacobi_svd_f64(C, W, m, n, cfg->b, cfg->eps_factor * OMEGA, cfg->nu_factor * OMEGA,
                                cfg->early_stop, cfg->max_sweeps, &sw, &rot, r0.off_hist, r0.rot_hist);
    r0.sweeps = sw; r0.rotations = rot; r0.status = st;
    int st2 = extract_svd(C, W, m, n, r0.normA, sig, U, V);
    if (rep) *rep = r0;
    free(C); free(W);
    return st ? st : st2;
}

/* Batched Alg. 3: `batch` independent n x n matrices, contiguous.  The     */
/* oracle simply loops (OpenMP across matrices is the only parallelism).    */
int orc_mp_evd_batched(const double *A, int n, int batch, const orc_cfg *cfg, double *lam,
                       double *V, int *sweeps, int *sweeps_low)
{
    /* step 1 as cfg->low_solver says (symmetric QR by default, reading R12') */
    orc_cfg c1 = *cfg;
    int worst = 0;
    _Pragma("omp parallel for schedule(dynamic,1) reduction(max:worst)")
    for (int k = 0; k < batch; ++k) {
        orc_report rep;
        int st = orc_mp_evd(A + (size_t)k * n * n, n, &c1, NULL, lam + (size_t)k * n,
                            V + (size_t)k * n * n, &rep);
        if (sweeps) sweeps[k] = rep.sweeps;
        if (sweeps_low) sweeps_low[k] = rep.sweeps_low;
        if (st > worst) worst = st;
    }
    return worst;
}

size_t orc_report_size(void) { return sizeof(orc_report); }
size_t orc_cfg_size(void) { return sizeof(orc_cfg); }
