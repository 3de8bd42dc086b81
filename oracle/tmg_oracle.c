/*
 * CPU ORACLE for the time-multigrid slab sweep -- TEST INFRASTRUCTURE ONLY.
 *
 * This file restates, in plain C, the arithmetic of the reference package's
 * hot path (arxiv/paper_1409_5254, `pkg/src/timemg/multigrid.py` and
 * `pkg/src/timemg/dg.py`), operation for operation, so that it reproduces the
 * reference's float64 results bit for bit.  It is used by `tests/` as the
 * parity checker, by `__graft_entry__.smoke()` as the checker and by
 * `bench.py` as the CPU baseline ("port") -- never by the product path.
 *
 * Rules that make the restatement bitwise (all verified against the golden
 * vectors in tests/golden, produced by running the reference itself):
 *   - every product and sum is a separately rounded IEEE double operation
 *     (compile with -ffp-contract=off, no -ffast-math);
 *   - block products sum over j in ascending order, first term is a product,
 *     then acc += mat[i,j]*x[j]           (multigrid.py:145-155);
 *   - residual order ((-(K+M)) u + f) + N u_prev   (multigrid.py:158-165);
 *   - LU solve: permute, forward, backward with true division (dg.py:153-168);
 *   - the coarse-grid `coupling @ out[n-1]` goes through OpenBLAS dgemv in the
 *     reference (multigrid.py:205); its summation tree is host dependent and is
 *     selected by `dot_variant` (see tmo_blas_dot_row);
 *   - norms: per-slab sum of squares (multigrid.py:193-197) followed by numpy's
 *     pairwise summation (np.sum, multigrid.py:459), restated in
 *     tmo_pairwise_sum.
 *
 * Parallelism: OpenMP over slabs inside each phase.  Every slab is computed by
 * the same code regardless of the thread that runs it, so results do not
 * depend on the thread count (the property the reference's worker team has,
 * multigrid.py:4-8).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TMO_MAXNT 8
#define TMO_MAXLEV 64
#define TMO_PAR_MIN 8192 /* below this many slabs a phase runs serially */

/* Per-level constants, copied verbatim from the reference objects:
 * A = LocalOperators.minus_step_matrix (dg.py:213-215), C = coupling
 * (dg.py:236), lu/perm = BlockLU (dg.py:144-151), omega = resolve_damping(
 * alpha(tau)) (smoothing.py:24-54), R1/R2 = build_transfers (transfers.py). */
typedef struct {
    int32_t nt;
    int32_t has_transfer;
    double A[TMO_MAXNT * TMO_MAXNT];
    double C[TMO_MAXNT * TMO_MAXNT];
    double lu[TMO_MAXNT * TMO_MAXNT];
    int32_t perm[TMO_MAXNT];
    double omega;
    double R1[TMO_MAXNT * TMO_MAXNT];
    double R2[TMO_MAXNT * TMO_MAXNT];
} tmo_level;

/* ---------------------------------------------------------------- slab math */

/* acc[i] = sum_j M[i,j] x[j], j ascending, mul then add (multigrid.py:148-151) */
static inline void block_acc(const double *M, int nt, const double *x, double *acc)
{
    for (int i = 0; i < nt; ++i) {
        double a = M[i * nt + 0] * x[0];
        for (int j = 1; j < nt; ++j) a += M[i * nt + j] * x[j];
        acc[i] = a;
    }
}

/* same with the transpose of M (prolongation uses r1.T, multigrid.py:189) */
static inline void block_acc_t(const double *M, int nt, const double *x, double *acc)
{
    for (int i = 0; i < nt; ++i) {
        double a = M[0 * nt + i] * x[0];
        for (int j = 1; j < nt; ++j) a += M[j * nt + i] * x[j];
        acc[i] = a;
    }
}

/* r = ((A u_n) + f_n) [+ C u_{n-1}]  -- multigrid.py:159-165 and 170-176 */
static inline void slab_residual(const tmo_level *L, const double *u, const double *f,
                                 const double *uprev, double *r)
{
    const int nt = L->nt;
    block_acc(L->A, nt, u, r);
    for (int i = 0; i < nt; ++i) r[i] += f[i];
    if (uprev) {
        double c[TMO_MAXNT];
        block_acc(L->C, nt, uprev, c);
        for (int i = 0; i < nt; ++i) r[i] += c[i];
    }
}

/* BlockLU.solve_rows for one row (dg.py:153-168), in place on y (= r on entry) */
static inline void slab_lu_solve(const tmo_level *L, const double *r, double *y)
{
    const int n = L->nt;
    const double *lu = L->lu;
    if (n == 1) {
        y[0] = r[0] / lu[0];
        return;
    }
    for (int i = 0; i < n; ++i) y[i] = r[L->perm[i]];
    for (int i = 1; i < n; ++i)
        for (int j = 0; j < i; ++j) y[i] -= lu[i * n + j] * y[j];
    for (int i = n - 1; i >= 0; --i) {
        for (int j = i + 1; j < n; ++j) y[i] -= lu[i * n + j] * y[j];
        y[i] /= lu[i * n + i];
    }
}

/* ------------------------------------------------------------ phase kernels */

/* _residual_slab (multigrid.py:158-165) over [a, b) */
void tmo_residual(const tmo_level *L, const double *f, const double *u, double *out,
                  int64_t a, int64_t b)
{
    const int nt = L->nt;
#pragma omp parallel for schedule(static) if (b - a >= TMO_PAR_MIN)
    for (int64_t n = a; n < b; ++n)
        slab_residual(L, u + n * nt, f + n * nt, n > 0 ? u + (n - 1) * nt : NULL, out + n * nt);
}

/* _sweep_slab (multigrid.py:168-180) over [a, b): dst = src + omega*LU^-1 r */
void tmo_sweep(const tmo_level *L, const double *f, const double *src, double *dst,
               int64_t a, int64_t b)
{
    const int nt = L->nt;
#pragma omp parallel for schedule(static) if (b - a >= TMO_PAR_MIN)
    for (int64_t n = a; n < b; ++n) {
        double r[TMO_MAXNT], c[TMO_MAXNT];
        slab_residual(L, src + n * nt, f + n * nt, n > 0 ? src + (n - 1) * nt : NULL, r);
        slab_lu_solve(L, r, c);
        for (int i = 0; i < nt; ++i) c[i] *= L->omega;
        for (int i = 0; i < nt; ++i) c[i] += src[n * nt + i];
        for (int i = 0; i < nt; ++i) dst[n * nt + i] = c[i];
    }
}

/* _restrict_slab (multigrid.py:183-185): coarse[c] = R1 fine[2c] + R2 fine[2c+1] */
void tmo_restrict(const tmo_level *L, const double *fine, double *coarse, int64_t ca, int64_t cb)
{
    const int nt = L->nt;
#pragma omp parallel for schedule(static) if (cb - ca >= TMO_PAR_MIN)
    for (int64_t c = ca; c < cb; ++c) {
        double a1[TMO_MAXNT], a2[TMO_MAXNT];
        block_acc(L->R1, nt, fine + (2 * c) * nt, a1);
        block_acc(L->R2, nt, fine + (2 * c + 1) * nt, a2);
        for (int i = 0; i < nt; ++i) coarse[c * nt + i] = a1[i] + a2[i];
    }
}

/* _prolong_add_slab (multigrid.py:188-190): fine[2c] += R1^T coarse[c], ... */
void tmo_prolong_add(const tmo_level *L, const double *coarse, double *fine, int64_t ca, int64_t cb)
{
    const int nt = L->nt;
#pragma omp parallel for schedule(static) if (cb - ca >= TMO_PAR_MIN)
    for (int64_t c = ca; c < cb; ++c) {
        double a1[TMO_MAXNT], a2[TMO_MAXNT];
        block_acc_t(L->R1, nt, coarse + c * nt, a1);
        block_acc_t(L->R2, nt, coarse + c * nt, a2);
        for (int i = 0; i < nt; ++i) fine[(2 * c) * nt + i] += a1[i];
        for (int i = 0; i < nt; ++i) fine[(2 * c + 1) * nt + i] += a2[i];
    }
}

/* _sqnorm_slab (multigrid.py:193-197) */
void tmo_sqnorm(const double *x, double *out, int nt, int64_t a, int64_t b)
{
#pragma omp parallel for schedule(static) if (b - a >= TMO_PAR_MIN)
    for (int64_t n = a; n < b; ++n) {
        double acc = x[n * nt] * x[n * nt];
        for (int j = 1; j < nt; ++j) acc += x[n * nt + j] * x[n * nt + j];
        out[n] = acc;
    }
}

/* numpy's pairwise summation as used by np.sum on a contiguous float64 vector
 * (the reduction in multigrid.py:459).  Blocks of <= 128 use eight
 * interleaved accumulators; larger ranges split at n/2 rounded down to a
 * multiple of 8.  Verified bit-exact against np.sum (tests/test_oracle.py). */
double tmo_pairwise_sum(const double *a, int64_t n)
{
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return tmo_pairwise_sum(a, n2) + tmo_pairwise_sum(a + n2, n - n2);
}

/* One row of `coupling @ x` as numpy computes it through OpenBLAS dgemv
 * (multigrid.py:205).  variant 0: the trees measured for OpenBLAS 0.3.30
 * (scipy-openblas, DYNAMIC_ARCH) on the Xeon host that produced the golden
 * vectors -- n=1: a0x0; n=2: fma(a0,x0,a1x1); n=3: fma(a2,x2,fma(a0,x0,a1x1));
 * n=4: (a0x0+a2x2)+(a1x1+a3x3); all results then get "+ 0.0" (rows of exact
 * zeros come out as +0).  variant 1: plain sequential mul/add.  variant 2:
 * sequential FMA chain t = fma(a_j, x_j, t).
 * Returns -1 status through *ok when the variant has no tree for n. */
double tmo_blas_dot_row(const double *a, const double *x, int n, int variant, int *ok)
{
    double t;
    *ok = 1;
    if (variant == 2) {
        t = a[0] * x[0];
        for (int j = 1; j < n; ++j) t = fma(a[j], x[j], t);
        return t + 0.0;
    }
    if (variant == 1 || n > 4) {
        if (variant != 1) *ok = 0;
        t = a[0] * x[0];
        for (int j = 1; j < n; ++j) t += a[j] * x[j];
        return t + 0.0;
    }
    switch (n) {
    case 1: t = a[0] * x[0]; break;
    case 2: t = fma(a[0], x[0], a[1] * x[1]); break;
    case 3: t = fma(a[2], x[2], fma(a[0], x[0], a[1] * x[1])); break;
    default: {
        double p0 = a[0] * x[0], p1 = a[1] * x[1], p2 = a[2] * x[2], p3 = a[3] * x[3];
        t = (p0 + p2) + (p1 + p3);
    }
    }
    return t + 0.0;
}

/* _forward_substitute (multigrid.py:200-205): exact block forward solve */
int tmo_forward_substitute(const tmo_level *L, const double *rhs, double *out, int64_t n,
                           int variant)
{
    const int nt = L->nt;
    int ok = 1;
    if (n <= 0) return 0;
    slab_lu_solve(L, rhs, out);
    for (int64_t k = 1; k < n; ++k) {
        double b[TMO_MAXNT];
        for (int i = 0; i < nt; ++i) {
            int ok_i;
            double cu = tmo_blas_dot_row(L->C + i * nt, out + (k - 1) * nt, nt, variant, &ok_i);
            ok &= ok_i;
            b[i] = rhs[k * nt + i] + cu;
        }
        slab_lu_solve(L, b, out + k * nt);
    }
    return ok ? 0 : 1;
}

/* The exact solution of the same block system (K+M) u_k = f_k + N u_{k-1}
 * (dg.py:290-303) in extended precision (x87 long double, 64-bit mantissa):
 * the yardstick for the parallel-scan solve, whose association differs from
 * the serial sweep's -- both are compared with this instead of with each
 * other when the recurrence is ill-conditioned (alpha -> 1 for small tau).
 * Not a restatement of reference arithmetic; test infrastructure only. */
int tmo_forward_substitute_ld(const tmo_level *L, const double *rhs, double *out, int64_t n)
{
    const int nt = L->nt;
    long double prev[TMO_MAXNT] = {0};
    for (int64_t k = 0; k < n; ++k) {
        long double y[TMO_MAXNT], b[TMO_MAXNT];
        for (int i = 0; i < nt; ++i) {
            long double c = 0.0L;
            if (k > 0)
                for (int j = 0; j < nt; ++j) c += (long double)L->C[i * nt + j] * prev[j];
            b[i] = (long double)rhs[k * nt + i] + c;
        }
        for (int i = 0; i < nt; ++i) y[i] = b[L->perm[i]];
        for (int i = 1; i < nt; ++i)
            for (int j = 0; j < i; ++j) y[i] -= (long double)L->lu[i * nt + j] * y[j];
        for (int i = nt - 1; i >= 0; --i) {
            for (int j = i + 1; j < nt; ++j) y[i] -= (long double)L->lu[i * nt + j] * y[j];
            y[i] /= (long double)L->lu[i * nt + i];
        }
        for (int i = 0; i < nt; ++i) {
            prev[i] = y[i];
            out[k * nt + i] = (double)y[i];
        }
    }
    return 0;
}

/* ------------------------------------------------------------------- cycles */

typedef struct {
    int depth;                 /* levels used by the cycle */
    const tmo_level *lev;      /* [depth] */
    const int64_t *n;          /* slabs per level */
    int nu1, nu2, gamma;       /* cycle kind: 1 V-cycle (reference); 2 W-cycle; 3 F-cycle */
    int dot_variant;
    double *u[TMO_MAXLEV][2];
    double *f[TMO_MAXLEV];
    double *r[TMO_MAXLEV];
} tmo_ws;

/* _cycle (multigrid.py:263-330), serial-slab form.  Kinds beyond the
 * reference's V-cycle (not in the reference, SPEC.md:430 -- these
 * compositions of the reference's own steps are the documented oracle for
 * them): W (kind 2) visits the coarser level twice, both visits W-cycles; F
 * (kind 3) visits it twice, an F-cycle and then a V-cycle.  The coarsest
 * level is solved once per visit of its parent whatever the kind. */
static int tmo_cycle_visits(int kind) { return kind == 1 ? 1 : 2; }
static int tmo_cycle_child(int kind, int visit) { return (kind == 3 && visit > 0) ? 1 : kind; }

static int tmo_cycle_rec(tmo_ws *w, int lev, int cur, int kind)
{
    const tmo_level *L = &w->lev[lev];
    const int nt = L->nt;
    const int64_t n = w->n[lev];
    for (int k = 0; k < w->nu1; ++k) {
        tmo_sweep(L, w->f[lev], w->u[lev][cur], w->u[lev][1 - cur], 0, n);
        cur ^= 1;
    }
    tmo_residual(L, w->f[lev], w->u[lev][cur], w->r[lev], 0, n);
    tmo_restrict(L, w->r[lev], w->f[lev + 1], 0, n / 2);
    int ccur;
    if (lev + 1 == w->depth - 1) {
        tmo_forward_substitute(&w->lev[lev + 1], w->f[lev + 1], w->u[lev + 1][0], w->n[lev + 1],
                               w->dot_variant);
        ccur = 0;
    } else {
        memset(w->u[lev + 1][0], 0, sizeof(double) * (size_t)(w->n[lev + 1] * nt));
        ccur = 0;
        for (int g = 0; g < tmo_cycle_visits(kind); ++g)
            ccur = tmo_cycle_rec(w, lev + 1, ccur, tmo_cycle_child(kind, g));
    }
    tmo_prolong_add(L, w->u[lev + 1][ccur], w->u[lev][cur], 0, n / 2);
    for (int k = 0; k < w->nu2; ++k) {
        tmo_sweep(L, w->f[lev], w->u[lev][cur], w->u[lev][1 - cur], 0, n);
        cur ^= 1;
    }
    return cur;
}

static int ws_alloc(tmo_ws *w)
{
    for (int l = 0; l < w->depth; ++l) {
        size_t sz = sizeof(double) * (size_t)(w->n[l] * w->lev[l].nt);
        w->u[l][0] = (double *)calloc(1, sz ? sz : 8);
        w->u[l][1] = (double *)calloc(1, sz ? sz : 8);
        w->f[l] = (double *)calloc(1, sz ? sz : 8);
        w->r[l] = (double *)calloc(1, sz ? sz : 8);
        if (!w->u[l][0] || !w->u[l][1] || !w->f[l] || !w->r[l]) return -1;
    }
    return 0;
}

static void ws_free(tmo_ws *w)
{
    for (int l = 0; l < w->depth; ++l) {
        free(w->u[l][0]);
        free(w->u[l][1]);
        free(w->f[l]);
        free(w->r[l]);
    }
}

/* One cycle from the finest level (v_cycle / two_grid_cycle via
 * _serial_cycle, multigrid.py:344-375): u_out = cycle(u_in, f). */
int tmo_cycle(const tmo_level *lev, const int64_t *n, int depth, int nu1, int nu2, int gamma,
              int dot_variant, const double *u_in, const double *f, double *u_out)
{
    if (depth < 2 || depth > TMO_MAXLEV || gamma < 1 || gamma > 3) return -1;
    tmo_ws w;
    memset(&w, 0, sizeof w);
    w.depth = depth; w.lev = lev; w.n = n;
    w.nu1 = nu1; w.nu2 = nu2; w.gamma = gamma; w.dot_variant = dot_variant;
    if (ws_alloc(&w)) { ws_free(&w); return -2; }
    size_t sz = sizeof(double) * (size_t)(n[0] * lev[0].nt);
    memcpy(w.u[0][0], u_in, sz);
    memcpy(w.f[0], f, sz);
    int cur = tmo_cycle_rec(&w, 0, 0, gamma);
    memcpy(u_out, w.u[0][cur], sz);
    ws_free(&w);
    return 0;
}

/* residual norm at the finest level: norm_at (multigrid.py:447-462) */
static double norm_at(tmo_ws *w, double *sq, int cur)
{
    const tmo_level *L = &w->lev[0];
    tmo_residual(L, w->f[0], w->u[0][cur], w->r[0], 0, w->n[0]);
    tmo_sqnorm(w->r[0], sq, L->nt, 0, w->n[0]);
    return sqrt(tmo_pairwise_sum(sq, w->n[0]));
}

/* _iterate (multigrid.py:427-500).  `floor_` is 1e-12*np.linalg.norm(f),
 * computed by the caller with numpy as the reference does (:445).
 * norms_out has room for max_iters+1 values; returns the iteration count. */
int tmo_iterate(const tmo_level *lev, const int64_t *n, int depth, int nu1, int nu2, int gamma,
                int dot_variant, const double *f, const double *u_init, double eps, double floor_,
                int max_iters, double *u_out, double *norms_out, int *n_norms)
{
    if (depth < 2 || depth > TMO_MAXLEV || gamma < 1 || gamma > 3) return -1;
    tmo_ws w;
    memset(&w, 0, sizeof w);
    w.depth = depth; w.lev = lev; w.n = n;
    w.nu1 = nu1; w.nu2 = nu2; w.gamma = gamma; w.dot_variant = dot_variant;
    if (ws_alloc(&w)) { ws_free(&w); return -2; }
    double *sq = (double *)malloc(sizeof(double) * (size_t)(n[0] ? n[0] : 1));
    size_t sz = sizeof(double) * (size_t)(n[0] * lev[0].nt);
    memcpy(w.u[0][0], u_init, sz);
    memcpy(w.f[0], f, sz);
    int cur = 0, iters = 0, k = 0;
    double r0 = norm_at(&w, sq, cur);
    norms_out[k++] = r0;
    double tol = eps * r0 > floor_ ? eps * r0 : floor_;
    double rk = r0;
    while (rk > tol && iters < max_iters) {
        cur = tmo_cycle_rec(&w, 0, cur, gamma);
        rk = norm_at(&w, sq, cur);
        iters += 1;
        norms_out[k++] = rk;
    }
    *n_norms = k;
    memcpy(u_out, w.u[0][cur], sz);
    free(sq);
    ws_free(&w);
    return iters;
}

/* block_jacobi_sweep (multigrid.py:208-220): nu sweeps with ping-pong */
int tmo_block_jacobi(const tmo_level *L, const double *u, const double *f, int64_t n, int nu,
                     double *out)
{
    size_t sz = sizeof(double) * (size_t)(n * L->nt);
    double *b0 = (double *)malloc(sz ? sz : 8), *b1 = (double *)malloc(sz ? sz : 8);
    if (!b0 || !b1) { free(b0); free(b1); return -2; }
    memcpy(b0, u, sz);
    double *buf[2] = {b0, b1};
    int cur = 0;
    for (int k = 0; k < nu; ++k) {
        tmo_sweep(L, f, buf[cur], buf[1 - cur], 0, n);
        cur ^= 1;
    }
    memcpy(out, buf[cur], sz);
    free(b0);
    free(b1);
    return 0;
}

/* The fused pass of BASELINE config 5, composed from the reference's own slab
 * functions: nu sweeps, residual, restriction (multigrid.py:274-285). */
int tmo_down_pass(const tmo_level *L, const double *u, const double *f, int64_t n, int nu,
                  double *u_out, double *f_coarse)
{
    size_t sz = sizeof(double) * (size_t)(n * L->nt);
    double *r = (double *)malloc(sz ? sz : 8);
    if (!r) return -2;
    int st = tmo_block_jacobi(L, u, f, n, nu, u_out);
    if (st) { free(r); return st; }
    tmo_residual(L, f, u_out, r, 0, n);
    tmo_restrict(L, r, f_coarse, 0, n / 2);
    free(r);
    return 0;
}

int tmo_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void tmo_set_num_threads(int t)
{
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}
