/*
 * timemg_b200 -- C ABI of the B200 time-multigrid slab-sweep library.
 *
 * The reference (arxiv/paper_1409_5254, Python package `timemg`) has no FFI:
 * its hot path is the private slab-kernel layer of pkg/src/timemg/multigrid.py
 * (signature style `(ops, omega, f, src, dst, a, b)`, in-place writes into
 * caller-owned arrays over slab ranges).  Each entry point below replaces one
 * of those functions (cited per declaration) for whole levels at once, for a
 * batch of independent problems that share one operator.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers owned by the caller; the library
 *    never frees them.  Layout: [batch][n_slabs][n_t], C-contiguous, slab
 *    major (the reference's (N, n_t) float64 arrays, multigrid.py:253-257),
 *    problem b at offset b * n_slabs * n_t.
 *  - dtype: TMG_F64 (bitwise parity with the reference) or TMG_F32.
 *  - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call is stream-ordered and asynchronous unless stated.
 *  - Return: 0 on success, a positive cudaError_t value for CUDA failures,
 *    or a negative TMG_E* code for argument errors.  tmg_last_error() gives a
 *    message for the calling thread.  Nothing throws across the ABI.
 *  - `active` (optional, may be NULL): int32 per problem; problems with
 *    active[b] == 0 are skipped (left untouched) -- the batched stopping mask.
 */
#ifndef TIMEMG_B200_H
#define TIMEMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TMG_MAXNT 8
#define TMG_F64 0
#define TMG_F32 1

#define TMG_E_ARG -1      /* invalid argument (reference raises ValueError) */
#define TMG_E_UNSUPPORTED -2
#define TMG_E_NOMEM -3

/* Per-level constants, copied verbatim from the reference objects:
 *   minus_step  = LocalOperators.minus_step_matrix      dg.py:213-215
 *   coupling    = LocalOperators.coupling               dg.py:236
 *   lu, perm    = BlockLU.lu / BlockLU.perm             dg.py:144-151
 *   omega       = resolve_damping(alpha(tau))           smoothing.py:24-54,
 *                                                       multigrid.py:339-341
 *   r1, r2      = Level.r1 / Level.r2 (transfers to the next coarser level,
 *                 zero on the coarsest level)           transfers.py:16-37
 * Matrices are row-major n_t x n_t in the first n_t*n_t entries. */
typedef struct tmg_level_desc {
    int32_t n_t;
    int32_t has_transfer;
    int64_t n_slabs;
    double omega;
    double minus_step[TMG_MAXNT * TMG_MAXNT];
    double coupling[TMG_MAXNT * TMG_MAXNT];
    double lu[TMG_MAXNT * TMG_MAXNT];
    double r1[TMG_MAXNT * TMG_MAXNT];
    double r2[TMG_MAXNT * TMG_MAXNT];
    int32_t perm[TMG_MAXNT];
} tmg_level_desc;

const char *tmg_last_error(void);
int tmg_version(void);
/* device capability probe: 0 if a GPU with sm_100 is usable */
int tmg_device_check(int device);

/* ---- slab kernels (one level, whole range [0, n_slabs)) -------------------- */

/* nu damped block-Jacobi sweeps, u_out = S^nu u_in.
 * Replaces block_jacobi_sweep / _sweep_slab (multigrid.py:168-180, 208-220).
 * u_in may equal NULL (zero initial guess).  u_in and u_out must not alias. */
int tmg_sweep(int dtype, const tmg_level_desc *lev, const void *f, const void *u_in, void *u_out,
              int64_t batch, int nu, const int32_t *active, void *stream);

/* r = f - L u  (the reference's ((-(K+M))u + f) + N u_prev order).
 * Replaces _residual_slab (multigrid.py:158-165). */
int tmg_residual(int dtype, const tmg_level_desc *lev, const void *f, const void *u, void *r,
                 int64_t batch, void *stream);

/* Fused down pass of one V-cycle level: nu1 sweeps, residual, restriction.
 *   u_out    = S^nu1 u_in                    (_sweep_slab x nu1, :274-277)
 *   f_coarse = R (f - L u_out)               (_residual_slab + _restrict_slab, :283-285)
 * u_in == NULL means the zero initial guess of a coarse level (:311-312).
 * The residual never reaches HBM. */
int tmg_down(int dtype, const tmg_level_desc *lev, const void *f, const void *u_in, void *u_out,
             void *f_coarse, int64_t batch, int nu1, const int32_t *active, void *stream);

/* Fused up pass: u_out = S^nu2 (u_in + P u_coarse)
 * (_prolong_add_slab + _sweep_slab x nu2, multigrid.py:317-327).
 * If sq_out != NULL the squared residual norm partials of u_out are written:
 * sq_out[b * n_slabs + n] = sum_j r[n,j]^2 (_sqnorm_slab, :193-197). */
int tmg_up(int dtype, const tmg_level_desc *lev, const void *f, const void *u_in,
           const void *u_coarse, void *u_out, double *sq_out, int64_t batch, int nu2,
           const int32_t *active, void *stream);

/* Exact coarsest-level solve L u = f.
 * method 0: block forward substitution, bitwise with _forward_substitute
 *           (multigrid.py:200-205); dot_variant selects the host-BLAS
 *           summation tree of `coupling @ u` (0 = OpenBLAS 0.3.30 trees of the
 *           golden host, 1 = sequential).
 * method 1: parallel associative scan of the rank-1 slab recurrence
 *           s_n = alpha s_{n-1} + e.LU^-1 f_n (not bitwise; ~1e-15 relative). */
int tmg_coarse_solve(int dtype, const tmg_level_desc *lev, const void *f, void *u,
                     int64_t batch, int method, int dot_variant, void *stream);

/* ||f - L u||_2 per problem with numpy's pairwise summation order
 * (norm_at, multigrid.py:447-462): norms_out[b] (device, float64). */
int tmg_resid_norm(int dtype, const tmg_level_desc *lev, const void *f, const void *u,
                   double *norms_out, int64_t batch, void *stream);

/* Raw numpy-order pairwise sum (no sqrt) of the per-slab squared residual
 * norms sum_j r[n,j]^2 over slabs [skip, n_slabs) of each problem:
 * sums_out[b] (device, float64).  One rank's share of norm_at
 * (multigrid.py:447-462) when a problem is sharded along time: a rank's slab
 * range preceded by `skip` halo slabs of its left neighbour (the residual of
 * the first owned slab couples to the last halo slab; the range is a subtree
 * of np.sum's pairwise recursion, so combining the ranks' sums in that tree
 * reproduces the single-device norm bit for bit). */
int tmg_resid_sqsum(int dtype, const tmg_level_desc *lev, const void *f, const void *u, int64_t skip,
                    double *sums_out, int64_t batch, void *stream);

/* Diagnostics: live per-kernel device times of the plan's own launches.
 * tmg_trace_enable(1) makes plans launch directly (no CUDA graph) with a CUDA
 * event recorded on the launch stream after every kernel; each finished solve
 * appends "kernel-description\tlaunches\ttotal_ms\n" lines (times between
 * consecutive events, i.e. kernel duration plus any launch gap) that
 * tmg_trace_read copies into buf (NUL-terminated, truncated to cap) and
 * clears.  Returns the text length.  tmg_trace_enable(0) restores graphs. */
int tmg_trace_enable(int on);
int64_t tmg_trace_read(char *buf, int64_t cap);

/* ---- right-hand side (rhs_moments, dg.py:265-287) ---------------------------
 * rhs[b][n][j] = sum_k fvals[b][n][k] * weights[j][k] (the fused multiply-add
 * chain from +0 of numpy's `fvals @ weights.T`, dg.py:284), then
 * rhs[b][0][j] += u0[b] * start[j] where u0[b] != 0 (dg.py:285-286).
 * nodes[s] (left Radau nodes c_k), weights[n_t * s] (tau * basis_values * b,
 * row-major) and start[n_t] (basis values at 0) are HOST arrays, the
 * reference's own; fvals, u0 (NULL = no initial value) and rhs are device
 * arrays.  s must equal n_t (the Radau rule, dg.py:276). */
int tmg_rhs_samples(const double *fvals, const double *u0, const double *nodes, const double *weights,
                    const double *start, int n_t, int s, double *rhs, int64_t n_slabs, int64_t batch,
                    void *stream);
/* The same moments of f(t) = sum_q amp[b][q] sin(freq[q] t / T + phase[b][q])
 * at t = t0 + (n + nodes[k]) tau, evaluated in the kernel (one launch for the
 * whole batch; freq[q] host, = 2 pi (q+1) as formed on the host).  CUDA's sin
 * (<= 2 ulp) stands in for the host libm: a few ulp from the host assembly. */
int tmg_rhs_sines(const double *amp, const double *phase, const double *u0, const double *freq, int n_terms,
                  double T, double tau, double t0, const double *nodes, const double *weights,
                  const double *start, int n_t, int s, double *rhs, int64_t n_slabs, int64_t batch,
                  void *stream);
const char *tmg_rhs_last_error(void);

/* ---- solver plan (the cycle / iteration driver, multigrid.py:263-500) ----- */

typedef struct tmg_plan tmg_plan;

typedef struct tmg_plan_opts {
    int32_t dtype;        /* TMG_F64 / TMG_F32 */
    int32_t nu1, nu2;     /* CycleConfig.nu1/nu2 */
    int32_t gamma;        /* cycle kind: 1 = V-cycle (reference), 2 = W-cycle, 3 = F-cycle */
    int32_t coarse;       /* 0 = serial (bitwise), 1 = scan, 2 = auto */
    int32_t dot_variant;  /* see tmg_coarse_solve */
    int32_t use_graph;    /* capture one cycle in a CUDA graph */
    int32_t tail_max_slabs; /* 0 = auto: levels with <= this many slabs per
                               problem run in the single-CTA engine */
} tmg_plan_opts;

/* levels: n_levels descriptors (the cycle depth), finest first. */
int tmg_plan_create(tmg_plan **plan, const tmg_level_desc *levels, int n_levels, int64_t batch,
                    const tmg_plan_opts *opts);
/* A batch of problems with DIFFERENT operators of the same shape (levels:
 * batch x n_levels descriptors, problem-major), e.g. a sweep of the two-grid
 * convergence factor over (p_t-fixed) step sizes and damping values
 * (measure_convergence_factor, multigrid.py:534-544; the paper's Fourier-vs-
 * measured experiment).  Supported when a whole problem fits one CTA
 * (TMG_E_UNSUPPORTED otherwise); solve/stats as for tmg_plan_create. */
int tmg_plan_create_multi(tmg_plan **plan, const tmg_level_desc *levels, int n_levels, int64_t batch,
                          const tmg_plan_opts *opts);
int tmg_plan_destroy(tmg_plan *plan);

/* One or more cycles without norms (v_cycle / two_grid_cycle,
 * multigrid.py:344-375): u is updated in place (u_in -> u_out). */
int tmg_plan_cycles(tmg_plan *plan, const void *f, void *u, int n_cycles, void *stream);

/* Iterate cycles until ||r_k|| <= max(eps ||r_0||, floor[b]) or max_iters
 * (_iterate, multigrid.py:427-500).  u: initial guess in, solution out.
 * floor_per_problem: host array [batch] (1e-12 * ||f_b||, multigrid.py:445).
 * Blocks until done. */
int tmg_plan_solve(tmg_plan *plan, const void *f, void *u, const double *floor_per_problem,
                   double eps, int max_iters, void *stream);

/* Host-buffer form of tmg_plan_solve -- the call a host-side binding of the
 * reference makes (numpy arrays in, numpy arrays out): f_host, u_init_host
 * (NULL = zero initial guess) and u_host are host arrays [batch][n_slabs][n_t]
 * (pinned memory gives full PCIe speed; u_init_host may equal u_host).
 * Copies in, solves, copies the solution into u_host; batches of >= 8
 * problems are pipelined in sub-batches on two streams so the PCIe copies of
 * one overlap the solve of the other.  Device buffers are owned by the plan.
 * Blocks until done. */
int tmg_plan_solve_host(tmg_plan *plan, const void *f_host, const void *u_init_host, void *u_host,
                        const double *floor_per_problem, double eps, int max_iters);

/* A stream of n_batches independent batches through host buffers, each
 * [batch][n_slabs][n_t] from the zero initial guess (the host-side call for
 * a producer of many right-hand-side batches): pipelined ACROSS batches --
 * batch k+1 is copied in and batch k-1 copied out while batch k is solved --
 * so in steady state a batch costs max(solve, H2D, D2H).  floor_per_problem:
 * [n_batches][batch]; results per batch: iterations[n_batches][batch],
 * norms[n_batches][batch][max_iters + 1], converged[n_batches][batch] (any of
 * the three may be NULL).  Blocks until every batch is done. */
int tmg_plan_solve_host_stream(tmg_plan *plan, int n_batches, const void *const *f_hosts, void *const *u_hosts,
                               const double *floor_per_problem, double eps, int max_iters, int32_t *iterations,
                               double *norms, int32_t *converged);

/* Results of the last tmg_plan_solve (host arrays):
 * iterations[batch], norms[batch * (max_iters + 1)] (first iterations[b]+1
 * valid per problem), converged[batch]. */
int tmg_plan_stats(const tmg_plan *plan, int32_t *iterations, double *norms, int32_t *converged);

/* Launch/timing info of the plan: number of kernels per cycle, number of
 * streaming (multi-CTA) levels, first tail level. */
int tmg_plan_info(const tmg_plan *plan, int32_t *kernels_per_cycle, int32_t *stream_levels,
                  int32_t *tail_level);

#ifdef __cplusplus
}
#endif
#endif /* TIMEMG_B200_H */
