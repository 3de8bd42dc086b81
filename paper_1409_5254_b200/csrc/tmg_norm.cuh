// Residual-norm finalisation and the stopping rule (multigrid.py:445-496).
// Included by exactly one translation unit (tmg_api.cu).
#pragma once
#include "tmg_pairwise.cuh"
#include "tmg_types.cuh"

namespace tmg {

// sum of a perfect binary tree of `m` values (m a power of two) per problem,
// one CTA per problem, then the stopping-rule update.
//   mode 0: r0 (initialises tol/active), mode 1: after a cycle.
__global__ void __launch_bounds__(1024)
    finalize_leaves_kernel(const double *leaves, long long m, ProbState *st, double *hist,
                           int hist_stride, const double *floor_, double eps, int mode)
{
    pdl_trigger();
    pdl_wait();
    __shared__ double part[1024];
    const int b = blockIdx.x;
    if (mode == 1 && !st[b].active) return;
    const double *lv = leaves + (size_t)b * m;
    const int T = blockDim.x;
    const int t = threadIdx.x;
    double v = 0.0;
    long long per = m > T ? m / T : 1;
    int used = (int)(m > T ? T : m);
    if (t < used) {
        if (per <= 32) {
            // the thread's perfect subtree in registers, 16 leaves at a time:
            // all loads first (no dependent load chain), then log2 rounds of
            // left + right; per = 32 is two such halves
            const int p = (int)(per < 16 ? per : 16);
            double half[2] = {0.0, 0.0};
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                if (hh * 16 < per) {
                    double x[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) x[i] = i < p ? lv[(long long)t * per + hh * 16 + i] : 0.0;
#pragma unroll
                    for (int w = 1; w < 16; w <<= 1) {
                        if (w < p) {
#pragma unroll
                            for (int i = 0; i < 16; i += 2 * w) x[i] = __dadd_rn(x[i], x[i + w]);
                        }
                    }
                    half[hh] = x[0];
                }
            }
            v = per > 16 ? __dadd_rn(half[0], half[1]) : half[0];
        } else {
            // bottom-up perfect tree over [t*per, (t+1)*per)
            double stack[40];
            for (long long i = 0; i < per; ++i) {
                double x = lv[t * per + i];
                int l = 0;
                while ((i >> l) & 1) { x = __dadd_rn(stack[l], x); ++l; }
                stack[l] = x;
            }
            int top = 0;
            while ((1LL << top) < per) ++top;
            v = stack[top];
        }
    }
    // the threads' values: the same left + right tree, five levels per warp by
    // shuffles (lane l holds node l of the level when l % (2 s) == 0), then
    // the warps' sums by warp 0  (used is a power of two, as m and T are)
#pragma unroll
    for (int s2 = 1; s2 < 32; s2 <<= 1) {
        const double o = __shfl_down_sync(0xffffffffu, v, s2);
        if (s2 < used) v = __dadd_rn(v, o);
    }
    if ((t & 31) == 0) part[t >> 5] = v;
    __syncthreads();
    if (t < 32) {
        const int nw = (used + 31) >> 5;
        double w = t < nw ? part[t] : 0.0;
#pragma unroll
        for (int s2 = 1; s2 < 32; s2 <<= 1) {
            const double o = __shfl_down_sync(0xffffffffu, w, s2);
            if (s2 < nw) w = __dadd_rn(w, o);
        }
        if (t == 0) part[0] = w;
    }
    if (t == 0) {
        double nrm = __dsqrt_rn(part[0]);
        ProbState &p = st[b];
        if (mode == 0) {
            hist[(size_t)b * hist_stride] = nrm;
            double e = __dmul_rn(eps, nrm);
            p.tol = e > floor_[b] ? e : floor_[b];
            p.iters = 0;
            p.active = (nrm > p.tol) && (p.max_iters > 0);
            p.converged = nrm <= p.tol;
        } else {
            p.iters += 1;
            hist[(size_t)b * hist_stride + p.iters] = nrm;
            p.converged = nrm <= p.tol;
            p.active = (nrm > p.tol) && (p.iters < p.max_iters);
        }
    }
}

// raw pairwise sum (np.sum order, no sqrt) of sq[b * stride + skip, + cnt):
// one rank's share of the norm of a time-sharded problem (its slab range is a
// subtree of numpy's pairwise recursion)
__global__ void __launch_bounds__(1024)
    range_sum_kernel(const double *sq, long long stride, long long skip, long long cnt, double *out)
{
    __shared__ double part[1024];
    const int b = blockIdx.x;
    const double s = block_pairwise(sq + (size_t)b * stride + skip, cnt, part);
    if (threadIdx.x == 0) out[b] = s;
}

// generic (any n) exact pairwise over per-slab squares
__global__ void __launch_bounds__(1024)
    finalize_sq_kernel(const double *sq, long long n, ProbState *st, double *hist, int hist_stride,
                       const double *floor_, double eps, int mode, double *norm_out)
{
    __shared__ double part[1024];
    const int b = blockIdx.x;
    if (st && mode == 1 && !st[b].active) return;
    double s = block_pairwise(sq + (size_t)b * n, n, part);
    if (threadIdx.x == 0) {
        double nrm = __dsqrt_rn(s);
        if (norm_out) norm_out[b] = nrm;
        if (st) {
            ProbState &p = st[b];
            if (mode == 0) {
                hist[(size_t)b * hist_stride] = nrm;
                double e = __dmul_rn(eps, nrm);
                p.tol = e > floor_[b] ? e : floor_[b];
                p.iters = 0;
                p.active = (nrm > p.tol) && (p.max_iters > 0);
                p.converged = nrm <= p.tol;
            } else {
                p.iters += 1;
                hist[(size_t)b * hist_stride + p.iters] = nrm;
                p.converged = nrm <= p.tol;
                p.active = (nrm > p.tol) && (p.iters < p.max_iters);
            }
        }
    }
}

// publish the per-problem active flags for the next cycle's kernels and,
// inside the solve graph, set the while-node condition (any problem active)
__global__ void __launch_bounds__(256)
    set_active_kernel(const ProbState *st, int *active, int *any_out, int batch,
                      cudaGraphConditionalHandle h, int use_handle)
{
    pdl_trigger();
    pdl_wait();
    int any = 0;
    for (int b = threadIdx.x; b < batch; b += blockDim.x) {
        const int a = st[b].active;
        active[b] = a;
        any |= a;
    }
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) {
        if (any_out) *any_out = any;
        if (use_handle) cudaGraphSetConditional(h, any ? 1u : 0u);
    }
}

}  // namespace tmg
