// Right-hand-side moments on the GPU: rhs_moments (reference dg.py:265-287)
//
//   rhs[n, j] = sum_k fvals[n, k] * weights[j, k]      (fvals @ weights.T)
//   fvals[n, k] = f(t0 + (n + c_k) tau)                 (left Radau nodes c_k)
//   rhs[0, j] += u0 * eval_start[j]                     (only when u0 != 0)
//
// with weights = tau * basis_values(c) * b (host, the reference's own array).
// Two entry points:
//  * tmg_rhs_samples: fvals given (e.g. a torch-evaluated forcing); the
//    product is the fused multiply-add chain from +0 that numpy's matmul
//    (OpenBLAS dgemm, small K) performs on the golden host, so host samples
//    give the reference's moments bit for bit (tests/test_gpu_scale_and_edges.py).
//  * tmg_rhs_sines: the benchmark problems' forcing
//    f(t) = sum_k amp_k sin(freq_k t / T + phase_k) evaluated in the kernel
//    (problems.py:make_forcing order: freq_k = RN(2 pi (k+1)) formed on the
//    host as numpy does, then RN(RN(freq_k t) / T) + phase_k, accumulated
//    from +0).  sin is CUDA's (<= 2 ulp) where numpy calls the host libm, so
//    the moments agree with the host assembly to a few ulp, not bitwise.
// One thread per (problem, slab); everything for a slab stays in registers
// and the slab's n_t moments are written once (HBM write-bound when the
// forcing is cheap; the sines make tmg_rhs_sines fp64-bound).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include <algorithm>
#include "timemg_b200.h"

namespace {

constexpr int RHS_MAXS = 8;      // quadrature nodes (s = n_t for the Radau rule)
constexpr int RHS_MAXNT = 8;
constexpr int RHS_MAXTERMS = 16;

struct RhsConst {
    double nodes[RHS_MAXS];
    double w[RHS_MAXNT * RHS_MAXS];  // weights[j][k], row-major n_t x s
    double start[RHS_MAXNT];
    double freq[RHS_MAXTERMS];
    double T, tau, t0;
    int n_t, s, n_terms, t_is_one;
};

thread_local std::string g_rhs_err;

int rfail(int code, const char *msg)
{
    g_rhs_err = msg;
    return code;
}

__device__ __forceinline__ double slab_time(const RhsConst &c, long long n, int k)
{
    // t0 + (n + c_k) * tau, numpy's order
    return __dadd_rn(c.t0, __dmul_rn(__dadd_rn((double)n, c.nodes[k]), c.tau));
}

template <int NT>
__device__ __forceinline__ void store_moments(double *dst, const double (&m)[NT])
{
    if constexpr (NT % 2 == 0) {
#pragma unroll
        for (int j = 0; j < NT; j += 2) *reinterpret_cast<double2 *>(dst + j) = make_double2(m[j], m[j + 1]);
    } else {
#pragma unroll
        for (int j = 0; j < NT; ++j) dst[j] = m[j];
    }
}

// u0 folded into slab 0: rhs[0] += u0 * eval_start (dg.py:285-286)
template <int NT>
__device__ __forceinline__ void fold_u0(const RhsConst &c, double u0, double (&m)[NT])
{
    if (u0 != 0.0) {
#pragma unroll
        for (int j = 0; j < NT; ++j) m[j] = __dadd_rn(m[j], __dmul_rn(u0, c.start[j]));
    }
}

// S consecutive samples of one slab (16-byte loads when the slab's samples
// are a multiple of 16 bytes and the array is 16-byte aligned)
template <int S> __device__ __forceinline__ void load_samples(const double *p, bool vec, double (&fv)[S])
{
    if constexpr (S % 2 == 0) {
        if (vec) {
#pragma unroll
            for (int k = 0; k < S; k += 2) {
                const double2 v = *reinterpret_cast<const double2 *>(p + k);
                fv[k] = v.x;
                fv[k + 1] = v.y;
            }
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < S; ++k) fv[k] = p[k];
}

// grid: x over the slabs of a problem (grid-stride), y over the problems
// (grid-stride) -- no integer division per element; one slab per thread and
// step, loads and stores of a warp contiguous
template <int NT, int S>
__global__ void __launch_bounds__(256) rhs_samples_kernel(const __grid_constant__ RhsConst c, const double *fvals,
                                                          const double *u0, double *rhs, long long n,
                                                          long long batch)
{
    const bool vec = (reinterpret_cast<uintptr_t>(fvals) & 15) == 0 && ((n * S) % 2 == 0 || batch == 1);
    for (long long b = blockIdx.y; b < batch; b += gridDim.y) {
        const double *fb = fvals + b * n * S;
        double *rb = rhs + b * n * NT;
        for (long long slab = (long long)blockIdx.x * blockDim.x + threadIdx.x; slab < n;
             slab += (long long)gridDim.x * blockDim.x) {
            double fv[S];
            load_samples<S>(fb + slab * S, vec, fv);
            double m[NT];
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < S; ++k) acc = __fma_rn(fv[k], c.w[j * S + k], acc);
                m[j] = acc;
            }
            if (slab == 0 && u0) fold_u0<NT>(c, u0[b], m);
            store_moments<NT>(rb + slab * NT, m);
        }
    }
}

template <int NT, int S>
__global__ void __launch_bounds__(256) rhs_sines_kernel(const __grid_constant__ RhsConst c, const double *amp,
                                                        const double *phase, const double *u0, double *rhs,
                                                        long long n, long long total)
{
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (long long)gridDim.x * blockDim.x) {
        const long long b = g / n;
        const long long slab = g - b * n;
        const double *a = amp + b * c.n_terms;
        const double *ph = phase + b * c.n_terms;
        double fv[S];
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const double t = slab_time(c, slab, k);
            double v = 0.0;
            for (int q = 0; q < c.n_terms; ++q) {
                double x = __dmul_rn(c.freq[q], t);
                if (!c.t_is_one) x = __ddiv_rn(x, c.T);
                x = __dadd_rn(x, ph[q]);
                v = __dadd_rn(v, __dmul_rn(a[q], sin(x)));
            }
            fv[k] = v;
        }
        double m[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < S; ++k) acc = __fma_rn(fv[k], c.w[j * S + k], acc);
            m[j] = acc;
        }
        if (slab == 0 && u0) fold_u0<NT>(c, u0[b], m);
        store_moments<NT>(rhs + g * NT, m);
    }
}

unsigned grid_for(long long total)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long blocks = (total + 255) / 256;
    const long long cap = (long long)sms * 8;  // 8 resident 256-thread CTAs per SM, grid-stride beyond
    return (unsigned)(blocks < cap ? blocks : cap);
}

template <int NT, int S, bool SINES>
int launch(const RhsConst &c, const double *fvals, const double *amp, const double *phase, const double *u0,
           double *rhs, long long n, long long total, cudaStream_t s)
{
    if (total == 0) return 0;
    const unsigned grid = grid_for(total);
    if constexpr (SINES) {
        rhs_sines_kernel<NT, S><<<grid, 256, 0, s>>>(c, amp, phase, u0, rhs, n, total);
    } else {
        // x: the slabs of one problem, y: problems; together about the same
        // number of CTAs as the flat grid
        const long long batch = total / n;
        const unsigned gx = (unsigned)std::min<long long>((n + 255) / 256, grid);
        const unsigned gy = (unsigned)std::min<long long>(batch, std::max<long long>(1, grid / gx));
        rhs_samples_kernel<NT, S><<<dim3(gx, std::min(gy, 65535u)), 256, 0, s>>>(c, fvals, u0, rhs, n, batch);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return rfail((int)e, cudaGetErrorString(e));
    return 0;
}

template <bool SINES>
int dispatch(const RhsConst &c, const double *fvals, const double *amp, const double *phase, const double *u0,
             double *rhs, long long n, long long total, cudaStream_t s)
{
    // the Radau rule has s = n_t nodes (dg.py:276); other (n_t, s) pairs are
    // not instantiated
    if (c.s != c.n_t) return rfail(TMG_E_UNSUPPORTED, "tmg_rhs: quadrature nodes s must equal n_t");
    switch (c.n_t) {
    case 1: return launch<1, 1, SINES>(c, fvals, amp, phase, u0, rhs, n, total, s);
    case 2: return launch<2, 2, SINES>(c, fvals, amp, phase, u0, rhs, n, total, s);
    case 3: return launch<3, 3, SINES>(c, fvals, amp, phase, u0, rhs, n, total, s);
    case 4: return launch<4, 4, SINES>(c, fvals, amp, phase, u0, rhs, n, total, s);
    }
    return rfail(TMG_E_UNSUPPORTED, "tmg_rhs: n_t must be 1..4");
}

int fill_const(RhsConst &c, const double *nodes, const double *weights, const double *start, int n_t, int s)
{
    if (n_t < 1 || n_t > RHS_MAXNT || s < 1 || s > RHS_MAXS)
        return rfail(TMG_E_ARG, "tmg_rhs: n_t and s must lie in 1..8");
    if (!weights || !start || !nodes) return rfail(TMG_E_ARG, "tmg_rhs: null quadrature data");
    c = RhsConst{};
    for (int k = 0; k < s; ++k) c.nodes[k] = nodes[k];
    for (int i = 0; i < n_t * s; ++i) c.w[i] = weights[i];
    for (int j = 0; j < n_t; ++j) c.start[j] = start[j];
    c.n_t = n_t;
    c.s = s;
    return 0;
}

}  // namespace

extern "C" {

const char *tmg_rhs_last_error(void) { return g_rhs_err.c_str(); }

int tmg_rhs_samples(const double *fvals, const double *u0, const double *nodes, const double *weights,
                    const double *start, int n_t, int s, double *rhs, int64_t n_slabs, int64_t batch,
                    void *stream)
{
    RhsConst c;
    if (int e = fill_const(c, nodes, weights, start, n_t, s)) return e;
    if (n_slabs < 0 || batch < 0 || (!fvals && n_slabs * batch > 0) || !rhs)
        return rfail(TMG_E_ARG, "tmg_rhs_samples: bad sizes or null arrays");
    return dispatch<false>(c, fvals, nullptr, nullptr, u0, rhs, n_slabs, n_slabs * batch, (cudaStream_t)stream);
}

int tmg_rhs_sines(const double *amp, const double *phase, const double *u0, const double *freq, int n_terms,
                  double T, double tau, double t0, const double *nodes, const double *weights,
                  const double *start, int n_t, int s, double *rhs, int64_t n_slabs, int64_t batch,
                  void *stream)
{
    RhsConst c;
    if (int e = fill_const(c, nodes, weights, start, n_t, s)) return e;
    if (n_terms < 0 || n_terms > RHS_MAXTERMS) return rfail(TMG_E_ARG, "tmg_rhs_sines: 0..16 terms");
    if (!(T > 0.0) || !(tau > 0.0)) return rfail(TMG_E_ARG, "tmg_rhs_sines: T and tau must be positive");
    if (n_slabs < 0 || batch < 0 || !rhs || (n_terms > 0 && (!amp || !phase || !freq)))
        return rfail(TMG_E_ARG, "tmg_rhs_sines: bad sizes or null arrays");
    for (int q = 0; q < n_terms; ++q) c.freq[q] = freq[q];
    c.n_terms = n_terms;
    c.T = T;
    c.tau = tau;
    c.t0 = t0;
    c.t_is_one = T == 1.0;
    return dispatch<true>(c, nullptr, amp, phase, u0, rhs, n_slabs, n_slabs * batch, (cudaStream_t)stream);
}

}  // extern "C"
