// Per-slab arithmetic of the time-multigrid hot path, sm_100a.
//
// Every function here reproduces the float64 operation order of the
// reference (arxiv/paper_1409_5254, pkg/src/timemg/multigrid.py and dg.py)
// with explicitly rounded IEEE operations (__dmul_rn / __dadd_rn / __dsub_rn /
// __ddiv_rn; the library is also compiled with -fmad=false), so the GPU
// iterates are bit-identical to the reference's:
//   bmat           _block_apply  multigrid.py:145-155 (j ascending, mul then add)
//   residual       _residual_slab multigrid.py:158-165 : ((A u) + f) + N u_prev
//   lu_solve       BlockLU.solve_rows dg.py:153-168 (perm, forward, backward, /)
//   sweep          _sweep_slab   multigrid.py:168-180 : (LU^-1 r) * omega + u
//   restrict_part  _restrict_slab multigrid.py:183-185 : R1 r_2c + R2 r_2c+1
//   prolong_part   _prolong_add_slab multigrid.py:188-190 : u += R^T u_c
//   sqnorm         _sqnorm_slab  multigrid.py:193-197
//   blas_dot       `coupling @ x` in _forward_substitute multigrid.py:205
//
// Coupling.  For the default radau_lagrange basis the coupling block
// N = outer(eval_start, eval_end) has nonzeros only in row 0 (eval_start = e0)
// -- the "sparse" path: a slab needs ONE scalar from its predecessor,
// s = sum_j N[0,j] u_prev[j] (same order as the reference's row-0 product),
// plus the sign bits of u_prev, which fix the sign of the exact zeros the
// reference adds to rows >= 1 (r_i + (+-0)).  That keeps the result bitwise
// identical including signed zeros.  Any other coupling (scaled_legendre)
// takes the "general" path that exchanges the whole predecessor slab.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifdef TMG_NO_EXPECT
#define TMG_UNLIKELY(x) (x)
#else
#define TMG_UNLIKELY(x) __builtin_expect(!!(x), 0)
#endif

namespace tmg {

template <typename T> struct FP;
template <> struct FP<double> {
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
    static __device__ __forceinline__ double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
    static __device__ __forceinline__ double sqrt_(double a) { return __dsqrt_rn(a); }
    static __device__ __forceinline__ unsigned sbit(double x) {
        return (unsigned)((unsigned long long)__double_as_longlong(x) >> 63);
    }
    static __device__ __forceinline__ double zero(bool neg) { return neg ? -0.0 : 0.0; }
};
template <> struct FP<float> {
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
    static __device__ __forceinline__ float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
    static __device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
    static __device__ __forceinline__ unsigned sbit(float x) { return (unsigned)__float_as_uint(x) >> 31; }
    static __device__ __forceinline__ float zero(bool neg) { return neg ? -0.0f : 0.0f; }
};

// fp32 is a throughput variant (BASELINE config 5: normwise 1e-5 against the
// fp64 reference), not a parity path: its slab arithmetic uses fused
// multiply-adds and the precomputed damped inverse WK instead of the
// reference's separately rounded operations and LU divisions.
template <typename T> __host__ __device__ constexpr bool fast_fp() { return sizeof(T) == 4; }

// a / d, correctly rounded, for a divisor d known ahead of time with
// rinv = RN(1/d): q0 = RN(a rinv) is within ~2 ulp, one fma correction makes
// it faithful, and a second correction gives RN(a/d) exactly (Markstein's
// theorem: rinv correctly rounded + faithful q => q + (a - d q) rinv rounds to
// the correctly rounded quotient; the remainders are exact fma results).
// Outside a safe exponent window (zeros, subnormals, huge values) it defers to
// the IEEE division, so the result always equals FP<T>::div(a, d) bit for bit.
// the IEEE divisions of the rare paths, out of line: inline they are ~40
// instructions each, and the single-CTA engine alone had 387 copies (640 KB of
// code around a hot path of a few hundred instructions per level pass)
static __device__ __noinline__ double ddiv_cold(double a, double d) { return __ddiv_rn(a, d); }
static __device__ __noinline__ float fdiv_cold(float a, float d) { return __fdiv_rn(a, d); }

__device__ __forceinline__ double divq(double a, double d, double rinv)
{
    double q0 = __dmul_rn(a, rinv);
    double q1 = __fma_rn(__fma_rn(-q0, d, a), rinv, q0);
    double q2 = __fma_rn(__fma_rn(-q1, d, a), rinv, q1);
    const unsigned e = (unsigned)(__double2hiint(a) >> 20) & 0x7ffu;
    if (__builtin_expect(e - 123u >= 1800u, 0)) q2 = ddiv_cold(a, d);  // |a| outside [2^-900, 2^900)
    return q2;
}
__device__ __forceinline__ float divq(float a, float d, float rinv)
{
    float q0 = __fmul_rn(a, rinv);
    float q1 = __fmaf_rn(__fmaf_rn(-q0, d, a), rinv, q0);
    float q2 = __fmaf_rn(__fmaf_rn(-q1, d, a), rinv, q1);
    const unsigned e = (__float_as_uint(a) >> 23) & 0xffu;
    if (__builtin_expect(e - 28u >= 200u, 0)) q2 = fdiv_cold(a, d);  // |a| outside [2^-99, 2^101)
    return q2;
}

// branch-free variant: the caller ORs `bad` over a whole LU solve and redoes
// the solve with IEEE division when any lane of the warp hit the window edge
__device__ __forceinline__ double divq_nb(double a, double d, double rinv, unsigned &bad)
{
    double q0 = __dmul_rn(a, rinv);
    double q1 = __fma_rn(__fma_rn(-q0, d, a), rinv, q0);
    // exponent field in place (one LOP3); the caller-side OR folds into a max
    const unsigned e = (unsigned)__double2hiint(a) & 0x7ff00000u;
    bad |= (unsigned)(e - (123u << 20) >= (1800u << 20));
    return __fma_rn(__fma_rn(-q1, d, a), rinv, q1);
}
__device__ __forceinline__ float divq_nb(float a, float d, float rinv, unsigned &bad)
{
    float q0 = __fmul_rn(a, rinv);
    float q1 = __fmaf_rn(__fmaf_rn(-q0, d, a), rinv, q0);
    const unsigned e = (__float_as_uint(a) >> 23) & 0xffu;
    bad |= (unsigned)(e - 28u >= 200u);
    return __fmaf_rn(__fmaf_rn(-q1, d, a), rinv, q1);
}

// Per-level constants in the compute type (kernel parameter / shared memory).
template <typename T, int NT> struct LevelC {
    T A[NT * NT];   // minus_step_matrix  (dg.py:213-215)
    T C[NT * NT];   // coupling           (dg.py:236)
    T lu[NT * NT];  // BlockLU.lu         (dg.py:145)
    T rinv[NT];     // RN(1 / lu[i,i]): divisor reciprocals for divq
    T PA[NT * NT];  // rows of A in LU-permutation order: PA[i] = A[perm[i]]
    T R1[NT * NT];  // Level.r1           (transfers.py:16-37)
    T R2[NT * NT];  // Level.r2
    T omega;        // resolve_damping(alpha(tau))
    // fp32 fast form (no parity order to keep): WK = omega (K+M)^-1 P^T, so the
    // damped update of a permuted residual y is u += WK y (FMA, no divisions)
    T WK[NT * NT];
    int perm[NT];   // BlockLU.perm       (dg.py:148-151)
    unsigned cneg[NT];  // sign bits of coupling row i (sparse path)
    int has_transfer;
    // rank-1 form of the coupling N = c e^T for the scan coarse solve:
    // s_k = e.u_k obeys s_k = calpha s_{k-1} + e.LU^-1 f_k and
    // u_k = LU^-1 f_k + s_{k-1} cw with cw = LU^-1 c, calpha = e.cw
    T ce[NT];
    T cw[NT];
    T calpha;
    double calpha_lo;  // alpha - calpha (double-double tail, for the grid-wide scan)
    int scan_ok;
};

// What a slab needs from its predecessor.
template <typename T, int NT, bool SPARSE> struct Cpl;
template <typename T, int NT> struct Cpl<T, NT, true> {
    T s;         // sum_j C[0,j] u_prev[j]
    unsigned m;  // sign bits of u_prev
};
template <typename T, int NT> struct Cpl<T, NT, false> {
    T u[NT];
};

template <typename T, int NT>
__device__ __forceinline__ void bmat(const T *M, const T (&x)[NT], T (&o)[NT])
{
    if constexpr (fast_fp<T>()) {
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            T a = M[i * NT] * x[0];
#pragma unroll
            for (int j = 1; j < NT; ++j) a = __fmaf_rn(M[i * NT + j], x[j], a);
            o[i] = a;
        }
        return;
    }
#pragma unroll
    for (int i = 0; i < NT; ++i) {
        T a = FP<T>::mul(M[i * NT], x[0]);
#pragma unroll
        for (int j = 1; j < NT; ++j) a = FP<T>::add(a, FP<T>::mul(M[i * NT + j], x[j]));
        o[i] = a;
    }
}

// Signed zeros of the sparse coupling.  Row i >= 1 of the reference's
// residual is r_i = ((A u)_i + f_i) + z_i with z_i = sum_j (+-0 * u_prev[j]) a
// signed zero; adding it changes r_i only when (A u)_i + f_i is -0, which in
// round-to-nearest needs f_i = -0.  So when no f_i (i >= 1) of the slabs at
// hand is -0 ("SZ = false", checked once per row of slabs), z_i is skipped
// and the predecessor's sign bits are not needed at all; otherwise (SZ =
// true) they are tracked exactly as before.  Both give the reference's bits.
template <typename T, int NT>
__device__ __forceinline__ bool neg_zero_rows(const T (&f)[NT])
{
    bool any = false;
    if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int i = 1; i < NT; ++i)
            any |= (unsigned long long)__double_as_longlong((double)f[i]) == 0x8000000000000000ull;
    }
    return any;
}

template <typename T, int NT, bool SPARSE, bool SZ = true>
__device__ __forceinline__ Cpl<T, NT, SPARSE> make_cpl(const LevelC<T, NT> &L, const T (&u)[NT])
{
    Cpl<T, NT, SPARSE> c;
    if constexpr (SPARSE && fast_fp<T>()) {
        T a = L.C[0] * u[0];
#pragma unroll
        for (int j = 1; j < NT; ++j) a = __fmaf_rn(L.C[j], u[j], a);
        c.s = a;
        c.m = 0;  // signed zeros are not tracked in the fast form
    } else if constexpr (SPARSE) {
        T a = FP<T>::mul(L.C[0], u[0]);
#pragma unroll
        for (int j = 1; j < NT; ++j) a = FP<T>::add(a, FP<T>::mul(L.C[j], u[j]));
        c.s = a;
        unsigned m = 0;
        if constexpr (SZ) {
#pragma unroll
            for (int j = 0; j < NT; ++j) m |= FP<T>::sbit(u[j]) << j;
        }
        c.m = m;
    } else {
#pragma unroll
        for (int j = 0; j < NT; ++j) c.u[j] = u[j];
    }
    return c;
}

template <typename T> __device__ __forceinline__ T shfl_up_t(T v, int d)
{
    return __shfl_up_sync(0xffffffffu, v, d);
}
template <typename T> __device__ __forceinline__ T shfl_t(T v, int src)
{
    return __shfl_sync(0xffffffffu, v, src);
}

template <typename T, int NT, bool SPARSE>
__device__ __forceinline__ Cpl<T, NT, SPARSE> cpl_shfl_up(const Cpl<T, NT, SPARSE> &c)
{
    Cpl<T, NT, SPARSE> o;
    if constexpr (SPARSE) {
        o.s = shfl_up_t(c.s, 1);
        o.m = shfl_up_t(c.m, 1);
    } else {
#pragma unroll
        for (int j = 0; j < NT; ++j) o.u[j] = shfl_up_t(c.u[j], 1);
    }
    return o;
}

template <typename T, int NT, bool SPARSE, bool SZ = true>
__device__ __forceinline__ Cpl<T, NT, SPARSE> cpl_shfl(const Cpl<T, NT, SPARSE> &c, int src)
{
    Cpl<T, NT, SPARSE> o;
    if constexpr (SPARSE) {
        o.s = shfl_t(c.s, src);
        o.m = SZ ? shfl_t(c.m, src) : 0u;
    } else {
#pragma unroll
        for (int j = 0; j < NT; ++j) o.u[j] = shfl_t(c.u[j], src);
    }
    return o;
}

template <typename T, int NT, bool SPARSE>
__device__ __forceinline__ void cpl_zero(Cpl<T, NT, SPARSE> &c)
{
    if constexpr (SPARSE) {
        c.s = T(0);
        c.m = 0;
    } else {
#pragma unroll
        for (int j = 0; j < NT; ++j) c.u[j] = T(0);
    }
}

template <typename T, int NT, bool SPARSE, bool SZ = true>
__device__ __forceinline__ void cpl_select(Cpl<T, NT, SPARSE> &dst, const Cpl<T, NT, SPARSE> &src,
                                           bool take)
{
    if constexpr (SPARSE) {
        dst.s = take ? src.s : dst.s;
        if constexpr (SZ) dst.m = take ? src.m : dst.m;
    } else {
#pragma unroll
        for (int j = 0; j < NT; ++j) dst.u[j] = take ? src.u[j] : dst.u[j];
    }
}

// r = ((A u) + f) [+ N u_prev if has_prev]   (multigrid.py:159-165)
template <typename T, int NT, bool SPARSE, bool SZ = true>
__device__ __forceinline__ void residual(const LevelC<T, NT> &L, const T (&u)[NT], const T (&f)[NT],
                                         const Cpl<T, NT, SPARSE> &p, bool has_prev, T (&r)[NT])
{
    if constexpr (fast_fp<T>()) {
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            T a = f[i];
#pragma unroll
            for (int j = 0; j < NT; ++j) a = __fmaf_rn(L.A[i * NT + j], u[j], a);
            r[i] = a;
        }
        if constexpr (SPARSE) {
            r[0] = has_prev ? r[0] + p.s : r[0];
        } else {
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                T a = r[i];
#pragma unroll
                for (int j = 0; j < NT; ++j) a = __fmaf_rn(L.C[i * NT + j], p.u[j], a);
                r[i] = has_prev ? a : r[i];
            }
        }
        return;
    }
    bmat<T, NT>(L.A, u, r);
#pragma unroll
    for (int i = 0; i < NT; ++i) r[i] = FP<T>::add(r[i], f[i]);
    if constexpr (SPARSE) {
        T r0 = FP<T>::add(r[0], p.s);
        r[0] = has_prev ? r0 : r[0];
        if constexpr (!SZ) return;  // no -0 among f[1..]: the zero terms change nothing
        const unsigned full = (1u << NT) - 1u;
#pragma unroll
        for (int i = 1; i < NT; ++i) {
            // the reference adds sum_j (+-0 * u_prev[j]): -0 iff every product is -0
            T ri = FP<T>::add(r[i], FP<T>::zero(((p.m ^ L.cneg[i]) & full) == full));
            r[i] = has_prev ? ri : r[i];
        }
    } else {
        T c[NT];
        bmat<T, NT>(L.C, p.u, c);
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            T ri = FP<T>::add(r[i], c[i]);
            r[i] = has_prev ? ri : r[i];
        }
    }
}

// y = LU^-1 r  (dg.py:153-168)
template <typename T, int NT>
__device__ __forceinline__ void lu_solve(const LevelC<T, NT> &L, const T (&r)[NT], T (&y)[NT])
{
    if constexpr (NT == 1) {
        y[0] = divq(r[0], L.lu[0], L.rinv[0]);
    } else {
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            T v = r[0];
#pragma unroll
            for (int q = 1; q < NT; ++q) v = (L.perm[i] == q) ? r[q] : v;
            y[i] = v;
        }
#pragma unroll
        for (int i = 1; i < NT; ++i)
#pragma unroll
            for (int j = 0; j < i; ++j) y[i] = FP<T>::sub(y[i], FP<T>::mul(L.lu[i * NT + j], y[j]));
#pragma unroll
        for (int i = NT - 1; i >= 0; --i) {
#pragma unroll
            for (int j = i + 1; j < NT; ++j) y[i] = FP<T>::sub(y[i], FP<T>::mul(L.lu[i * NT + j], y[j]));
            y[i] = divq(y[i], L.lu[i * NT + i], L.rinv[i]);
        }
    }
}

// one damped block-Jacobi update of slab n in place (multigrid.py:169-180).
// Branch-free divisions; the rare out-of-window numerator redoes the LU solve
// with IEEE division (one branch per slab instead of one per division).
template <typename T, int NT, bool SPARSE>
__device__ __forceinline__ void sweep(const LevelC<T, NT> &L, T (&u)[NT], const T (&f)[NT],
                                      const Cpl<T, NT, SPARSE> &p, bool has_prev);

// lane-selected transfer product: odd ? R2 r : R1 r   (multigrid.py:184-185)
template <typename T, int NT>
__device__ __forceinline__ void restrict_part(const LevelC<T, NT> &L, const T (&r)[NT], bool odd,
                                              T (&o)[NT])
{
#pragma unroll
    for (int i = 0; i < NT; ++i) {
        T a = FP<T>::mul(odd ? L.R2[i * NT] : L.R1[i * NT], r[0]);
#pragma unroll
        for (int j = 1; j < NT; ++j)
            a = FP<T>::add(a, FP<T>::mul(odd ? L.R2[i * NT + j] : L.R1[i * NT + j], r[j]));
        o[i] = a;
    }
}

// u += (odd ? R2 : R1)^T uc   (multigrid.py:189-190)
template <typename T, int NT>
__device__ __forceinline__ void prolong_part(const LevelC<T, NT> &L, const T (&uc)[NT], bool odd,
                                             T (&u)[NT])
{
#pragma unroll
    for (int i = 0; i < NT; ++i) {
        T a = FP<T>::mul(odd ? L.R2[i] : L.R1[i], uc[0]);
#pragma unroll
        for (int j = 1; j < NT; ++j) a = FP<T>::add(a, FP<T>::mul(odd ? L.R2[j * NT + i] : L.R1[j * NT + i], uc[j]));
        u[i] = FP<T>::add(u[i], a);
    }
}

template <typename T, int NT> __device__ __forceinline__ T sqnorm(const T (&r)[NT])
{
    if constexpr (fast_fp<T>()) {
        T a = r[0] * r[0];
#pragma unroll
        for (int j = 1; j < NT; ++j) a = __fmaf_rn(r[j], r[j], a);
        return a;
    }
    T a = FP<T>::mul(r[0], r[0]);
#pragma unroll
    for (int j = 1; j < NT; ++j) a = FP<T>::add(a, FP<T>::mul(r[j], r[j]));
    return a;
}

// One row of `coupling @ x` as numpy/OpenBLAS computes it (multigrid.py:205).
// variant 0: trees measured on the golden host (OpenBLAS 0.3.30); 1: sequential;
// 2: sequential FMA chain.  The host picks the variant by measuring its own
// numpy (paper_1409_5254_b200/blas_tree.py).
template <typename T, int NT>
__device__ __forceinline__ T blas_dot(const T *a, const T (&x)[NT], int variant)
{
    T t;
    if (variant == 2) {
        t = FP<T>::mul(a[0], x[0]);
#pragma unroll
        for (int j = 1; j < NT; ++j) t = FP<T>::fma(a[j], x[j], t);
    } else if (variant == 1 || NT > 4) {
        t = FP<T>::mul(a[0], x[0]);
#pragma unroll
        for (int j = 1; j < NT; ++j) t = FP<T>::add(t, FP<T>::mul(a[j], x[j]));
    } else if constexpr (NT == 1) {
        t = FP<T>::mul(a[0], x[0]);
    } else if constexpr (NT == 2) {
        t = FP<T>::fma(a[0], x[0], FP<T>::mul(a[1], x[1]));
    } else if constexpr (NT == 3) {
        t = FP<T>::fma(a[2], x[2], FP<T>::fma(a[0], x[0], FP<T>::mul(a[1], x[1])));
    } else {
        T p0 = FP<T>::mul(a[0], x[0]), p1 = FP<T>::mul(a[1], x[1]);
        T p2 = FP<T>::mul(a[2], x[2]), p3 = FP<T>::mul(a[3 % NT], x[3 % NT]);
        t = FP<T>::add(FP<T>::add(p0, p2), FP<T>::add(p1, p3));
    }
    return FP<T>::add(t, T(0));
}

// ---- slab I/O helpers ------------------------------------------------------

template <typename T, int NT>
__device__ __forceinline__ void load_slab(const T *p, T (&x)[NT])
{
    if constexpr (sizeof(T) == 8 && NT % 2 == 0) {
#pragma unroll
        for (int j = 0; j < NT; j += 2) {
            double2 v = *reinterpret_cast<const double2 *>(p + j);
            x[j] = v.x;
            x[j + 1] = v.y;
        }
    } else if constexpr (sizeof(T) == 4 && NT == 4) {
        float4 v = *reinterpret_cast<const float4 *>(p);
        x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else if constexpr (sizeof(T) == 4 && NT == 2) {
        float2 v = *reinterpret_cast<const float2 *>(p);
        x[0] = v.x; x[1] = v.y;
    } else {
#pragma unroll
        for (int j = 0; j < NT; ++j) x[j] = p[j];
    }
}

template <typename T, int NT>
__device__ __forceinline__ void store_slab(T *p, const T (&x)[NT])
{
    if constexpr (sizeof(T) == 8 && NT % 2 == 0) {
#pragma unroll
        for (int j = 0; j < NT; j += 2) *reinterpret_cast<double2 *>(p + j) = make_double2(x[j], x[j + 1]);
    } else if constexpr (sizeof(T) == 4 && NT == 4) {
        *reinterpret_cast<float4 *>(p) = make_float4(x[0], x[1], x[2], x[3]);
    } else if constexpr (sizeof(T) == 4 && NT == 2) {
        *reinterpret_cast<float2 *>(p) = make_float2(x[0], x[1]);
    } else {
#pragma unroll
        for (int j = 0; j < NT; ++j) p[j] = x[j];
    }
}

template <typename T, int NT>
__device__ __forceinline__ void load_slab_scalar(const T *p, T (&x)[NT])
{
#pragma unroll
    for (int j = 0; j < NT; ++j) x[j] = p[j];
}

template <typename T, int NT> __device__ __forceinline__ void zero_slab(T (&x)[NT])
{
#pragma unroll
    for (int j = 0; j < NT; ++j) x[j] = T(0);
}

}  // namespace tmg

namespace tmg {

// ---- fast-path variants used by the streaming kernels ---------------------
// LU row permutation as a compile-time pattern: the reference's factors use
// perm = (1, 2, .., n_t-1, 0) for small steps and the identity for large ones
// (other patterns fall back to runtime selects).
enum PermKind { P_GEN = 0, P_ID = 1, P_ROT = 2 };

// y_i = r_{perm[i]} with r = ((A u) + f) [+ N u_prev]: each row computed in
// exactly the reference's order, just stored in the order the LU solve reads.
template <typename T, int NT, bool SPARSE, int PERM, bool SZ = true>
__device__ __forceinline__ void residual_perm(const LevelC<T, NT> &L, const T (&u)[NT], const T (&f)[NT],
                                              const Cpl<T, NT, SPARSE> &p, bool has_prev, T (&y)[NT])
{
    if constexpr (PERM == P_GEN || fast_fp<T>()) {
        T r[NT];
        residual<T, NT, SPARSE, SZ>(L, u, f, p, has_prev, r);
        if constexpr (PERM == P_ROT) {
#pragma unroll
            for (int i = 0; i < NT; ++i) y[i] = r[(i + 1) % NT];
            return;
        } else if constexpr (PERM == P_ID) {
#pragma unroll
            for (int i = 0; i < NT; ++i) y[i] = r[i];
            return;
        }
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            T v = r[0];
#pragma unroll
            for (int q = 1; q < NT; ++q) v = (L.perm[i] == q) ? r[q] : v;
            y[i] = v;
        }
    } else {
        const unsigned full = (1u << NT) - 1u;
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            const int src = (PERM == P_ROT) ? (i + 1) % NT : i;
            T a = FP<T>::mul(L.A[src * NT], u[0]);
#pragma unroll
            for (int j = 1; j < NT; ++j) a = FP<T>::add(a, FP<T>::mul(L.A[src * NT + j], u[j]));
            a = FP<T>::add(a, f[src]);
            T c;
            if constexpr (SPARSE) {
                if (!SZ && src != 0) {  // zero term skipped (see neg_zero_rows)
                    y[i] = a;
                    continue;
                }
                c = (src == 0) ? p.s : FP<T>::zero(((p.m ^ L.cneg[src]) & full) == full);
            } else {
                c = FP<T>::mul(L.C[src * NT], p.u[0]);
#pragma unroll
                for (int j = 1; j < NT; ++j) c = FP<T>::add(c, FP<T>::mul(L.C[src * NT + j], p.u[j]));
            }
            T ac = FP<T>::add(a, c);
            y[i] = has_prev ? ac : a;
        }
    }
}

// forward + backward substitution on an already permuted right-hand side
template <typename T, int NT> __device__ __forceinline__ void lu_apply(const LevelC<T, NT> &L, T (&y)[NT])
{
#pragma unroll
    for (int i = 1; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < i; ++j) y[i] = FP<T>::sub(y[i], FP<T>::mul(L.lu[i * NT + j], y[j]));
#pragma unroll
    for (int i = NT - 1; i >= 0; --i) {
#pragma unroll
        for (int j = i + 1; j < NT; ++j) y[i] = FP<T>::sub(y[i], FP<T>::mul(L.lu[i * NT + j], y[j]));
        y[i] = divq(y[i], L.lu[i * NT + i], L.rinv[i]);
    }
}

// LU solve with branch-free divisions; `bad` flags lanes that need the IEEE path
template <typename T, int NT>
__device__ __forceinline__ void lu_apply_nb(const LevelC<T, NT> &L, T (&y)[NT], unsigned &bad)
{
#pragma unroll
    for (int i = 1; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < i; ++j) y[i] = FP<T>::sub(y[i], FP<T>::mul(L.lu[i * NT + j], y[j]));
#pragma unroll
    for (int i = NT - 1; i >= 0; --i) {
#pragma unroll
        for (int j = i + 1; j < NT; ++j) y[i] = FP<T>::sub(y[i], FP<T>::mul(L.lu[i * NT + j], y[j]));
        y[i] = divq_nb(y[i], L.lu[i * NT + i], L.rinv[i], bad);
    }
}

// a / d, exact, for the fallback of the branch-free LU solves: a zero
// numerator gives the correctly signed zero a * RN(1/d) (sign(a) xor sign(d),
// as IEEE division) without the slow division; numerators outside the
// Markstein window take the IEEE division; the rest the two-correction form
__device__ __forceinline__ double divq_exact(double a, double d, double rinv)
{
    if (a == 0.0) return __dmul_rn(a, rinv);
    return divq(a, d, rinv);
}
__device__ __forceinline__ float divq_exact(float a, float d, float rinv)
{
    if (a == 0.0f) return __fmul_rn(a, rinv);
    return divq(a, d, rinv);
}

// exact LU solve (the fallback of lu_apply_nb when a numerator left the window)
template <typename T, int NT> __device__ __forceinline__ void lu_apply_fallback(const LevelC<T, NT> &L, T (&y)[NT])
{
#pragma unroll
    for (int i = 1; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < i; ++j) y[i] = FP<T>::sub(y[i], FP<T>::mul(L.lu[i * NT + j], y[j]));
#pragma unroll
    for (int i = NT - 1; i >= 0; --i) {
#pragma unroll
        for (int j = i + 1; j < NT; ++j) y[i] = FP<T>::sub(y[i], FP<T>::mul(L.lu[i * NT + j], y[j]));
        y[i] = divq_exact(y[i], L.lu[i * NT + i], L.rinv[i]);
    }
}

// exact-IEEE LU solve (the rare fallback of lu_apply_nb)
template <typename T, int NT> __device__ __forceinline__ void lu_apply_ieee(const LevelC<T, NT> &L, T (&y)[NT])
{
#pragma unroll
    for (int i = 1; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < i; ++j) y[i] = FP<T>::sub(y[i], FP<T>::mul(L.lu[i * NT + j], y[j]));
#pragma unroll
    for (int i = NT - 1; i >= 0; --i) {
#pragma unroll
        for (int j = i + 1; j < NT; ++j) y[i] = FP<T>::sub(y[i], FP<T>::mul(L.lu[i * NT + j], y[j]));
        y[i] = FP<T>::div(y[i], L.lu[i * NT + i]);
    }
}

// the exact fallback out of line: J permuted right-hand sides and the LU constants by value
template <typename T, int NT, int J> struct LuPack { T v[J][NT]; };
template <typename T, int NT> struct LuConst { T lu[NT * NT]; T rinv[NT]; };
template <typename T, int NT, int J>
__device__ __noinline__ LuPack<T, NT, J> lu_fallback_byvalue(LuPack<T, NT, J> y, LuConst<T, NT> c)
{
#pragma unroll 1
    for (int q = 0; q < J; ++q) {
#pragma unroll
        for (int i = 1; i < NT; ++i)
#pragma unroll
            for (int j = 0; j < i; ++j) y.v[q][i] = FP<T>::sub(y.v[q][i], FP<T>::mul(c.lu[i * NT + j], y.v[q][j]));
#pragma unroll
        for (int i = NT - 1; i >= 0; --i) {
#pragma unroll
            for (int j = i + 1; j < NT; ++j) y.v[q][i] = FP<T>::sub(y.v[q][i], FP<T>::mul(c.lu[i * NT + j], y.v[q][j]));
            y.v[q][i] = divq_exact(y.v[q][i], c.lu[i * NT + i], c.rinv[i]);
        }
    }
    return y;
}

// the same for one slab with the level constants behind a pointer (the
// single-CTA engine keeps them in shared memory): one pointer and n_t doubles
// per call site instead of n_t^2 + 2 n_t doubles
template <typename T, int NT>
__device__ __noinline__ LuPack<T, NT, 1> lu_fallback_ptr(const LevelC<T, NT> *L, LuPack<T, NT, 1> y)
{
#pragma unroll
    for (int i = 1; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < i; ++j) y.v[0][i] = FP<T>::sub(y.v[0][i], FP<T>::mul(L->lu[i * NT + j], y.v[0][j]));
#pragma unroll
    for (int i = NT - 1; i >= 0; --i) {
#pragma unroll
        for (int j = i + 1; j < NT; ++j) y.v[0][i] = FP<T>::sub(y.v[0][i], FP<T>::mul(L->lu[i * NT + j], y.v[0][j]));
        y.v[0][i] = divq_exact(y.v[0][i], L->lu[i * NT + i], L->rinv[i]);
    }
    return y;
}

// LU solve + damped update for J slabs whose permuted residuals y are given
template <typename T, int NT, int J>
__device__ __forceinline__ void finish_j(const LevelC<T, NT> &L, T (&u)[J][NT], T (&y)[J][NT])
{
    if constexpr (fast_fp<T>()) {
#pragma unroll
        for (int q = 0; q < J; ++q)
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                T a = u[q][i];
#pragma unroll
                for (int j = 0; j < NT; ++j) a = __fmaf_rn(L.WK[i * NT + j], y[q][j], a);
                u[q][i] = a;
            }
        return;
    }
    T ys[J][NT];
    unsigned bad = 0;
#pragma unroll
    for (int q = 0; q < J; ++q)
#pragma unroll
        for (int i = 0; i < NT; ++i) ys[q][i] = y[q][i];
#pragma unroll
    for (int q = 0; q < J; ++q) lu_apply_nb<T, NT>(L, y[q], bad);
    if (TMG_UNLIKELY(__any_sync(0xffffffffu, bad))) {
#ifndef TMG_INLINE_FALLBACK
      if constexpr (NT <= 2) {
        // out of line, so the hot loop's code stays dense (-3 % on the headline;
        // n_t >= 3 would pass 20+ doubles and measured 5 % slower: inline there).
        // Operands by value in registers: passing them through a local-memory
        // block instead measured 4 % SLOWER (ptxas then reloads the level
        // constants with LDC in the hot path).
        LuPack<T, NT, J> in;
        LuConst<T, NT> lc;
#pragma unroll
        for (int i = 0; i < NT * NT; ++i) lc.lu[i] = L.lu[i];
#pragma unroll
        for (int i = 0; i < NT; ++i) lc.rinv[i] = L.rinv[i];
#pragma unroll
        for (int q = 0; q < J; ++q)
#pragma unroll
            for (int i = 0; i < NT; ++i) in.v[q][i] = ys[q][i];
        LuPack<T, NT, J> out = lu_fallback_byvalue<T, NT, J>(in, lc);
#pragma unroll
        for (int q = 0; q < J; ++q)
#pragma unroll
            for (int i = 0; i < NT; ++i) y[q][i] = out.v[q][i];
      } else
#endif
      {
#pragma unroll
        for (int q = 0; q < J; ++q) {
#pragma unroll
            for (int i = 0; i < NT; ++i) y[q][i] = ys[q][i];
            lu_apply_fallback<T, NT>(L, y[q]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < J; ++q)
#pragma unroll
        for (int i = 0; i < NT; ++i) u[q][i] = FP<T>::add(FP<T>::mul(y[q][i], L.omega), u[q][i]);
}

// J independent slabs (one per row of a stage) swept together: two dependency
// chains per lane hide the fp64 latency of the strictly ordered arithmetic
template <typename T, int NT, bool SPARSE, int PERM, int J, bool SZ = true>
__device__ __forceinline__ void sweep_j(const LevelC<T, NT> &L, T (&u)[J][NT], const T (&f)[J][NT],
                                        const Cpl<T, NT, SPARSE> (&p)[J], const bool (&hp)[J])
{
    T y[J][NT];
#pragma unroll
    for (int q = 0; q < J; ++q) residual_perm<T, NT, SPARSE, PERM, SZ>(L, u[q], f[q], p[q], hp[q], y[q]);
    finish_j<T, NT, J>(L, u, y);
}

// the first sweep from the zero initial guess: with u = +0 the residual equals
// f up to the signs of zero entries, which cannot change any nonzero value of
// the LU solve, and the update (c omega) + (+0) maps every zero to +0 -- so
// u = (omega LU^-1 f) + 0 is bitwise the full sweep, without the matrix
// products and without the predecessor exchange
template <typename T, int NT, int PERM, int J>
__device__ __forceinline__ void sweep_zero_j(const LevelC<T, NT> &L, T (&u)[J][NT], const T (&f)[J][NT])
{
    T y[J][NT];
#pragma unroll
    for (int q = 0; q < J; ++q) {
        if constexpr (PERM == P_GEN) {
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                T v = f[q][0];
#pragma unroll
                for (int c = 1; c < NT; ++c) v = (L.perm[i] == c) ? f[q][c] : v;
                y[q][i] = v;
            }
        } else {
#pragma unroll
            for (int i = 0; i < NT; ++i) y[q][i] = f[q][(PERM == P_ROT) ? (i + 1) % NT : i];
        }
#pragma unroll
        for (int i = 0; i < NT; ++i) u[q][i] = T(0);
    }
    finish_j<T, NT, J>(L, u, y);
}

// undo the row permutation of residual_perm: r[perm[i]] = y[i]
template <typename T, int NT, int PERM>
__device__ __forceinline__ void unpermute(const LevelC<T, NT> &L, const T (&y)[NT], T (&r)[NT])
{
    if constexpr (PERM == P_ROT) {
#pragma unroll
        for (int j = 0; j < NT; ++j) r[j] = y[(j + NT - 1) % NT];
    } else if constexpr (PERM == P_ID) {
#pragma unroll
        for (int j = 0; j < NT; ++j) r[j] = y[j];
    } else {
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            T v = y[0];
#pragma unroll
            for (int i = 1; i < NT; ++i) v = (L.perm[i] == j) ? y[i] : v;
            r[j] = v;
        }
    }
}

template <typename T, int NT, bool SPARSE, int PERM>
__device__ __forceinline__ void sweep_p(const LevelC<T, NT> &L, T (&u)[NT], const T (&f)[NT],
                                        const Cpl<T, NT, SPARSE> &p, bool has_prev)
{
    T y[NT];
    residual_perm<T, NT, SPARSE, PERM>(L, u, f, p, has_prev, y);
    lu_apply<T, NT>(L, y);
#pragma unroll
    for (int i = 0; i < NT; ++i) u[i] = FP<T>::add(FP<T>::mul(y[i], L.omega), u[i]);
}

// transfer products with the lane's own block held in registers
template <typename T, int NT>
__device__ __forceinline__ void restrict_reg(const T (&R)[NT * NT], const T (&r)[NT], T (&o)[NT])
{
    if constexpr (fast_fp<T>()) {
        bmat<T, NT>(R, r, o);
        return;
    }
#pragma unroll
    for (int i = 0; i < NT; ++i) {
        T a = FP<T>::mul(R[i * NT], r[0]);
#pragma unroll
        for (int j = 1; j < NT; ++j) a = FP<T>::add(a, FP<T>::mul(R[i * NT + j], r[j]));
        o[i] = a;
    }
}
template <typename T, int NT>
__device__ __forceinline__ void prolong_reg(const T (&R)[NT * NT], const T (&uc)[NT], T (&u)[NT])
{
    if constexpr (fast_fp<T>()) {
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            T a = u[i];
#pragma unroll
            for (int j = 0; j < NT; ++j) a = __fmaf_rn(R[j * NT + i], uc[j], a);
            u[i] = a;
        }
        return;
    }
#pragma unroll
    for (int i = 0; i < NT; ++i) {
        T a = FP<T>::mul(R[i], uc[0]);
#pragma unroll
        for (int j = 1; j < NT; ++j) a = FP<T>::add(a, FP<T>::mul(R[j * NT + i], uc[j]));
        u[i] = FP<T>::add(u[i], a);
    }
}

template <typename T, int NT>
__device__ __forceinline__ void restrict_ptr(const T *R, const T (&r)[NT], T (&o)[NT])
{
    if constexpr (fast_fp<T>()) {
        bmat<T, NT>(R, r, o);
        return;
    }
#pragma unroll
    for (int i = 0; i < NT; ++i) {
        T a = FP<T>::mul(R[i * NT], r[0]);
#pragma unroll
        for (int j = 1; j < NT; ++j) a = FP<T>::add(a, FP<T>::mul(R[i * NT + j], r[j]));
        o[i] = a;
    }
}
template <typename T, int NT>
__device__ __forceinline__ void prolong_ptr(const T *R, const T (&uc)[NT], T (&u)[NT])
{
    if constexpr (fast_fp<T>()) {
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            T a = u[i];
#pragma unroll
            for (int j = 0; j < NT; ++j) a = __fmaf_rn(R[j * NT + i], uc[j], a);
            u[i] = a;
        }
        return;
    }
#pragma unroll
    for (int i = 0; i < NT; ++i) {
        T a = FP<T>::mul(R[i], uc[0]);
#pragma unroll
        for (int j = 1; j < NT; ++j) a = FP<T>::add(a, FP<T>::mul(R[j * NT + i], uc[j]));
        u[i] = FP<T>::add(u[i], a);
    }
}

// rotate-shuffle: lane l receives lane (l-1) mod 32's value; lane 0 receives
// lane 31's, i.e. exactly the carry the NEXT row's lane 0 needs
template <typename T, int NT, bool SPARSE>
__device__ __forceinline__ Cpl<T, NT, SPARSE> cpl_rot(const Cpl<T, NT, SPARSE> &c, int src)
{
    return cpl_shfl<T, NT, SPARSE>(c, src);
}

template <typename T, int NT, bool SPARSE>
__device__ __forceinline__ void sweep(const LevelC<T, NT> &L, T (&u)[NT], const T (&f)[NT],
                                      const Cpl<T, NT, SPARSE> &p, bool has_prev)
{
    T y[NT], ys[NT];
    residual_perm<T, NT, SPARSE, P_GEN>(L, u, f, p, has_prev, y);
    if constexpr (fast_fp<T>()) {
        T uu[1][NT], yy[1][NT];
#pragma unroll
        for (int i = 0; i < NT; ++i) {
            uu[0][i] = u[i];
            yy[0][i] = y[i];
        }
        finish_j<T, NT, 1>(L, uu, yy);
#pragma unroll
        for (int i = 0; i < NT; ++i) u[i] = uu[0][i];
        return;
    }
#pragma unroll
    for (int i = 0; i < NT; ++i) ys[i] = y[i];
    unsigned bad = 0;
    lu_apply_nb<T, NT>(L, y, bad);
    if (__builtin_expect(bad != 0, 0)) {
        // per thread (no warp vote: the single-CTA engine's chunks differ), out of line
        LuPack<T, NT, 1> in;
#pragma unroll
        for (int i = 0; i < NT; ++i) in.v[0][i] = ys[i];
        const LuPack<T, NT, 1> out = lu_fallback_ptr<T, NT>(&L, in);
#pragma unroll
        for (int i = 0; i < NT; ++i) y[i] = out.v[0][i];
    }
#pragma unroll
    for (int i = 0; i < NT; ++i) u[i] = FP<T>::add(FP<T>::mul(y[i], L.omega), u[i]);
}

}  // namespace tmg
