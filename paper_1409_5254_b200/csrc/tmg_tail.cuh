// Single-CTA multilevel engine (coarse tail / whole small solves) and the
// serial coarse solve.
//
// Levels below a few thousand slabs are latency bound: a level pass costs
// less than a kernel launch.  One CTA per problem therefore runs the rest of
// the cycle -- every remaining level down to the coarsest solve and back --
// with the level arrays resident in shared memory and __syncthreads between
// phases (the reference's team barriers, multigrid.py:277-327).  For small
// problems (config 1, N = 2^10) the same engine runs the WHOLE solve
// (_iterate, multigrid.py:427-500) in one launch, residual norms included.
//
// Threads own contiguous, even-length chunks of slabs; a sweep first
// publishes each chunk's last old slab (the only cross-thread dependency),
// then updates the chunk in place.  Results are independent of the split.
#pragma once
#include "tmg_pairwise.cuh"
#include "tmg_types.cuh"

namespace tmg {


// ---------------------------------------------------------------------------
// coarse solve: block forward substitution (multigrid.py:200-205), one thread
// per problem; bitwise with the reference for the calibrated dot variant.
template <typename T, int NT, bool SPARSE>
__device__ void forward_substitute(const LevelC<T, NT> &L, const T *f, T *u, long long n,
                                   int variant)
{
    if (n <= 0) return;
    T x[NT], y[NT];
    load_slab_scalar<T, NT>(f, x);
    lu_solve<T, NT>(L, x, y);
#pragma unroll
    for (int j = 0; j < NT; ++j) u[j] = y[j];
    for (long long k = 1; k < n; ++k) {
        T b[NT];
#pragma unroll
        for (int i = 0; i < NT; ++i) b[i] = FP<T>::add(f[k * NT + i], blas_dot<T, NT>(L.C + i * NT, y, variant));
        lu_solve<T, NT>(L, b, y);
#pragma unroll
        for (int j = 0; j < NT; ++j) u[k * NT + j] = y[j];
    }
}

template <typename T, int NT, bool SPARSE>
__global__ void coarse_serial_kernel(const __grid_constant__ LevelC<T, NT> L, const T *f, T *u,
                                     long long n, int batch, int variant, const int *active)
{
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    if (active && !active[b]) return;
    forward_substitute<T, NT, SPARSE>(L, f + (size_t)b * n * NT, u + (size_t)b * n * NT, n, variant);
}

// ---------------------------------------------------------------------------
// the single-CTA engine

// Exact coarse solve L u = f as a CTA-wide associative scan of the rank-1
// slab recurrence (north star: "the coarsest-level forward solve done as a
// parallel associative scan"): with g_k = LU^-1 f_k and h_k = e.g_k,
//   s_k = alpha s_{k-1} + h_k,   u_k = g_k + s_{k-1} w      (s_{-1} = 0)
// Threads scan contiguous chunks, the chunk maps x -> A x + H are combined
// with a Hillis-Steele scan in shared memory, then each chunk is replayed with
// its incoming s.  Mathematically equal to _forward_substitute
// (multigrid.py:200-205) but associated differently: ~1e-15 relative, not
// bitwise.  |alpha| = |R(-tau)| <= 1 keeps it stable.  f may alias nothing;
// u receives the solution.  sA, sH: blockDim.x scratch values each.
template <typename T, int NT>
__device__ void cta_scan_solve(const LevelC<T, NT> &L, const T *f, T *u, long long n, T *sA, T *sH)
{
    const int t = threadIdx.x, P = blockDim.x;
    const long long m = (n + P - 1) / P;
    const long long a = min(n, (long long)t * m), e = min(n, a + m);
    T s = T(0), A = T(1);
    for (long long k = a; k < e; ++k) {
        T x[NT], g[NT];
        load_slab_scalar<T, NT>(f + k * NT, x);
        lu_solve<T, NT>(L, x, g);
        T h = FP<T>::mul(L.ce[0], g[0]);
#pragma unroll
        for (int j = 1; j < NT; ++j) h = FP<T>::fma(L.ce[j], g[j], h);
#pragma unroll
        for (int j = 0; j < NT; ++j) u[k * NT + j] = g[j];
        s = FP<T>::fma(L.calpha, s, h);
        A = FP<T>::mul(A, L.calpha);
    }
    sA[t] = A;
    sH[t] = s;
    __syncthreads();
    for (int off = 1; off < P; off <<= 1) {
        T pa = T(1), ph = T(0);
        if (t >= off) {
            pa = sA[t - off];
            ph = sH[t - off];
        }
        __syncthreads();
        if (t >= off) {
            // (A, H) o (pa, ph): x -> A (pa x + ph) + H
            sH[t] = FP<T>::fma(sA[t], ph, sH[t]);
            sA[t] = FP<T>::mul(sA[t], pa);
        }
        __syncthreads();
    }
    s = t == 0 ? T(0) : sH[t - 1];
    __syncthreads();
    for (long long k = a; k < e; ++k) {
        T g[NT];
        load_slab_scalar<T, NT>(u + k * NT, g);
        T h = FP<T>::mul(L.ce[0], g[0]);
#pragma unroll
        for (int j = 1; j < NT; ++j) h = FP<T>::fma(L.ce[j], g[j], h);
#pragma unroll
        for (int j = 0; j < NT; ++j) u[k * NT + j] = FP<T>::fma(s, L.cw[j], g[j]);
        s = FP<T>::fma(L.calpha, s, h);
    }
    __syncthreads();
}

template <typename T, int NT>
__global__ void __launch_bounds__(1024)
    coarse_scan_kernel(const __grid_constant__ LevelC<T, NT> L, const T *f, T *u, long long n, int batch,
                       const int *active)
{
    __shared__ T sA[1024], sH[1024];
    const int b = blockIdx.x;
    if (b >= batch || (active && !active[b])) return;
    cta_scan_solve<T, NT>(L, f + (size_t)b * n * NT, u + (size_t)b * n * NT, n, sA, sH);
}

template <typename T, int NT, bool SPARSE> struct Engine {
    const LevelC<T, NT> *L;  // shared copy
    T *u[MAXLEV];
    T *f[MAXLEV];
    long long n[MAXLEV];
    T *xch;        // [blockDim][NT+1]
    double *part;  // [blockDim]
    double *sq;    // [n0] (full mode)

    __device__ __forceinline__ void chunk(long long nn, long long &a, long long &e) const
    {
        long long m = (nn + blockDim.x - 1) / blockDim.x;
        m += m & 1;
        a = min(nn, (long long)threadIdx.x * m);
        e = min(nn, a + m);
    }
    __device__ __forceinline__ void put(const Cpl<T, NT, SPARSE> &c) const
    {
        T *x = xch + threadIdx.x * (NT + 1);
        if constexpr (SPARSE) {
            x[0] = c.s;
            x[1] = (T)c.m;
        } else {
#pragma unroll
            for (int j = 0; j < NT; ++j) x[j] = c.u[j];
        }
    }
    __device__ __forceinline__ Cpl<T, NT, SPARSE> get(int t) const
    {
        const T *x = xch + t * (NT + 1);
        Cpl<T, NT, SPARSE> c;
        if constexpr (SPARSE) {
            c.s = x[0];
            c.m = (unsigned)x[1];
        } else {
#pragma unroll
            for (int j = 0; j < NT; ++j) c.u[j] = x[j];
        }
        return c;
    }
    __device__ void publish_last(int l) const
    {
        long long a, e;
        chunk(n[l], a, e);
        if (a < e) {
            T x[NT];
            load_slab_scalar<T, NT>(u[l] + (e - 1) * NT, x);
            put(make_cpl<T, NT, SPARSE>(L[l], x));
        }
        __syncthreads();
    }
    __device__ void sweep_level(int l) const
    {
        publish_last(l);
        long long a, e;
        chunk(n[l], a, e);
        if (a < e) {
            const LevelC<T, NT> &Lv = L[l];
            Cpl<T, NT, SPARSE> prev;
            cpl_zero(prev);
            if (a > 0) prev = get(threadIdx.x - 1);
            for (long long k = a; k < e; ++k) {
                T x[NT], ff[NT];
                load_slab_scalar<T, NT>(u[l] + k * NT, x);
                load_slab_scalar<T, NT>(f[l] + k * NT, ff);
                Cpl<T, NT, SPARSE> own = make_cpl<T, NT, SPARSE>(Lv, x);
                sweep<T, NT, SPARSE>(Lv, x, ff, prev, k > 0);
#pragma unroll
                for (int j = 0; j < NT; ++j) u[l][k * NT + j] = x[j];
                prev = own;
            }
        }
        __syncthreads();
    }
    // residual + restriction into level l+1; zero initial guess there
    __device__ void restrict_level(int l) const
    {
        publish_last(l);
        long long a, e;
        chunk(n[l], a, e);
        const LevelC<T, NT> &Lv = L[l];
        const long long nc = n[l] >> 1;
        if (a < e) {
            Cpl<T, NT, SPARSE> prev;
            cpl_zero(prev);
            if (a > 0) prev = get(threadIdx.x - 1);
            for (long long c = a >> 1; c < (e >> 1) && c < nc; ++c) {
                T x0[NT], x1[NT], f0[NT], f1[NT], r0[NT], r1[NT], p0[NT], p1[NT];
                load_slab_scalar<T, NT>(u[l] + (2 * c) * NT, x0);
                load_slab_scalar<T, NT>(u[l] + (2 * c + 1) * NT, x1);
                load_slab_scalar<T, NT>(f[l] + (2 * c) * NT, f0);
                load_slab_scalar<T, NT>(f[l] + (2 * c + 1) * NT, f1);
                residual<T, NT, SPARSE>(Lv, x0, f0, prev, 2 * c > 0, r0);
                Cpl<T, NT, SPARSE> c0 = make_cpl<T, NT, SPARSE>(Lv, x0);
                residual<T, NT, SPARSE>(Lv, x1, f1, c0, true, r1);
                prev = make_cpl<T, NT, SPARSE>(Lv, x1);
                restrict_part<T, NT>(Lv, r0, false, p0);
                restrict_part<T, NT>(Lv, r1, true, p1);
#pragma unroll
                for (int i = 0; i < NT; ++i) {
                    f[l + 1][c * NT + i] = FP<T>::add(p0[i], p1[i]);
                    u[l + 1][c * NT + i] = T(0);
                }
            }
        }
        __syncthreads();
    }
    __device__ void prolong_level(int l) const
    {
        long long a, e;
        chunk(n[l], a, e);
        const LevelC<T, NT> &Lv = L[l];
        const long long nc = n[l] >> 1;
        for (long long c = a >> 1; c < (e >> 1) && c < nc; ++c) {
            T uc[NT], x0[NT], x1[NT];
            load_slab_scalar<T, NT>(u[l + 1] + c * NT, uc);
            load_slab_scalar<T, NT>(u[l] + (2 * c) * NT, x0);
            load_slab_scalar<T, NT>(u[l] + (2 * c + 1) * NT, x1);
            prolong_part<T, NT>(Lv, uc, false, x0);
            prolong_part<T, NT>(Lv, uc, true, x1);
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                u[l][(2 * c) * NT + j] = x0[j];
                u[l][(2 * c + 1) * NT + j] = x1[j];
            }
        }
        __syncthreads();
    }
    int scan = 0;  // coarsest solve: 0 = serial forward substitution (bitwise), 1 = scan

    __device__ void coarse_level(int l, int variant) const
    {
        if (scan) {
            cta_scan_solve<T, NT>(L[l], f[l], u[l], n[l], xch, xch + blockDim.x);
            return;
        }
        if (threadIdx.x == 0) forward_substitute<T, NT, SPARSE>(L[l], f[l], u[l], n[l], variant);
        __syncthreads();
    }
    // gamma-cycle from level l0 (multigrid.py:263-330); iterative, no recursion
    __device__ void cycle(int l0, int last, int nu1, int nu2, int gamma, int variant) const
    {
        int cnt[MAXLEV];
        int l = l0;
        for (int k = 0; k < nu1; ++k) sweep_level(l);
        restrict_level(l);
        cnt[l] = 0;
        while (true) {
            if (l + 1 == last) {
                coarse_level(last, variant);
                cnt[l] = gamma;
            }
            if (cnt[l] < gamma) {
                cnt[l] += 1;
                l += 1;
                for (int k = 0; k < nu1; ++k) sweep_level(l);
                restrict_level(l);
                cnt[l] = 0;
                continue;
            }
            prolong_level(l);
            for (int k = 0; k < nu2; ++k) sweep_level(l);
            if (l == l0) break;
            l -= 1;
        }
    }
    // ||f - L u|| at level l with numpy pairwise order (norm_at, :447-462)
    __device__ double norm(int l) const
    {
        publish_last(l);
        long long a, e;
        chunk(n[l], a, e);
        const LevelC<T, NT> &Lv = L[l];
        if (a < e) {
            Cpl<T, NT, SPARSE> prev;
            cpl_zero(prev);
            if (a > 0) prev = get(threadIdx.x - 1);
            for (long long k = a; k < e; ++k) {
                T x[NT], ff[NT], r[NT];
                load_slab_scalar<T, NT>(u[l] + k * NT, x);
                load_slab_scalar<T, NT>(f[l] + k * NT, ff);
                residual<T, NT, SPARSE>(Lv, x, ff, prev, k > 0, r);
                prev = make_cpl<T, NT, SPARSE>(Lv, x);
                sq[k] = (double)sqnorm<T, NT>(r);
            }
        }
        __syncthreads();
        return __dsqrt_rn(block_pairwise(sq, n[l], part));
    }
};


template <typename T, int NT, bool SPARSE>
__global__ void __launch_bounds__(TAIL_THREADS)
    tail_kernel(const __grid_constant__ TailArgs<T, NT> a)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int b = blockIdx.x;
    if (a.active && !a.active[b]) return;
    const int nlev = a.depth - a.l0;
    LevelC<T, NT> *Ls = reinterpret_cast<LevelC<T, NT> *>(smem);
    for (int i = threadIdx.x; i < (int)(sizeof(LevelC<T, NT>) * nlev / 4); i += blockDim.x)
        reinterpret_cast<uint32_t *>(Ls)[i] = reinterpret_cast<const uint32_t *>(a.levels + a.l0)[i];
    unsigned char *p = smem + sizeof(LevelC<T, NT>) * nlev;
    Engine<T, NT, SPARSE> E;
    E.L = Ls - a.l0;  // index by absolute level
    E.scan = a.coarse_scan;
    E.xch = reinterpret_cast<T *>(p);
    p += sizeof(T) * TAIL_THREADS * (NT + 1);
    E.part = reinterpret_cast<double *>(p);
    p += sizeof(double) * TAIL_THREADS;
    p = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
    T *store = a.in_smem ? reinterpret_cast<T *>(p) : a.gstore + (size_t)b * a.store_elems;
    for (int l = a.l0; l < a.depth; ++l) {
        E.n[l] = a.n[l];
        E.u[l] = store + a.off[l];
        E.f[l] = store + a.off[l] + a.n[l] * NT;
    }
    E.sq = reinterpret_cast<double *>(store + a.store_elems);
    __syncthreads();

    const long long n0 = a.n[a.l0];
    const long long ne = n0 * NT;
    const T *fin = a.f_in + (size_t)b * ne;
    for (long long i = threadIdx.x; i < ne; i += blockDim.x) {
        E.f[a.l0][i] = fin[i];
        E.u[a.l0][i] = a.u_in ? a.u_in[(size_t)b * ne + i] : T(0);
    }
    __syncthreads();
    const int last = a.depth - 1;

    if (!a.full) {
        for (int c = 0; c < a.n_cycles; ++c) {
            if (a.l0 == last) E.coarse_level(last, a.dot_variant);
            else E.cycle(a.l0, last, a.nu1, a.nu2, a.gamma, a.dot_variant);
        }
    } else {
        // _iterate (multigrid.py:476-492) on one problem
        double *hist = a.hist + (size_t)b * (a.max_iters + 1);
        double r0 = E.norm(a.l0);
        double e = __dmul_rn(a.eps, r0);
        double tol = e > a.floor_[b] ? e : a.floor_[b];
        double rk = r0;
        int iters = 0;
        if (threadIdx.x == 0) hist[0] = r0;
        while (rk > tol && iters < a.max_iters) {
            E.cycle(a.l0, last, a.nu1, a.nu2, a.gamma, a.dot_variant);
            rk = E.norm(a.l0);
            iters += 1;
            if (threadIdx.x == 0) hist[iters] = rk;
        }
        if (threadIdx.x == 0 && a.st) {
            a.st[b].tol = tol;
            a.st[b].iters = iters;
            a.st[b].active = 0;
            a.st[b].converged = rk <= tol;
        }
    }
    __syncthreads();
    for (long long i = threadIdx.x; i < ne; i += blockDim.x) a.u_out[(size_t)b * ne + i] = E.u[a.l0][i];
}

}  // namespace tmg
