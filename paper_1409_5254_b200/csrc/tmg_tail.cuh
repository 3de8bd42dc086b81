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
__device__ __forceinline__ void group_sync(int P)
{
    if (P <= 32) __syncwarp();
    else __syncthreads();
}

template <typename T, int NT>
__device__ void cta_scan_solve(const LevelC<T, NT> &L, const T *f, T *u, long long n, T *sA, T *sH,
                               int P = 0)
{
    if (P == 0) P = blockDim.x;
    const int t = threadIdx.x;
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
    group_sync(P);
    for (int off = 1; off < P; off <<= 1) {
        T pa = T(1), ph = T(0);
        if (t >= off) {
            pa = sA[t - off];
            ph = sH[t - off];
        }
        group_sync(P);
        if (t >= off) {
            // (A, H) o (pa, ph): x -> A (pa x + ph) + H
            sH[t] = FP<T>::fma(sA[t], ph, sH[t]);
            sA[t] = FP<T>::mul(sA[t], pa);
        }
        group_sync(P);
    }
    s = t == 0 ? T(0) : sH[t - 1];
    group_sync(P);
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
    group_sync(P);
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

// dynamic shared memory of the tail kernel (all extern __shared__ arrays alias)
extern __shared__ __align__(128) unsigned char tmg_tail_smem[];

constexpr int WARP_MAX = 64;  // levels this small run in warp 0 only (no block barriers)
constexpr int TAIL_MAXNU = 4;

// Shared-memory layout (byte offsets from tmg_tail_smem):
//   LevelC[nlev] | int meta[4*nlev] (u, f, p offsets, n) | T scan scratch[2][TT]
//   | double part[TT] | level store (when SMEM): per level u, f, p (n*NT each)
//   | sq[n_l0] (full mode)
//
// Per level three arrays: f (right-hand side), p (the iterate after the
// pre-sweeps) and u (the level's result: iterate or coarse correction).  A
// level pass reads one set and writes another, so a pass needs ONE barrier
// and no halo publication: a thread re-derives the few slabs left of its
// chunk that its chunk depends on (Jacobi couples slab n to n-1 only; after
// k sweeps from a slab without its predecessor, every slab >= k further is
// exact), with the level constants in registers:
//   down(l):  nu1 sweeps (from zero, or from u) + residual + restriction ->
//             f(l+1), p(l) (+ the norm leaves of the INPUT's residual at l0)
//   up(l):    u(l) = S^nu2 (p(l) + P u(l+1))
// Levels of <= WARP_MAX slabs run in warp 0 with warp barriers only.
template <typename T, int NT, bool SPARSE, bool SMEM> struct Engine {
    using C = Cpl<T, NT, SPARSE>;
    int l0;            // first (finest) level handled here
    uint32_t o_meta, o_scan, o_part, o_store;
    T *gbase;          // level store in global memory (!SMEM)
    double *sq;        // per-slab squared residual norms of level l0 (full mode)
    int scan = 0;      // coarsest solve: 0 = serial forward substitution (bitwise), 1 = scan
    bool prev_warp = false;  // the previous pass ran in warp mode
    unsigned long long *trace = nullptr;  // [phase kind][level] cycle totals (thread 0 of block 0)
    long long t_mark = 0;

    // phase kinds for the trace: 0 down, 2 up, 3 coarse, 4 norm
    __device__ __forceinline__ void tick(int kind, int l)
    {
        if (trace && threadIdx.x == 0) {
            long long now = clock64();
            atomicAdd(trace + kind * MAXLEV + l, (unsigned long long)(now - t_mark));
            t_mark = now;
        }
    }

    __device__ __forceinline__ const LevelC<T, NT> &Lv(int l) const
    {
        return reinterpret_cast<const LevelC<T, NT> *>(tmg_tail_smem)[l - l0];
    }
    __device__ __forceinline__ const int *meta() const
    {
        return reinterpret_cast<const int *>(tmg_tail_smem + o_meta);
    }
    __device__ __forceinline__ T *arr(int off) const
    {
        if constexpr (SMEM) return reinterpret_cast<T *>(tmg_tail_smem + o_store) + off;
        else return gbase + off;
    }
    __device__ __forceinline__ T *U(int l) const { return arr(meta()[4 * (l - l0)]); }
    __device__ __forceinline__ T *F(int l) const { return arr(meta()[4 * (l - l0) + 1]); }
    __device__ __forceinline__ T *Pre(int l) const { return arr(meta()[4 * (l - l0) + 2]); }
    __device__ __forceinline__ int N(int l) const { return meta()[4 * (l - l0) + 3]; }
    __device__ __forceinline__ double *part() const
    {
        return reinterpret_cast<double *>(tmg_tail_smem + o_part);
    }

    // contiguous, even-length chunk of this thread at a level of n slabs
    __device__ __forceinline__ void chunk(int n, int &a, int &e) const
    {
        const int tt = (int)blockDim.x;
        int m = (n + tt - 1) / tt;
        m += m & 1;
        a = min(n, (int)threadIdx.x * m);
        e = min(n, a + m);
    }
    __device__ __forceinline__ static bool warp_level(int n) { return n <= WARP_MAX; }
    // entering a pass: block passes after warp-0 passes need a block barrier
    // first; in warp mode the other warps skip the pass
    __device__ __forceinline__ bool enter(int n)
    {
        const bool w = warp_level(n);
        if (!w && prev_warp) __syncthreads();
        prev_warp = w;
        return !w || threadIdx.x < 32;
    }
    __device__ __forceinline__ void leave(int n) const
    {
        if (warp_level(n)) __syncwarp();
        else __syncthreads();
    }
    __device__ __forceinline__ void load(const T *p, T (&x)[NT]) const
    {
#pragma unroll
        for (int j = 0; j < NT; ++j) x[j] = p[j];
    }
    __device__ __forceinline__ void store(T *p, const T (&x)[NT]) const
    {
#pragma unroll
        for (int j = 0; j < NT; ++j) p[j] = x[j];
    }

    // one damped sweep of two consecutive slabs (two dependency chains): the
    // pair's old values couple the second to the first; pin = the old value
    // of the slab before the pair.  Exact IEEE divisions when a numerator
    // leaves the Markstein window (per thread: no warp vote, chunks differ)
    __device__ __forceinline__ void sweep2(const LevelC<T, NT> &L, T (&x0)[NT], T (&x1)[NT], const T (&f0)[NT],
                                           const T (&f1)[NT], const C &pin, bool hp0, C &o1) const
    {
        const C o0 = make_cpl<T, NT, SPARSE>(L, x0);
        o1 = make_cpl<T, NT, SPARSE>(L, x1);
        sweep<T, NT, SPARSE>(L, x0, f0, pin, hp0);
        sweep<T, NT, SPARSE>(L, x1, f1, o0, true);
    }
    // the first sweep from the zero guess: u = (omega LU^-1 f) + 0 (bitwise
    // the full sweep, see sweep_zero_j)
    __device__ __forceinline__ void sweep_zero1(const LevelC<T, NT> &L, T (&x)[NT], const T (&f)[NT]) const
    {
        T u[1][NT], ff[1][NT];
#pragma unroll
        for (int i = 0; i < NT; ++i) ff[0][i] = f[i];
        if constexpr (fast_fp<T>()) {
            sweep_zero_j<T, NT, P_GEN, 1>(L, u, ff);
        } else {
            // per-thread IEEE fallback (sweep_zero_j votes over the warp)
            T y[NT], ys[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                T v = f[0];
#pragma unroll
                for (int c = 1; c < NT; ++c) v = (L.perm[i] == c) ? f[c] : v;
                y[i] = v;
                ys[i] = v;
            }
            unsigned bad = 0;
            lu_apply_nb<T, NT>(L, y, bad);
            if (__builtin_expect(bad != 0, 0)) {
                LuPack<T, NT, 1> in;
#pragma unroll
                for (int i = 0; i < NT; ++i) in.v[0][i] = ys[i];
                const LuPack<T, NT, 1> out = lu_fallback_ptr<T, NT>(&L, in);
#pragma unroll
                for (int i = 0; i < NT; ++i) y[i] = out.v[0][i];
            }
#pragma unroll
            for (int i = 0; i < NT; ++i) u[0][i] = FP<T>::add(FP<T>::mul(y[i], L.omega), T(0));
        }
#pragma unroll
        for (int i = 0; i < NT; ++i) x[i] = u[0][i];
    }

    // Levels of <= 64 slabs: warp 0, lane t owns the slab pair (2t, 2t+1);
    // the predecessor of a lane's first slab comes from lane t-1 by a
    // shuffle (no re-derived halo).  Lanes past the level compute on zeros
    // and store nothing; every lane takes part in the shuffles.
    __device__ void down_warp(int l, int n, bool zg, int nu, bool norm)
    {
        const int lane = threadIdx.x;
        const bool act = 2 * lane < n;
        const LevelC<T, NT> &L = Lv(l);
        const int j = 2 * lane;
        T x0[NT], x1[NT], f0[NT], f1[NT];
        zero_slab<T, NT>(x0);
        zero_slab<T, NT>(x1);
        zero_slab<T, NT>(f0);
        zero_slab<T, NT>(f1);
        if (act) {
            load(F(l) + j * NT, f0);
            load(F(l) + (j + 1) * NT, f1);
            if (!zg) {
                load(U(l) + j * NT, x0);
                load(U(l) + (j + 1) * NT, x1);
            }
        }
        const bool hp = lane > 0;
#pragma unroll
        for (int k = 0; k < TAIL_MAXNU; ++k) {
            if (k >= nu) break;
            if (k == 0 && zg) {
                if (act) {
                    sweep_zero1(L, x0, f0);
                    sweep_zero1(L, x1, f1);
                }
                continue;
            }
            const C o0 = make_cpl<T, NT, SPARSE>(L, x0);
            const C pin = cpl_shfl_up<T, NT, SPARSE>(make_cpl<T, NT, SPARSE>(L, x1));
            if (act) {
                if (k == 0 && norm) {
                    T r0[NT], r1[NT];
                    residual<T, NT, SPARSE>(L, x0, f0, pin, hp, r0);
                    residual<T, NT, SPARSE>(L, x1, f1, o0, true, r1);
                    sq[j] = (double)sqnorm<T, NT>(r0);
                    sq[j + 1] = (double)sqnorm<T, NT>(r1);
                }
                sweep<T, NT, SPARSE>(L, x0, f0, pin, hp);
                sweep<T, NT, SPARSE>(L, x1, f1, o0, true);
            }
        }
        T r0[NT], r1[NT];
        const C o0 = make_cpl<T, NT, SPARSE>(L, x0);
        const C pin = cpl_shfl_up<T, NT, SPARSE>(make_cpl<T, NT, SPARSE>(L, x1));
        residual<T, NT, SPARSE>(L, x0, f0, pin, hp, r0);
        residual<T, NT, SPARSE>(L, x1, f1, o0, true, r1);
        if (act) {
            if (norm && nu == 0) {
                sq[j] = (double)sqnorm<T, NT>(r0);
                sq[j + 1] = (double)sqnorm<T, NT>(r1);
            }
            store(Pre(l) + j * NT, x0);
            store(Pre(l) + (j + 1) * NT, x1);
            T p0[NT], p1[NT];
            restrict_part<T, NT>(L, r0, false, p0);
            restrict_part<T, NT>(L, r1, true, p1);
            T *fc = F(l + 1);
#pragma unroll
            for (int i = 0; i < NT; ++i) fc[lane * NT + i] = FP<T>::add(p0[i], p1[i]);
        }
        __syncwarp();
    }

    __device__ void up_warp(int l, int n, int nu)
    {
        const int lane = threadIdx.x;
        const bool act = 2 * lane < n;
        const LevelC<T, NT> &L = Lv(l);
        const int j = 2 * lane;
        T x0[NT], x1[NT], f0[NT], f1[NT];
        zero_slab<T, NT>(x0);
        zero_slab<T, NT>(x1);
        zero_slab<T, NT>(f0);
        zero_slab<T, NT>(f1);
        if (act) {
            T c[NT];
            load(Pre(l) + j * NT, x0);
            load(Pre(l) + (j + 1) * NT, x1);
            load(U(l + 1) + lane * NT, c);
            prolong_part<T, NT>(L, c, false, x0);
            prolong_part<T, NT>(L, c, true, x1);
            if (nu > 0) {
                load(F(l) + j * NT, f0);
                load(F(l) + (j + 1) * NT, f1);
            }
        }
        const bool hp = lane > 0;
#pragma unroll
        for (int k = 0; k < TAIL_MAXNU; ++k) {
            if (k >= nu) break;
            const C o0 = make_cpl<T, NT, SPARSE>(L, x0);
            const C pin = cpl_shfl_up<T, NT, SPARSE>(make_cpl<T, NT, SPARSE>(L, x1));
            if (act) {
                sweep<T, NT, SPARSE>(L, x0, f0, pin, hp);
                sweep<T, NT, SPARSE>(L, x1, f1, o0, true);
            }
        }
        if (act) {
            store(U(l) + j * NT, x0);
            store(U(l) + (j + 1) * NT, x1);
        }
        __syncwarp();
    }

    // down pass of level l (multigrid.py:274-285): nu sweeps from the zero
    // guess (zg) or from U(l), the residual, the restriction into F(l+1); the
    // pre-smoothed iterate into Pre(l).  norm: the per-slab squared residual
    // norms of the INPUT iterate (its first sweep's residual; norm_at,
    // :447-459) into sq.
    __device__ void down(int l, bool zg, int nu, bool norm)
    {
        const int n = N(l);
        if (warp_level(n)) {
            if (enter(n)) down_warp(l, n, zg, nu, norm);
            tick(0, l);
            return;
        }
        if (enter(n)) {
            int a, e;
            chunk(n, a, e);
            if (a < e) {
                const LevelC<T, NT> &L = Lv(l);
                int hs = max(0, a - (nu + 1)) & ~1;
                const T *f = F(l), *u = U(l);
                T *pre = Pre(l), *fc = F(l + 1);
                C cin[TAIL_MAXNU], cres;  // predecessor data per sweep / for the residual
#pragma unroll
                for (int k = 0; k < TAIL_MAXNU; ++k) cpl_zero(cin[k]);
                cpl_zero(cres);
                if (zg && nu == 1 && a > 0) {
                    // one sweep from the zero guess has no predecessor: all the
                    // chunk needs from its left is the swept slab a-1 (for the
                    // residual of slab a) -- one zero-guess sweep instead of a
                    // re-derived pair with its residuals
                    T fh[NT], xh[NT];
                    load(f + (a - 1) * NT, fh);
                    zero_slab<T, NT>(xh);
                    sweep_zero1(L, xh, fh);
                    cres = make_cpl<T, NT, SPARSE>(L, xh);
                    hs = a;
                }
                for (int j = hs; j < e; j += 2) {
                    T x0[NT], x1[NT], f0[NT], f1[NT];
                    load(f + j * NT, f0);
                    load(f + (j + 1) * NT, f1);
                    if (zg) {
                        zero_slab<T, NT>(x0);
                        zero_slab<T, NT>(x1);
                    } else {
                        load(u + j * NT, x0);
                        load(u + (j + 1) * NT, x1);
                    }
                    const bool hp = j > 0;
#pragma unroll
                    for (int k = 0; k < TAIL_MAXNU; ++k) {
                        if (k >= nu) break;
                        if (k == 0 && zg) {
                            sweep_zero1(L, x0, f0);
                            sweep_zero1(L, x1, f1);
                            continue;
                        }
                        if (k == 0 && norm && j >= a) {
                            T r0[NT], r1[NT];
                            const C o0 = make_cpl<T, NT, SPARSE>(L, x0);
                            residual<T, NT, SPARSE>(L, x0, f0, cin[0], hp, r0);
                            residual<T, NT, SPARSE>(L, x1, f1, o0, true, r1);
                            sq[j] = (double)sqnorm<T, NT>(r0);
                            sq[j + 1] = (double)sqnorm<T, NT>(r1);
                        }
                        C o1;
                        sweep2(L, x0, x1, f0, f1, cin[k], hp, o1);
                        cin[k] = o1;
                    }
                    T r0[NT], r1[NT];
                    const C o0 = make_cpl<T, NT, SPARSE>(L, x0);
                    residual<T, NT, SPARSE>(L, x0, f0, cres, hp, r0);
                    residual<T, NT, SPARSE>(L, x1, f1, o0, true, r1);
                    cres = make_cpl<T, NT, SPARSE>(L, x1);
                    if (j >= a) {
                        if (norm && nu == 0) {
                            sq[j] = (double)sqnorm<T, NT>(r0);
                            sq[j + 1] = (double)sqnorm<T, NT>(r1);
                        }
                        store(pre + j * NT, x0);
                        store(pre + (j + 1) * NT, x1);
                        T p0[NT], p1[NT];
                        restrict_part<T, NT>(L, r0, false, p0);
                        restrict_part<T, NT>(L, r1, true, p1);
#pragma unroll
                        for (int i = 0; i < NT; ++i) fc[(j >> 1) * NT + i] = FP<T>::add(p0[i], p1[i]);
                    }
                }
            }
            leave(n);
        }
        tick(0, l);
    }

    // up pass of level l (multigrid.py:317-327): u(l) = S^nu (Pre(l) + P u(l+1))
    __device__ void up(int l, int nu)
    {
        const int n = N(l);
        if (warp_level(n)) {
            if (enter(n)) up_warp(l, n, nu);
            tick(2, l);
            return;
        }
        if (enter(n)) {
            int a, e;
            chunk(n, a, e);
            if (a < e) {
                const LevelC<T, NT> &L = Lv(l);
                int hs = max(0, a - nu) & ~1;
                const T *f = F(l), *pre = Pre(l), *uc = U(l + 1);
                T *u = U(l);
                C cin[TAIL_MAXNU];
#pragma unroll
                for (int k = 0; k < TAIL_MAXNU; ++k) cpl_zero(cin[k]);
                if (nu == 1 && a > 0) {
                    // one post-sweep: the chunk needs only the prolongated
                    // (unswept) slab a-1 from its left -- no re-derived pair
                    T xh[NT], c[NT];
                    load(pre + (a - 1) * NT, xh);
                    load(uc + ((a - 1) >> 1) * NT, c);
                    prolong_part<T, NT>(L, c, true, xh);   // a is even: slab a-1 is odd
                    cin[0] = make_cpl<T, NT, SPARSE>(L, xh);
                    hs = a;
                }
                for (int j = hs; j < e; j += 2) {
                    T x0[NT], x1[NT], f0[NT], f1[NT], c[NT];
                    load(pre + j * NT, x0);
                    load(pre + (j + 1) * NT, x1);
                    load(uc + (j >> 1) * NT, c);
                    prolong_part<T, NT>(L, c, false, x0);
                    prolong_part<T, NT>(L, c, true, x1);
                    if (nu > 0) {
                        load(f + j * NT, f0);
                        load(f + (j + 1) * NT, f1);
                    }
                    const bool hp = j > 0;
#pragma unroll
                    for (int k = 0; k < TAIL_MAXNU; ++k) {
                        if (k >= nu) break;
                        C o1;
                        sweep2(L, x0, x1, f0, f1, cin[k], hp, o1);
                        cin[k] = o1;
                    }
                    if (j >= a) {
                        store(u + j * NT, x0);
                        store(u + (j + 1) * NT, x1);
                    }
                }
            }
            leave(n);
        }
        tick(2, l);
    }

    __device__ void coarse_level(int l, int variant)
    {
        const int n = N(l);
        if (scan) {
            if (prev_warp) __syncthreads();
            prev_warp = false;
            T *xs = reinterpret_cast<T *>(tmg_tail_smem + o_scan);
            cta_scan_solve<T, NT>(Lv(l), F(l), U(l), n, xs, xs + blockDim.x, (int)blockDim.x);
            tick(3, l);
            return;
        }
        if (enter(n)) {
            if (threadIdx.x == 0) forward_substitute<T, NT, SPARSE>(Lv(l), F(l), U(l), n, variant);
            leave(n);
        }
        tick(3, l);
    }

    // the rest of a cycle of the given kind (1 V, 2 W, 3 F) whose down pass
    // at lstart is done (multigrid.py:263-330 for V; W and F as the oracle's
    // tmo_cycle_rec: a W visits the coarser level twice with W-cycles, an F
    // with an F-cycle and then a V-cycle), iterative: cnt[l] = visits of
    // level l+1 so far, kd[l] = the kind of level l's current cycle
    __device__ static int visits(int kind) { return kind == 1 ? 1 : 2; }
    __device__ static int child_kind(int kind, int visit) { return (kind == 3 && visit > 0) ? 1 : kind; }
    __device__ void cycle_rest(int lstart, int last, int nu1, int nu2, int kind, int variant)
    {
        int cnt[MAXLEV];
        unsigned char kd[MAXLEV];
        int l = lstart;
        cnt[l] = 0;
        kd[l] = (unsigned char)kind;
        while (true) {
            if (l + 1 == last) {
                coarse_level(last, variant);
                cnt[l] = visits(kd[l]);
            }
            if (cnt[l] < visits(kd[l])) {
                const bool zg = cnt[l] == 0;  // first visit: zero initial guess (:311-312)
                const int ck = child_kind(kd[l], cnt[l]);
                cnt[l] += 1;
                l += 1;
                down(l, zg, nu1, false);
                cnt[l] = 0;
                kd[l] = (unsigned char)ck;
                continue;
            }
            up(l, nu2);
            if (l == lstart) break;
            l -= 1;
        }
    }

    // ||r|| of level l0's INPUT iterate from sq (written by down(l0, .., norm))
    __device__ double norm_reduce(int l)
    {
        __syncthreads();
        prev_warp = false;
        const double nrm = __dsqrt_rn(block_pairwise_auto(sq, N(l), part()));
        tick(4, l);
        return nrm;
    }
};

template <typename T, int NT, bool SPARSE, bool SMEM>
__device__ void tail_body(const TailArgs<T, NT> &a)
{
    const int b = blockIdx.x;
    const int nlev = a.depth - a.l0;
    // constants and level metadata into shared memory
    for (int i = threadIdx.x; i < (int)(sizeof(LevelC<T, NT>) * nlev / 4); i += blockDim.x)
        reinterpret_cast<uint32_t *>(tmg_tail_smem)[i] = reinterpret_cast<const uint32_t *>(a.levels + (size_t)b * a.levels_stride + a.l0)[i];
    Engine<T, NT, SPARSE, SMEM> E;
    E.l0 = a.l0;
    E.scan = a.coarse_scan;
    E.trace = blockIdx.x == 0 ? a.trace : nullptr;
    E.t_mark = clock64();
    uint32_t o = (uint32_t)(sizeof(LevelC<T, NT>) * nlev);
    E.o_meta = o;
    o += (uint32_t)(sizeof(int) * 4 * nlev);
    o = (o + 15) & ~15u;
    E.o_scan = o;
    o += (uint32_t)(sizeof(T) * 2 * blockDim.x);
    o = (o + 15) & ~15u;
    E.o_part = o;
    o += (uint32_t)(sizeof(double) * blockDim.x);
    o = (o + 15) & ~15u;
    E.o_store = o;
    E.gbase = SMEM ? nullptr : a.gstore + (size_t)b * a.store_elems;
    int *meta = reinterpret_cast<int *>(tmg_tail_smem + E.o_meta);
    for (int l = a.l0 + threadIdx.x; l < a.depth; l += blockDim.x) {
        const int nn = (int)a.n[l];
        meta[4 * (l - a.l0)] = (int)a.off[l];
        meta[4 * (l - a.l0) + 1] = (int)(a.off[l] + (long long)nn * NT);
        meta[4 * (l - a.l0) + 2] = (int)(a.off[l] + 2LL * nn * NT);
        meta[4 * (l - a.l0) + 3] = nn;
    }
    E.sq = reinterpret_cast<double *>(E.arr((int)a.store_elems));
    __syncthreads();

    const int n0 = (int)a.n[a.l0];
    const int ne = n0 * NT;
    const T *fin = a.f_in + (size_t)b * ne;
    T *u0 = E.U(a.l0), *f0 = E.F(a.l0);
    for (int i = threadIdx.x; i < ne; i += blockDim.x) {
        f0[i] = fin[i];
        u0[i] = a.u_in ? a.u_in[(size_t)b * ne + i] : T(0);
    }
    __syncthreads();
    const int last = a.depth - 1;

    if (!a.full) {
        // each_kind: n_cycles cycles of kind gamma; else gamma is the kind of
        // the calling (streamed) level's cycle and its n_cycles visits of
        // level l0 are cycles of the child kinds
        for (int c = 0; c < a.n_cycles; ++c) {
            if (a.l0 == last) {
                E.coarse_level(last, a.dot_variant);
            } else {
                E.down(a.l0, c == 0 && !a.u_in, a.nu1, false);
                const int kind = a.each_kind ? a.gamma : E.child_kind(a.gamma, c);
                E.cycle_rest(a.l0, last, a.nu1, a.nu2, kind, a.dot_variant);
            }
        }
    } else {
        // _iterate (multigrid.py:476-492) on one problem; the norm of each
        // iterate comes from the next cycle's down pass (its first sweep's
        // residual), which is discarded when the stopping test ends the solve
        double *hist = a.hist + (size_t)b * (a.max_iters + 1);
        E.down(a.l0, false, a.nu1, true);
        const double r0 = E.norm_reduce(a.l0);
        const double e = __dmul_rn(a.eps, r0);
        const double tol = e > a.floor_[b] ? e : a.floor_[b];
        double rk = r0;
        int iters = 0;
        if (threadIdx.x == 0) hist[0] = r0;
        while (rk > tol && iters < a.max_iters) {
            E.cycle_rest(a.l0, last, a.nu1, a.nu2, a.gamma, a.dot_variant);
            E.down(a.l0, false, a.nu1, true);
            rk = E.norm_reduce(a.l0);
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
    for (int i = threadIdx.x; i < ne; i += blockDim.x) a.u_out[(size_t)b * ne + i] = u0[i];
}

template <typename T, int NT, bool SPARSE>
__global__ void __launch_bounds__(TAIL_THREADS)
    tail_kernel(const __grid_constant__ TailArgs<T, NT> a)
{
    pdl_trigger();
    pdl_wait();
    if (a.active && !a.active[blockIdx.x]) return;
    if (a.in_smem) tail_body<T, NT, SPARSE, true>(a);
    else tail_body<T, NT, SPARSE, false>(a);
}

}  // namespace tmg
