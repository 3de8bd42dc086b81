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

// Shared-memory layout (byte offsets from tmg_tail_smem):
//   LevelC[nlev] | int meta[3*nlev] (u offset, f offset, n) | T xv[2][TT][NT]
//   | unsigned xm[2][TT] | double part[TT] | level store (when SMEM)
template <typename T, int NT, bool SPARSE, bool SMEM> struct Engine {
    using C = Cpl<T, NT, SPARSE>;
    int l0;            // first (finest) level handled here
    uint32_t o_meta, o_xv, o_xm, o_part, o_store;
    T *gbase;          // level store in global memory (!SMEM)
    double *sq;        // per-slab squares for the norm
    int xp = 0;        // halo buffer currently valid
    int nthr;          // participating threads: blockDim.x, or 32 in warp mode (a power of two)
    int lgthr;         // log2(nthr)
    int scan = 0;      // coarsest solve: 0 = serial forward substitution (bitwise), 1 = scan
    unsigned long long *trace = nullptr;  // [phase kind][level] cycle totals (thread 0 of block 0)
    long long t_mark = 0;

    // phase kinds for the trace: 0 sweep, 1 restrict, 2 prolong, 3 coarse, 4 norm, 5 warp handoff
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
    __device__ __forceinline__ T *U(int l) const { return arr(meta()[3 * (l - l0)]); }
    __device__ __forceinline__ T *F(int l) const { return arr(meta()[3 * (l - l0) + 1]); }
    __device__ __forceinline__ int N(int l) const { return meta()[3 * (l - l0) + 2]; }
    __device__ __forceinline__ T *xv(int w, int t) const
    {
        return reinterpret_cast<T *>(tmg_tail_smem + o_xv) + ((size_t)w * blockDim.x + t) * NT;
    }
    __device__ __forceinline__ unsigned *xm(int w, int t) const
    {
        return reinterpret_cast<unsigned *>(tmg_tail_smem + o_xm) + (size_t)w * blockDim.x + t;
    }
    __device__ __forceinline__ double *part() const
    {
        return reinterpret_cast<double *>(tmg_tail_smem + o_part);
    }
    __device__ __forceinline__ void sync() const { group_sync(nthr); }

    // contiguous, even-length chunk of the participating thread
    __device__ __forceinline__ void chunk(int nn, int &a, int &e) const
    {
        int m = (nn + nthr - 1) >> lgthr;
        m += m & 1;
        a = min(nn, (int)threadIdx.x * m);
        e = min(nn, a + m);
    }
    // Halo exchange.  Invariant: before a phase that needs level l's halo,
    // buffer xp holds, per thread, the coupling data of the CURRENT last slab
    // of its chunk at level l.  Each phase that changes a level publishes its
    // own last slab into the other buffer and flips xp, so the barrier ending
    // the phase also publishes the halo: one barrier per sweep.
    __device__ __forceinline__ void put(const C &c, int w) const
    {
        if constexpr (SPARSE) {
            xv(w, threadIdx.x)[0] = c.s;
            *xm(w, threadIdx.x) = c.m;
        } else {
#pragma unroll
            for (int j = 0; j < NT; ++j) xv(w, threadIdx.x)[j] = c.u[j];
        }
    }
    __device__ __forceinline__ C get(int t) const
    {
        C c;
        if constexpr (SPARSE) {
            c.s = xv(xp, t)[0];
            c.m = *xm(xp, t);
        } else {
#pragma unroll
            for (int j = 0; j < NT; ++j) c.u[j] = xv(xp, t)[j];
        }
        return c;
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

    __device__ void publish_last(int l)
    {
        int a, e;
        chunk(N(l), a, e);
        if (a < e) {
            T x[NT];
            load(U(l) + (e - 1) * NT, x);
            put(make_cpl<T, NT, SPARSE>(Lv(l), x), xp);
        }
        sync();
    }

    __device__ void sweep_level(int l)
    {
        int a, e;
        chunk(N(l), a, e);
        if (a < e) {
            const LevelC<T, NT> &L = Lv(l);
            T *u = U(l);
            const T *f = F(l);
            C prev;
            cpl_zero(prev);
            if (a > 0) prev = get(threadIdx.x - 1);
            T last[NT];
            int k = a;
            // slab pairs: two independent dependency chains per thread
            for (; k + 1 < e; k += 2) {
                T x0[NT], x1[NT], f0[NT], f1[NT];
                load(u + k * NT, x0);
                load(u + (k + 1) * NT, x1);
                load(f + k * NT, f0);
                load(f + (k + 1) * NT, f1);
                C o0 = make_cpl<T, NT, SPARSE>(L, x0);
                C o1 = make_cpl<T, NT, SPARSE>(L, x1);
                sweep<T, NT, SPARSE>(L, x0, f0, prev, k > 0);
                sweep<T, NT, SPARSE>(L, x1, f1, o0, true);
                store(u + k * NT, x0);
                store(u + (k + 1) * NT, x1);
#pragma unroll
                for (int j = 0; j < NT; ++j) last[j] = x1[j];
                prev = o1;
            }
            if (k < e) {
                T x[NT], ff[NT];
                load(u + k * NT, x);
                load(f + k * NT, ff);
                sweep<T, NT, SPARSE>(L, x, ff, prev, k > 0);
                store(u + k * NT, x);
#pragma unroll
                for (int j = 0; j < NT; ++j) last[j] = x[j];
            }
            put(make_cpl<T, NT, SPARSE>(L, last), xp ^ 1);
        }
        xp ^= 1;
        sync();
        tick(0, l);
    }

    // residual + restriction into level l+1 (multigrid.py:283-285) and the
    // zero initial guess there (:312)
    __device__ void restrict_level(int l)
    {
        int a, e;
        chunk(N(l), a, e);
        const LevelC<T, NT> &L = Lv(l);
        const int nc = N(l) >> 1;
        const T *u = U(l), *f = F(l);
        T *fc = F(l + 1), *uc = U(l + 1);
        if (a < e) {
            C prev;
            cpl_zero(prev);
            if (a > 0) prev = get(threadIdx.x - 1);
            for (int c = a >> 1; c < (e >> 1) && c < nc; ++c) {
                T x0[NT], x1[NT], f0[NT], f1[NT], r0[NT], r1[NT], p0[NT], p1[NT];
                load(u + (2 * c) * NT, x0);
                load(u + (2 * c + 1) * NT, x1);
                load(f + (2 * c) * NT, f0);
                load(f + (2 * c + 1) * NT, f1);
                residual<T, NT, SPARSE>(L, x0, f0, prev, 2 * c > 0, r0);
                C c0 = make_cpl<T, NT, SPARSE>(L, x0);
                residual<T, NT, SPARSE>(L, x1, f1, c0, true, r1);
                prev = make_cpl<T, NT, SPARSE>(L, x1);
                restrict_part<T, NT>(L, r0, false, p0);
                restrict_part<T, NT>(L, r1, true, p1);
#pragma unroll
                for (int i = 0; i < NT; ++i) {
                    fc[c * NT + i] = FP<T>::add(p0[i], p1[i]);
                    uc[c * NT + i] = T(0);
                }
            }
        }
        int ac, ec;
        chunk(N(l + 1), ac, ec);
        if (ac < ec) {
            T z[NT];
            zero_slab<T, NT>(z);
            put(make_cpl<T, NT, SPARSE>(Lv(l + 1), z), xp ^ 1);
        }
        xp ^= 1;
        sync();
        tick(1, l);
    }

    // u_l += P u_{l+1} (multigrid.py:317)
    __device__ void prolong_level(int l)
    {
        int a, e;
        chunk(N(l), a, e);
        const LevelC<T, NT> &L = Lv(l);
        const int nc = N(l) >> 1;
        T *u = U(l);
        const T *uc = U(l + 1);
        for (int c = a >> 1; c < (e >> 1) && c < nc; ++c) {
            T cc[NT], x0[NT], x1[NT];
            load(uc + c * NT, cc);
            load(u + (2 * c) * NT, x0);
            load(u + (2 * c + 1) * NT, x1);
            prolong_part<T, NT>(L, cc, false, x0);
            prolong_part<T, NT>(L, cc, true, x1);
            store(u + (2 * c) * NT, x0);
            store(u + (2 * c + 1) * NT, x1);
        }
        if (a < e) {
            T x[NT];
            load(u + (e - 1) * NT, x);
            put(make_cpl<T, NT, SPARSE>(L, x), xp ^ 1);
        }
        xp ^= 1;
        sync();
        tick(2, l);
    }

    __device__ void coarse_level(int l, int variant)
    {
        if (scan) {
            T *xs = reinterpret_cast<T *>(tmg_tail_smem + o_xv);
            cta_scan_solve<T, NT>(Lv(l), F(l), U(l), N(l), xs, xs + blockDim.x, nthr);
            tick(3, l);
            return;
        }
        if (threadIdx.x == 0) forward_substitute<T, NT, SPARSE>(Lv(l), F(l), U(l), N(l), variant);
        sync();
        tick(3, l);
    }

    // gamma-cycle from level l0 (multigrid.py:263-330), iterative.  In block
    // mode, the coarse-grid correction of the first level with <= WARP_MAX
    // slabs below it is handed to warp 0 (warp-synchronous, no block barriers).
    template <bool WARP>
    __device__ void cycle(int lstart, int last, int nu1, int nu2, int gamma, int variant)
    {
        int cnt[MAXLEV];
        int l = lstart;
        for (int k = 0; k < nu1; ++k) sweep_level(l);
        restrict_level(l);
        cnt[l] = 0;
        while (true) {
            if (l + 1 == last) {
                coarse_level(last, variant);
                cnt[l] = gamma;
            } else if (!WARP && cnt[l] == 0 && N(l + 1) <= WARP_MAX) {
                const int xp0 = xp;
                if (threadIdx.x < 32) {
                    const int nt0 = nthr, lg0 = lgthr;
                    nthr = 32;
                    lgthr = 5;
                    publish_last(l + 1);
                    for (int g = 0; g < gamma; ++g) cycle<true>(l + 1, last, nu1, nu2, gamma, variant);
                    nthr = nt0;
                    lgthr = lg0;
                }
                xp = xp0;  // the next phase (prolong) publishes afresh
                __syncthreads();
                tick(5, l + 1);
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
            if (l == lstart) break;
            l -= 1;
        }
    }

    // ||f - L u|| at level l with numpy pairwise order (norm_at, :447-462)
    __device__ double norm(int l) const
    {
        int a, e;
        chunk(N(l), a, e);
        const LevelC<T, NT> &L = Lv(l);
        const T *u = U(l), *f = F(l);
        if (a < e) {
            C prev;
            cpl_zero(prev);
            if (a > 0) prev = get(threadIdx.x - 1);
            for (int k = a; k < e; ++k) {
                T x[NT], ff[NT], r[NT];
                load(u + k * NT, x);
                load(f + k * NT, ff);
                residual<T, NT, SPARSE>(L, x, ff, prev, k > 0, r);
                prev = make_cpl<T, NT, SPARSE>(L, x);
                sq[k] = (double)sqnorm<T, NT>(r);
            }
        }
        __syncthreads();
        double nrm = __dsqrt_rn(block_pairwise_auto(sq, N(l), part()));
        const_cast<Engine *>(this)->tick(4, l);
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
    E.nthr = blockDim.x;
    E.lgthr = 31 - __clz((int)blockDim.x);
    E.scan = a.coarse_scan;
    E.trace = blockIdx.x == 0 ? a.trace : nullptr;
    E.t_mark = clock64();
    uint32_t o = (uint32_t)(sizeof(LevelC<T, NT>) * nlev);
    E.o_meta = o;
    o += (uint32_t)(sizeof(int) * 3 * nlev);
    o = (o + 15) & ~15u;
    E.o_xv = o;
    o += (uint32_t)(sizeof(T) * 2 * blockDim.x * NT);
    E.o_xm = o;
    o += (uint32_t)(sizeof(unsigned) * 2 * blockDim.x);
    o = (o + 15) & ~15u;
    E.o_part = o;
    o += (uint32_t)(sizeof(double) * blockDim.x);
    o = (o + 15) & ~15u;
    E.o_store = o;
    E.gbase = SMEM ? nullptr : a.gstore + (size_t)b * a.store_elems;
    int *meta = reinterpret_cast<int *>(tmg_tail_smem + E.o_meta);
    for (int l = a.l0 + threadIdx.x; l < a.depth; l += blockDim.x) {
        meta[3 * (l - a.l0)] = (int)a.off[l];
        meta[3 * (l - a.l0) + 1] = (int)(a.off[l] + a.n[l] * NT);
        meta[3 * (l - a.l0) + 2] = (int)a.n[l];
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
    E.publish_last(a.l0);
    const int last = a.depth - 1;

    if (!a.full) {
        for (int c = 0; c < a.n_cycles; ++c) {
            if (a.l0 == last) E.coarse_level(last, a.dot_variant);
            else E.template cycle<false>(a.l0, last, a.nu1, a.nu2, a.gamma, a.dot_variant);
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
            E.template cycle<false>(a.l0, last, a.nu1, a.nu2, a.gamma, a.dot_variant);
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
