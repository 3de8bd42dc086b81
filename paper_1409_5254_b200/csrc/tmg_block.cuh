// Single-CTA multilevel engine, exact norms and coarse solves.
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
#include "tmg_slab.cuh"

namespace tmg {

constexpr int TAIL_THREADS = 512;
constexpr int MAXLEV = 48;

// ---------------------------------------------------------------------------
// numpy pairwise summation (np.sum, multigrid.py:459), exact for any n.
// Serial form for one thread:
__device__ __forceinline__ double pw_leaf(const double *a, long long n)
{
    if (n < 8) {
        double res = 0.0;
        for (long long i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    long long i;
    for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
}

// serial pairwise over [0, n) with an explicit stack (no device recursion)
__device__ double pw_serial(const double *a, long long n)
{
    // depth <= log2(n / 128) + 1; 40 covers any int64 length
    struct Node { long long off, len; double left; int state; };
    Node st[40];
    int sp = 0;
    st[0] = {0, n, 0.0, 0};
    double ret = 0.0;
    while (sp >= 0) {
        Node &nd = st[sp];
        if (nd.len <= 128) {
            ret = pw_leaf(a + nd.off, nd.len);
            --sp;
            continue;
        }
        long long n2 = nd.len / 2;
        n2 -= n2 % 8;
        if (nd.state == 0) {
            nd.state = 1;
            st[sp + 1] = {nd.off, n2, 0.0, 0};
            ++sp;
        } else if (nd.state == 1) {
            nd.left = ret;
            nd.state = 2;
            st[sp + 1] = {nd.off + n2, nd.len - n2, 0.0, 0};
            ++sp;
        } else {
            ret = __dadd_rn(nd.left, ret);
            --sp;
        }
    }
    return ret;
}

// CTA-wide exact pairwise sum; all threads get the result.  `part` has
// blockDim.x doubles of shared scratch; blockDim.x must be a power of two.
__device__ double block_pairwise(const double *a, long long n, double *part)
{
    const int T = blockDim.x;
    int D = 0;
    while ((1 << D) < T) ++D;
    const int t = threadIdx.x;
    long long off = 0, len = n;
    int d = 0;
    while (d < D && len > 128) {
        long long n2 = len / 2;
        n2 -= n2 % 8;
        if ((t >> (D - 1 - d)) & 1) { off += n2; len -= n2; }
        else len = n2;
        ++d;
    }
    const bool owner = (d == D) || ((t & ((1 << (D - d)) - 1)) == 0);
    if (owner) part[t] = (d == D) ? pw_serial(a + off, len) : pw_leaf(a + off, len);
    __syncthreads();
    if (t == 0) {
        // re-walk the top of the tree, combining owners' partials
        struct Node { long long len; double left; int d, p, state; };
        Node st[24];  // depth <= D + 1 <= 11
        int sp = 0;
        st[0] = {n, 0.0, 0, 0, 0};
        double ret = 0.0;
        while (sp >= 0) {
            Node &nd = st[sp];
            if (nd.d == D || nd.len <= 128) {
                ret = part[nd.p << (D - nd.d)];
                --sp;
                continue;
            }
            long long n2 = nd.len / 2;
            n2 -= n2 % 8;
            if (nd.state == 0) {
                nd.state = 1;
                st[sp + 1] = {n2, 0.0, nd.d + 1, nd.p << 1, 0};
                ++sp;
            } else if (nd.state == 1) {
                nd.left = ret;
                nd.state = 2;
                st[sp + 1] = {nd.len - n2, 0.0, nd.d + 1, (nd.p << 1) | 1, 0};
                ++sp;
            } else {
                ret = __dadd_rn(nd.left, ret);
                --sp;
            }
        }
        part[0] = ret;
    }
    __syncthreads();
    double s = part[0];
    __syncthreads();
    return s;
}

// ---------------------------------------------------------------------------
// per-problem iteration state (multigrid.py:481-496)
struct ProbState {
    double tol;
    int iters;
    int active;
    int max_iters;
    int converged;
};

// sum of a perfect binary tree of `m` values (m a power of two) per problem,
// one CTA per problem, then the stopping-rule update.
//   mode 0: r0 (initialises tol/active), mode 1: after a cycle.
__global__ void __launch_bounds__(1024)
    finalize_leaves_kernel(const double *leaves, long long m, ProbState *st, double *hist,
                           int hist_stride, const double *floor_, double eps, int mode)
{
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
    part[t] = v;
    __syncthreads();
    for (int s = 1; s < used; s <<= 1) {
        if ((t % (2 * s)) == 0 && t + s < used) part[t] = __dadd_rn(part[t], part[t + s]);
        __syncthreads();
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

__global__ void active_flags_kernel(const ProbState *st, int *active, int *any, int batch)
{
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < batch) {
        int a = st[b].active;
        active[b] = a;
        if (a) atomicOr(any, 1);
    }
}

__global__ void copy_active_kernel(const ProbState *st, int *active, int batch)
{
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < batch) active[b] = st[b].active;
}

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

template <typename T, int NT> struct TailArgs {
    const LevelC<T, NT> *levels;  // [depth] device array (copied to shared memory)
    int l0, depth;                // runs levels l0 .. depth-1 (depth-1 = coarsest)
    long long n[MAXLEV];          // slabs per level
    long long off[MAXLEV];        // element offset of level l's u (and f) in the store
    long long store_elems;        // per problem: elements of one level-array set
    const T *f_in;                // f at l0, [B][n_l0][NT]
    const T *u_in;                // u at l0 (cycle mode: NULL = zero guess; full: initial guess)
    T *u_out;                     // u at l0 after the work
    T *gstore;                    // global level store when not in shared memory
    int in_smem;
    int nu1, nu2, gamma, dot_variant;
    int full;                     // 1: _iterate with norms; 0: n_cycles cycles
    int n_cycles;
    // full mode
    double eps;
    const double *floor_;
    int max_iters;
    double *hist;                 // [B][max_iters+1]
    ProbState *st;
    const int *active;
};

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
    __device__ void coarse_level(int l, int variant) const
    {
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

template <typename T, int NT>
__host__ __device__ constexpr size_t tail_fixed_smem(int nlev)
{
    return sizeof(LevelC<T, NT>) * (size_t)nlev + sizeof(T) * TAIL_THREADS * (NT + 1) +
           sizeof(double) * TAIL_THREADS + 64;
}

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
