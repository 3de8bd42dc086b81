// Grid-wide exact solve of the block lower-bidiagonal system L u = f as an
// associative scan (forward_solve, dg.py:290-303, and the coarsest-level
// solve, multigrid.py:200-205, method "scan").
//
// The sparse coupling N = outer(eval_start, eval_end) is rank one, so with
// g_k = LU^-1 f_k and h_k = e.g_k the block recurrence collapses to a scalar
// affine one (LevelC::ce, cw, calpha):
//     s_k = alpha s_{k-1} + h_k,      u_k = g_k + s_{k-1} w,      s_{-1} = 0.
// Three passes, no waiting between warps at all; a tile is one WARP's 32 K
// consecutive slabs.  Loads and stores are coalesced 32-slab rows; a
// per-warp shared-memory transpose gives every lane a strip of K consecutive
// slabs, so the recurrence runs K steps in registers and only once per 32 K
// slabs across the lanes:
// A warp owns runs of `run` consecutive tiles (the host picks run so that a
// problem has at most SCAN_MAX_RUNS runs and the grid stays balanced):
//   1. scan_agg_kernel: g, h per slab; each lane's strip sum, then the lanes'
//      inclusive sums by 5 shuffle steps with the constant multipliers
//      alpha^(K 2^q); the tile's map x -> A x + H (A = alpha^(slabs)); the
//      run's tiles composed in double-double, the run's H written;
//   2. scan_carry_kernel: one CTA per problem scans the runs' maps (staged in
//      shared memory; blocks per thread, then the CTA) into each run's
//      incoming s;
//   3. scan_replay_kernel: every run again (f re-read, g recomputed), the
//      incoming s carried from tile to tile in double-double, the lanes'
//      s_prev from it, u = g + s_prev w written once.
// HBM: f twice, u once (3 n_t s bytes per slab against 2 for one pass).
// The maps are composed in double-double with alpha itself in double-double
// (LevelC::calpha + calpha_lo, formed on the host): alpha is applied ~N times,
// so a rounded alpha (or alpha^k) would be a SYSTEMATIC error growing
// linearly along the recurrence -- for alpha -> 1 (small tau) ~1e-11 relative
// at 2^20.  In double-double the scan agrees with the extended-precision
// solution of the same system to a few ulp per slab (tests: scan vs
// long-double substitution), i.e. it is more accurate than the serial sweep,
// whose own error grows like sqrt(N) ulp.  Not bitwise with the serial
// substitution (different association).
#pragma once
#include "tmg_slab.cuh"
#include "tmg_types.cuh"

namespace tmg {

// K: consecutive slabs per lane (the g values of a strip stay in registers)
template <int NT> __host__ __device__ constexpr int scan_groups() { return NT <= 2 ? 8 : 4; }
constexpr int SCAN_WARPS = 8;     // warps per CTA

// The maps are composed in double-double with alpha itself in double-double
// (LevelC::calpha + calpha_lo, formed on the host): alpha is applied ~N times,
// so a rounded alpha (or a rounded alpha^k) would be a SYSTEMATIC error
// growing linearly along the recurrence -- for alpha -> 1 (small tau) that
// alone is ~1e-11 relative at 2^20.  In double-double the scan agrees with
// the extended-precision solution of the same system to a few ulp per slab
// (tests: scan vs long-double substitution), i.e. it is more accurate than
// the serial sweep, whose own error grows like sqrt(N) ulp.

struct DD {
    double hi, lo;
};
__device__ __forceinline__ DD dd_two_sum(double a, double b)
{
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}
__device__ __forceinline__ DD dd_fast(double hi, double lo)
{
    const double s = __dadd_rn(hi, lo);
    return {s, __dsub_rn(lo, __dsub_rn(s, hi))};
}
// (a_hi + a_lo)(b_hi + b_lo)
__device__ __forceinline__ DD dd_mul(DD a, DD b)
{
    const double p = __dmul_rn(a.hi, b.hi);
    double e = __fma_rn(a.hi, b.hi, -p);
    e = __fma_rn(a.hi, b.lo, e);
    e = __fma_rn(a.lo, b.hi, e);
    return dd_fast(p, e);
}
// a * b + c (all double-double)
__device__ __forceinline__ DD dd_mul_add(DD a, DD b, DD c)
{
    const DD p = dd_mul(a, b);
    DD s = dd_two_sum(p.hi, c.hi);
    return dd_fast(s.hi, __dadd_rn(s.lo, __dadd_rn(p.lo, c.lo)));
}


template <typename T, int NT> struct ScanTile {
    static constexpr int GROUPS = scan_groups<NT>();    // K: consecutive slabs per lane
    static constexpr int LOGK = GROUPS == 8 ? 3 : 2;
    static constexpr long long SLABS = 32LL * GROUPS;   // a tile is one warp's slabs
    // per-warp transpose buffer: lane l's strip of K slabs at l * STRIDE
    // elements.  The pad (one vector of the slab's access width) makes both
    // the row-wise access (lane <-> slab 32 j + lane, as the global loads
    // and stores go) and the strip-wise access bank-conflict free.
    static constexpr int SLAB_BYTES = NT * (int)sizeof(T);
    static constexpr int PAD_BYTES = SLAB_BYTES % 16 == 0 ? 16 : SLAB_BYTES % 8 == 0 ? 8 : 4;
    static constexpr int STRIDE = GROUPS * NT + PAD_BYTES / (int)sizeof(T);
    static constexpr int WARP_ELEMS = 32 * STRIDE;
    static __device__ __forceinline__ int pos(int sl) { return (sl >> LOGK) * STRIDE + (sl & (GROUPS - 1)) * NT; }
};

// alpha^(2^k): the multipliers of a lane's strip (k = LOGK), of the shuffle
// scan over the lanes (LOGK + q, q < 5) and of a tile (LOGK + 5)
struct ScanPowers {
    DD p[16];
};
__device__ __forceinline__ ScanPowers scan_powers(const DD &alpha, int kmax)
{
    ScanPowers P;
    P.p[0] = alpha;
    for (int k = 1; k <= kmax && k < 16; ++k) P.p[k] = dd_mul(P.p[k - 1], P.p[k - 1]);
    return P;
}

// g = LU^-1 f for the K slabs of a lane's strip, g holding the right-hand
// sides already in LU row order (P f): branch-free divisions, the rare
// out-of-window numerator redoes the strip exactly, out of line
template <typename T, int NT, int K>
__device__ __forceinline__ void scan_lu(const LevelC<T, NT> &L, T (&g)[K][NT])
{
    if constexpr (fast_fp<T>()) {
#pragma unroll
        for (int i = 0; i < K; ++i) lu_apply<T, NT>(L, g[i]);
    } else {
        unsigned bad = 0;
        T ys[K][NT];
#pragma unroll
        for (int i = 0; i < K; ++i)
#pragma unroll
            for (int r = 0; r < NT; ++r) ys[i][r] = g[i][r];
#pragma unroll
        for (int i = 0; i < K; ++i) lu_apply_nb<T, NT>(L, g[i], bad);
        if (TMG_UNLIKELY(__any_sync(0xffffffffu, bad))) {
            LuPack<T, NT, K> in;
            LuConst<T, NT> lc;
#pragma unroll
            for (int i = 0; i < NT * NT; ++i) lc.lu[i] = L.lu[i];
#pragma unroll
            for (int i = 0; i < NT; ++i) lc.rinv[i] = L.rinv[i];
#pragma unroll
            for (int i = 0; i < K; ++i)
#pragma unroll
                for (int r = 0; r < NT; ++r) in.v[i][r] = ys[i][r];
            LuPack<T, NT, K> out = lu_fallback_byvalue<T, NT, K>(in, lc);
#pragma unroll
            for (int i = 0; i < K; ++i)
#pragma unroll
                for (int r = 0; r < NT; ++r) g[i][r] = out.v[i][r];
        }
    }
}

// one warp's 32 K slabs.  Global loads go row-wise (lane <-> slab 32 j + lane:
// coalesced; cp.async straight into the padded buffer, the NEXT tile's fetch
// in flight under this tile's arithmetic), the buffer hands every lane its strip of K
// CONSECUTIVE slabs: g and h per slab (K independent LU solves), the strip's
// sum H = sum_i alpha^(K-1-i) h_i as a K-step recurrence in registers, then
// ONE 5-step shuffle scan over the lanes' sums per 32 K slabs (multipliers
// alpha^(K 2^q)).  Returns the lane's inclusive sum iH (slabs up to the end of
// its strip) and the warp's H (all lanes).  Slabs past the end of the problem
// read as f = 0 (g = h = 0).
// ---- tile fetch: global -> the warp's padded transpose buffer ---------------
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait()
{
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
template <int BYTES> __device__ __forceinline__ void cp_async_piece(void *dst, const void *src)
{
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d), "l"(src), "n"(BYTES) : "memory");
}
// asynchronous fetch of the tile at s0 (row-wise: lane <-> slab 32 j + lane;
// slabs past the end are zero-filled by plain stores); ONE commit group.
// fb must be aligned to ScanTile::PAD_BYTES (the piece size).
template <typename T, int NT>
__device__ __forceinline__ void scan_fetch_async(const T *fb, long long n, long long s0, int lane, T *sm)
{
    using Tile = ScanTile<T, NT>;
    constexpr int PIECE = Tile::PAD_BYTES;
#pragma unroll
    for (int j = 0; j < Tile::GROUPS; ++j) {
        const long long k = s0 + 32LL * j + lane;
        T *dst = sm + Tile::pos(32 * j + lane);
        if (k < n) {
            const char *src = reinterpret_cast<const char *>(fb + k * NT);
#pragma unroll
            for (int o = 0; o < Tile::SLAB_BYTES; o += PIECE)
                cp_async_piece<PIECE>(reinterpret_cast<char *>(dst) + o, src + o);
        } else {
#pragma unroll
            for (int i = 0; i < NT; ++i) dst[i] = T(0);
        }
    }
    cp_async_commit();
}
// synchronous fetch (any alignment)
template <typename T, int NT>
__device__ __forceinline__ void scan_fetch_sync(const T *fb, long long n, long long s0, int lane, T *sm)
{
    using Tile = ScanTile<T, NT>;
    constexpr int K = Tile::GROUPS;
    T x[K][NT];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const long long k = s0 + 32LL * j + lane;
#pragma unroll
        for (int i = 0; i < NT; ++i) x[j][i] = k < n ? fb[k * NT + i] : T(0);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) store_slab<T, NT>(sm + Tile::pos(32 * j + lane), x[j]);
}

// the tile in sm (all lanes' fetches complete and visible: the caller has
// waited and synchronised the warp) -> g, h, iH, the warp's H
template <typename T, int NT>
__device__ __forceinline__ double scan_warp(const LevelC<T, NT> &L, const ScanPowers &P, int lane, const T *sm,
                                            T (&g)[ScanTile<T, NT>::GROUPS][NT],
                                            double (&h)[ScanTile<T, NT>::GROUPS], double &iH)
{
    using Tile = ScanTile<T, NT>;
    constexpr int K = Tile::GROUPS;
    T x[K][NT];
    // the strip, rows in LU order (y_r = f_perm[r]): for n_t <= 2 one vector
    // load and a select, above scalar loads at the permuted offsets (register
    // arrays indexed by perm[] would go to local memory)
    if constexpr (NT <= 2) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
            load_slab<T, NT>(sm + lane * Tile::STRIDE + i * NT, x[i]);
#pragma unroll
            for (int r = 0; r < NT; ++r) {
                T v = x[i][0];
#pragma unroll
                for (int q = 1; q < NT; ++q) v = (L.perm[r] == q) ? x[i][q] : v;
                g[i][r] = v;
            }
        }
    } else {
#pragma unroll
        for (int r = 0; r < NT; ++r) {
            const T *src = sm + lane * Tile::STRIDE + L.perm[r];
#pragma unroll
            for (int i = 0; i < K; ++i) g[i][r] = src[i * NT];
        }
    }
    __syncwarp();
    scan_lu<T, NT, K>(L, g);
    const double a1 = P.p[0].hi;
    double H = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        T hh = FP<T>::mul(L.ce[0], g[i][0]);
#pragma unroll
        for (int r = 1; r < NT; ++r) hh = FP<T>::fma(L.ce[r], g[i][r], hh);
        h[i] = (double)hh;
        H = i == 0 ? h[0] : __fma_rn(a1, H, h[i]);
    }
    // across the lanes in double (its rounding stays local to the warp's
    // slabs); the tile and carry compositions, which run along the whole
    // recurrence with the same multiplier, in double-double
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const int off = 1 << q;
        const double ph = __shfl_up_sync(0xffffffffu, H, off);
        if (lane >= off) H = __fma_rn(P.p[Tile::LOGK + q].hi, ph, H);  // H_l += alpha^(K off) H_{l-off}
    }
    iH = H;
    return __shfl_sync(0xffffffffu, H, 31);
}

// (a_hi + a_lo)^r, r >= 0
__device__ __forceinline__ DD dd_pow(DD a, long long r)
{
    DD out{1.0, 0.0};
    while (r > 0) {
        if (r & 1) out = dd_mul(out, a);
        a = dd_mul(a, a);
        r >>= 1;
    }
    return out;
}

// The sequence of tiles a warp walks: runs t = w0, w0 + stride, ... (grid-
// stride over all problems' runs), `run` tiles each.  Advanced incrementally
// (one 32-bit division per run, none per tile).
struct ScanItem {
    int t, b, r, q;      // run (global index), problem, run within the problem, tile within the run
    long long s0;        // first slab of the tile
    bool valid;
};
template <typename T, int NT>
__device__ __forceinline__ void scan_item_place(ScanItem &it, int total, int runs_per, int run, long long n,
                                                const int *active)
{
    if (it.q == 0 && it.t < total) {
        it.b = it.t / runs_per;
        it.r = it.t - it.b * runs_per;
    }
    it.s0 = ((long long)it.r * run + it.q) * ScanTile<T, NT>::SLABS;
    it.valid = it.t < total && it.s0 < n && !(active && !active[it.b]);
}
template <typename T, int NT>
__device__ __forceinline__ ScanItem scan_item_next(ScanItem it, int stride, int total, int runs_per, int run,
                                                   long long n, const int *active)
{
    if (++it.q == run) {
        it.q = 0;
        it.t = it.t < total ? it.t + stride : it.t;
    }
    scan_item_place<T, NT>(it, total, runs_per, run, n, active);
    return it;
}

// pass 1: a warp owns RUNS of `run` consecutive tiles; it walks a run tile by
// tile, composing the tiles' maps in double-double, and writes the run's H.
// No CTA barrier anywhere: the warps of a CTA drift apart.  Dynamic shared
// memory: two transpose buffers per warp.
template <typename T, int NT>
__global__ void __launch_bounds__(SCAN_WARPS * 32)
    scan_agg_kernel(const __grid_constant__ LevelC<T, NT> L, const T *f, long long n, int batch,
                    long long runs_per, int run, double *maps, const int *active)
{
    using Tile = ScanTile<T, NT>;
    constexpr int G = Tile::GROUPS;
    extern __shared__ __align__(16) unsigned char scan_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T *buf = reinterpret_cast<T *>(scan_smem) + warp * 2 * Tile::WARP_ELEMS;
    const ScanPowers P = scan_powers(DD{(double)L.calpha, L.calpha_lo}, Tile::LOGK + 5);
    const DD PT = P.p[Tile::LOGK + 5];  // alpha^(tile)
    const int total = (int)(runs_per * batch);
    const int w0 = blockIdx.x * SCAN_WARPS + warp, stride = gridDim.x * SCAN_WARPS;
    // programmatic dependent launch: everything above ran under the previous
    // kernel's tail; no global memory is touched before this wait
    pdl_trigger();
    pdl_wait();
    if (w0 >= total) return;
    const int items = ((total - w0 + stride - 1) / stride) * run;
    const bool async = (((uintptr_t)f | (uintptr_t)((size_t)n * NT * sizeof(T))) & (Tile::PAD_BYTES - 1)) == 0;
    ScanItem cur{w0, 0, 0, 0, 0, false};
    scan_item_place<T, NT>(cur, total, (int)runs_per, run, n, active);
    if (async && cur.valid) scan_fetch_async<T, NT>(f + (size_t)cur.b * n * NT, n, cur.s0, lane, buf);
    else cp_async_commit();
    DD RH{0.0, 0.0};
    for (int i = 0; i < items; ++i) {
        const ScanItem nxt = scan_item_next<T, NT>(cur, stride, total, (int)runs_per, run, n, active);
        T *sm = buf + (i & 1) * Tile::WARP_ELEMS;
        if (async && i + 1 < items && nxt.valid)
            scan_fetch_async<T, NT>(f + (size_t)nxt.b * n * NT, n, nxt.s0, lane, buf + ((i + 1) & 1) * Tile::WARP_ELEMS);
        else cp_async_commit();
        double WH = 0.0;
        if (cur.valid) {
            if (!async) scan_fetch_sync<T, NT>(f + (size_t)cur.b * n * NT, n, cur.s0, lane, sm);
            cp_async_wait<1>();
            __syncwarp();
            T g[G][NT];
            double h[G], iH;
            WH = scan_warp<T, NT>(L, P, lane, sm, g, h, iH);
            __syncwarp();
        }
        RH = dd_mul_add(PT, RH, DD{WH, 0.0});
        if (cur.q == run - 1) {
            if (lane == 0 && cur.t < total && !(active && !active[cur.b])) maps[cur.t] = __dadd_rn(RH.hi, RH.lo);
            RH = DD{0.0, 0.0};
        }
        cur = nxt;
    }
    cp_async_wait<0>();
}

// pass 2, one CTA per problem: the runs' maps x -> A x + H_k (A = alpha^(run
// slabs)) composed into each run's incoming s, in double-double.  The maps
// are staged in shared memory by coalesced loads (a thread's strided walk over
// global memory is bound by the load unit of the one SM this CTA runs on); a
// thread owns 4 sub-runs of m4 consecutive maps and walks them as 4
// independent chains (the double-double multiply-add is a ~18-deep dependent
// chain); the threads' maps are scanned across the CTA; the carries go back
// through the same buffer.  maps and carry may be the same array.
constexpr int SCAN_CARRY_THREADS = 1024;
constexpr int SCAN_MAX_RUNS = 16384;   // per problem (shared-memory staging)
// maps per sub-run: the smallest power of two with 4 m4 threads covering runs_per
__host__ __device__ inline int scan_carry_logm4(int runs_per, int threads)
{
    int lg = 0;
    while ((4 * threads) << lg < runs_per) ++lg;
    return lg;
}
// threads of the carry CTA: a power of two, 4 maps per thread until 1024
inline int scan_carry_threads(long long runs_per)
{
    int th = 32;
    while (th < SCAN_CARRY_THREADS && 4LL * th < runs_per) th <<= 1;
    return th;
}
template <typename T, int NT>
__global__ void __launch_bounds__(SCAN_CARRY_THREADS)
    scan_carry_kernel(const __grid_constant__ LevelC<T, NT> L, int runs_per, int run, const double *maps,
                      double *carry, const int *active)
{
    using Tile = ScanTile<T, NT>;
    extern __shared__ double stage[];
    __shared__ double sAh[SCAN_CARRY_THREADS], sAl[SCAN_CARRY_THREADS], sHh[SCAN_CARRY_THREADS],
        sHl[SCAN_CARRY_THREADS];
    const int b = blockIdx.x;
    const ScanPowers P = scan_powers(DD{(double)L.calpha, L.calpha_lo}, Tile::LOGK + 5);
    const DD TA = dd_pow(P.p[Tile::LOGK + 5], run);   // alpha^(run slabs)
    pdl_trigger();
    pdl_wait();   // the maps (pass 1) are complete and visible from here on
    if (active && !active[b]) return;
    const int t = threadIdx.x;
    const int Pn = blockDim.x;
    const double *mb = maps + (size_t)b * runs_per;
    double *cb = carry + (size_t)b * runs_per;
    const int lg = scan_carry_logm4(runs_per, Pn), m4 = 1 << lg;
    const int lgS = lg + 2;                             // a thread's block: S = 4 m4 maps
    // one pad element per block: odd stride between the threads' blocks
    for (int k = t; k < runs_per; k += Pn) stage[k + (k >> lgS)] = mb[k];
    __syncthreads();
    const int a = t << lgS;
    double *mine = stage + a + t;
    DD A4{1.0, 0.0}, Hc[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) Hc[c] = DD{0.0, 0.0};
    for (int i = 0; i < m4; ++i) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int k = (c << lg) + i;
            const double q = a + k < runs_per ? mine[k] : 0.0;
            Hc[c] = dd_mul_add(TA, Hc[c], DD{q, 0.0});
        }
        A4 = dd_mul(TA, A4);
    }
    // the thread's map: its 4 sub-runs in sequence
    DD H = Hc[0];
#pragma unroll
    for (int c = 1; c < 4; ++c) H = dd_mul_add(A4, H, Hc[c]);
    DD A = dd_mul(A4, A4);
    A = dd_mul(A, A);
    sAh[t] = A.hi;
    sAl[t] = A.lo;
    sHh[t] = H.hi;
    sHl[t] = H.lo;
    __syncthreads();
    for (int off = 1; off < Pn; off <<= 1) {  // inclusive scan of the threads' maps
        DD pa{1.0, 0.0}, ph{0.0, 0.0};
        if (t >= off) {
            pa = DD{sAh[t - off], sAl[t - off]};
            ph = DD{sHh[t - off], sHl[t - off]};
        }
        __syncthreads();
        if (t >= off) {
            H = dd_mul_add(A, ph, H);
            A = dd_mul(A, pa);
            sAh[t] = A.hi;
            sAl[t] = A.lo;
            sHh[t] = H.hi;
            sHl[t] = H.lo;
        }
        __syncthreads();
    }
    // s before each sub-run, then along the sub-runs (4 chains again)
    DD sc[4];
    sc[0] = t == 0 ? DD{0.0, 0.0} : DD{sHh[t - 1], sHl[t - 1]};  // s_{-1} = 0
#pragma unroll
    for (int c = 1; c < 4; ++c) sc[c] = dd_mul_add(A4, sc[c - 1], Hc[c - 1]);
    for (int i = 0; i < m4; ++i) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int k = (c << lg) + i;
            if (a + k < runs_per) {
                const double q = mine[k];
                mine[k] = __dadd_rn(sc[c].hi, sc[c].lo);
                sc[c] = dd_mul_add(TA, sc[c], DD{q, 0.0});
            }
        }
    }
    __syncthreads();
    for (int k = t; k < runs_per; k += Pn) cb[k] = stage[k + (k >> lgS)];
}

// pass 3: every run again (f re-read, g recomputed), u = g + s_prev w; the
// incoming s moves from tile to tile in double-double
template <typename T, int NT>
__global__ void __launch_bounds__(SCAN_WARPS * 32)
    scan_replay_kernel(const __grid_constant__ LevelC<T, NT> L, const T *f, T *u, long long n, int batch,
                       long long runs_per, int run, const double *carry, const int *active)
{
    using Tile = ScanTile<T, NT>;
    constexpr int G = Tile::GROUPS;
    extern __shared__ __align__(16) unsigned char scan_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T *buf = reinterpret_cast<T *>(scan_smem) + warp * 2 * Tile::WARP_ELEMS;
    const ScanPowers P = scan_powers(DD{(double)L.calpha, L.calpha_lo}, Tile::LOGK + 5);
    const DD PT = P.p[Tile::LOGK + 5];
    // alpha^(K (lane+1)): the multiplier of the tile's incoming s at the end of a lane's strip
    DD laneA_dd{1.0, 0.0};
#pragma unroll
    for (int q = 0; q < 6; ++q)
        if ((lane + 1) & (1 << q)) laneA_dd = dd_mul(laneA_dd, P.p[Tile::LOGK + q]);
    const double laneA = laneA_dd.hi;
    const double a1 = P.p[0].hi;
    const int total = (int)(runs_per * batch);
    const int w0 = blockIdx.x * SCAN_WARPS + warp, stride = gridDim.x * SCAN_WARPS;
    // programmatic dependent launch: everything above ran under the previous
    // kernel's tail; no global memory is touched before this wait
    pdl_trigger();
    pdl_wait();
    if (w0 >= total) return;
    const int items = ((total - w0 + stride - 1) / stride) * run;
    const bool async = (((uintptr_t)f | (uintptr_t)((size_t)n * NT * sizeof(T))) & (Tile::PAD_BYTES - 1)) == 0;
    ScanItem cur{w0, 0, 0, 0, 0, false};
    scan_item_place<T, NT>(cur, total, (int)runs_per, run, n, active);
    if (async && cur.valid) scan_fetch_async<T, NT>(f + (size_t)cur.b * n * NT, n, cur.s0, lane, buf);
    else cp_async_commit();
    DD sdd{0.0, 0.0};
    for (int i = 0; i < items; ++i) {
        const ScanItem nxt = scan_item_next<T, NT>(cur, stride, total, (int)runs_per, run, n, active);
        T *sm = buf + (i & 1) * Tile::WARP_ELEMS;
        if (async && i + 1 < items && nxt.valid)
            scan_fetch_async<T, NT>(f + (size_t)nxt.b * n * NT, n, nxt.s0, lane, buf + ((i + 1) & 1) * Tile::WARP_ELEMS);
        else cp_async_commit();
        if (cur.valid) {
            if (cur.q == 0) sdd = DD{carry[cur.t], 0.0};   // s before the run
            if (!async) scan_fetch_sync<T, NT>(f + (size_t)cur.b * n * NT, n, cur.s0, lane, sm);
            cp_async_wait<1>();
            __syncwarp();
            T g[G][NT];
            double h[G], iH;
            const double WH = scan_warp<T, NT>(L, P, lane, sm, g, h, iH);
            __syncwarp();
            const double sg = __dadd_rn(sdd.hi, sdd.lo);    // the tile's incoming s
            const double s_incl = __fma_rn(laneA, sg, iH);  // s after this lane's strip
            double s = __shfl_up_sync(0xffffffffu, s_incl, 1);
            if (lane == 0) s = sg;
            // along the strip: u_i = g_i + s_{i-1} w, s_i = alpha s_{i-1} + h_i
#pragma unroll
            for (int k = 0; k < G; ++k) {
                T o[NT];
#pragma unroll
                for (int r = 0; r < NT; ++r) o[r] = (T)__fma_rn(s, (double)L.cw[r], (double)g[k][r]);
                store_slab<T, NT>(sm + lane * Tile::STRIDE + k * NT, o);
                s = __fma_rn(a1, s, h[k]);
            }
            __syncwarp();
            T *ub = u + (size_t)cur.b * n * NT;
#pragma unroll
            for (int j = 0; j < G; ++j) {
                const long long k = cur.s0 + 32LL * j + lane;
                T o[NT];
                load_slab<T, NT>(sm + Tile::pos(32 * j + lane), o);
                if (k < n) store_slab<T, NT>(ub + k * NT, o);
            }
            __syncwarp();
            sdd = dd_mul_add(PT, sdd, DD{WH, 0.0});
        }
        cur = nxt;
    }
    cp_async_wait<0>();
}

}  // namespace tmg
