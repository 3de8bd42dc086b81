// Grid-wide exact solve of the block lower-bidiagonal system L u = f as an
// associative scan (forward_solve, dg.py:290-303, and the coarsest-level
// solve, multigrid.py:200-205, method "scan").
//
// The sparse coupling N = outer(eval_start, eval_end) is rank one, so with
// g_k = LU^-1 f_k and h_k = e.g_k the block recurrence collapses to a scalar
// affine one (LevelC::ce, cw, calpha):
//     s_k = alpha s_{k-1} + h_k,      u_k = g_k + s_{k-1} w,      s_{-1} = 0.
// Three passes, no inter-CTA waiting; a tile is one CTA: SCAN_WARPS warps of
// SCAN_GROUPS x 32 consecutive slabs (one slab per lane per group, so loads
// and stores are coalesced 32-slab rows):
//   1. scan_agg_kernel: g, h per slab; each lane's inclusive sum over its
//      group  H_l = sum_{i <= l} alpha^(l-i) h_i  by 5 shuffle steps with the
//      constant multipliers alpha^(2^k); the groups', warps' and tile's maps
//      x -> A x + H (A = alpha^(slabs)); only the tile's H is written;
//   2. scan_carry_kernel: one CTA per problem scans the tiles' maps (chunks
//      per thread, then the CTA) into each tile's incoming s;
//   3. scan_replay_kernel: every tile again (f re-read, g recomputed), each
//      warp's incoming s from the tile's and the preceding warps' maps, the
//      lanes' s_prev, u = g + s_prev w written once.
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

namespace tmg {

// 32-slab groups per warp tile (the g values of a tile stay in registers)
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
struct ScanTileMap {
    double Hhi, Hlo;            // the tile's map x -> alpha^(slabs) x + H
};
struct ScanCarry {
    double hi, lo;              // s before the tile
};

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
    static constexpr int GROUPS = scan_groups<NT>();
    static constexpr long long WARP_SLABS = 32LL * GROUPS;
    static constexpr long long SLABS = WARP_SLABS * SCAN_WARPS;
};

// alpha^(2^k), k = 0..log2(SCAN_WARPS * WARP_SLABS): the multipliers of the
// shuffle scan (k < 5), of a group (k = 5), of a warp and of a tile
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

// one warp's slabs: g (registers), the lanes' inclusive sums per group, the
// warp's H (all lanes); lanes past the end of the problem contribute h = 0
template <typename T, int NT>
__device__ __forceinline__ DD scan_warp(const LevelC<T, NT> &L, const ScanPowers &P, const T *fb, long long n,
                                        long long s0, int lane, T (&g)[ScanTile<T, NT>::GROUPS][NT],
                                        double (&iH)[ScanTile<T, NT>::GROUPS])
{
    constexpr int G = ScanTile<T, NT>::GROUPS;
    DD WH{0.0, 0.0};
#pragma unroll
    for (int j = 0; j < G; ++j) {
        const long long k = s0 + 32LL * j + lane;
        T x[NT];
        if (k < n) {
            load_slab<T, NT>(fb + k * NT, x);
        } else {
#pragma unroll
            for (int i = 0; i < NT; ++i) x[i] = T(0);
        }
        lu_solve<T, NT>(L, x, g[j]);
        T h = FP<T>::mul(L.ce[0], g[j][0]);
#pragma unroll
        for (int i = 1; i < NT; ++i) h = FP<T>::fma(L.ce[i], g[j][i], h);
        // within a warp in double (its rounding stays local to the warp's
        // slabs); the tile and carry compositions, which run along the whole
        // recurrence with the same multiplier, in double-double
        double H = k < n ? (double)h : 0.0;
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const int off = 1 << q;
            const double ph = __shfl_up_sync(0xffffffffu, H, off);
            if (lane >= off) H = __fma_rn(P.p[q].hi, ph, H);  // H_l += alpha^off H_{l-off}
        }
        iH[j] = H;
        WH.hi = __fma_rn(P.p[5].hi, WH.hi, __shfl_sync(0xffffffffu, H, 31));  // x -> alpha^32 x + H_group
    }
    return WH;
}

template <typename T, int NT>
__global__ void __launch_bounds__(SCAN_WARPS * 32)
    scan_agg_kernel(const __grid_constant__ LevelC<T, NT> L, const T *f, long long n, int batch,
                    long long tiles_per, ScanTileMap *maps, const int *active)
{
    constexpr int G = ScanTile<T, NT>::GROUPS;
    constexpr int LOGW = 31 - __builtin_clz((unsigned)ScanTile<T, NT>::WARP_SLABS);
    __shared__ double sh[SCAN_WARPS], sl[SCAN_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const ScanPowers P = scan_powers(DD{(double)L.calpha, L.calpha_lo}, LOGW);
    const long long total = tiles_per * batch;
    for (long long t = blockIdx.x; t < total; t += gridDim.x) {
        const long long b = t / tiles_per, tile = t - b * tiles_per;
        if (active && !active[b]) continue;
        T g[G][NT];
        double iH[G];
        const DD WH = scan_warp<T, NT>(L, P, f + (size_t)b * n * NT, n,
                                       tile * ScanTile<T, NT>::SLABS + warp * ScanTile<T, NT>::WARP_SLABS, lane,
                                       g, iH);
        if (lane == 0) {
            sh[warp] = WH.hi;
            sl[warp] = WH.lo;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            DD TH{0.0, 0.0};
            for (int w = 0; w < SCAN_WARPS; ++w) TH = dd_mul_add(P.p[LOGW], TH, DD{sh[w], sl[w]});
            maps[t] = ScanTileMap{TH.hi, TH.lo};
        }
        __syncthreads();
    }
}

// one CTA per problem: each thread composes a contiguous run of tile maps
// (x -> A x + H_k, A = alpha^tile), the runs are scanned across the CTA,
// each thread then writes its tiles' incoming s (all in double-double)
constexpr int SCAN_CARRY_THREADS = 512;
template <typename T, int NT>
__global__ void __launch_bounds__(SCAN_CARRY_THREADS)
    scan_carry_kernel(const __grid_constant__ LevelC<T, NT> L, long long tiles_per, const ScanTileMap *maps,
                      ScanCarry *carry, const int *active)
{
    constexpr int LOGT = 31 - __builtin_clz((unsigned)ScanTile<T, NT>::SLABS);
    __shared__ double sAh[SCAN_CARRY_THREADS], sAl[SCAN_CARRY_THREADS], sHh[SCAN_CARRY_THREADS],
        sHl[SCAN_CARRY_THREADS];
    const int b = blockIdx.x;
    if (active && !active[b]) return;
    const ScanPowers P = scan_powers(DD{(double)L.calpha, L.calpha_lo}, LOGT);
    const DD TA = P.p[LOGT];
    const int t = threadIdx.x, Pn = blockDim.x;
    const ScanTileMap *mb = maps + (size_t)b * tiles_per;
    ScanCarry *cb = carry + (size_t)b * tiles_per;
    const long long m = (tiles_per + Pn - 1) / Pn;
    const long long a = min(tiles_per, (long long)t * m), e = min(tiles_per, a + m);
    DD A{1.0, 0.0}, H{0.0, 0.0};  // the run's map
    for (long long k = a; k < e; ++k) {
        const ScanTileMap q = mb[k];
        H = dd_mul_add(TA, H, DD{q.Hhi, q.Hlo});
        A = dd_mul(TA, A);
    }
    sAh[t] = A.hi;
    sAl[t] = A.lo;
    sHh[t] = H.hi;
    sHl[t] = H.lo;
    __syncthreads();
    for (int off = 1; off < Pn; off <<= 1) {  // inclusive scan of the runs' maps
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
    DD s = t == 0 ? DD{0.0, 0.0} : DD{sHh[t - 1], sHl[t - 1]};  // s before the run (s_{-1} = 0)
    for (long long k = a; k < e; ++k) {
        cb[k] = ScanCarry{s.hi, s.lo};
        const ScanTileMap q = mb[k];
        s = dd_mul_add(TA, s, DD{q.Hhi, q.Hlo});
    }
}

template <typename T, int NT>
__global__ void __launch_bounds__(SCAN_WARPS * 32)
    scan_replay_kernel(const __grid_constant__ LevelC<T, NT> L, const T *f, T *u, long long n, int batch,
                       long long tiles_per, const ScanCarry *carry, const int *active)
{
    constexpr int G = ScanTile<T, NT>::GROUPS;
    constexpr int LOGW = 31 - __builtin_clz((unsigned)ScanTile<T, NT>::WARP_SLABS);
    __shared__ double sh[SCAN_WARPS], sl[SCAN_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const ScanPowers P = scan_powers(DD{(double)L.calpha, L.calpha_lo}, LOGW);
    // alpha^(lane+1): a lane's inclusive multiplier within its group
    DD laneA_dd{1.0, 0.0};
#pragma unroll
    for (int q = 0; q < 5; ++q)
        if ((lane + 1) & (1 << q)) laneA_dd = dd_mul(laneA_dd, P.p[q]);
    if (lane == 31) laneA_dd = P.p[5];
    const double laneA = laneA_dd.hi;
    const long long total = tiles_per * batch;
    for (long long t = blockIdx.x; t < total; t += gridDim.x) {
        const long long b = t / tiles_per, tile = t - b * tiles_per;
        if (active && !active[b]) continue;
        T g[G][NT];
        double iH[G];
        const long long s0 = tile * ScanTile<T, NT>::SLABS + warp * ScanTile<T, NT>::WARP_SLABS;
        const DD WH = scan_warp<T, NT>(L, P, f + (size_t)b * n * NT, n, s0, lane, g, iH);
        if (lane == 0) {
            sh[warp] = WH.hi;
            sl[warp] = WH.lo;
        }
        __syncthreads();
        // this warp's incoming s: the tile's, then the preceding warps' maps
        DD sin{carry[t].hi, carry[t].lo};
        for (int w = 0; w < warp; ++w) sin = dd_mul_add(P.p[LOGW], sin, DD{sh[w], sl[w]});
        __syncthreads();
        T *ub = u + (size_t)b * n * NT;
        double sg = __dadd_rn(sin.hi, sin.lo);  // the warp's incoming s, then each group's (local)
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const double s_incl = __fma_rn(laneA, sg, iH[j]);  // s after this lane's slab
            double s_prev = __shfl_up_sync(0xffffffffu, s_incl, 1);
            if (lane == 0) s_prev = sg;
            const long long k = s0 + 32LL * j + lane;
            if (k < n) {
                T o[NT];
#pragma unroll
                for (int i = 0; i < NT; ++i) o[i] = (T)__fma_rn(s_prev, (double)L.cw[i], (double)g[j][i]);
                store_slab<T, NT>(ub + k * NT, o);
            }
            sg = __shfl_sync(0xffffffffu, s_incl, 31);
        }
    }
}

}  // namespace tmg
