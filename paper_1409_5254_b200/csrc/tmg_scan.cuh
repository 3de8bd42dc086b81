// Grid-wide exact solve of the block lower-bidiagonal system L u = f as an
// associative scan with decoupled look-back (forward_solve, dg.py:290-303,
// and the coarsest-level solve, multigrid.py:200-205, method "scan").
//
// The sparse coupling N = outer(eval_start, eval_end) is rank one, so with
// g_k = LU^-1 f_k and h_k = e.g_k the block recurrence collapses to a scalar
// affine one (LevelC::ce, cw, calpha):
//     s_k = alpha s_{k-1} + h_k,      u_k = g_k + s_{k-1} w,      s_{-1} = 0.
// Each warp owns a tile of SCAN_GROUPS x 32 consecutive slabs (a power of two;
// one slab per lane per group, so every load and store is a coalesced
// 32-slab row):
//   1. g, h per slab; warp-inclusive scan of the maps x -> alpha x + h per
//      group (5 shuffle steps); the tile's map (A, H) by composing the groups;
//   2. publish (A, H), look back over the preceding tiles of the problem,
//      32 at a time (aggregates until an inclusive prefix) for the incoming
//      s, publish the tile's inclusive s;
//   3. replay: u = g + s_prev w from the registers (f is read once, u
//      written once: 2 n_t s bytes per slab, HBM-bound).
// Tiles are handed out in order by an atomic counter, so every tile a warp
// waits for is already running (no deadlock).  Not bitwise with the serial
// substitution (different association; |alpha| <= 1 keeps it stable): the
// result agrees with the extended-precision solution to a few ulp per slab.
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
struct ScanTileState {
    double Ahi, Alo, Hhi, Hlo;  // the tile's map x -> A x + H (flag >= 1)
    double Shi, Slo;            // s after the tile (flag 2)
    int flag;                   // 0: nothing yet, 1: aggregate, 2: aggregate + inclusive
    int pad;
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


// spin with relaxed loads (an acquire load per poll would invalidate L1 every
// iteration); the caller fences once after seeing the flag set
__device__ __forceinline__ int scan_flag_poll(const int *p)
{
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void scan_fence_acquire()
{
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void scan_flag_store(int *p, int v)
{
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename T, int NT>
__global__ void __launch_bounds__(SCAN_WARPS * 32, 2)
    scan_solve_kernel(const __grid_constant__ LevelC<T, NT> L, const T *f, T *u, long long n, int batch,
                      long long tiles_per, ScanTileState *st, unsigned long long *counter, const int *active)
{
    const int lane = threadIdx.x & 31;
    const long long total = tiles_per * batch;
    constexpr int SCAN_GROUPS = scan_groups<NT>();
    const long long TILE = 32LL * SCAN_GROUPS;
    const DD alpha{(double)L.calpha, L.calpha_lo};
    while (true) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(counter, 1ULL);
        t = __shfl_sync(0xffffffffu, t, 0);
        if ((long long)t >= total) return;
        const long long b = (long long)t / tiles_per;
        const long long tile = (long long)t - b * tiles_per;
        if (active && !active[b]) continue;
        const T *fb = f + (size_t)b * n * NT;
        T *ub = u + (size_t)b * n * NT;
        ScanTileState *sb = st + b * tiles_per;
        const long long s0 = tile * TILE;

        // 1. per group: g, h; inclusive double-double scan of the maps
        //    x -> alpha x + h over the lanes (past the end: identity)
        T g[SCAN_GROUPS][NT];
        DD iH[SCAN_GROUPS], gA[SCAN_GROUPS];  // per group: lanes' inclusive H, the group's multiplier
        DD laneA{1.0, 0.0};                   // alpha^(lane+1): a lane's inclusive multiplier
#pragma unroll
        for (int j = 0; j < SCAN_GROUPS; ++j) {
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
            DD A = k < n ? alpha : DD{1.0, 0.0}, H{k < n ? (double)h : 0.0, 0.0};
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const DD pa{__shfl_up_sync(0xffffffffu, A.hi, off), __shfl_up_sync(0xffffffffu, A.lo, off)};
                const DD ph{__shfl_up_sync(0xffffffffu, H.hi, off), __shfl_up_sync(0xffffffffu, H.lo, off)};
                if (lane >= off) {
                    H = dd_mul_add(A, ph, H);  // (A, H) o (pa, ph): x -> A (pa x + ph) + H
                    A = dd_mul(A, pa);
                }
            }
            if (j == 0) laneA = A;
            iH[j] = H;
            gA[j] = DD{__shfl_sync(0xffffffffu, A.hi, 31), __shfl_sync(0xffffffffu, A.lo, 31)};
        }
        // the tile's map: the groups' maps composed in order
        DD TA{1.0, 0.0}, TH{0.0, 0.0};
#pragma unroll
        for (int j = 0; j < SCAN_GROUPS; ++j) {
            const DD gh{__shfl_sync(0xffffffffu, iH[j].hi, 31), __shfl_sync(0xffffffffu, iH[j].lo, 31)};
            TH = dd_mul_add(gA[j], TH, gh);
            TA = dd_mul(gA[j], TA);
        }

        // 2. decoupled look-back for the incoming s (double-double), one
        //    window of 32 preceding tiles per step (a tile per lane): the
        //    nearest tile with its inclusive s ends the walk, the aggregates
        //    before it are composed with a shuffle tree
        if (lane == 0 && tile > 0) {
            sb[tile].Ahi = TA.hi;
            sb[tile].Alo = TA.lo;
            sb[tile].Hhi = TH.hi;
            sb[tile].Hlo = TH.lo;
            scan_flag_store(&sb[tile].flag, 1);
        }
        DD accA{1.0, 0.0}, accH{0.0, 0.0};  // s_in = accA * (s after the window) + accH
        for (long long w0 = tile - 1; w0 >= 0; w0 -= 32) {
            const long long p = w0 - lane;
            int fl = 2;
            DD a{0.0, 0.0}, h{0.0, 0.0};  // before the problem start: s = 0 (a constant map)
            if (p >= 0) {
                while ((fl = scan_flag_poll(&sb[p].flag)) == 0) {
                }
                scan_fence_acquire();
                if (fl == 2) {
                    h = DD{*(volatile double *)&sb[p].Shi, *(volatile double *)&sb[p].Slo};
                } else {
                    a = DD{*(volatile double *)&sb[p].Ahi, *(volatile double *)&sb[p].Alo};
                    h = DD{*(volatile double *)&sb[p].Hhi, *(volatile double *)&sb[p].Hlo};
                }
            }
            const unsigned m2 = __ballot_sync(0xffffffffu, fl == 2);
            const int k = m2 ? __ffs(m2) - 1 : 32;
            if (lane > k) {  // beyond the nearest inclusive tile: not needed
                a = DD{1.0, 0.0};
                h = DD{0.0, 0.0};
            }
            // map_0 o map_1 o ... o map_31 (lane 0 = the nearest tile, applied last)
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const DD pa{__shfl_down_sync(0xffffffffu, a.hi, off), __shfl_down_sync(0xffffffffu, a.lo, off)};
                const DD ph{__shfl_down_sync(0xffffffffu, h.hi, off), __shfl_down_sync(0xffffffffu, h.lo, off)};
                if (lane + off < 32) {
                    h = dd_mul_add(a, ph, h);
                    a = dd_mul(a, pa);
                }
            }
            accH = dd_mul_add(accA, h, accH);  // meaningful in lane 0
            accA = dd_mul(accA, a);
            if (k < 32) break;
        }
        DD sin{__shfl_sync(0xffffffffu, accH.hi, 0), __shfl_sync(0xffffffffu, accH.lo, 0)};
        if (lane == 0) {
            const DD sout = dd_mul_add(TA, sin, TH);
            sb[tile].Ahi = TA.hi;
            sb[tile].Alo = TA.lo;
            sb[tile].Hhi = TH.hi;
            sb[tile].Hlo = TH.lo;
            sb[tile].Shi = sout.hi;
            sb[tile].Slo = sout.lo;
            scan_flag_store(&sb[tile].flag, 2);
        }

        // 3. replay from the registers: u = g + s_prev w, s_prev in double-double
#pragma unroll
        for (int j = 0; j < SCAN_GROUPS; ++j) {
            // valid lanes' inclusive multiplier is alpha^(lane+1) in every group
            const DD s_incl = dd_mul_add(laneA, sin, iH[j]);
            DD s_prev{__shfl_up_sync(0xffffffffu, s_incl.hi, 1), __shfl_up_sync(0xffffffffu, s_incl.lo, 1)};
            if (lane == 0) s_prev = sin;
            const long long k = s0 + 32LL * j + lane;
            if (k < n) {
                T o[NT];
#pragma unroll
                for (int i = 0; i < NT; ++i)
                    o[i] = (T)__fma_rn(s_prev.hi, (double)L.cw[i],
                                       __fma_rn(s_prev.lo, (double)L.cw[i], (double)g[j][i]));
                store_slab<T, NT>(ub + k * NT, o);
            }
            sin = DD{__shfl_sync(0xffffffffu, s_incl.hi, 31), __shfl_sync(0xffffffffu, s_incl.lo, 31)};
        }
    }
}

}  // namespace tmg
