// Plain data shared by the host driver and the kernels.
#pragma once
#include "tmg_slab.cuh"

namespace tmg {

constexpr int TAIL_THREADS = 512;

// Programmatic dependent launch (the plan's kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): a kernel lets its
// successor be scheduled as soon as all of its CTAs have started, and waits
// for its predecessor's completion (and memory) before its first global
// access.  Launch latency and CTA rasterisation overlap the previous kernel's
// tail; without the attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
constexpr int MAXLEV = 48;

// streaming kernels: consecutive slabs owned by one lane (a row is 32*P slabs).
// Two slabs give each lane two independent dependency chains and make the
// restriction pairs lane-local; larger fp64 blocks would spill.
#ifndef TMG_WIDE_FP64
#define TMG_WIDE_FP64 0  // experiment: two-slab lanes for n_t >= 3 fp64 too (one 8-warp CTA per SM)
#endif
template <typename T, int NT> constexpr int slabs_per_lane() { return (NT <= 2 || sizeof(T) == 4 || TMG_WIDE_FP64) ? 2 : 1; }
// fine slabs per TMA ring stage (a multiple of the row): the per-stage work
// (mbarrier wait, proxy fence, refill) is ~80 instructions, so two-slab lanes
// take two 64-slab rows per stage; one-slab lanes keep 2 rows of 32 slabs
// (larger fp64 stages would not leave two CTAs per SM)
#ifndef TMG_STAGE_SLABS_P2
#define TMG_STAGE_SLABS_P2 128
#endif
template <typename T, int NT> constexpr int stage_slabs() { return slabs_per_lane<T, NT>() == 2 ? TMG_STAGE_SLABS_P2 : 64; }

// per-problem iteration state (multigrid.py:481-496)
struct ProbState {
    double tol;
    int iters;
    int active;
    int max_iters;
    int converged;
};

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
    int nu1, nu2, dot_variant;
    int gamma;                    // cycle kind (1 V, 2 W, 3 F): full mode, each_kind; else the caller's
    int each_kind;                // cycle mode: 1 = every cycle is of kind gamma; 0 = the caller's visits
    int coarse_scan;              // coarsest solve by the CTA scan (not bitwise)
    int levels_stride;            // 0: one operator for the batch; else problem b's levels at b*stride
    unsigned long long *trace;    // optional: per-phase SM-cycle totals of problem 0 (diagnostics)
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


template <typename T, int NT>
__host__ __device__ constexpr size_t tail_fixed_smem(int nlev)
{
    // LevelC[nlev] | meta[4 nlev] | scan scratch [2][TT] | part[TT] (+ alignment)
    return sizeof(LevelC<T, NT>) * (size_t)nlev + sizeof(int) * 4 * (size_t)nlev + sizeof(T) * 2 * TAIL_THREADS +
           sizeof(double) * TAIL_THREADS + 64;
}

}  // namespace tmg
