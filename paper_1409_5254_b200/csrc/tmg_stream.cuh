// Streaming level kernels: one warp walks a contiguous chunk of slabs, one
// "row" of 32*P slabs at a time.  Lane l owns the P consecutive slabs
// P*l .. P*l+P-1 of the row (P = 2 for n_t <= 2 in fp64 and for fp32, else 1)
// and keeps their n_t values in registers through all sweeps of the pass:
//
//   down:  nu1 sweeps -> residual -> restriction        (multigrid.py:274-285)
//   up:    prolong-add -> nu2 sweeps [-> residual norm] (multigrid.py:317-327,
//                                                         447-459)
//
// Jacobi reads only slab n and n-1 of the previous iterate (multigrid.py:
// 168-180).  A lane's second slab takes its predecessor from the lane's first
// slab; the first slab's predecessor is one rotate-shuffle away: lane l
// receives lane l-1's last slab and lane 0 receives lane 31's -- the value the
// NEXT row's lane 0 will need -- so lane 0 swaps it with the carry it kept
// from the previous row.  With P = 2 a restriction pair (2i, 2i+1) and the two
// fine slabs of a prolongation live in one lane: no shuffles there at all.
// A chunk that does not start at slab 0 first runs one "warm-up" row over the
// 32*P slabs before it (after k sweeps only slabs >= k of it are valid; the
// last one needs nu+1 <= 32*P of them), so warps never synchronise with each
// other: the pass is one HBM read of u, f (and u_coarse) and one write of u
// (and f_coarse) per slab.
//
// Rows arrive in a per-warp shared-memory ring (stage_slabs() per stage) filled by
// the TMA engine (cp.async.bulk global->shared, completion on an mbarrier, L2
// evict-first); lane 0 refills a stage as soon as the warp has read it.
// Interior rows run a specialised path (every slab valid, every slab has a
// predecessor); the problem's first row and a ragged last row take the
// general path.
#pragma once
#include "tmg_slab.cuh"
#include "tmg_types.cuh"

namespace tmg {

constexpr int SW_STAGES = 4;        // max ring stages per warp
constexpr int SW_LEAF_BATCH = 4;    // numpy leaves reduced together (one per 8 lanes)
#ifndef TMG_P2_WARPS
#define TMG_P2_WARPS 8
#endif
#ifndef TMG_P2_MINB
#define TMG_P2_MINB 2
#endif
// CTA shape: 2 CTAs of 8 warps per SM (~110 registers per thread).  3 CTAs of
// 6 warps (96 registers) measured no faster: the passes are issue-bound, not
// latency-bound, at this occupancy.
template <typename T, int NT> struct CtaShape {
    static constexpr bool PAIR = slabs_per_lane<T, NT>() == 2;
    // two fp64 slabs of n_t >= 3 per lane need > 128 registers: one CTA per SM
    static constexpr bool WIDE = PAIR && sizeof(T) == 8 && NT >= 3;
    static constexpr int WARPS = WIDE ? 8 : PAIR ? TMG_P2_WARPS : 8;
    static constexpr int MINB = WIDE ? 1 : PAIR ? TMG_P2_MINB : 2;
    // shared memory per CTA that keeps MINB CTAs resident (227 KB per SM,
    // 1 KB reserved per CTA)
    static constexpr size_t CAP = WIDE ? 200 * 1024 : PAIR ? (TMG_P2_MINB >= 3 ? 72 * 1024 : 104 * 1024) : 110 * 1024;
};

enum StreamFlags : int {
    SF_ZERO_GUESS = 1,   // u_in is the zero vector: not read
    SF_RESTRICT = 2,     // residual + restriction -> fc
    SF_WRITE_U = 4,      // store the smoothed iterate
    SF_PROLONG = 8,      // u += P uc before the sweeps
    SF_NORM_LEAF = 16,   // residual -> numpy pairwise leaf sums -> leaf_out
    SF_NORM_SQ = 32,     // residual -> per-slab squared norms -> sq_out
    SF_WRITE_R = 64,     // residual -> r_out
    SF_TMA = 128,        // all problem bases are 16-byte aligned: use the bulk-copy ring
};

// kernel specialisations: the plan's hot passes get their flags at compile time
// K_DOWNNORM: a down pass that also returns the residual norm of its INPUT
// (taken from the first sweep's residual -- the stopping test of the previous
// cycle comes for free with the next cycle's first pass)
// K_UP2: an up pass that RECOMPUTES the nu pre-sweeps from the level's
// original iterate (bitwise the same values the down pass had) instead of
// reading a stored pre-smoothed iterate -- the down pass then writes no u.
// K_UP2NORM: K_UP2 that also returns the residual norm of its OUTPUT (the
// stopping test of the cycle it ends, multigrid.py:447-459)
// K_UP2DOWN: the finest up pass of cycle k FUSED with the finest down pass of
// cycle k+1 (K_UP2 then K_DOWNNORM on the same rows in registers): u is read
// and f read once for both, the new iterate stored once; the down part is
// speculative exactly like the separate K_DOWNNORM was (discarded when the
// stopping test ends the solve).  Halo rows alternate between two buffers by
// cycle parity (the up part reads the previous cycle's, the down part writes
// the next one's).
enum Kind : int { K_GENERIC = 0, K_DOWN = 1, K_UP = 2, K_UPNORM = 3, K_DOWNNORM = 4, K_UP2 = 5, K_UP2NORM = 6,
                  K_UP2DOWN = 7 };

template <typename T> struct StreamArgs {
    const T *f;
    const T *f_alt;        // K_DOWN at level 1 under the vertical fusion: f double-buffered by cycle parity
    const T *f1;           // stream_kernel_v: level-1 right-hand side, buffer A (parity 0 reads A, writes B)
    T *f1_alt;             // stream_kernel_v: buffer B
    const T *u_in;
    T *u_out;
    const T *uc;
    T *fc;
    T *r_out;
    T *halo;               // [batch][chunks][32*P][NT]: each chunk's last row of the ORIGINAL
                           // iterate (written by down passes, read by K_UP2 warm-up rows)
    T *halo_alt;           // K_UP2DOWN: the second halo buffer
    const int *iters;      // K_UP2DOWN: per-problem cycle counter (parity picks the halo buffer)
    int iters_stride;      // in ints
    double *sq_out;
    double *leaf_out;
    const int *active;
    long long n;           // fine slabs per problem
    long long chunks;      // chunks per problem
    int batch;
    int rows_per_chunk;    // rows of 32*P slabs; a multiple of the stage and of leaf_rows
    int leaf_rows;         // rows per numpy pairwise leaf (SF_NORM_LEAF)
    int flags;
};

// ---- PTX helpers (mbarrier + bulk async copy) -------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// TMG_LONG_WARMUP: the row-wise warm-up everywhere (A/B)
__device__ __forceinline__ constexpr bool warm_short()
{
#ifdef TMG_LONG_WARMUP
    return false;
#else
    return true;
#endif
}

template <int KIND> struct KindProlongs {
    static constexpr bool value = KIND != K_DOWN && KIND != K_DOWNNORM;
};
template <int KIND> struct KindLeaf {
    static constexpr bool value =
        KIND == K_GENERIC || KIND == K_UPNORM || KIND == K_DOWNNORM || KIND == K_UP2NORM || KIND == K_UP2DOWN;
};

// vector load/store of one lane's P*NT consecutive elements (16-byte pieces
// when the lane stride allows, else 8-byte, else scalar)
template <typename T, int NE> struct LaneVec {
    static constexpr int BYTES = NE * (int)sizeof(T);
    static constexpr int VB = (BYTES % 16 == 0) ? 16 : (BYTES % 8 == 0) ? 8 : (int)sizeof(T);
    static constexpr int PER = VB / (int)sizeof(T);
};
template <typename T, int NE> __device__ __forceinline__ void vload(const T *p, T (&x)[NE])
{
    constexpr int PER = LaneVec<T, NE>::PER;
#pragma unroll
    for (int i = 0; i < NE; i += PER) {
        if constexpr (sizeof(T) == 8 && PER == 2) {
            double2 v = *reinterpret_cast<const double2 *>(p + i);
            x[i] = v.x; x[i + 1] = v.y;
        } else if constexpr (sizeof(T) == 4 && PER == 4) {
            float4 v = *reinterpret_cast<const float4 *>(p + i);
            x[i] = v.x; x[i + 1] = v.y; x[i + 2] = v.z; x[i + 3] = v.w;
        } else if constexpr (sizeof(T) == 4 && PER == 2) {
            float2 v = *reinterpret_cast<const float2 *>(p + i);
            x[i] = v.x; x[i + 1] = v.y;
        } else {
            x[i] = p[i];
        }
    }
}
template <typename T, int NE> __device__ __forceinline__ void vstore(T *p, const T (&x)[NE])
{
    constexpr int PER = LaneVec<T, NE>::PER;
#pragma unroll
    for (int i = 0; i < NE; i += PER) {
        if constexpr (sizeof(T) == 8 && PER == 2) {
            *reinterpret_cast<double2 *>(p + i) = make_double2(x[i], x[i + 1]);
        } else if constexpr (sizeof(T) == 4 && PER == 4) {
            *reinterpret_cast<float4 *>(p + i) = make_float4(x[i], x[i + 1], x[i + 2], x[i + 3]);
        } else if constexpr (sizeof(T) == 4 && PER == 2) {
            *reinterpret_cast<float2 *>(p + i) = make_float2(x[i], x[i + 1]);
        } else {
            p[i] = x[i];
        }
    }
}
template <typename T, int NT, int P> __device__ __forceinline__ void load_lane(const T *p, T (&x)[P][NT])
{
    T v[P * NT];
    vload<T, P * NT>(p, v);
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
        for (int i = 0; i < NT; ++i) x[q][i] = v[q * NT + i];
}
template <typename T, int NT, int P> __device__ __forceinline__ void store_lane(T *p, const T (&x)[P][NT])
{
    T v[P * NT];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
        for (int i = 0; i < NT; ++i) v[q * NT + i] = x[q][i];
    vstore<T, P * NT>(p, v);
}

template <typename T, int NT, bool WITH_C, bool LEAF> struct RowLayout {
    static constexpr int P = slabs_per_lane<T, NT>();
    static constexpr int W = 32 * P;                // slabs per row
    static constexpr int G = stage_slabs<T, NT>() / W;  // rows per ring stage
    static constexpr int ROW = W * NT;              // elements of one fine row
    static constexpr int HALF = ROW / 2;            // elements of the matching coarse half-row
    static constexpr int OFF_F = G * ROW;
    static constexpr int OFF_C = 2 * G * ROW;
    static constexpr int STAGE = G * (2 * ROW + (WITH_C ? HALF : 0));
    // per-warp numpy leaf buffer: LB leaves of <= 128 slab norms each
    static constexpr int LB = P == 2 ? SW_LEAF_BATCH : 2;
    static constexpr int LEAFBUF = LEAF ? LB * 128 : 0;
    static constexpr size_t LBYTES = sizeof(T) * LEAFBUF;
    // per-warp copy of (R1, R2) for n_t >= 3 with one slab per lane (R2 padded
    // by 2 elements so the even and odd half-warps read different banks)
    static constexpr int RELEMS = (P == 1 && NT >= 3) ? 2 * NT * NT + 2 : 0;
    static constexpr int RSTRIDE = NT * NT + 2;
    static constexpr size_t RBYTES = ((sizeof(T) * RELEMS + 15) / 16) * 16;
    // signed-zero record (fp64): up to 3 nu + 1 = 13 exchanges per row
    static constexpr size_t RECBYTES = sizeof(T) == 8 ? ((13 * NT * 4 + 15) / 16) * 16 : 0;
    // ring depth from the per-CTA budget of the CTA shape: 2..4 stages
    static constexpr int WARPS = CtaShape<T, NT>::WARPS;
    static constexpr size_t WARP_CAP = CtaShape<T, NT>::CAP / WARPS - LBYTES - RBYTES - RECBYTES;
    static constexpr int ST_RAW = (int)(WARP_CAP / (sizeof(T) * STAGE));
    static constexpr int ST = ST_RAW < 2 ? 2 : (ST_RAW > SW_STAGES ? SW_STAGES : ST_RAW);
    static constexpr size_t BYTES_PER_WARP = sizeof(T) * STAGE * ST + RBYTES + LBYTES + RECBYTES;
    // mbarrier block (one 8-byte barrier per warp and stage), padded to 128 B
    static constexpr size_t BAR_BYTES = ((WARPS * ST * 8 + 127) / 128) * 128;
    static constexpr size_t SMEM_BYTES = BAR_BYTES + BYTES_PER_WARP * WARPS;
};

// RTREG: the restriction blocks (R1, R2) of a two-slab lane held in ordinary
// registers, opaque to the compiler (see transfer_regs)
template <typename T, int NT, int NU, bool SPARSE, int KIND, int PERM, bool RTREG = false> struct Streamer {
    using C = Cpl<T, NT, SPARSE>;
    static constexpr int CF = KIND == K_DOWN ? (SF_RESTRICT | SF_WRITE_U)
                              : KIND == K_UP ? (SF_PROLONG | SF_WRITE_U)
                              : KIND == K_UPNORM ? (SF_PROLONG | SF_WRITE_U | SF_NORM_LEAF)
                              : KIND == K_DOWNNORM ? (SF_RESTRICT | SF_WRITE_U | SF_NORM_LEAF)
                              : KIND == K_UP2 ? (SF_PROLONG | SF_WRITE_U)
                              : KIND == K_UP2NORM ? (SF_PROLONG | SF_WRITE_U | SF_NORM_LEAF)
                              : KIND == K_UP2DOWN ? (SF_PROLONG | SF_WRITE_U | SF_RESTRICT | SF_NORM_LEAF)
                                                  : 0;
    // pre-sweeps recomputed before the prolongation (K_UP2, K_UP2NORM, K_UP2DOWN)
    static constexpr int NPRE = (KIND == K_UP2 || KIND == K_UP2NORM || KIND == K_UP2DOWN) ? NU : 0;
    // sweeps of the next cycle's down pass after the up pass (K_UP2DOWN; nu1 == nu2)
    static constexpr int NPOST = KIND == K_UP2DOWN ? NU : 0;
    // norm of the pass's input (K_DOWNNORM) rather than of its output
    static constexpr bool NORM_IN = KIND == K_DOWNNORM && NU > 0;
    static constexpr int P = slabs_per_lane<T, NT>();
    static constexpr int W = 32 * P;
    static constexpr int LB = RowLayout<T, NT, true, true>::LB;
    const LevelC<T, NT> &L;
    const StreamArgs<T> &a;
    int lane;
    int flags;
    // one slab per lane: this lane's transfer block (odd lanes R2, even lanes
    // R1) in registers for n_t <= 2, a per-warp shared-memory copy above
    static constexpr bool RREG = P == 1 && NT * NT * sizeof(T) <= 64;
    // exact signed zeros of the sparse coupling (see neg_zero_rows): rows
    // whose f has no -0 skip them; the others need the sign bits of the
    // previous row's last slab at every exchange, which lane 31 leaves in
    // `rec` (the high words of its slab: one store per exchange)
    static constexpr bool TRACK = SPARSE && !fast_fp<T>();
    static constexpr int NX = NPRE + NU + NPOST + 1;  // exchanges per row
    T Rm[RREG ? NT * NT : 1];
    T Rr1[RTREG ? NT * NT : 1], Rr2[RTREG ? NT * NT : 1];
    const T *Rs;
    unsigned *rec;           // [NX][NT] (TRACK)
    C carry[NPRE + NU + NPOST + 1];  // lane 0: predecessor data of the next row, per sweep
    T *leafbuf;              // per-warp numpy leaf buffer (SF_NORM_LEAF)
    int leaf_q;              // rows buffered in leafbuf
    int lb = LB;             // leaves per flush (the buffer's capacity)
    long long leaf0;         // leaf_out index of the first buffered leaf (leaf_begin)
    long long nc;
    bool write_u;            // the pass stores u (u_out given)
    bool vec_out;            // u_out rows are 16-byte aligned (vector stores)
    T *halo_w;               // K_UP2DOWN: this lane's slot of the chunk's halo row (last row only)

    // ptxas treats kernel-parameter constants as uniform values: in the coarse
    // down pairs it parks (R1, R2) in ordinary registers outside the row loop
    // and then, every row, spills four uniform registers and moves the twelve
    // halves back into uniform registers (R2UR) just to use each once as a
    // uniform operand -- 20 of the pass's 284 instructions per row.  Values
    // that came out of a shuffle are not "uniform" any more and are used
    // straight from their registers.
    __device__ __forceinline__ void transfer_regs()
    {
        if constexpr (RTREG) {
#pragma unroll
            for (int i = 0; i < NT * NT; ++i) {
                // (a select against a lane-dependent value under a condition
                // that always holds: the result is the constant, but not
                // provably uniform)
                Rr1[i] = a.n > 0 ? L.R1[i] : (T)lane;
                Rr2[i] = a.n > 0 ? L.R2[i] : (T)lane;
            }
        }
    }
    __device__ __forceinline__ bool has(int f) const
    {
        return KIND == K_GENERIC ? (flags & f) != 0 : (CF & f) != 0;
    }
    __device__ __forceinline__ bool need_r() const
    {
        return has(SF_RESTRICT) || has(SF_NORM_LEAF) || has(SF_NORM_SQ) || has(SF_WRITE_R);
    }

    // numpy pairwise leaves (np.sum over the slab norms, multigrid.py:459):
    // accumulator j of a leaf sums its slabs j, j+8, j+16, ... in order; the
    // 8 accumulators combine as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)).  Slab
    // norms go to shared memory; every LB leaves, lane 8l+j runs accumulator
    // j of leaf l (a 16-term sequential sum) and 3 shuffle steps combine them.
    __device__ __forceinline__ void leaf_flush(int b)
    {
        __syncwarp();
        // (no integer divisions on the full-buffer path: they are subroutine calls)
        const int nl = leaf_q == lb * a.leaf_rows ? lb : leaf_q / a.leaf_rows;
        const int m = a.leaf_rows * W;
        const int l = lane >> 3, j = lane & 7;
        T acc = T(0);
        if (l < nl) {
            const T *p = leafbuf + l * m + j;
            acc = p[0];
            for (int i = 8; i < m; i += 8) acc = FP<T>::add(acc, p[i]);
        }
        T t1 = FP<T>::add(acc, __shfl_down_sync(0xffffffffu, acc, 1));
        T t2 = FP<T>::add(t1, __shfl_down_sync(0xffffffffu, t1, 2));
        T t3 = FP<T>::add(t2, __shfl_down_sync(0xffffffffu, t2, 4));
        if (j == 0 && l < nl) a.leaf_out[leaf0 + l] = (double)t3;
        __syncwarp();
        leaf_q = 0;
        leaf0 += nl;
    }
    // leaf cursor of a warp whose first row is row0 (a multiple of leaf_rows):
    // index into leaf_out of the next leaf to flush, advanced by every flush
    __device__ __forceinline__ void leaf_begin(long long row0, int b)
    {
        leaf_q = 0;
        leaf0 = (long long)b * (a.n / ((long long)W * a.leaf_rows)) + row0 / a.leaf_rows;
    }
    __device__ __forceinline__ void leaf_row(const T (&r)[P][NT], long long row, int b)
    {
        T sq[P];
#pragma unroll
        for (int q = 0; q < P; ++q) sq[q] = sqnorm<T, NT>(r[q]);
        vstore<T, P>(leafbuf + leaf_q * W + lane * P, sq);
        if (++leaf_q == lb * a.leaf_rows) leaf_flush(b);
    }

    // predecessor data of the row's P slabs at sweep k: the lane's own earlier
    // slab, or (first slab) lane-1's last slab / the carry from the previous row
    template <bool SZ>
    __device__ __forceinline__ void exchange(const T (&u)[P][NT], int k, C (&prev)[P])
    {
        C own[P];
#pragma unroll
        for (int q = 0; q < P; ++q) own[q] = make_cpl<T, NT, SPARSE, SZ>(L, u[q]);
        C x = cpl_shfl<T, NT, SPARSE, SZ>(own[P - 1], (lane + 31) & 31);
        prev[0] = x;
        cpl_select<T, NT, SPARSE, SZ>(prev[0], carry[k], lane == 0);
        if constexpr (TRACK && SZ) {
            // lane 0's predecessor is the previous row's last slab: its sign
            // bits from the record (the carry holds only its coupling sum
            // when that row skipped the signed zeros)
            __syncwarp();
            if (lane == 0) {
                unsigned m = 0;
#pragma unroll
                for (int j = 0; j < NT; ++j) m |= (rec[k * NT + j] >> 31) << j;
                prev[0].m = m;
            }
            __syncwarp();
        }
#pragma unroll
        for (int q = 1; q < P; ++q) prev[q] = own[q - 1];
        carry[k] = x;
        if constexpr (TRACK) {
            if (lane == 31) {
                {
#pragma unroll
                    for (int j = 0; j < NT; ++j) rec[k * NT + j] = (unsigned)__double2hiint((double)u[P - 1][j]);
                }
            }
        }
    }

    // one row; slab0 = this lane's first slab.  INTERIOR: every slab exists
    // and none is slab 0 of the problem.  uo / fco: this lane's u_out /
    // f_coarse elements of the row.
    template <bool INTERIOR>
    __device__ __forceinline__ void row(T (&u)[P][NT], const T (&f)[P][NT], const T (&uc)[NT], long long slab0,
                                        long long row_idx, bool warm, int b, T *uo, T *fco, bool zg)
    {
        if constexpr (TRACK) {
            bool nz = false;
#pragma unroll
            for (int q = 0; q < P; ++q) nz |= neg_zero_rows<T, NT>(f[q]);
            // (inlined: an out-of-line exact path would take the row arrays
            // by reference and force them into local memory -- 3x slower)
            if (TMG_UNLIKELY(__any_sync(0xffffffffu, nz))) {
                row_impl<INTERIOR, true>(u, f, uc, slab0, row_idx, warm, b, uo, fco, zg);
                return;
            }
        }
        row_impl<INTERIOR, false>(u, f, uc, slab0, row_idx, warm, b, uo, fco, zg);
    }

    template <bool INTERIOR, bool SZ>
    __device__ __forceinline__ void row_impl(T (&u)[P][NT], const T (&f)[P][NT], const T (&uc)[NT],
                                             long long slab0, long long row_idx, bool warm, int b, T *uo,
                                             T *fco, bool zg)
    {
        bool valid[P], hp[P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            valid[q] = INTERIOR || slab0 + q < a.n;
            hp[q] = INTERIOR || slab0 + q > 0;
        }
        // K_UP2: the down pass's pre-sweeps, recomputed (same bits)
#pragma unroll
        for (int k = 0; k < NPRE; ++k) {
            if (k == 0 && zg) {
                sweep_zero_j<T, NT, PERM, P>(L, u, f);
                continue;
            }
            C prev[P];
            exchange<SZ>(u, k, prev);
            sweep_j<T, NT, SPARSE, PERM, P, SZ>(L, u, f, prev, hp);
        }
        if (has(SF_PROLONG)) {
#pragma unroll
            for (int q = 0; q < P; ++q) {
                if (INTERIOR || slab0 + q < 2 * nc) {
                    if constexpr (P == 2) {
                        if (q == 0) prolong_reg<T, NT>(L.R1, uc, u[q]);
                        else prolong_reg<T, NT>(L.R2, uc, u[q]);
                    } else if constexpr (RREG) prolong_reg<T, NT>(Rm, uc, u[q]);
                    else prolong_ptr<T, NT>(Rs, uc, u[q]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < NU; ++k) {
            if (!NORM_IN && NPRE == 0 && k == 0 && zg) {
                sweep_zero_j<T, NT, PERM, P>(L, u, f);
                continue;
            }
            C prev[P];
            exchange<SZ>(u, NPRE + k, prev);
            if (NORM_IN && k == 0) {
                // the first sweep's residual IS the input's residual: take its norm
                T y[P][NT];
#pragma unroll
                for (int q = 0; q < P; ++q) residual_perm<T, NT, SPARSE, PERM, SZ>(L, u[q], f[q], prev[q], hp[q], y[q]);
                if (!warm) {
                    T r[P][NT];
#pragma unroll
                    for (int q = 0; q < P; ++q) unpermute<T, NT, PERM>(L, y[q], r[q]);
                    leaf_row(r, row_idx, b);
                }
                finish_j<T, NT, P>(L, u, y);
            } else {
                sweep_j<T, NT, SPARSE, PERM, P, SZ>(L, u, f, prev, hp);
            }
        }
        if constexpr (NPOST > 0) {
            // the up pass is complete: store this cycle's result (and, on the
            // chunk's last row, its halo for the next cycle's up pass)
            if (!warm && write_u) {
                if (INTERIOR && vec_out) {
                    store_lane<T, NT, P>(uo, u);
                } else {
#pragma unroll
                    for (int q = 0; q < P; ++q)
                        if (valid[q]) store_slab<T, NT>(uo + q * NT, u[q]);
                }
            }
            if (!warm && halo_w) store_lane<T, NT, P>(halo_w, u);
            // the next cycle's down pass; its first sweep's residual is the
            // stopping norm of the result just stored
#pragma unroll
            for (int k = 0; k < NPOST; ++k) {
                C prev[P];
                exchange<SZ>(u, NPRE + NU + k, prev);
                if (k == 0) {
                    T y[P][NT];
#pragma unroll
                    for (int q = 0; q < P; ++q) residual_perm<T, NT, SPARSE, PERM, SZ>(L, u[q], f[q], prev[q], hp[q], y[q]);
                    if (!warm) {
                        T r[P][NT];
#pragma unroll
                        for (int q = 0; q < P; ++q) unpermute<T, NT, PERM>(L, y[q], r[q]);
                        leaf_row(r, row_idx, b);
                    }
                    finish_j<T, NT, P>(L, u, y);
                } else {
                    sweep_j<T, NT, SPARSE, PERM, P, SZ>(L, u, f, prev, hp);
                }
            }
        }
        if (need_r()) {
            C prev[P];
            exchange<SZ>(u, NPRE + NU + NPOST, prev);
            if (!warm) {
                T r[P][NT];
#pragma unroll
                for (int q = 0; q < P; ++q) residual<T, NT, SPARSE, SZ>(L, u[q], f[q], prev[q], hp[q], r[q]);
                if (has(SF_WRITE_R)) {
#pragma unroll
                    for (int q = 0; q < P; ++q)
                        if (valid[q]) store_slab<T, NT>(a.r_out + ((size_t)b * a.n + slab0 + q) * NT, r[q]);
                }
                if (has(SF_RESTRICT)) {
                    T p[NT];
                    bool st;
                    if constexpr (P == 2) {
                        T p1[NT];
                        if constexpr (RTREG) {
                            restrict_reg<T, NT>(Rr1, r[0], p);
                            restrict_reg<T, NT>(Rr2, r[1], p1);
                        } else {
                            restrict_reg<T, NT>(L.R1, r[0], p);
                            restrict_reg<T, NT>(L.R2, r[1], p1);
                        }
#pragma unroll
                        for (int i = 0; i < NT; ++i) p[i] = FP<T>::add(p[i], p1[i]);
                        st = true;
                    } else {
                        T qq[NT];
                        if constexpr (RREG) restrict_reg<T, NT>(Rm, r[0], p);
                        else restrict_ptr<T, NT>(Rs, r[0], p);
#pragma unroll
                        for (int i = 0; i < NT; ++i) qq[i] = __shfl_down_sync(0xffffffffu, p[i], 1);
#pragma unroll
                        for (int i = 0; i < NT; ++i) p[i] = FP<T>::add(p[i], qq[i]);
                        st = !(lane & 1);
                    }
                    if (st && (INTERIOR || (slab0 >> 1) < nc)) store_slab<T, NT>(fco, p);
                }
                if (has(SF_NORM_SQ)) {
#pragma unroll
                    for (int q = 0; q < P; ++q)
                        if (valid[q]) a.sq_out[(size_t)b * a.n + slab0 + q] = (double)sqnorm<T, NT>(r[q]);
                }
                if (!NORM_IN && NPOST == 0 && has(SF_NORM_LEAF)) leaf_row(r, row_idx, b);
            }
        }
        if (NPOST == 0 && has(SF_WRITE_U) && !warm && write_u) {
            if (INTERIOR && vec_out) {
                store_lane<T, NT, P>(uo, u);
            } else {
#pragma unroll
                for (int q = 0; q < P; ++q)
                    if (valid[q]) store_slab<T, NT>(uo + q * NT, u[q]);
            }
        }
    }
};

template <typename T, int NT, int NU, bool SPARSE, int KIND, int PERM>
__global__ void __launch_bounds__(CtaShape<T, NT>::WARPS * 32, CtaShape<T, NT>::MINB)
    stream_kernel(const __grid_constant__ LevelC<T, NT> L, const __grid_constant__ StreamArgs<T> a)
{
    constexpr bool WITH_C = KindProlongs<KIND>::value;
    using Lay = RowLayout<T, NT, WITH_C, KindLeaf<KIND>::value>;
    using S = Streamer<T, NT, NU, SPARSE, KIND, PERM, KIND == K_DOWN && Lay::P == 2 && sizeof(T) == 8>;
    constexpr int P = S::P;
    constexpr int W = Lay::W;
    constexpr int G = Lay::G;
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const long long gw = (long long)blockIdx.x * Lay::WARPS + warp;
    if (gw >= (long long)a.batch * a.chunks) return;
    const int b = (int)(gw / a.chunks);
    const long long chunk = gw - (long long)b * a.chunks;
    if (a.active && !a.active[b]) return;

    S st{L, a, lane, a.flags};
    st.transfer_regs();
    const long long n = a.n;
    st.nc = n >> 1;
    const long long nrows = (n + W - 1) / W;
    const long long row0 = chunk * a.rows_per_chunk;
    const int rows = (int)min((long long)a.rows_per_chunk, nrows - row0);
    const int ngroups = (rows + G - 1) / G;
    const bool zero_guess = a.flags & SF_ZERO_GUESS;
    const bool tma = a.flags & SF_TMA;
    const bool prolong = WITH_C && st.has(SF_PROLONG);
    const int lofs = lane * P;  // this lane's first slab within a row

    const T *fsrc = (a.f_alt && (a.iters[(size_t)b * a.iters_stride] & 1)) ? a.f_alt : a.f;
    const T *fb = fsrc + (size_t)b * n * NT;
    const T *ub = zero_guess ? nullptr : a.u_in + (size_t)b * n * NT;
    const T *ucb = prolong ? a.uc + (size_t)b * st.nc * NT : nullptr;

    constexpr int ST = Lay::ST;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem) + warp * ST;
    unsigned char *wbase = smem + Lay::BAR_BYTES + (size_t)warp * Lay::BYTES_PER_WARP;
    T *ring = reinterpret_cast<T *>(wbase + Lay::RBYTES + Lay::LBYTES + Lay::RECBYTES);
    st.leafbuf = reinterpret_cast<T *>(wbase + Lay::RBYTES);
    st.rec = reinterpret_cast<unsigned *>(wbase + Lay::RBYTES + Lay::LBYTES);
    if constexpr (P == 1) {
        if (st.has(SF_RESTRICT) || prolong) {
            const bool odd = lane & 1;
            if constexpr (S::RREG) {
#pragma unroll
                for (int i = 0; i < NT * NT; ++i) st.Rm[i] = odd ? L.R2[i] : L.R1[i];
            } else {
                T *rs = reinterpret_cast<T *>(wbase);
                for (int i = lane; i < NT * NT; i += 32) {
                    rs[i] = L.R1[i];
                    rs[Lay::RSTRIDE + i] = L.R2[i];
                }
                __syncwarp();
                st.Rs = rs + (odd ? Lay::RSTRIDE : 0);
            }
        }
    }
#pragma unroll
    for (int k = 0; k <= S::NPRE + NU + S::NPOST; ++k) cpl_zero(st.carry[k]);
    st.halo_w = nullptr;
    // halo buffers: K_UP2DOWN alternates them by the problem's cycle parity
    T *halo_in = a.halo, *halo_next = nullptr;
    if constexpr (S::NPOST > 0) {
        if (a.iters[(size_t)b * a.iters_stride] & 1) {
            halo_in = a.halo_alt;
            halo_next = a.halo;
        } else {
            halo_next = a.halo_alt;
        }
    }
    st.leaf_q = 0;
    st.leaf0 = 0;
    if (KindLeaf<KIND>::value && st.has(SF_NORM_LEAF)) st.leaf_begin(row0, b);

    // groups [0, g_full) consist of G whole rows (and go through the ring when
    // TMA is on); groups [g_int0, g_full) are interior (no slab 0, all valid)
    const int g_full = (int)max(0LL, min((long long)(rows / G), (n / W - row0) / G));
    const int g_int0 = row0 == 0 ? 1 : 0;
    auto group_tma = [&](int g) -> bool { return tma && g < g_full; };
    // per-lane output cursors (advanced by one row at a time)
    st.write_u = st.has(SF_WRITE_U) && a.u_out != nullptr;
    st.vec_out = st.write_u && (((uintptr_t)a.u_out & 15) == 0) && (((n * NT * sizeof(T)) & 15) == 0);
    T *uo = st.write_u ? a.u_out + ((size_t)b * n + (size_t)row0 * W + lofs) * NT : nullptr;
    T *fco = st.has(SF_RESTRICT) ? a.fc + ((size_t)b * st.nc + (((size_t)row0 * W + lofs) >> 1)) * NT : nullptr;
    uint64_t pol = 0;
    if (lane == 0 && tma) {
#pragma unroll
        for (int s = 0; s < ST; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        pol = policy_evict_first();
    }
    __syncwarp();
    auto issue = [&](int g) {  // lane 0 only
        if (!group_tma(g)) return;
        T *stg = ring + (size_t)(g % ST) * Lay::STAGE;
        uint64_t *bar = &bars[g % ST];
        const long long s0 = (row0 + (long long)g * G) * W;
        const uint32_t bytes = (uint32_t)(G * Lay::ROW * sizeof(T));
        const uint32_t cbytes = prolong ? (uint32_t)(G * Lay::HALF * sizeof(T)) : 0u;
        mbar_expect_tx(bar, bytes * (zero_guess ? 1u : 2u) + cbytes);
        bulk_g2s(stg + Lay::OFF_F, fb + s0 * NT, bytes, bar, pol);
        if (!zero_guess) bulk_g2s(stg, ub + s0 * NT, bytes, bar, pol);
        if (cbytes) bulk_g2s(stg + Lay::OFF_C, ucb + (s0 >> 1) * NT, cbytes, bar, pol);
    };
    if (lane == 0 && tma)
        for (int g = 0; g < ngroups && g < ST; ++g) issue(g);

    // general (bounds-checked) load of one row
    auto load_row_gen = [&](long long r, T (&u)[P][NT], T (&f)[P][NT], T (&uc)[NT], bool with_u) {
        const long long s0 = r * W + lofs;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            zero_slab<T, NT>(u[q]);
            zero_slab<T, NT>(f[q]);
            if (s0 + q < n) {
                load_slab_scalar<T, NT>(fb + (s0 + q) * NT, f[q]);
                if (with_u) load_slab_scalar<T, NT>(ub + (s0 + q) * NT, u[q]);
            }
        }
        zero_slab<T, NT>(uc);
        if (prolong && (s0 >> 1) < st.nc) load_slab_scalar<T, NT>(ucb + (s0 >> 1) * NT, uc);
    };

    // warm-up: the row before the chunk, for the carries only
    if (row0 > 0) {
        T u[P][NT], f[P][NT], uc[NT];
        const long long wr = row0 - 1;
        load_row_gen(wr, u, f, uc, !zero_guess && S::NPRE == 0);
        if (S::NPRE > 0 && !zero_guess)  // the neighbour chunk may already have overwritten this row
            load_lane<T, NT, P>(halo_in + ((size_t)b * a.chunks + chunk - 1) * Lay::ROW + lofs * NT, u);
        if (wr > 0) st.template row<true>(u, f, uc, wr * W + lofs, wr, true, b, nullptr, nullptr, zero_guess);
        else st.template row<false>(u, f, uc, wr * W + lofs, wr, true, b, nullptr, nullptr, zero_guess);
    }

    const bool halo_out = a.halo && !zero_guess && chunk + 1 < a.chunks && !S::NPRE;
    for (int g = 0; g < ngroups; ++g) {
        const bool gt = group_tma(g);
        const T *stg = ring + (size_t)(g % ST) * Lay::STAGE;
        const bool interior = g >= g_int0 && g < g_full;
        if (gt) mbar_wait(&bars[g % ST], (uint32_t)((g / ST) & 1));
#pragma unroll 1
        for (int qq = 0; qq < G; ++qq) {
            const int rr = g * G + qq;  // row within the chunk
            if (G > 1 && rr >= rows) break;
            const long long ridx = row0 + rr;
            T u[P][NT], f[P][NT], uc[NT];
            if (gt) {
                load_lane<T, NT, P>(stg + Lay::OFF_F + qq * Lay::ROW + lofs * NT, f);
                if (zero_guess) {
#pragma unroll
                    for (int q = 0; q < P; ++q) zero_slab<T, NT>(u[q]);
                } else {
                    load_lane<T, NT, P>(stg + qq * Lay::ROW + lofs * NT, u);
                }
                if (prolong) load_slab<T, NT>(stg + Lay::OFF_C + qq * Lay::HALF + (lofs >> 1) * NT, uc);
                else zero_slab<T, NT>(uc);
                if (qq == G - 1) {
                    // the stage is fully read: hand it back to the copy engine.
                    // Every lane orders its shared-memory reads of the stage
                    // before the bulk copy (async proxy) that overwrites it.
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0 && g + ST < ngroups) issue(g + ST);
                }
            } else {
                load_row_gen(ridx, u, f, uc, !zero_guess);
            }
            if (halo_out && rr == rows - 1) {
                // the chunk's last row: the next chunk's up-pass warm-up input
                store_lane<T, NT, P>(a.halo + ((size_t)b * a.chunks + chunk) * Lay::ROW + lofs * NT, u);
            }
            if constexpr (S::NPOST > 0)
                st.halo_w = (rr == rows - 1 && chunk + 1 < a.chunks)
                                ? halo_next + ((size_t)b * a.chunks + chunk) * Lay::ROW + lofs * NT
                                : nullptr;
            if (interior)
                st.template row<true>(u, f, uc, ridx * W + lofs, ridx, false, b, uo, fco, zero_guess);
            else
                st.template row<false>(u, f, uc, ridx * W + lofs, ridx, false, b, uo, fco, zero_guess);
            if (st.write_u) uo += Lay::ROW;
            if (fco) fco += Lay::HALF;
        }
    }
    if (KindLeaf<KIND>::value && st.has(SF_NORM_LEAF) && st.leaf_q > 0) st.leaf_flush(b);
}


// ---------------------------------------------------------------------------
// Vertical fusion at the finest level (two-slab lanes): the level-1 up pass
// (zero original iterate: omega LU^-1 f pre-sweep, prolong-add of u_2, nu2
// sweeps) runs INSIDE the fused finest pass.  Per ring stage: one coarse row
// of level 1 (64 slabs) is computed into a per-warp shared-memory row, then
// the two fine rows it covers run the K_UP2DOWN row with their u_c taken from
// that row -- so u_1 is never stored nor re-read.  f_1 alternates between two
// buffers by cycle parity (this cycle's is read here and by nothing later;
// the next cycle's is written here and read by the level-1 down pass), like
// the halo rows.  Warm-up: the coarse row before the chunk, then the fine row
// before it (its u_c is that coarse row's exact second half).
template <typename T, int NT, bool FINEST = true> struct RowLayoutV {
    static constexpr int P = slabs_per_lane<T, NT>();
    static constexpr int W = 32 * P;
    static constexpr int ROW = W * NT;       // elements of a 64-slab row (fine or coarse)
    static constexpr int HALF = ROW / 2;
    // stage: [u rows (FINEST only)] | f rows | coarse f row | coarse-coarse u half row
    static constexpr int OFF_U = 0;
    static constexpr int OFF_F = FINEST ? 2 * ROW : 0;
    static constexpr int OFF_F1 = OFF_F + 2 * ROW;
    static constexpr int OFF_C2 = OFF_F1 + ROW;
    static constexpr int STAGE = OFF_C2 + HALF;
    static constexpr int ST = FINEST ? 2 : 3;
    static constexpr int LB = P == 2 ? 2 : 1;  // numpy leaves per flush (smem budget)
    static constexpr int LEAFBUF = FINEST ? LB * 128 : 0;
    static constexpr int RSTRIDE = NT * NT + 2;
    static constexpr int RELEMS = P == 1 ? 2 * (2 * RSTRIDE) : 0;  // both levels' (R1, R2), one-slab lanes
    static constexpr int WARPS = CtaShape<T, NT>::WARPS;
    // signed-zero records (fp64, nu <= 2): 3 nu + 1 exchanges per fine row, 2 nu + 1 per coarse row
    static constexpr int REC_FINE = 7 * NT, REC_COARSE = 5 * NT;
    static constexpr size_t RECBYTES = sizeof(T) == 8 ? (((REC_FINE + REC_COARSE) * 4 + 15) / 16) * 16 : 0;
    static constexpr size_t BYTES_PER_WARP = sizeof(T) * (STAGE * ST + ROW + LEAFBUF + RELEMS) + RECBYTES;
    static constexpr size_t BAR_BYTES = ((WARPS * ST * 8 + 127) / 128) * 128;
    static constexpr size_t SMEM_BYTES = BAR_BYTES + BYTES_PER_WARP * WARPS;
};

// FINEST: level 0 (K_UP2DOWN rows, in-place u, halo rows and f_1 by cycle
// parity, norm leaves).  !FINEST: a coarse pair (levels l, l+1 >= 1, both from
// the zero guess): K_UP2 rows at level l with u_c from the level-(l+1) row in
// shared memory, u_l written for the next finer level's up pass.
template <typename T, int NT, int NU, bool SPARSE, int PERM, bool FINEST = true>
__global__ void __launch_bounds__(CtaShape<T, NT>::WARPS * 32, CtaShape<T, NT>::MINB)
    stream_kernel_v(const __grid_constant__ LevelC<T, NT> L, const __grid_constant__ LevelC<T, NT> L1,
                    const __grid_constant__ StreamArgs<T> a, const __grid_constant__ StreamArgs<T> a1)
{
    using Lay = RowLayoutV<T, NT, FINEST>;
    using S = Streamer<T, NT, NU, SPARSE, FINEST ? K_UP2DOWN : K_UP2, PERM>;
    using S1 = Streamer<T, NT, NU, SPARSE, K_UP2, PERM>;
    constexpr int P = S::P, W = 32 * P;
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const long long gw = (long long)blockIdx.x * Lay::WARPS + warp;
    if (gw >= (long long)a.batch * a.chunks) return;
    const int b = (int)(gw / a.chunks);
    const long long chunk = gw - (long long)b * a.chunks;
    if (a.active && !a.active[b]) return;

    const long long n = a.n, n1 = n >> 1, n2 = n >> 2;
    S st{L, a, lane, a.flags};
    st.nc = n1;
    S1 s1{L1, a1, lane, a1.flags};
    s1.nc = n2;
    const long long row0 = chunk * a.rows_per_chunk;          // even; every row full (n % 128 == 0)
    const int rows = (int)min((long long)a.rows_per_chunk, n / W - row0);
    const int ngroups = rows >> 1;
    const int lofs = lane * P;
    const bool par = FINEST && (a.iters[(size_t)b * a.iters_stride] & 1);
    T *halo_in = par ? a.halo_alt : a.halo;
    T *halo_next = par ? a.halo : a.halo_alt;
    const T *f1b = (par ? a.f1_alt : a.f1) + (size_t)b * n1 * NT;   // this cycle's level-(l+1) f
    T *fcb = FINEST ? (par ? (T *)a.f1 : a.f1_alt) + (size_t)b * n1 * NT : nullptr;  // next cycle's f_1
    const T *fb = a.f + (size_t)b * n * NT;
    const T *ub = FINEST ? a.u_in + (size_t)b * n * NT : nullptr;
    const T *u2b = a.uc + (size_t)b * n2 * NT;

    uint64_t *bars = reinterpret_cast<uint64_t *>(smem) + warp * Lay::ST;
    unsigned char *wbase = smem + Lay::BAR_BYTES + (size_t)warp * Lay::BYTES_PER_WARP;
    st.leafbuf = reinterpret_cast<T *>(wbase);
    st.lb = Lay::LB;
    T *u1row = reinterpret_cast<T *>(wbase) + Lay::LEAFBUF;
    T *ring = u1row + Lay::ROW;
    {
        unsigned *rec = reinterpret_cast<unsigned *>(wbase + Lay::BYTES_PER_WARP - Lay::RECBYTES);
        st.rec = rec;
        s1.rec = rec + Lay::REC_FINE;
    }
    if constexpr (P == 1) {
        T *rs = ring + Lay::STAGE * Lay::ST;
        for (int i = lane; i < NT * NT; i += 32) {
            rs[i] = L.R1[i];
            rs[Lay::RSTRIDE + i] = L.R2[i];
            rs[2 * Lay::RSTRIDE + i] = L1.R1[i];
            rs[3 * Lay::RSTRIDE + i] = L1.R2[i];
        }
        __syncwarp();
        st.Rs = rs + ((lane & 1) ? Lay::RSTRIDE : 0);
        s1.Rs = rs + 2 * Lay::RSTRIDE + ((lane & 1) ? Lay::RSTRIDE : 0);
    }
#pragma unroll
    for (int k = 0; k <= S::NPRE + NU + S::NPOST; ++k) cpl_zero(st.carry[k]);
#pragma unroll
    for (int k = 0; k <= S1::NPRE + NU; ++k) cpl_zero(s1.carry[k]);
    st.leaf_q = 0;
    st.leaf0 = 0;
    if constexpr (FINEST) st.leaf_begin(row0, b);
    st.halo_w = nullptr;
    st.write_u = true;
    st.vec_out = true;
    s1.leaf_q = 0;
    s1.leaf0 = 0;
    s1.halo_w = nullptr;
    s1.write_u = true;
    s1.vec_out = true;
    T *uo = a.u_out + ((size_t)b * n + (size_t)row0 * W + lofs) * NT;
    T *fco = FINEST ? fcb + (((size_t)row0 * W + lofs) >> 1) * NT : nullptr;
    uint64_t pol = 0;
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < Lay::ST; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        pol = policy_evict_first();
    }
    __syncwarp();
    auto issue = [&](int g) {  // lane 0 only
        T *stg = ring + (size_t)(g % Lay::ST) * Lay::STAGE;
        uint64_t *bar = &bars[g % Lay::ST];
        const long long s0 = (row0 + 2LL * g) * W;      // first fine slab of the stage
        const long long c0 = s0 >> 1;                   // first coarse slab
        const uint32_t fine = (uint32_t)(2 * Lay::ROW * sizeof(T));
        const uint32_t crow = (uint32_t)(Lay::ROW * sizeof(T));
        const uint32_t chalf = (uint32_t)(Lay::HALF * sizeof(T));
        mbar_expect_tx(bar, (FINEST ? 2 : 1) * fine + crow + chalf);
        if (FINEST) bulk_g2s(stg + Lay::OFF_U, ub + s0 * NT, fine, bar, pol);
        bulk_g2s(stg + Lay::OFF_F, fb + s0 * NT, fine, bar, pol);
        bulk_g2s(stg + Lay::OFF_F1, f1b + c0 * NT, crow, bar, pol);
        bulk_g2s(stg + Lay::OFF_C2, u2b + (c0 >> 1) * NT, chalf, bar, pol);
    };
    if (lane == 0)
        for (int g = 0; g < ngroups && g < Lay::ST; ++g) issue(g);

    // coarse row cr (zero original iterate) into u1row
    auto coarse_row = [&](long long cr, const T (&f1)[P][NT], const T (&u2)[NT]) {
        T u[P][NT];
#pragma unroll
        for (int q = 0; q < P; ++q) zero_slab<T, NT>(u[q]);
        if (cr > 0) s1.template row<true>(u, f1, u2, cr * W + lofs, cr, false, b, u1row + lofs * NT, nullptr, true);
        else s1.template row<false>(u, f1, u2, cr * W + lofs, cr, false, b, u1row + lofs * NT, nullptr, true);
        __syncwarp();
    };

    if (row0 > 0 && !FINEST && NU == 1 && warm_short()) {
        // both levels from the zero guess with nu = 1: the pre-sweep needs no
        // predecessor, so the carries depend on two level-(l+1) slabs and one
        // level-l slab before the chunk (same functions, same bits as the rows)
        using C = typename S::C;
        const long long g0 = row0 * W;
        const long long jc = (g0 >> 1) - 1;    // odd; jc - 1 is its even partner under one level-(l+2) slab
        T fa[1][NT], fbb[1][NT], u2[NT], ua[1][NT], ub[1][NT];
        load_slab_scalar<T, NT>(f1b + (jc - 1) * NT, fa[0]);
        load_slab_scalar<T, NT>(f1b + jc * NT, fbb[0]);
        load_slab_scalar<T, NT>(u2b + (jc >> 1) * NT, u2);
        sweep_zero_j<T, NT, PERM, 1>(L1, ua, fa);
        sweep_zero_j<T, NT, PERM, 1>(L1, ub, fbb);
        prolong_reg<T, NT>(L1.R1, u2, ua[0]);
        prolong_reg<T, NT>(L1.R2, u2, ub[0]);
        const C ca[1] = {make_cpl<T, NT, SPARSE, true>(L1, ua[0])};
        s1.carry[1] = make_cpl<T, NT, SPARSE, true>(L1, ub[0]);
        T ubm[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) ubm[j] = ub[0][j];
        const bool hp1[1] = {true};
        sweep_j<T, NT, SPARSE, PERM, 1, true>(L1, ub, fbb, ca, hp1);   // level-(l+1) result at slab jc
        T ff[1][NT], um[1][NT];
        load_slab_scalar<T, NT>(fb + (g0 - 1) * NT, ff[0]);
        sweep_zero_j<T, NT, PERM, 1>(L, um, ff);
        prolong_reg<T, NT>(L.R2, ub[0], um[0]);
        st.carry[1] = make_cpl<T, NT, SPARSE, true>(L, um[0]);
        if constexpr (S::TRACK) {
            if (lane == 0) {
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    s1.rec[NT + j] = (unsigned)__double2hiint((double)ubm[j]);
                    st.rec[NT + j] = (unsigned)__double2hiint((double)um[0][j]);
                }
            }
        }
        __syncwarp();
    } else if (row0 > 0) {
        // warm-up: the coarse row before the chunk, then the fine row before it
        const long long cw = (row0 >> 1) - 1;
        T f1[P][NT], u2[NT];
#pragma unroll
        for (int q = 0; q < P; ++q) load_slab_scalar<T, NT>(f1b + (cw * W + lofs + q) * NT, f1[q]);
        load_slab_scalar<T, NT>(u2b + ((cw * W + lofs) >> 1) * NT, u2);
        coarse_row(cw, f1, u2);
        const long long wr = row0 - 1;
        T u[P][NT], f[P][NT], uc[NT];
#pragma unroll
        for (int q = 0; q < P; ++q) load_slab_scalar<T, NT>(fb + (wr * W + lofs + q) * NT, f[q]);
        if constexpr (FINEST) {
            load_lane<T, NT, P>(halo_in + ((size_t)b * a.chunks + chunk - 1) * Lay::ROW + lofs * NT, u);
        } else {
#pragma unroll
            for (int q = 0; q < P; ++q) zero_slab<T, NT>(u[q]);
        }
        load_slab<T, NT>(u1row + Lay::HALF + (lofs >> 1) * NT, uc);
        st.template row<true>(u, f, uc, wr * W + lofs, wr, true, b, nullptr, nullptr, !FINEST);
        __syncwarp();
    }

    // loop invariants of the per-row bookkeeping as 32-bit row numbers
    const int halo_rr = (FINEST && chunk + 1 < a.chunks) ? rows - 1 : -1;   // row whose result is the chunk's halo
    T *halo_slot = FINEST ? halo_next + ((size_t)b * a.chunks + chunk) * Lay::ROW + lofs * NT : nullptr;
    const int first_rr = row0 == 0 ? 0 : -1;                               // the problem's first row (general path)
    for (int g = 0; g < ngroups; ++g) {
        const T *stg = ring + (size_t)(g % Lay::ST) * Lay::STAGE;
        mbar_wait(&bars[g % Lay::ST], (uint32_t)((g / Lay::ST) & 1));
        {
            T f1[P][NT], u2[NT];
            load_lane<T, NT, P>(stg + Lay::OFF_F1 + lofs * NT, f1);
            load_slab<T, NT>(stg + Lay::OFF_C2 + (lofs >> 1) * NT, u2);
            coarse_row((row0 >> 1) + g, f1, u2);
        }
#pragma unroll 1
        for (int qq = 0; qq < 2; ++qq) {
            const int rr = 2 * g + qq;
            const long long ridx = row0 + rr;
            T u[P][NT], f[P][NT], uc[NT];
            load_lane<T, NT, P>(stg + Lay::OFF_F + qq * Lay::ROW + lofs * NT, f);
            if constexpr (FINEST) {
                load_lane<T, NT, P>(stg + Lay::OFF_U + qq * Lay::ROW + lofs * NT, u);
            } else {
#pragma unroll
                for (int q = 0; q < P; ++q) zero_slab<T, NT>(u[q]);
            }
            load_slab<T, NT>(u1row + qq * Lay::HALF + (lofs >> 1) * NT, uc);
            if (qq == 1) {
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0 && g + Lay::ST < ngroups) issue(g + Lay::ST);
            }
            if constexpr (FINEST) st.halo_w = rr == halo_rr ? halo_slot : nullptr;
            if (rr != first_rr) st.template row<true>(u, f, uc, ridx * W + lofs, ridx, false, b, uo, fco, !FINEST);
            else st.template row<false>(u, f, uc, ridx * W + lofs, ridx, false, b, uo, fco, !FINEST);
            uo += Lay::ROW;
            if constexpr (FINEST) fco += Lay::HALF;
        }
        __syncwarp();  // every lane is done with u1row before the next coarse row overwrites it
    }
    if constexpr (FINEST)
        if (st.leaf_q > 0) st.leaf_flush(b);
}


// ---------------------------------------------------------------------------
// Coarse down-pass pairs (two-slab lanes, both levels from the zero guess):
// per ring stage the two level-l rows' down passes (nu1 sweeps, residual,
// restriction) leave their restricted rows in a per-warp shared-memory row,
// which is stored as f_{l+1} and at once swept as one level-(l+1) row (its own
// down pass: f_{l+2}) -- one launch instead of two, f_{l+1} not re-read.
// Warm-up: three level-l rows before the chunk (the first for the carries,
// the next two for the level-(l+1) row before the chunk), then that row.
template <typename T, int NT> struct RowLayoutD {
    static constexpr int P = slabs_per_lane<T, NT>();
    static constexpr int W = 32 * P;
    static constexpr int ROW = W * NT;
    static constexpr int HALF = ROW / 2;
    static constexpr int STAGE = 2 * ROW;    // two level-l f rows
    static constexpr int ST = 3;
    // one-slab lanes keep both levels' transfer blocks in shared memory
    static constexpr int RSTRIDE = NT * NT + 2;
    static constexpr int RELEMS = P == 1 ? 2 * (2 * RSTRIDE) : 0;
    static constexpr int WARPS = CtaShape<T, NT>::WARPS;
    // signed-zero records (fp64, nu <= 2): nu + 1 exchanges per row, both levels
    static constexpr int REC_ONE = 3 * NT;
    static constexpr size_t RECBYTES = sizeof(T) == 8 ? ((2 * REC_ONE * 4 + 15) / 16) * 16 : 0;
    static constexpr size_t BYTES_PER_WARP = sizeof(T) * (STAGE * ST + ROW + RELEMS) + RECBYTES;
    static constexpr size_t BAR_BYTES = ((WARPS * ST * 8 + 127) / 128) * 128;
    static constexpr size_t SMEM_BYTES = BAR_BYTES + BYTES_PER_WARP * WARPS;
};

template <typename T, int NT, int NU, bool SPARSE, int PERM>
__global__ void __launch_bounds__(CtaShape<T, NT>::WARPS * 32, CtaShape<T, NT>::MINB)
    stream_kernel_d(const __grid_constant__ LevelC<T, NT> L, const __grid_constant__ LevelC<T, NT> L1,
                    const __grid_constant__ StreamArgs<T> a, const __grid_constant__ StreamArgs<T> a1)
{
    using Lay = RowLayoutD<T, NT>;
#ifdef TMG_NO_RTREG
    using S0 = Streamer<T, NT, NU, SPARSE, K_DOWN, PERM>;
#else
    using S0 = Streamer<T, NT, NU, SPARSE, K_DOWN, PERM, RowLayoutD<T, NT>::P == 2 && sizeof(T) == 8>;
#endif
    using S = Streamer<T, NT, NU, SPARSE, K_DOWN, PERM>;
    constexpr int P = S::P, W = 32 * P;
    extern __shared__ __align__(128) unsigned char smem[];
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const long long gw = (long long)blockIdx.x * Lay::WARPS + warp;
    if (gw >= (long long)a.batch * a.chunks) return;
    const int b = (int)(gw / a.chunks);
    const long long chunk = gw - (long long)b * a.chunks;
    if (a.active && !a.active[b]) return;

    const long long n = a.n, n1 = n >> 1, n2 = n >> 2;
    S0 st{L, a, lane, a.flags};
    st.nc = n1;
    st.transfer_regs();
    S s1{L1, a1, lane, a1.flags};
    s1.nc = n2;
    const long long row0 = chunk * a.rows_per_chunk;          // even; every row full (n % 128 == 0)
    const int rows = (int)min((long long)a.rows_per_chunk, n / W - row0);
    const int ngroups = rows >> 1;
    const int lofs = lane * P;
    const T *fsrc = (a.f_alt && (a.iters[(size_t)b * a.iters_stride] & 1)) ? a.f_alt : a.f;
    const T *fb = fsrc + (size_t)b * n * NT;
    T *f1b = a.fc + (size_t)b * n1 * NT;     // f_{l+1} (stored)
    T *f2b = a1.fc + (size_t)b * n2 * NT;    // f_{l+2}

    uint64_t *bars = reinterpret_cast<uint64_t *>(smem) + warp * Lay::ST;
    unsigned char *wbase = smem + Lay::BAR_BYTES + (size_t)warp * Lay::BYTES_PER_WARP;
    T *c1row = reinterpret_cast<T *>(wbase);
    T *ring = c1row + Lay::ROW;
    {
        unsigned *rec = reinterpret_cast<unsigned *>(wbase + Lay::BYTES_PER_WARP - Lay::RECBYTES);
        st.rec = rec;
        s1.rec = rec + Lay::REC_ONE;
    }
    if constexpr (P == 1) {
        // per-warp copies of both levels' (R1, R2); odd lanes use R2
        T *rs = ring + Lay::STAGE * Lay::ST;
        for (int i = lane; i < NT * NT; i += 32) {
            rs[i] = L.R1[i];
            rs[Lay::RSTRIDE + i] = L.R2[i];
            rs[2 * Lay::RSTRIDE + i] = L1.R1[i];
            rs[3 * Lay::RSTRIDE + i] = L1.R2[i];
        }
        __syncwarp();
        st.Rs = rs + ((lane & 1) ? Lay::RSTRIDE : 0);
        s1.Rs = rs + 2 * Lay::RSTRIDE + ((lane & 1) ? Lay::RSTRIDE : 0);
    }
#pragma unroll
    for (int k = 0; k <= NU; ++k) {
        cpl_zero(st.carry[k]);
        cpl_zero(s1.carry[k]);
    }
    st.leaf_q = s1.leaf_q = 0;
    st.leaf0 = s1.leaf0 = 0;
    st.halo_w = s1.halo_w = nullptr;
    st.write_u = s1.write_u = false;
    st.vec_out = s1.vec_out = false;
    uint64_t pol = 0;
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < Lay::ST; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        pol = policy_evict_first();
    }
    __syncwarp();
    auto issue = [&](int g) {  // lane 0 only
        T *stg = ring + (size_t)(g % Lay::ST) * Lay::STAGE;
        uint64_t *bar = &bars[g % Lay::ST];
        const long long s0 = (row0 + 2LL * g) * W;
        const uint32_t bytes = (uint32_t)(Lay::STAGE * sizeof(T));
        mbar_expect_tx(bar, bytes);
        bulk_g2s(stg, fb + s0 * NT, bytes, bar, pol);
    };
    if (lane == 0)
        for (int g = 0; g < ngroups && g < Lay::ST; ++g) issue(g);

    // one level-l row from f (zero guess); its restricted row half -> c1row
    auto fine_row = [&](long long r, const T (&f)[P][NT], int half, bool warm) {
        T u[P][NT], uc[NT];
#pragma unroll
        for (int q = 0; q < P; ++q) zero_slab<T, NT>(u[q]);
        zero_slab<T, NT>(uc);
        T *dst = warm ? nullptr : c1row + half * Lay::HALF + (lofs >> 1) * NT;
        if (r > 0) st.template row<true>(u, f, uc, r * W + lofs, r, warm, b, nullptr, dst, true);
        else st.template row<false>(u, f, uc, r * W + lofs, r, warm, b, nullptr, dst, true);
    };
    // the level-(l+1) row cr from c1row: store it as f_{l+1} (unless a warm-up
    // row of the previous chunk), then its own down pass -> f_{l+2}
    auto coarse_row = [&](long long cr, bool store) {
        __syncwarp();
        T f[P][NT], u[P][NT], uc[NT];
        load_lane<T, NT, P>(c1row + lofs * NT, f);
        if (store) store_lane<T, NT, P>(f1b + (cr * W + lofs) * NT, f);
#pragma unroll
        for (int q = 0; q < P; ++q) zero_slab<T, NT>(u[q]);
        zero_slab<T, NT>(uc);
        T *fco2 = store ? f2b + ((cr * W + lofs) >> 1) * NT : nullptr;
        if (cr > 0) s1.template row<true>(u, f, uc, cr * W + lofs, cr, !store, b, nullptr, fco2, true);
        else s1.template row<false>(u, f, uc, cr * W + lofs, cr, !store, b, nullptr, fco2, true);
        __syncwarp();
    };

    if (row0 > 0 && NU == 1 && warm_short()) {
        // nu1 = 1 from the zero guess: the first sweep needs no predecessor, so
        // the chunk depends on only THREE level-l slabs before it -- their
        // zero-guess sweeps, the residuals of the last two, their restriction
        // and that level-(l+1) slab's zero-guess sweep give both levels'
        // carries (every lane computes the same scalars; same functions, same
        // bits as the row path) instead of three level-l rows and one
        // level-(l+1) row: the small levels' kernels are mostly warm-up.
        using C = typename S::C;
        const long long g0 = row0 * W;
        T f3[3][NT], u3[3][NT];
#pragma unroll
        for (int i = 0; i < 3; ++i) load_slab_scalar<T, NT>(fb + (g0 - 3 + i) * NT, f3[i]);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            T uu[1][NT], ff[1][NT];
#pragma unroll
            for (int j = 0; j < NT; ++j) ff[0][j] = f3[i][j];
            sweep_zero_j<T, NT, PERM, 1>(L, uu, ff);
#pragma unroll
            for (int j = 0; j < NT; ++j) u3[i][j] = uu[0][j];
        }
        const C c0 = make_cpl<T, NT, SPARSE, true>(L, u3[0]);
        const C c1 = make_cpl<T, NT, SPARSE, true>(L, u3[1]);
        st.carry[NU] = make_cpl<T, NT, SPARSE, true>(L, u3[2]);
        T r0[NT], r1[NT], pc[1][NT], p1[NT], uc1[1][NT];
        residual<T, NT, SPARSE, true>(L, u3[1], f3[1], c0, true, r0);
        residual<T, NT, SPARSE, true>(L, u3[2], f3[2], c1, true, r1);
        restrict_reg<T, NT>(L.R1, r0, pc[0]);
        restrict_reg<T, NT>(L.R2, r1, p1);
#pragma unroll
        for (int j = 0; j < NT; ++j) pc[0][j] = FP<T>::add(pc[0][j], p1[j]);
        sweep_zero_j<T, NT, PERM, 1>(L1, uc1, pc);
        s1.carry[NU] = make_cpl<T, NT, SPARSE, true>(L1, uc1[0]);
        if constexpr (S::TRACK) {
            if (lane == 0) {
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    st.rec[NU * NT + j] = (unsigned)__double2hiint((double)u3[2][j]);
                    s1.rec[NU * NT + j] = (unsigned)__double2hiint((double)uc1[0][j]);
                }
            }
        }
        __syncwarp();
    } else if (row0 > 0) {
        // warm-up: level-l rows row0-3 (carries only), row0-2 and row0-1 (the
        // level-(l+1) row before the chunk), then that row (carries only)
        for (long long r = max(0LL, row0 - 3); r < row0; ++r) {
            T f[P][NT];
#pragma unroll
            for (int q = 0; q < P; ++q) load_slab_scalar<T, NT>(fb + (r * W + lofs + q) * NT, f[q]);
            fine_row(r, f, (int)(r & 1), r == row0 - 3);
        }
        coarse_row((row0 >> 1) - 1, false);
    }

    for (int g = 0; g < ngroups; ++g) {
        const T *stg = ring + (size_t)(g % Lay::ST) * Lay::STAGE;
        mbar_wait(&bars[g % Lay::ST], (uint32_t)((g / Lay::ST) & 1));
#pragma unroll 1
        for (int qq = 0; qq < 2; ++qq) {
            T f[P][NT];
            load_lane<T, NT, P>(stg + qq * Lay::ROW + lofs * NT, f);
            if (qq == 1) {
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0 && g + Lay::ST < ngroups) issue(g + Lay::ST);
            }
            fine_row(row0 + 2 * g + qq, f, qq, false);
        }
        coarse_row((row0 >> 1) + g, true);
    }
}

}  // namespace tmg
