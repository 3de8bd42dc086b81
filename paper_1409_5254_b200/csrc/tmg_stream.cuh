// Streaming level kernels: one warp walks a contiguous chunk of slabs, 32
// slabs (one "row") at a time.  Lane l owns slab 32*row + l of the row and
// keeps its n_t values in registers through all sweeps of the pass:
//
//   down:  nu1 sweeps -> residual -> restriction        (multigrid.py:274-285)
//   up:    prolong-add -> nu2 sweeps [-> residual norm] (multigrid.py:317-327,
//                                                         447-459)
//
// Jacobi reads only slab n and n-1 of the previous iterate (multigrid.py:
// 168-180).  What slab n needs from slab n-1 at sweep k is one rotate-shuffle
// away: lane l receives lane l-1's value and lane 0 receives lane 31's -- the
// value the NEXT row's lane 0 will need -- so lane 0 swaps it with the carry
// it kept from the previous row.  A chunk that does not start at slab 0 first
// runs one "warm-up" row over the 32 slabs before it (only lanes >= k are
// valid after k sweeps; lane 31 needs nu+1 <= 32 of them), so warps never
// synchronise with each other: the pass is one HBM read of u, f (and u_coarse)
// and one write of u (and f_coarse) per slab.
//
// Rows arrive two at a time in a per-warp shared-memory ring filled by the
// TMA engine (cp.async.bulk global->shared, completion on an mbarrier, L2
// evict-first); lane 0 refills a stage as soon as the warp has read it.
// Interior rows run a specialised path (every lane valid, every slab has a
// predecessor); the problem's first row and a ragged last row take the
// general path.
#pragma once
#include "tmg_slab.cuh"

namespace tmg {

constexpr int SW_WARPS = 8;   // warps per CTA
constexpr int SW_STAGES = 4;  // ring stages per warp (3 for the up passes: larger stages)
constexpr int SW_GROUP = 2;   // rows per stage
#ifndef TMG_MINB
#define TMG_MINB(NT) 2
#endif

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
enum Kind : int { K_GENERIC = 0, K_DOWN = 1, K_UP = 2, K_UPNORM = 3, K_DOWNNORM = 4, K_UP2 = 5 };

template <typename T> struct StreamArgs {
    const T *f;
    const T *u_in;
    T *u_out;
    const T *uc;
    T *fc;
    T *r_out;
    T *halo;               // [batch][chunks][J rows][32][NT]: each chunk's last J rows of the
                           // ORIGINAL iterate (written by down passes, read by K_UP2 warm-ups)
    double *sq_out;
    double *leaf_out;
    const int *active;
    long long n;           // fine slabs per problem
    long long chunks;      // chunks per problem
    int batch;
    int rows_per_chunk;    // multiple of SW_GROUP and of leaf_rows
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

template <typename T, int NT, bool WITH_C> struct RowLayout {
    static constexpr int ROW = 32 * NT;   // elements of one fine row
    static constexpr int HALF = 16 * NT;  // elements of the matching coarse half-row
    static constexpr int OFF_F = SW_GROUP * ROW;
    static constexpr int OFF_C = 2 * SW_GROUP * ROW;
    static constexpr int STAGE = SW_GROUP * (2 * ROW + (WITH_C ? HALF : 0));
    // ring depth from a per-CTA budget that keeps the register-limited
    // occupancy (3 CTAs/SM for n_t <= 2, 2 CTAs/SM above): 2..4 stages
    static constexpr size_t BUDGET = NT <= 2 ? 72 * 1024 : 100 * 1024;
    static constexpr int ST_RAW = (int)(BUDGET / (SW_WARPS * sizeof(T) * STAGE));
    static constexpr int ST = ST_RAW < 2 ? 2 : (ST_RAW > SW_STAGES ? SW_STAGES : ST_RAW);
    // per-warp copy of (R1, R2) for n_t >= 3 (R2 padded by 2 elements so the
    // even and odd half-warps read different banks)
    static constexpr int RELEMS = NT >= 3 ? 2 * NT * NT + 2 : 0;
    static constexpr int RSTRIDE = NT * NT + 2;
    static constexpr size_t RBYTES = ((sizeof(T) * RELEMS + 15) / 16) * 16;
    static constexpr size_t BYTES_PER_WARP = sizeof(T) * STAGE * ST + RBYTES;
    // mbarrier block (one 8-byte barrier per warp and stage), padded to 128 B
    static constexpr size_t BAR_BYTES = ((SW_WARPS * ST * 8 + 127) / 128) * 128;
    static constexpr size_t SMEM_BYTES = BAR_BYTES + BYTES_PER_WARP * SW_WARPS;
};

template <int KIND> struct KindProlongs {
    static constexpr bool value = KIND != K_DOWN && KIND != K_DOWNNORM;
};
// rows processed jointly (must agree between a level's down and up passes:
// the halo holds J rows)
template <typename T, int NT> struct JointRows {
    static constexpr int value = (NT <= 2 || sizeof(T) == 4) ? 2 : 1;
};

template <typename T, int NT, int NU, bool SPARSE, int KIND, int PERM> struct Streamer {
    using C = Cpl<T, NT, SPARSE>;
    static constexpr int CF = KIND == K_DOWN ? (SF_RESTRICT | SF_WRITE_U)
                              : KIND == K_UP ? (SF_PROLONG | SF_WRITE_U)
                              : KIND == K_UPNORM ? (SF_PROLONG | SF_WRITE_U | SF_NORM_LEAF)
                              : KIND == K_DOWNNORM ? (SF_RESTRICT | SF_WRITE_U | SF_NORM_LEAF)
                              : KIND == K_UP2 ? (SF_PROLONG | SF_WRITE_U)
                                              : 0;
    // pre-sweeps recomputed before the prolongation (K_UP2)
    static constexpr int NPRE = KIND == K_UP2 ? NU : 0;
    // norm of the pass's input (K_DOWNNORM) rather than of its output
    static constexpr bool NORM_IN = KIND == K_DOWNNORM && NU > 0;
    // rows swept jointly per lane (two dependency chains hide fp64 latency);
    // larger blocks have enough independent work per row already
    static constexpr int J = JointRows<T, NT>::value;
    const LevelC<T, NT> &L;
    const StreamArgs<T> &a;
    int lane;
    int flags;
    // this lane's transfer block (odd lanes R2, even lanes R1): registers for
    // n_t <= 2, a per-warp shared-memory copy for larger blocks
    static constexpr bool RREG = NT * NT * sizeof(T) <= 64;
    T Rm[RREG ? NT * NT : 1];
    const T *Rs;
    C carry[NPRE + NU + 1];  // lane 0: predecessor data of the next row, per sweep
    T leaf_acc;
    int leaf_q;         // row position inside the current numpy leaf
    long long nc;
    bool write_u;       // the pass stores u (u_out given)

    __device__ __forceinline__ bool has(int f) const
    {
        return KIND == K_GENERIC ? (flags & f) != 0 : (CF & f) != 0;
    }
    __device__ __forceinline__ bool need_r() const
    {
        return has(SF_RESTRICT) || has(SF_NORM_LEAF) || has(SF_NORM_SQ) || has(SF_WRITE_R);
    }

    // numpy pairwise leaf (np.sum, multigrid.py:459): accumulator j sums leaf
    // elements j, j+8, j+16, ... in order; 8 accumulators combined as
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) at the leaf's last row
    __device__ __forceinline__ void leaf_add(const T (&r)[NT], long long row, int b)
    {
        T sq = sqnorm<T, NT>(r);
        T v1 = __shfl_down_sync(0xffffffffu, sq, 8);
        T v2 = __shfl_down_sync(0xffffffffu, sq, 16);
        T v3 = __shfl_down_sync(0xffffffffu, sq, 24);
        leaf_acc = (leaf_q == 0) ? sq : FP<T>::add(leaf_acc, sq);
        leaf_acc = FP<T>::add(leaf_acc, v1);
        leaf_acc = FP<T>::add(leaf_acc, v2);
        leaf_acc = FP<T>::add(leaf_acc, v3);
        if (leaf_q == a.leaf_rows - 1) {
            T t1 = FP<T>::add(leaf_acc, __shfl_down_sync(0xffffffffu, leaf_acc, 1));
            T t2 = FP<T>::add(t1, __shfl_down_sync(0xffffffffu, t1, 2));
            T t3 = FP<T>::add(t2, __shfl_down_sync(0xffffffffu, t2, 4));
            const long long nleaves = a.n / (32LL * a.leaf_rows);
            if (lane == 0) a.leaf_out[(size_t)b * nleaves + row / a.leaf_rows] = (double)t3;
            leaf_q = 0;
        } else {
            leaf_q += 1;
        }
    }

    // predecessor data for JJ consecutive rows at sweep k (rotate-shuffle + carry)
    template <int JJ>
    __device__ __forceinline__ void exchange(const T (&u)[JJ][NT], int k, C (&prev)[JJ])
    {
        C x[JJ];
#pragma unroll
        for (int q = 0; q < JJ; ++q) {
            C own = make_cpl<T, NT, SPARSE>(L, u[q]);
            x[q] = cpl_shfl<T, NT, SPARSE>(own, (lane + 31) & 31);
        }
        prev[0] = x[0];
        cpl_select<T, NT, SPARSE>(prev[0], carry[k], lane == 0);
#pragma unroll
        for (int q = 1; q < JJ; ++q) {
            prev[q] = x[q];
            cpl_select<T, NT, SPARSE>(prev[q], x[q - 1], lane == 0);
        }
        carry[k] = x[JJ - 1];
    }

    // JJ rows starting at slab0 (this lane's slab in the first row);
    // INTERIOR: every slab exists and none is slab 0 of the problem.
    // Rows q >= nrow are beyond the chunk: computed but never stored.
    // uo/fco: this lane's u_out / f_coarse element for the first row (row
    // stride 32*NT / 16*NT elements), advanced by the caller
    template <bool INTERIOR, int JJ>
    __device__ __forceinline__ void rows(T (&u)[JJ][NT], const T (&f)[JJ][NT], const T (&uc)[JJ][NT],
                                         long long slab0, long long row_idx0, int nrow, bool warm, int b,
                                         T *uo, T *fco, bool zg)
    {
        bool valid[JJ], hp[JJ];
#pragma unroll
        for (int q = 0; q < JJ; ++q) {
            const long long sl = slab0 + 32 * q;
            valid[q] = INTERIOR || (q < nrow && sl < a.n);
            hp[q] = INTERIOR || sl > 0;
        }
        // K_UP2: the down pass's pre-sweeps, recomputed (same bits)
#pragma unroll
        for (int k = 0; k < NPRE; ++k) {
            if (k == 0 && zg) {
                sweep_zero_j<T, NT, PERM, JJ>(L, u, f);
                continue;
            }
            C prev[JJ];
            exchange<JJ>(u, k, prev);
            sweep_j<T, NT, SPARSE, PERM, JJ>(L, u, f, prev, hp);
        }
#pragma unroll
        for (int q = 0; q < JJ; ++q) {
            const long long sl = slab0 + 32 * q;
            if (has(SF_PROLONG)) {
                if (INTERIOR || sl < 2 * nc) {
                    if constexpr (RREG) prolong_reg<T, NT>(Rm, uc[q], u[q]);
                    else prolong_ptr<T, NT>(Rs, uc[q], u[q]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < NU; ++k) {
            if (!NORM_IN && NPRE == 0 && k == 0 && zg) {
                sweep_zero_j<T, NT, PERM, JJ>(L, u, f);
                continue;
            }
            C prev[JJ];
            exchange<JJ>(u, NPRE + k, prev);
            if (NORM_IN && k == 0) {
                // the first sweep's residual IS the input's residual: take its norm
                T y[JJ][NT];
#pragma unroll
                for (int q = 0; q < JJ; ++q) residual_perm<T, NT, SPARSE, PERM>(L, u[q], f[q], prev[q], hp[q], y[q]);
                if (!warm) {
#pragma unroll
                    for (int q = 0; q < JJ; ++q) {
                        if (INTERIOR || q < nrow) {
                            T r[NT];
                            unpermute<T, NT, PERM>(L, y[q], r);
                            leaf_add(r, row_idx0 + q, b);
                        }
                    }
                }
                finish_j<T, NT, JJ>(L, u, y);
            } else {
                sweep_j<T, NT, SPARSE, PERM, JJ>(L, u, f, prev, hp);
            }
        }
        if (need_r()) {
            C prev[JJ];
            exchange<JJ>(u, NPRE + NU, prev);
            if (!warm) {
#pragma unroll
                for (int q = 0; q < JJ; ++q) {
                    const long long sl = slab0 + 32 * q;
                    T r[NT];
                    residual<T, NT, SPARSE>(L, u[q], f[q], prev[q], hp[q], r);
                    if (has(SF_WRITE_R) && valid[q]) store_slab<T, NT>(a.r_out + ((size_t)b * a.n + sl) * NT, r);
                    if (has(SF_RESTRICT)) {
                        T p[NT], qq[NT];
                        if constexpr (RREG) restrict_reg<T, NT>(Rm, r, p);
                        else restrict_ptr<T, NT>(Rs, r, p);
#pragma unroll
                        for (int i = 0; i < NT; ++i) qq[i] = __shfl_down_sync(0xffffffffu, p[i], 1);
#pragma unroll
                        for (int i = 0; i < NT; ++i) p[i] = FP<T>::add(p[i], qq[i]);
                        const long long cidx = sl >> 1;
                        if (!(lane & 1) && (INTERIOR || (valid[q] && cidx < nc)))
                            store_slab<T, NT>(fco + q * 16 * NT, p);
                    }
                    if (has(SF_NORM_SQ)) {
                        if (valid[q]) a.sq_out[(size_t)b * a.n + sl] = (double)sqnorm<T, NT>(r);
                    }
                    if (!NORM_IN && has(SF_NORM_LEAF) && (INTERIOR || q < nrow)) leaf_add(r, row_idx0 + q, b);
                }
            }
        }
        if (has(SF_WRITE_U) && !warm && write_u) {
#pragma unroll
            for (int q = 0; q < JJ; ++q)
                if (valid[q]) store_slab<T, NT>(uo + q * 32 * NT, u[q]);
        }
    }
};

template <typename T, int NT>
__device__ __forceinline__ void load_row(const T *src, T (&x)[NT], bool vec)
{
    if (vec) load_slab<T, NT>(src, x);
    else load_slab_scalar<T, NT>(src, x);
}

template <typename T, int NT, int NU, bool SPARSE, int KIND, int PERM>
__global__ void __launch_bounds__(SW_WARPS * 32, TMG_MINB(NT))
    stream_kernel(const __grid_constant__ LevelC<T, NT> L, const __grid_constant__ StreamArgs<T> a)
{
    constexpr bool WITH_C = KindProlongs<KIND>::value;
    using Lay = RowLayout<T, NT, WITH_C>;
    using S = Streamer<T, NT, NU, SPARSE, KIND, PERM>;
    constexpr int J = S::J;
    constexpr int G = SW_GROUP;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const long long gw = (long long)blockIdx.x * SW_WARPS + warp;
    if (gw >= (long long)a.batch * a.chunks) return;
    const int b = (int)(gw / a.chunks);
    const long long chunk = gw - (long long)b * a.chunks;
    if (a.active && !a.active[b]) return;

    S st{L, a, lane, a.flags};
    const long long n = a.n;
    st.nc = n >> 1;
    const long long nrows = (n + 31) >> 5;
    const long long row0 = chunk * a.rows_per_chunk;
    const int rows = (int)min((long long)a.rows_per_chunk, nrows - row0);
    const int ngroups = (rows + G - 1) / G;
    const bool zero_guess = a.flags & SF_ZERO_GUESS;
    const bool tma = a.flags & SF_TMA;
    const bool prolong = WITH_C && st.has(SF_PROLONG);

    const T *fb = a.f + (size_t)b * n * NT;
    const T *ub = zero_guess ? nullptr : a.u_in + (size_t)b * n * NT;
    const T *ucb = prolong ? a.uc + (size_t)b * st.nc * NT : nullptr;

    constexpr int ST = Lay::ST;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem) + warp * ST;
    unsigned char *wbase = smem + Lay::BAR_BYTES + (size_t)warp * Lay::BYTES_PER_WARP;
    T *ring = reinterpret_cast<T *>(wbase + Lay::RBYTES);
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
#pragma unroll
    for (int k = 0; k <= S::NPRE + NU; ++k) cpl_zero(st.carry[k]);
    st.leaf_acc = T(0);
    st.leaf_q = 0;

    // groups [0, g_full) consist of G whole rows (and go through the ring when
    // TMA is on); groups [g_int0, g_full) are interior (no slab 0, all valid)
    const int g_full = (int)max(0LL, min((long long)(rows / G), (n / 32 - row0) / G));
    const int g_int0 = row0 == 0 ? 1 : 0;
    auto group_tma = [&](int g) -> bool { return tma && g < g_full; };
    // per-lane output cursors (advanced by G rows per group)
    st.write_u = st.has(SF_WRITE_U) && a.u_out != nullptr;
    T *uo = st.write_u ? a.u_out + ((size_t)b * n + (size_t)row0 * 32 + lane) * NT : nullptr;
    T *fco = st.has(SF_RESTRICT) ? a.fc + ((size_t)b * st.nc + (size_t)row0 * 16 + (lane >> 1)) * NT : nullptr;
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
        const long long s0 = (row0 + (long long)g * G) * 32;
        const uint32_t bytes = (uint32_t)(G * Lay::ROW * sizeof(T));
        const uint32_t cbytes = prolong ? (uint32_t)(G * Lay::HALF * sizeof(T)) : 0u;
        mbar_expect_tx(bar, bytes * (zero_guess ? 1u : 2u) + cbytes);
        bulk_g2s(stg + Lay::OFF_F, fb + s0 * NT, bytes, bar, pol);
        if (!zero_guess) bulk_g2s(stg, ub + s0 * NT, bytes, bar, pol);
        if (cbytes) bulk_g2s(stg + Lay::OFF_C, ucb + (s0 >> 1) * NT, cbytes, bar, pol);
    };
    if (lane == 0 && tma)
        for (int g = 0; g < ngroups && g < ST; ++g) issue(g);

    // warm-up: the J rows before the chunk, for the carries only
    if (row0 > 0) {
        T u[J][NT], f[J][NT], uc[J][NT];
        const long long wr0 = row0 - J;
#pragma unroll
        for (int q = 0; q < J; ++q) {
            const long long sl = (wr0 + q) * 32 + lane;
            zero_slab<T, NT>(u[q]);
            zero_slab<T, NT>(uc[q]);
            load_row<T, NT>(fb + sl * NT, f[q], tma);
            if (!zero_guess) {
                if (S::NPRE > 0)  // the neighbour chunk may already have overwritten these rows
                    load_row<T, NT>(a.halo + (((size_t)b * a.chunks + chunk - 1) * J + q) * 32 * NT + lane * NT,
                                    u[q], tma);
                else
                    load_row<T, NT>(ub + sl * NT, u[q], tma);
            }
            if (prolong) load_row<T, NT>(ucb + (sl >> 1) * NT, uc[q], tma);
        }
        if (wr0 > 0) st.template rows<true, J>(u, f, uc, wr0 * 32 + lane, wr0, J, true, b, nullptr, nullptr, zero_guess);
        else st.template rows<false, J>(u, f, uc, wr0 * 32 + lane, wr0, J, true, b, nullptr, nullptr, zero_guess);
    }

    for (int g = 0; g < ngroups; ++g) {
        const bool gt = group_tma(g);
        const T *stg = ring + (size_t)(g % ST) * Lay::STAGE;
        const long long r0g = row0 + (long long)g * G;
        const int nrow = min(G, rows - g * G);
        const bool interior = g >= g_int0 && g < g_full;
        if (gt) mbar_wait(&bars[g % ST], (uint32_t)((g / ST) & 1));
#pragma unroll
        for (int q0 = 0; q0 < G; q0 += J) {
            T u[J][NT], f[J][NT], uc[J][NT];
#pragma unroll
            for (int q = 0; q < J; ++q) {
                const int qq = q0 + q;
                const long long sl = (r0g + qq) * 32 + lane;
                if (gt) {
                    load_slab<T, NT>(stg + Lay::OFF_F + qq * Lay::ROW + lane * NT, f[q]);
                    if (zero_guess) zero_slab<T, NT>(u[q]);
                    else load_slab<T, NT>(stg + qq * Lay::ROW + lane * NT, u[q]);
                    if (prolong) load_slab<T, NT>(stg + Lay::OFF_C + qq * Lay::HALF + (lane >> 1) * NT, uc[q]);
                    else zero_slab<T, NT>(uc[q]);
                } else {
                    zero_slab<T, NT>(u[q]);
                    zero_slab<T, NT>(f[q]);
                    zero_slab<T, NT>(uc[q]);
                    if (qq < nrow && sl < n) {
                        load_slab_scalar<T, NT>(fb + sl * NT, f[q]);
                        if (!zero_guess) load_slab_scalar<T, NT>(ub + sl * NT, u[q]);
                        if (prolong && sl < 2 * st.nc) load_slab_scalar<T, NT>(ucb + (sl >> 1) * NT, uc[q]);
                    }
                }
            }
            if (a.halo && !zero_guess && chunk + 1 < a.chunks && !S::NPRE) {
                // last J rows of the chunk: the next chunk's up-pass warm-up input
#pragma unroll
                for (int q = 0; q < J; ++q) {
                    const int rr = g * G + q0 + q;
                    if (rr >= rows - J && rr < rows)
                        store_slab<T, NT>(a.halo + (((size_t)b * a.chunks + chunk) * J + (rr - (rows - J))) * 32 * NT +
                                              lane * NT, u[q]);
                }
            }
            if (q0 + J >= G) {
                // the stage is fully read: hand it back to the copy engine
                __syncwarp();
                if (gt && lane == 0 && g + ST < ngroups) issue(g + ST);
            }
            if (q0 < nrow) {
                if (interior)
                    st.template rows<true, J>(u, f, uc, (r0g + q0) * 32 + lane, r0g + q0, J, false, b, uo, fco,
                                              zero_guess);
                else
                    st.template rows<false, J>(u, f, uc, (r0g + q0) * 32 + lane, r0g + q0, nrow - q0, false, b,
                                               uo, fco, zero_guess);
            }
            if (st.write_u) uo += J * 32 * NT;
            if (fco) fco += J * 16 * NT;
        }
    }
}

}  // namespace tmg
