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
constexpr int SW_STAGES = 4;  // ring stages per warp
constexpr int SW_GROUP = 2;   // rows per stage

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
enum Kind : int { K_GENERIC = 0, K_DOWN = 1, K_UP = 2, K_UPNORM = 3 };

template <typename T> struct StreamArgs {
    const T *f;
    const T *u_in;
    T *u_out;
    const T *uc;
    T *fc;
    T *r_out;
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

template <typename T, int NT> struct RowLayout {
    static constexpr int ROW = 32 * NT;   // elements of one fine row
    static constexpr int HALF = 16 * NT;  // elements of the matching coarse half-row
    static constexpr int OFF_F = SW_GROUP * ROW;
    static constexpr int OFF_C = 2 * SW_GROUP * ROW;
    static constexpr int STAGE = SW_GROUP * (2 * ROW + HALF);
    // per-warp copy of (R1, R2) for n_t >= 3 (R2 padded by 2 elements so the
    // even and odd half-warps read different banks)
    static constexpr int RELEMS = NT >= 3 ? 2 * NT * NT + 2 : 0;
    static constexpr int RSTRIDE = NT * NT + 2;
    static constexpr size_t RBYTES = ((sizeof(T) * RELEMS + 15) / 16) * 16;
    static constexpr size_t BYTES_PER_WARP = sizeof(T) * STAGE * SW_STAGES + RBYTES;
    // mbarrier block (one 8-byte barrier per warp and stage), padded to 128 B
    static constexpr size_t BAR_BYTES = ((SW_WARPS * SW_STAGES * 8 + 127) / 128) * 128;
    static constexpr size_t SMEM_BYTES = BAR_BYTES + BYTES_PER_WARP * SW_WARPS;
};

template <typename T, int NT, int NU, bool SPARSE, int KIND, int PERM> struct Streamer {
    using C = Cpl<T, NT, SPARSE>;
    static constexpr int CF = KIND == K_DOWN ? (SF_RESTRICT | SF_WRITE_U)
                              : KIND == K_UP ? (SF_PROLONG | SF_WRITE_U)
                              : KIND == K_UPNORM ? (SF_PROLONG | SF_WRITE_U | SF_NORM_LEAF)
                                                 : 0;
    const LevelC<T, NT> &L;
    const StreamArgs<T> &a;
    int lane;
    int flags;
    // this lane's transfer block (odd lanes R2, even lanes R1): registers for
    // n_t <= 2, a per-warp shared-memory copy for larger blocks
    static constexpr bool RREG = NT <= 2;
    T Rm[RREG ? NT * NT : 1];
    const T *Rs;
    C carry[NU + 1];    // lane 0: predecessor data of the next row, per sweep
    T leaf_acc;
    int leaf_q;         // row position inside the current numpy leaf
    long long nc;

    __device__ __forceinline__ bool has(int f) const
    {
        return KIND == K_GENERIC ? (flags & f) != 0 : (CF & f) != 0;
    }
    __device__ __forceinline__ bool need_r() const
    {
        return has(SF_RESTRICT) || has(SF_NORM_LEAF) || has(SF_NORM_SQ) || has(SF_WRITE_R);
    }

    __device__ __forceinline__ void exchange(const T (&u)[NT], int k, C &prev)
    {
        C own = make_cpl<T, NT, SPARSE>(L, u);
        C x = cpl_shfl<T, NT, SPARSE>(own, (lane + 31) & 31);
        prev = x;
        cpl_select<T, NT, SPARSE>(prev, carry[k], lane == 0);
        carry[k] = x;
    }

    // one row; INTERIOR: all 32 slabs exist and none is slab 0 of the problem
    template <bool INTERIOR>
    __device__ __forceinline__ void row(T (&u)[NT], const T (&f)[NT], const T (&uc)[NT], long long slab,
                                        long long row_idx, bool warm, int b)
    {
        const bool valid = INTERIOR || slab < a.n;
        const bool hp = INTERIOR || slab > 0;
        if (has(SF_PROLONG)) {
            if (INTERIOR || slab < 2 * nc) {
                if constexpr (RREG) prolong_reg<T, NT>(Rm, uc, u);
                else prolong_ptr<T, NT>(Rs, uc, u);
            }
        }
#pragma unroll
        for (int k = 0; k < NU; ++k) {
            C prev;
            exchange(u, k, prev);
            sweep_p<T, NT, SPARSE, PERM>(L, u, f, prev, hp);
        }
        if (need_r()) {
            C prev;
            exchange(u, NU, prev);
            if (!warm) {
                T r[NT];
                residual<T, NT, SPARSE>(L, u, f, prev, hp, r);
                if (has(SF_WRITE_R) && valid) store_slab<T, NT>(a.r_out + ((size_t)b * a.n + slab) * NT, r);
                if (has(SF_RESTRICT)) {
                    T p[NT], q[NT];
                    if constexpr (RREG) restrict_reg<T, NT>(Rm, r, p);
                    else restrict_ptr<T, NT>(Rs, r, p);
#pragma unroll
                    for (int i = 0; i < NT; ++i) q[i] = __shfl_down_sync(0xffffffffu, p[i], 1);
#pragma unroll
                    for (int i = 0; i < NT; ++i) p[i] = FP<T>::add(p[i], q[i]);
                    const long long cidx = slab >> 1;
                    if (!(lane & 1) && (INTERIOR || cidx < nc))
                        store_slab<T, NT>(a.fc + ((size_t)b * nc + cidx) * NT, p);
                }
                if (has(SF_NORM_SQ)) {
                    if (valid) a.sq_out[(size_t)b * a.n + slab] = (double)sqnorm<T, NT>(r);
                }
                if (has(SF_NORM_LEAF)) {
                    // numpy pairwise leaf (np.sum, multigrid.py:459): 8 accumulators,
                    // accumulator j sums elements j, j+8, j+16, ... of the leaf in order
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
                        if (lane == 0) a.leaf_out[(size_t)b * nleaves + row_idx / a.leaf_rows] = (double)t3;
                        leaf_q = 0;
                    } else {
                        leaf_q += 1;
                    }
                }
            }
        }
        if (has(SF_WRITE_U) && !warm && valid) store_slab<T, NT>(a.u_out + ((size_t)b * a.n + slab) * NT, u);
    }
};

template <typename T, int NT, int NU, bool SPARSE, int KIND, int PERM>
__global__ void __launch_bounds__(SW_WARPS * 32, NT <= 2 ? 3 : 2)
    stream_kernel(const __grid_constant__ LevelC<T, NT> L, const __grid_constant__ StreamArgs<T> a)
{
    using Lay = RowLayout<T, NT>;
    using S = Streamer<T, NT, NU, SPARSE, KIND, PERM>;
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
    const int ngroups = (rows + SW_GROUP - 1) / SW_GROUP;
    const bool zero_guess = a.flags & SF_ZERO_GUESS;
    const bool tma = a.flags & SF_TMA;
    const bool prolong = st.has(SF_PROLONG);

    const T *fb = a.f + (size_t)b * n * NT;
    const T *ub = zero_guess ? nullptr : a.u_in + (size_t)b * n * NT;
    const T *ucb = prolong ? a.uc + (size_t)b * st.nc * NT : nullptr;

    uint64_t *bars = reinterpret_cast<uint64_t *>(smem) + warp * SW_STAGES;
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
    for (int k = 0; k <= NU; ++k) cpl_zero(st.carry[k]);
    st.leaf_acc = T(0);
    st.leaf_q = 0;

    // a group goes through the ring iff it consists of SW_GROUP whole rows
    auto group_tma = [&](int g) -> bool {
        return tma && (g + 1) * SW_GROUP <= rows && (row0 + (long long)(g + 1) * SW_GROUP) * 32 <= n;
    };
    uint64_t pol = 0;
    if (lane == 0 && tma) {
#pragma unroll
        for (int s = 0; s < SW_STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        pol = policy_evict_first();
    }
    __syncwarp();
    auto issue = [&](int g) {  // lane 0 only
        if (!group_tma(g)) return;
        T *stg = ring + (size_t)(g % SW_STAGES) * Lay::STAGE;
        uint64_t *bar = &bars[g % SW_STAGES];
        const long long s0 = (row0 + (long long)g * SW_GROUP) * 32;
        const uint32_t bytes = (uint32_t)(SW_GROUP * Lay::ROW * sizeof(T));
        const uint32_t cbytes = prolong ? (uint32_t)(SW_GROUP * Lay::HALF * sizeof(T)) : 0u;
        mbar_expect_tx(bar, bytes * (zero_guess ? 1u : 2u) + cbytes);
        bulk_g2s(stg + Lay::OFF_F, fb + s0 * NT, bytes, bar, pol);
        if (!zero_guess) bulk_g2s(stg, ub + s0 * NT, bytes, bar, pol);
        if (cbytes) bulk_g2s(stg + Lay::OFF_C, ucb + (s0 >> 1) * NT, cbytes, bar, pol);
    };
    if (lane == 0 && tma)
        for (int g = 0; g < ngroups && g < SW_STAGES; ++g) issue(g);

    // warm-up row (the 32 slabs before the chunk): carries only, no outputs
    if (row0 > 0) {
        const long long slab = (row0 - 1) * 32 + lane;
        T u[NT], f[NT], uc[NT];
        zero_slab<T, NT>(u);
        zero_slab<T, NT>(uc);
        if (tma) {
            load_slab<T, NT>(fb + slab * NT, f);
            if (!zero_guess) load_slab<T, NT>(ub + slab * NT, u);
            if (prolong) load_slab<T, NT>(ucb + (slab >> 1) * NT, uc);
        } else {
            load_slab_scalar<T, NT>(fb + slab * NT, f);
            if (!zero_guess) load_slab_scalar<T, NT>(ub + slab * NT, u);
            if (prolong) load_slab_scalar<T, NT>(ucb + (slab >> 1) * NT, uc);
        }
        if (row0 - 1 > 0) st.template row<true>(u, f, uc, slab, row0 - 1, true, b);
        else st.template row<false>(u, f, uc, slab, row0 - 1, true, b);
    }

    for (int g = 0; g < ngroups; ++g) {
        const bool gt = group_tma(g);
        const T *stg = ring + (size_t)(g % SW_STAGES) * Lay::STAGE;
        if (gt) mbar_wait(&bars[g % SW_STAGES], (uint32_t)((g / SW_STAGES) & 1));
#pragma unroll
        for (int q = 0; q < SW_GROUP; ++q) {
            const int rr = g * SW_GROUP + q;
            if (rr >= rows) break;
            const long long row_idx = row0 + rr;
            const long long slab = row_idx * 32 + lane;
            T u[NT], f[NT], uc[NT];
            if (gt) {
                load_slab<T, NT>(stg + Lay::OFF_F + q * Lay::ROW + lane * NT, f);
                if (zero_guess) zero_slab<T, NT>(u);
                else load_slab<T, NT>(stg + q * Lay::ROW + lane * NT, u);
                if (prolong) load_slab<T, NT>(stg + Lay::OFF_C + q * Lay::HALF + (lane >> 1) * NT, uc);
                else zero_slab<T, NT>(uc);
            } else {
                zero_slab<T, NT>(u);
                zero_slab<T, NT>(f);
                zero_slab<T, NT>(uc);
                if (slab < n) {
                    load_slab_scalar<T, NT>(fb + slab * NT, f);
                    if (!zero_guess) load_slab_scalar<T, NT>(ub + slab * NT, u);
                    if (prolong && slab < 2 * st.nc) load_slab_scalar<T, NT>(ucb + (slab >> 1) * NT, uc);
                }
            }
            if (q == SW_GROUP - 1 || rr + 1 >= rows) {
                // the stage is fully read: hand it back to the copy engine
                __syncwarp();
                if (gt && lane == 0 && g + SW_STAGES < ngroups) issue(g + SW_STAGES);
            }
            if (row_idx > 0 && (row_idx + 1) * 32 <= n) st.template row<true>(u, f, uc, slab, row_idx, false, b);
            else st.template row<false>(u, f, uc, slab, row_idx, false, b);
        }
    }
}

}  // namespace tmg
