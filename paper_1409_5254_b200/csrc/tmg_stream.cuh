// Streaming level kernels: one warp walks a contiguous chunk of slabs, 32
// slabs (one "row") at a time.  Lane l owns slab 32*row + l of the row and
// keeps its n_t values in registers through all sweeps of the pass:
//
//   down:  nu1 sweeps -> residual -> restriction      (multigrid.py:274-285)
//   up:    prolong-add -> nu2 sweeps [-> residual norm] (multigrid.py:317-327,
//                                                       447-459)
//
// Jacobi reads only slab n and n-1 of the previous iterate (multigrid.py:
// 168-180), so the value a lane needs from its left neighbour at sweep k is a
// warp shuffle away; lane 0 takes it from a per-sweep carry that lane 31 of
// the previous row left behind.  A chunk that does not start at slab 0 first
// runs one "warm-up" row over the 32 slabs before it (only lanes >= k are
// valid after k sweeps, and lane 31 needs nu+1 <= 32 of them), so warps never
// synchronise with each other: the whole pass is one HBM read of u, f (and
// u_coarse) and one write of u (and f_coarse) per slab.
//
// Rows arrive in a per-warp shared-memory ring filled by the TMA engine
// (cp.async.bulk global->shared, completion on an mbarrier); lane 0 issues
// the copy for row i+STAGES as soon as the warp has consumed row i.
#pragma once
#include "tmg_slab.cuh"

namespace tmg {

constexpr int SW_WARPS = 8;   // warps per CTA
constexpr int SW_STAGES = 4;  // rows in flight per warp

enum StreamFlags : int {
    SF_ZERO_GUESS = 1,   // u_in is the zero vector: not read
    SF_RESTRICT = 2,     // residual + restriction -> fc
    SF_WRITE_U = 4,      // store the smoothed iterate
    SF_PROLONG = 8,      // u += P uc before the sweeps
    SF_NORM_LEAF = 16,   // residual -> numpy pairwise leaf sums -> leaf_out
    SF_NORM_SQ = 32,     // residual -> per-slab squared norms -> sq_out
    SF_WRITE_R = 64,     // residual -> r_out
    SF_TMA = 128,        // all row bases are 16-byte aligned: use the bulk-copy ring
};

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
    int rows_per_chunk;
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
    static constexpr int STAGE = 2 * ROW + HALF;
    static constexpr size_t BYTES_PER_WARP = sizeof(T) * STAGE * SW_STAGES;
    // mbarrier block (one 8-byte barrier per warp and stage), padded to 128 B
    static constexpr size_t BAR_BYTES = ((SW_WARPS * SW_STAGES * 8 + 127) / 128) * 128;
    static constexpr size_t SMEM_BYTES = BAR_BYTES + BYTES_PER_WARP * SW_WARPS;
};

template <typename T, int NT, int NU, bool SPARSE, bool UP>
__global__ void __launch_bounds__(SW_WARPS * 32)
    stream_kernel(const __grid_constant__ LevelC<T, NT> L, const __grid_constant__ StreamArgs<T> a)
{
    using Lay = RowLayout<T, NT>;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const long long gw = (long long)blockIdx.x * SW_WARPS + warp;
    if (gw >= (long long)a.batch * a.chunks) return;
    const int b = (int)(gw / a.chunks);
    const long long chunk = gw - (long long)b * a.chunks;
    if (a.active && !a.active[b]) return;

    const long long n = a.n;
    const long long nc = n >> 1;
    const long long nrows = (n + 31) >> 5;
    const long long row0 = chunk * a.rows_per_chunk;
    const int rows = (int)min((long long)a.rows_per_chunk, nrows - row0);
    const int it0 = row0 > 0 ? -1 : 0;
    const int flags = a.flags;
    const bool zero_guess = flags & SF_ZERO_GUESS;
    const bool prolong = UP && (flags & SF_PROLONG);
    const bool need_r = flags & (SF_RESTRICT | SF_NORM_LEAF | SF_NORM_SQ | SF_WRITE_R);

    const T *fb = a.f + (size_t)b * n * NT;
    const T *ub = zero_guess ? nullptr : a.u_in + (size_t)b * n * NT;
    const T *ucb = prolong ? a.uc + (size_t)b * nc * NT : nullptr;

    uint64_t *bars = reinterpret_cast<uint64_t *>(smem) + warp * SW_STAGES;
    T *ring = reinterpret_cast<T *>(smem + Lay::BAR_BYTES) + (size_t)warp * Lay::STAGE * SW_STAGES;
    const bool tma = flags & SF_TMA;

    // a row goes through the ring iff all its pieces are 16-byte multiples
    auto row_tma = [&](long long row) -> bool {
        if (!tma) return false;
        long long cnt = min(32LL, n - row * 32);
        if ((cnt * NT * (long long)sizeof(T)) & 15) return false;
        if (prolong) {
            long long cc = min(16LL, nc - row * 16);
            if (cc > 0 && ((cc * NT * (long long)sizeof(T)) & 15)) return false;
        }
        return true;
    };
    uint64_t pol = 0;
    if (lane == 0 && tma) {
#pragma unroll
        for (int s = 0; s < SW_STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        pol = policy_evict_first();
    }
    __syncwarp();

    auto issue = [&](int it) {  // lane 0 only
        const long long row = row0 + it;
        if (!row_tma(row)) return;
        const int st = (it - it0) % SW_STAGES;
        T *stg = ring + (size_t)st * Lay::STAGE;
        const long long s0 = row * 32;
        const uint32_t bytes = (uint32_t)(min(32LL, n - s0) * NT * sizeof(T));
        long long cc = prolong ? min(16LL, nc - row * 16) : 0;
        const uint32_t cbytes = cc > 0 ? (uint32_t)(cc * NT * sizeof(T)) : 0u;
        mbar_expect_tx(&bars[st], bytes * (zero_guess ? 1u : 2u) + cbytes);
        bulk_g2s(stg + Lay::ROW, fb + s0 * NT, bytes, &bars[st], pol);
        if (!zero_guess) bulk_g2s(stg, ub + s0 * NT, bytes, &bars[st], pol);
        if (cbytes) bulk_g2s(stg + 2 * Lay::ROW, ucb + row * 16 * NT, cbytes, &bars[st], pol);
    };

    if (lane == 0 && tma)
        for (int it = it0; it < rows && it < it0 + SW_STAGES; ++it) issue(it);

    Cpl<T, NT, SPARSE> carry[NU + 1];
#pragma unroll
    for (int k = 0; k <= NU; ++k) cpl_zero(carry[k]);
    T leaf_acc = T(0);
    const bool odd = lane & 1;

    for (int it = it0; it < rows; ++it) {
        const long long row = row0 + it;
        const long long slab = row * 32 + lane;
        const bool valid = slab < n;
        T u[NT], f[NT], uc[NT];
        zero_slab<T, NT>(u);
        zero_slab<T, NT>(f);
        zero_slab<T, NT>(uc);
        const bool pro_ok = prolong && slab < 2 * nc;
        if (row_tma(row)) {
            const int st = (it - it0) % SW_STAGES;
            const T *stg = ring + (size_t)st * Lay::STAGE;
            mbar_wait(&bars[st], (uint32_t)(((it - it0) / SW_STAGES) & 1));
            if (valid) {
                load_slab<T, NT>(stg + Lay::ROW + lane * NT, f);
                if (!zero_guess) load_slab<T, NT>(stg + lane * NT, u);
                if (pro_ok) load_slab<T, NT>(stg + 2 * Lay::ROW + (lane >> 1) * NT, uc);
            }
            __syncwarp();
            if (lane == 0 && it + SW_STAGES < rows) issue(it + SW_STAGES);
        } else {
            if (valid) {
                load_slab_scalar<T, NT>(fb + slab * NT, f);
                if (!zero_guess) load_slab_scalar<T, NT>(ub + slab * NT, u);
                if (pro_ok) load_slab_scalar<T, NT>(ucb + (slab >> 1) * NT, uc);
            }
            __syncwarp();
            if (lane == 0 && tma && it + SW_STAGES < rows) issue(it + SW_STAGES);
        }

        if (UP && pro_ok) prolong_part<T, NT>(L, uc, odd, u);

        const bool has_prev = slab > 0;
#pragma unroll
        for (int k = 0; k < NU; ++k) {
            Cpl<T, NT, SPARSE> own = make_cpl<T, NT, SPARSE>(L, u);
            Cpl<T, NT, SPARSE> prev = cpl_shfl_up<T, NT, SPARSE>(own);
            cpl_select<T, NT, SPARSE>(prev, carry[k], lane == 0);
            carry[k] = cpl_shfl<T, NT, SPARSE>(own, 31);
            sweep<T, NT, SPARSE>(L, u, f, prev, has_prev);
        }

        if (need_r) {
            Cpl<T, NT, SPARSE> own = make_cpl<T, NT, SPARSE>(L, u);
            Cpl<T, NT, SPARSE> prev = cpl_shfl_up<T, NT, SPARSE>(own);
            cpl_select<T, NT, SPARSE>(prev, carry[NU], lane == 0);
            carry[NU] = cpl_shfl<T, NT, SPARSE>(own, 31);
            if (it >= 0) {
                T r[NT];
                residual<T, NT, SPARSE>(L, u, f, prev, has_prev, r);
                if (flags & SF_WRITE_R) {
                    if (valid) store_slab<T, NT>(a.r_out + ((size_t)b * n + slab) * NT, r);
                }
                if (flags & SF_RESTRICT) {
                    T p[NT], q[NT];
                    restrict_part<T, NT>(L, r, odd, p);
#pragma unroll
                    for (int i = 0; i < NT; ++i) q[i] = __shfl_down_sync(0xffffffffu, p[i], 1);
#pragma unroll
                    for (int i = 0; i < NT; ++i) p[i] = FP<T>::add(p[i], q[i]);
                    const long long cidx = slab >> 1;
                    if (!odd && cidx < nc) store_slab<T, NT>(a.fc + ((size_t)b * nc + cidx) * NT, p);
                }
                if (flags & (SF_NORM_LEAF | SF_NORM_SQ)) {
                    T sq = sqnorm<T, NT>(r);
                    if (flags & SF_NORM_SQ) {
                        if (valid) a.sq_out[(size_t)b * n + slab] = (double)sq;
                    } else {
                        // numpy pairwise leaf: 8 strided accumulators over the leaf
                        const int q = (int)(row % a.leaf_rows);
                        T v1 = __shfl_down_sync(0xffffffffu, sq, 8);
                        T v2 = __shfl_down_sync(0xffffffffu, sq, 16);
                        T v3 = __shfl_down_sync(0xffffffffu, sq, 24);
                        leaf_acc = (q == 0) ? sq : FP<T>::add(leaf_acc, sq);
                        leaf_acc = FP<T>::add(leaf_acc, v1);
                        leaf_acc = FP<T>::add(leaf_acc, v2);
                        leaf_acc = FP<T>::add(leaf_acc, v3);
                        if (q == a.leaf_rows - 1) {
                            T t1 = FP<T>::add(leaf_acc, __shfl_down_sync(0xffffffffu, leaf_acc, 1));
                            T t2 = FP<T>::add(t1, __shfl_down_sync(0xffffffffu, t1, 2));
                            T t3 = FP<T>::add(t2, __shfl_down_sync(0xffffffffu, t2, 4));
                            const long long nleaves = n / (32LL * a.leaf_rows);
                            if (lane == 0) a.leaf_out[(size_t)b * nleaves + row / a.leaf_rows] = (double)t3;
                        }
                    }
                }
            }
        }
        if ((flags & SF_WRITE_U) && it >= 0 && valid)
            store_slab<T, NT>(a.u_out + ((size_t)b * n + slab) * NT, u);
    }
}

}  // namespace tmg
