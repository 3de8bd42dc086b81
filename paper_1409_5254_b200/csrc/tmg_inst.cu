// Kernel instantiations for one (dtype, n_t) pair: compile with
//   -DTMG_T=double|float -DTMG_NT=1..4 -DTMG_PART=0..3
// The instantiations of a pair are split over four translation units so the
// build runs them in parallel:
//   part 0  the dispatcher, generic (runtime-flag) passes, down passes
// (the single-CTA tail engine and the coarse solves: tmg_inst_tail.cu)
//   part 1  up passes with separately stored pre-sweeps (K_UP, K_UPNORM) and
//           K_UP2NORM
//   part 2  the recomputing up passes (K_UP2, K_UP2DOWN)
//   part 3  the multi-level kernels (vertical fusion, coarse pairs)
#define TMG_INST_UNIT 1
#include "tmg_launch.cuh"
#include "tmg_stream.cuh"

#ifndef TMG_T
#error "define TMG_T and TMG_NT"
#endif
#ifndef TMG_PART
#define TMG_PART -1  // all parts in one unit
#endif
#define TMG_IN_PART(k) (TMG_PART < 0 || TMG_PART == (k))

namespace tmg {

// one stream-kernel kind (all nu, all LU-permutation patterns); defined in
// the part that owns the kind
template <typename T, int NT, int KIND>
int launch_kind(const LevelC<T, NT> &L, const StreamArgs<T> &a, int nu, int perm, cudaStream_t s);

namespace {

template <typename T, int NT, int NU, bool SP, int KIND, int PERM>
int launch_one(const LevelC<T, NT> &L, const StreamArgs<T> &a, cudaStream_t s)
{
    auto k = stream_kernel<T, NT, NU, SP, KIND, PERM>;
    constexpr size_t smem = RowLayout<T, NT, KindProlongs<KIND>::value, KindLeaf<KIND>::value>::SMEM_BYTES;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        attr = true;
    }
    const long long warps = (long long)a.batch * a.chunks;
    constexpr int WARPS = CtaShape<T, NT>::WARPS;
    const long long grid = (warps + WARPS - 1) / WARPS;
    if (grid <= 0) return 0;
    return (int)launch_pdl(k, dim3((unsigned)grid), dim3(WARPS * 32), smem, s, L, a);
}

template <typename T, int NT, bool SP, int KIND, int PERM>
int by_nu(const LevelC<T, NT> &L, const StreamArgs<T> &a, int nu, cudaStream_t s)
{
    switch (nu) {
    case 0: return launch_one<T, NT, 0, SP, KIND, PERM>(L, a, s);
    case 1: return launch_one<T, NT, 1, SP, KIND, PERM>(L, a, s);
    case 2: return launch_one<T, NT, 2, SP, KIND, PERM>(L, a, s);
    case 3: return launch_one<T, NT, 3, SP, KIND, PERM>(L, a, s);
    case 4: return launch_one<T, NT, 4, SP, KIND, PERM>(L, a, s);
    }
    return -2;
}

template <typename T, int NT, int KIND>
int by_perm(const LevelC<T, NT> &L, const StreamArgs<T> &a, int nu, int perm, cudaStream_t s)
{
    if constexpr (NT == 1) {
        return by_nu<T, NT, true, KIND, P_ID>(L, a, nu, s);  // n_t = 1: the only permutation
    } else {
        switch (perm) {
        case P_ID: return by_nu<T, NT, true, KIND, P_ID>(L, a, nu, s);
        case P_ROT: return by_nu<T, NT, true, KIND, P_ROT>(L, a, nu, s);
        default: return by_nu<T, NT, true, KIND, P_GEN>(L, a, nu, s);
        }
    }
}

}  // namespace

template <typename T, int NT, int KIND>
int launch_kind(const LevelC<T, NT> &L, const StreamArgs<T> &a, int nu, int perm, cudaStream_t s)
{
    return by_perm<T, NT, KIND>(L, a, nu, perm, s);
}

#if TMG_IN_PART(0)
template int launch_kind<TMG_T, TMG_NT, K_DOWN>(const LevelC<TMG_T, TMG_NT> &, const StreamArgs<TMG_T> &, int,
                                                int, cudaStream_t);
template int launch_kind<TMG_T, TMG_NT, K_DOWNNORM>(const LevelC<TMG_T, TMG_NT> &, const StreamArgs<TMG_T> &,
                                                    int, int, cudaStream_t);
#endif
#if TMG_IN_PART(1)
template int launch_kind<TMG_T, TMG_NT, K_UP>(const LevelC<TMG_T, TMG_NT> &, const StreamArgs<TMG_T> &, int, int,
                                              cudaStream_t);
template int launch_kind<TMG_T, TMG_NT, K_UPNORM>(const LevelC<TMG_T, TMG_NT> &, const StreamArgs<TMG_T> &, int,
                                                  int, cudaStream_t);
template int launch_kind<TMG_T, TMG_NT, K_UP2NORM>(const LevelC<TMG_T, TMG_NT> &, const StreamArgs<TMG_T> &, int,
                                                   int, cudaStream_t);
#endif
#if TMG_IN_PART(2)
template int launch_kind<TMG_T, TMG_NT, K_UP2>(const LevelC<TMG_T, TMG_NT> &, const StreamArgs<TMG_T> &, int, int,
                                               cudaStream_t);
template int launch_kind<TMG_T, TMG_NT, K_UP2DOWN>(const LevelC<TMG_T, TMG_NT> &, const StreamArgs<TMG_T> &, int,
                                                   int, cudaStream_t);
#endif

// kinds instantiated in other parts: no implicit instantiation here
#define TMG_EXTERN_KIND(K)                                                                                    \
    extern template int launch_kind<TMG_T, TMG_NT, K>(const LevelC<TMG_T, TMG_NT> &, const StreamArgs<TMG_T> &, \
                                                      int, int, cudaStream_t);
#if TMG_PART > 0
TMG_EXTERN_KIND(K_DOWN)
TMG_EXTERN_KIND(K_DOWNNORM)
#endif
#if TMG_PART == 0 || TMG_PART > 1
TMG_EXTERN_KIND(K_UP)
TMG_EXTERN_KIND(K_UPNORM)
TMG_EXTERN_KIND(K_UP2NORM)
#endif
#if TMG_PART >= 0 && TMG_PART != 2
TMG_EXTERN_KIND(K_UP2)
TMG_EXTERN_KIND(K_UP2DOWN)
#endif

#if TMG_IN_PART(0)
template <typename T, int NT>
int stream_launch(const LevelC<T, NT> &L, const StreamArgs<T> &a, int nu, int kind, int perm, bool sparse,
                  cudaStream_t s)
{
    if (!sparse || kind == K_GENERIC) {
        // runtime-flag kernel (general coupling, the single-level API entry points)
        return sparse ? by_nu<T, NT, true, K_GENERIC, P_GEN>(L, a, nu, s)
                      : by_nu<T, NT, false, K_GENERIC, P_GEN>(L, a, nu, s);
    }
    switch (kind) {
    case K_DOWN: return launch_kind<T, NT, K_DOWN>(L, a, nu, perm, s);
    case K_UP: return launch_kind<T, NT, K_UP>(L, a, nu, perm, s);
    case K_UPNORM: return launch_kind<T, NT, K_UPNORM>(L, a, nu, perm, s);
    case K_DOWNNORM: return launch_kind<T, NT, K_DOWNNORM>(L, a, nu, perm, s);
    case K_UP2: return launch_kind<T, NT, K_UP2>(L, a, nu, perm, s);
    case K_UP2NORM: return launch_kind<T, NT, K_UP2NORM>(L, a, nu, perm, s);
    case K_UP2DOWN: return launch_kind<T, NT, K_UP2DOWN>(L, a, nu, perm, s);
    }
    return -1;
}

template <typename T, int NT> size_t stream_smem_bytes() { return RowLayout<T, NT, true, true>::SMEM_BYTES; }

template int stream_launch<TMG_T, TMG_NT>(const LevelC<TMG_T, TMG_NT> &, const StreamArgs<TMG_T> &, int, int,
                                          int, bool, cudaStream_t);
template size_t stream_smem_bytes<TMG_T, TMG_NT>();
#endif

namespace {
template <typename T, int NT, int NU, int PERM, bool FINEST>
int launch_v(const LevelC<T, NT> &L0, const LevelC<T, NT> &L1, const StreamArgs<T> &a, const StreamArgs<T> &a1,
             cudaStream_t s)
{
    auto k = stream_kernel_v<T, NT, NU, true, PERM, FINEST>;
    constexpr size_t smem = RowLayoutV<T, NT, FINEST>::SMEM_BYTES;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        attr = true;
    }
    const long long warps = (long long)a.batch * a.chunks;
    constexpr int WARPS = CtaShape<T, NT>::WARPS;
    const long long grid = (warps + WARPS - 1) / WARPS;
    if (grid <= 0) return 0;
    return (int)launch_pdl(k, dim3((unsigned)grid), dim3(WARPS * 32), smem, s, L0, L1, a, a1);
}
template <typename T, int NT, int PERM, bool FINEST>
int v_by_nu(const LevelC<T, NT> &L0, const LevelC<T, NT> &L1, const StreamArgs<T> &a, const StreamArgs<T> &a1,
            int nu, cudaStream_t s)
{
    switch (nu) {
    case 1: return launch_v<T, NT, 1, PERM, FINEST>(L0, L1, a, a1, s);
    case 2: return launch_v<T, NT, 2, PERM, FINEST>(L0, L1, a, a1, s);
    }
    return -1;
}
}  // namespace

namespace {
template <typename T, int NT, int NU, int PERM>
int launch_d(const LevelC<T, NT> &L0, const LevelC<T, NT> &L1, const StreamArgs<T> &a, const StreamArgs<T> &a1,
             cudaStream_t s)
{
    auto k = stream_kernel_d<T, NT, NU, true, PERM>;
    constexpr size_t smem = RowLayoutD<T, NT>::SMEM_BYTES;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        attr = true;
    }
    const long long warps = (long long)a.batch * a.chunks;
    constexpr int WARPS = CtaShape<T, NT>::WARPS;
    const long long grid = (warps + WARPS - 1) / WARPS;
    if (grid <= 0) return 0;
    return (int)launch_pdl(k, dim3((unsigned)grid), dim3(WARPS * 32), smem, s, L0, L1, a, a1);
}
template <typename T, int NT, int PERM>
int d_by_nu(const LevelC<T, NT> &L0, const LevelC<T, NT> &L1, const StreamArgs<T> &a, const StreamArgs<T> &a1,
            int nu, cudaStream_t s)
{
    // the multi-level kernels are built for nu <= 2 (BASELINE's sweep counts;
    // larger nu takes the per-level kernels) to bound the build time
    switch (nu) {
    case 1: return launch_d<T, NT, 1, PERM>(L0, L1, a, a1, s);
    case 2: return launch_d<T, NT, 2, PERM>(L0, L1, a, a1, s);
    }
    return -1;
}
}  // namespace

#if TMG_IN_PART(3)
// coarse down-pass pairs (two-slab lanes, fp64, sparse coupling; -1 = not available)
template <typename T, int NT>
int stream_d_launch(const LevelC<T, NT> &L0, const LevelC<T, NT> &L1, const StreamArgs<T> &a,
                    const StreamArgs<T> &a1, int nu, int perm, cudaStream_t s)
{
    if constexpr (sizeof(T) != 8) {
        return -1;
    } else {
        switch (perm) {
        case P_ID: return d_by_nu<T, NT, P_ID>(L0, L1, a, a1, nu, s);
        case P_ROT: return d_by_nu<T, NT, P_ROT>(L0, L1, a, a1, nu, s);
        default: return d_by_nu<T, NT, P_GEN>(L0, L1, a, a1, nu, s);
        }
    }
}

// the finest pass with the level-1 up pass fused in (fp64, sparse
// coupling only; -1 = not available for this (dtype, n_t): use the separate passes)
template <typename T, int NT>
int stream_v_launch(const LevelC<T, NT> &L0, const LevelC<T, NT> &L1, const StreamArgs<T> &a,
                    const StreamArgs<T> &a1, int nu, int perm, bool finest, cudaStream_t s)
{
    if constexpr (sizeof(T) != 8) {
        return -1;
    } else {
        if (finest) {
            switch (perm) {
            case P_ID: return v_by_nu<T, NT, P_ID, true>(L0, L1, a, a1, nu, s);
            case P_ROT: return v_by_nu<T, NT, P_ROT, true>(L0, L1, a, a1, nu, s);
            default: return v_by_nu<T, NT, P_GEN, true>(L0, L1, a, a1, nu, s);
            }
        }
        switch (perm) {
        case P_ID: return v_by_nu<T, NT, P_ID, false>(L0, L1, a, a1, nu, s);
        case P_ROT: return v_by_nu<T, NT, P_ROT, false>(L0, L1, a, a1, nu, s);
        default: return v_by_nu<T, NT, P_GEN, false>(L0, L1, a, a1, nu, s);
        }
    }
}

#endif  // part 3


#if TMG_IN_PART(3)
template int stream_d_launch<TMG_T, TMG_NT>(const LevelC<TMG_T, TMG_NT> &, const LevelC<TMG_T, TMG_NT> &,
                                            const StreamArgs<TMG_T> &, const StreamArgs<TMG_T> &, int, int,
                                            cudaStream_t);
template int stream_v_launch<TMG_T, TMG_NT>(const LevelC<TMG_T, TMG_NT> &, const LevelC<TMG_T, TMG_NT> &,
                                            const StreamArgs<TMG_T> &, const StreamArgs<TMG_T> &, int, int,
                                            bool, cudaStream_t);
#endif

}  // namespace tmg
