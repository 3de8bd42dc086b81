// Launchers of the templated kernels.  Each (dtype, n_t) pair is compiled in
// its own translation unit (tmg_inst.cu built with -DTMG_T/-DTMG_NT) so the
// ~140 specialisations build in parallel; tmg_api.cu only sees these
// declarations.  All return 0 or a cudaError_t value (TMG_E_* for bad args).
#pragma once
#include <cuda_runtime.h>

#include "tmg_slab.cuh"
#include "tmg_types.cuh"

#include <cstdlib>
#include <utility>

namespace tmg {

// TMG_NO_PDL=1 launches without the programmatic-serialisation attribute (A/B)
inline bool pdl_enabled()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TMG_NO_PDL");
        v = (e && *e && *e != '0') ? 0 : 1;
    }
    return v == 1;
}

// kernel launch with programmatic dependent launch on the stream
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

template <typename T> struct StreamArgs;

// kind: Kind (tmg_stream.cuh); perm: PermKind (tmg_slab.cuh)
template <typename T, int NT>
int stream_launch(const LevelC<T, NT> &L, const StreamArgs<T> &a, int nu, int kind, int perm, bool sparse,
                  cudaStream_t s);
template <typename T, int NT> size_t stream_smem_bytes();
template <typename T, int NT>
int stream_d_launch(const LevelC<T, NT> &L0, const LevelC<T, NT> &L1, const StreamArgs<T> &a,
                    const StreamArgs<T> &a1, int nu, int perm, cudaStream_t s);
template <typename T, int NT>
int stream_v_launch(const LevelC<T, NT> &L0, const LevelC<T, NT> &L1, const StreamArgs<T> &a,
                    const StreamArgs<T> &a1, int nu, int perm, bool finest, cudaStream_t s);
template <typename T, int NT> int tail_prepare(bool sparse, size_t smem);
template <typename T, int NT>
int tail_launch(const TailArgs<T, NT> &t, bool sparse, unsigned grid, size_t smem, cudaStream_t s);
template <typename T, int NT>
int coarse_serial_launch(const LevelC<T, NT> &L, bool sparse, const T *f, T *u, long long n, int batch,
                         int variant, const int *active, cudaStream_t s);

template <typename T, int NT>
int coarse_scan_launch(const LevelC<T, NT> &L, const T *f, T *u, long long n, int batch, const int *active,
                       cudaStream_t s);
// Workspace of the scan solve on stream s (defined in tmg_api.cu): one
// grow-only device buffer per stream, reused by every call on that stream
// (work on one stream is ordered).  A stream-ordered allocation per call
// (cudaMallocAsync / cudaFreeAsync) cost 50-250 us and made the timings
// erratic; it remains the path under stream capture, where *owned is set
// and the caller frees with cudaFreeAsync.  nullptr on failure.
void *scan_workspace(size_t bytes, cudaStream_t s, bool *owned);

#define TMG_DECLARE(T, NT)                                                                              \
    extern template int stream_launch<T, NT>(const LevelC<T, NT> &, const StreamArgs<T> &, int, int, int, \
                                             bool, cudaStream_t);                                       \
    extern template size_t stream_smem_bytes<T, NT>();                                                  \
    extern template int stream_d_launch<T, NT>(const LevelC<T, NT> &, const LevelC<T, NT> &,             \
                                               const StreamArgs<T> &, const StreamArgs<T> &, int, int,    \
                                               cudaStream_t);                                             \
    extern template int stream_v_launch<T, NT>(const LevelC<T, NT> &, const LevelC<T, NT> &,             \
                                               const StreamArgs<T> &, const StreamArgs<T> &, int, int,    \
                                               bool, cudaStream_t);                                       \
    extern template int tail_prepare<T, NT>(bool, size_t);                                              \
    extern template int tail_launch<T, NT>(const TailArgs<T, NT> &, bool, unsigned, size_t, cudaStream_t); \
    extern template int coarse_serial_launch<T, NT>(const LevelC<T, NT> &, bool, const T *, T *, long long, \
                                                    int, int, const int *, cudaStream_t);     \
    extern template int coarse_scan_launch<T, NT>(const LevelC<T, NT> &, const T *, T *, long long, int, \
                                                  const int *, cudaStream_t);
#ifndef TMG_INST_UNIT
TMG_DECLARE(double, 1)
TMG_DECLARE(double, 2)
TMG_DECLARE(double, 3)
TMG_DECLARE(double, 4)
TMG_DECLARE(float, 1)
TMG_DECLARE(float, 2)
TMG_DECLARE(float, 3)
TMG_DECLARE(float, 4)
#endif

}  // namespace tmg
