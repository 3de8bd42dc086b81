// Instantiations of the single-CTA tail engine and the exact coarse solves
// (serial substitution, grid-wide scan) for one (dtype, n_t) pair:
//   -DTMG_T=double|float -DTMG_NT=1..4
// A translation unit of its own: edits of the tail rebuild nothing else.
#define TMG_INST_UNIT 1
#include "tmg_launch.cuh"
#include "tmg_tail.cuh"
#include "tmg_scan.cuh"

#include <algorithm>

#ifndef TMG_T
#error "define TMG_T and TMG_NT"
#endif

namespace tmg {

template <typename T, int NT> int tail_prepare(bool sparse, size_t smem)
{
    cudaError_t e = sparse ? cudaFuncSetAttribute(tail_kernel<T, NT, true>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                           : cudaFuncSetAttribute(tail_kernel<T, NT, false>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return (int)e;
}

template <typename T, int NT>
int tail_launch(const TailArgs<T, NT> &t, bool sparse, unsigned grid, size_t smem, cudaStream_t s)
{
    if (sparse) return (int)launch_pdl(tail_kernel<T, NT, true>, dim3(grid), dim3(TAIL_THREADS), smem, s, t);
    return (int)launch_pdl(tail_kernel<T, NT, false>, dim3(grid), dim3(TAIL_THREADS), smem, s, t);
}

template <typename T, int NT>
int coarse_serial_launch(const LevelC<T, NT> &L, bool sparse, const T *f, T *u, long long n, int batch,
                         int variant, const int *active, cudaStream_t s)
{
    const unsigned grid = (unsigned)((batch + 31) / 32);
    if (sparse) coarse_serial_kernel<T, NT, true><<<grid, 32, 0, s>>>(L, f, u, n, batch, variant, active);
    else coarse_serial_kernel<T, NT, false><<<grid, 32, 0, s>>>(L, f, u, n, batch, variant, active);
    return (int)cudaGetLastError();
}

// exact solve by the grid-wide decoupled look-back scan (tmg_scan.cuh): the
// tile states and the tile counter live in a stream-ordered allocation
template <typename T, int NT>
int coarse_scan_launch(const LevelC<T, NT> &L, const T *f, T *u, long long n, int batch, const int *active,
                       cudaStream_t s)
{
    if (n <= 0 || batch <= 0) return 0;
    const long long tile = 32LL * scan_groups<NT>();
    const long long tiles_per = (n + tile - 1) / tile;
    const size_t st_bytes = sizeof(ScanTileState) * (size_t)tiles_per * batch;
    void *ws = nullptr;
    cudaError_t e = cudaMallocAsync(&ws, st_bytes + 16, s);
    if (e != cudaSuccess) return (int)e;
    e = cudaMemsetAsync(ws, 0, st_bytes + 16, s);
    if (e == cudaSuccess) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const long long warps = tiles_per * batch;
        const long long ctas = std::min<long long>((warps + SCAN_WARPS - 1) / SCAN_WARPS, (long long)sms * 8);
        scan_solve_kernel<T, NT><<<(unsigned)ctas, SCAN_WARPS * 32, 0, s>>>(
            L, f, u, n, batch, tiles_per, reinterpret_cast<ScanTileState *>(ws),
            reinterpret_cast<unsigned long long *>(static_cast<char *>(ws) + st_bytes), active);
        e = cudaGetLastError();
    }
    cudaError_t e2 = cudaFreeAsync(ws, s);
    return (int)(e != cudaSuccess ? e : e2);
}

template int coarse_scan_launch<TMG_T, TMG_NT>(const LevelC<TMG_T, TMG_NT> &, const TMG_T *, TMG_T *, long long,
                                               int, const int *, cudaStream_t);
template int tail_prepare<TMG_T, TMG_NT>(bool, size_t);
template int tail_launch<TMG_T, TMG_NT>(const TailArgs<TMG_T, TMG_NT> &, bool, unsigned, size_t, cudaStream_t);
template int coarse_serial_launch<TMG_T, TMG_NT>(const LevelC<TMG_T, TMG_NT> &, bool, const TMG_T *, TMG_T *,
                                                 long long, int, int, const int *, cudaStream_t);

}  // namespace tmg
