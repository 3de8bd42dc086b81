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

// exact solve by the grid-wide three-pass scan (tmg_scan.cuh): tile maps and
// carries in a stream-ordered allocation
template <typename T, int NT>
int coarse_scan_launch(const LevelC<T, NT> &L, const T *f, T *u, long long n, int batch, const int *active,
                       cudaStream_t s)
{
    if (n <= 0 || batch <= 0) return 0;
    const long long tiles_per = (n + ScanTile<T, NT>::SLABS - 1) / ScanTile<T, NT>::SLABS;
    const size_t maps_bytes = sizeof(ScanTileMap) * (size_t)tiles_per * batch;
    const size_t carry_bytes = sizeof(ScanCarry) * (size_t)tiles_per * batch;
    void *ws = nullptr;
    cudaError_t e = cudaMallocAsync(&ws, maps_bytes + carry_bytes, s);
    if (e != cudaSuccess) return (int)e;
    auto *maps = reinterpret_cast<ScanTileMap *>(ws);
    auto *carry = reinterpret_cast<ScanCarry *>(static_cast<char *>(ws) + maps_bytes);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned ctas = (unsigned)std::min<long long>(tiles_per * batch, (long long)sms * 4);
    scan_agg_kernel<T, NT><<<ctas, SCAN_WARPS * 32, 0, s>>>(L, f, n, batch, tiles_per, maps, active);
    scan_carry_kernel<T, NT><<<(unsigned)batch, SCAN_CARRY_THREADS, 0, s>>>(L, tiles_per, maps, carry, active);
    scan_replay_kernel<T, NT><<<ctas, SCAN_WARPS * 32, 0, s>>>(L, f, u, n, batch, tiles_per, carry, active);
    e = cudaGetLastError();
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
