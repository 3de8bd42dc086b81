// Instantiations of the single-CTA tail engine and the exact coarse solves
// (serial substitution, grid-wide scan) for one (dtype, n_t) pair:
//   -DTMG_T=double|float -DTMG_NT=1..4
// A translation unit of its own: edits of the tail rebuild nothing else.
#define TMG_INST_UNIT 1
#include <cstdlib>
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

// exact solve by the grid-wide three-pass scan (tmg_scan.cuh): the runs' maps /
// carries (one array, converted in place) in a stream-ordered allocation
template <typename T, int NT>
int coarse_scan_launch(const LevelC<T, NT> &L, const T *f, T *u, long long n, int batch, const int *active,
                       cudaStream_t s)
{
    if (n <= 0 || batch <= 0) return 0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long tiles_per = (n + ScanTile<T, NT>::SLABS - 1) / ScanTile<T, NT>::SLABS;
    // tiles per run: at most SCAN_MAX_RUNS runs per problem and at most 32
    // tiles per run; among those the value that leaves the resident warps
    // (2 CTAs per SM, static grid-stride) the least uneven share, ties to
    // the longer run (fewer maps)
    const long long warps = (long long)sms * 2 * SCAN_WARPS;
    const long long cap = (tiles_per + SCAN_MAX_RUNS - 1) / SCAN_MAX_RUNS;
    int run = (int)cap;
    long long best = -1;
    for (long long c = cap; c <= std::max<long long>(cap, 32); ++c) {
        const long long runs = ((tiles_per + c - 1) / c) * batch;
        const long long worst = ((runs + warps - 1) / warps) * c;   // tiles of the busiest warp
        if (best < 0 || worst <= best) {
            best = worst;
            run = (int)c;
        }
    }
    if (const char *ev = getenv("TMG_SCAN_RUN")) {   // experiments
        const int v = atoi(ev);
        if (v >= cap && v <= 64) run = v;
    }
    const long long runs_per = (tiles_per + run - 1) / run;
    // workspace: the runs' maps, converted to carries in place
    bool ws_owned = false;
    void *ws = scan_workspace(sizeof(double) * (size_t)runs_per * batch, s, &ws_owned);
    if (!ws) return (int)cudaErrorMemoryAllocation;
    cudaError_t e = cudaSuccess;
    auto *maps = reinterpret_cast<double *>(ws);
    const int cth = scan_carry_threads(runs_per);
    const int lgS = scan_carry_logm4((int)runs_per, cth) + 2;
    const size_t stage_bytes = sizeof(double) * (size_t)(runs_per + (runs_per >> lgS) + 1);
    // two transpose buffers per warp; padded so that at most two CTAs share an
    // SM whatever n_t: with room to spare, the NEXT kernel's CTAs (programmatic
    // dependent launch) become resident early and shrink the L1 under the
    // running pass (p_t = 0: 532 us instead of 331 us at 4 x 2^24)
    const size_t tile_bytes = std::max<size_t>(sizeof(T) * 2 * SCAN_WARPS * ScanTile<T, NT>::WARP_ELEMS, 80 * 1024);
    static bool attr_done = false;
    if (!attr_done) {
        e = cudaFuncSetAttribute(scan_agg_kernel<T, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_bytes);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(scan_replay_kernel<T, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)tile_bytes);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(scan_carry_kernel<T, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(double) * (SCAN_MAX_RUNS + SCAN_MAX_RUNS / 4 + 2)));
        if (e != cudaSuccess) return (int)e;
        attr_done = true;
    }
    const unsigned ctas = (unsigned)std::min<long long>((runs_per * batch + SCAN_WARPS - 1) / SCAN_WARPS,
                                                       (long long)sms * 2);
    e = launch_pdl(scan_agg_kernel<T, NT>, dim3(ctas), dim3(SCAN_WARPS * 32), tile_bytes, s, L, f, n, batch, runs_per,
                   run, maps, active);
    if (e == cudaSuccess)
        e = launch_pdl(scan_carry_kernel<T, NT>, dim3((unsigned)batch), dim3(cth), stage_bytes, s, L, (int)runs_per,
                       run, (const double *)maps, maps, active);
    if (e == cudaSuccess)
        e = launch_pdl(scan_replay_kernel<T, NT>, dim3(ctas), dim3(SCAN_WARPS * 32), tile_bytes, s, L, f, u, n, batch,
                       runs_per, run, (const double *)maps, active);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (ws_owned) {
        cudaError_t e2 = cudaFreeAsync(ws, s);
        if (e == cudaSuccess) e = e2;
    }
    return (int)e;
}

template int coarse_scan_launch<TMG_T, TMG_NT>(const LevelC<TMG_T, TMG_NT> &, const TMG_T *, TMG_T *, long long,
                                               int, const int *, cudaStream_t);
template int tail_prepare<TMG_T, TMG_NT>(bool, size_t);
template int tail_launch<TMG_T, TMG_NT>(const TailArgs<TMG_T, TMG_NT> &, bool, unsigned, size_t, cudaStream_t);
template int coarse_serial_launch<TMG_T, TMG_NT>(const LevelC<TMG_T, TMG_NT> &, bool, const TMG_T *, TMG_T *,
                                                 long long, int, int, const int *, cudaStream_t);

}  // namespace tmg
