// Microbenchmark: latency of the tail engine's building blocks on one warp
// (n_t = 2, fp64, constants in shared memory as in the tail): one slab sweep,
// a sweep of a slab pair, a pair + residual + restriction (a down pass's
// compute), each as a dependent chain repeated N times.
#include <cstdio>
#include <cuda_runtime.h>
#include "tmg_slab.cuh"
using namespace tmg;
// Keeps the dependent chains finite (the constants are not a consistent
// factorisation, so the iteration need not contract): non-finite values would
// send every sweep down the exact-division fallback and time that instead.
__device__ __forceinline__ void clamp2(double *x)
{
    x[0] = fmin(fmax(x[0], -1e3), 1e3);
    x[1] = fmin(fmax(x[1], -1e3), 1e3);
}
__global__ void bench(const LevelC<double, 2> *Lg, double *out, long long *cyc, int n)
{
    __shared__ LevelC<double, 2> Ls;
    if (threadIdx.x == 0) Ls = *Lg;
    __syncthreads();
    const LevelC<double, 2> &L = Ls;
    double x0[2] = {0.3 + threadIdx.x, 0.7}, x1[2] = {0.1, 0.2}, f0[2] = {1.0, 2.0}, f1[2] = {0.5, 0.25};
    Cpl<double, 2, true> p;
    p.s = 0.1;
    p.m = 0;
    long long c0 = clock64();
    sweep<double, 2, true>(L, x0, f0, p, true);
    clamp2(x0);
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        sweep<double, 2, true>(L, x0, f0, p, true);
        clamp2(x0);
    }
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) {
        const Cpl<double, 2, true> o0 = make_cpl<double, 2, true>(L, x0);
        sweep<double, 2, true>(L, x0, f0, p, true);
        sweep<double, 2, true>(L, x1, f1, o0, true);
        clamp2(x0);
        clamp2(x1);
    }
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) {
        const Cpl<double, 2, true> o0 = make_cpl<double, 2, true>(L, x0);
        sweep<double, 2, true>(L, x0, f0, p, true);
        sweep<double, 2, true>(L, x1, f1, o0, true);
        double r0[2], r1[2], q0[2], q1[2];
        const Cpl<double, 2, true> c0 = make_cpl<double, 2, true>(L, x0);
        residual<double, 2, true>(L, x0, f0, p, true, r0);
        residual<double, 2, true>(L, x1, f1, c0, true, r1);
        restrict_part<double, 2>(L, r0, false, q0);
        restrict_part<double, 2>(L, r1, true, q1);
        f0[0] = q0[0] + q1[0];
        f1[1] = q0[1] + q1[1];
        clamp2(x0);
        clamp2(x1);
        clamp2(f0);
        clamp2(f1);
    }
    long long t3 = clock64();
    out[threadIdx.x] = x0[0] + x1[1] + f0[0] + f1[1];
    if (threadIdx.x == 0) {
        cyc[3] = t0 - c0;
        cyc[0] = (t1 - t0) / n;
        cyc[1] = (t2 - t1) / n;
        cyc[2] = (t3 - t2) / n;
    }
}
int main()
{
    LevelC<double, 2> h{};
    double A[4] = {-1.1, 0.3, -0.2, -1.4}, lu[4] = {0.9, 0.2, 0.3, 1.1};
    for (int i = 0; i < 4; ++i) { h.A[i] = A[i]; h.lu[i] = lu[i]; h.R1[i] = 0.5; h.R2[i] = 0.25; }
    h.C[0] = 1.0; h.C[1] = -1.0;
    h.rinv[0] = 1.0 / 0.9; h.rinv[1] = 1.0 / 1.1;
    h.perm[0] = 1; h.perm[1] = 0;
    h.omega = 0.5;
    LevelC<double, 2> *d;
    double *o;
    long long *c;
    cudaMalloc(&d, sizeof(h));
    cudaMemcpy(d, &h, sizeof(h), cudaMemcpyHostToDevice);
    cudaMalloc(&o, 32 * 8);
    cudaMallocManaged(&c, 4 * 8);
    for (int r = 0; r < 2; ++r) {
        bench<<<1, 32>>>(d, o, c, 1000);
        cudaDeviceSynchronize();
    }
    printf("cycles per: sweep %lld, pair sweep %lld, pair sweep+residual+restrict %lld\n", c[0], c[1], c[2]);
    printf("first (cold instruction cache) single sweep: %lld cycles\n", c[3]);
    double ho[32];
    cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
    printf("final values (finite => the fast path ran): %g %g\n", ho[0], ho[31]);
    return 0;
}
