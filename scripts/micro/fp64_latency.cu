// Microbenchmark: dependent-chain latency of fp64 ops on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double *out, long long *cyc, double a, double b, int n)
{
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
    long long t1 = clock64();
    double y = a;
    for (int i = 0; i < n; ++i) y = __dmul_rn(y, b);
    long long t2 = clock64();
    double z = a;
    for (int i = 0; i < n; ++i) z = __fma_rn(z, b, a);
    long long t3 = clock64();
    double w = a;
    for (int i = 0; i < n; ++i) w = __ddiv_rn(w, b);
    long long t4 = clock64();
    float fx = (float)a;
    for (int i = 0; i < n; ++i) fx = __fadd_rn(fx, (float)b);
    long long t5 = clock64();
    out[0] = x + y + z + w + fx;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
}
int main()
{
    double *o; long long *c;
    cudaMalloc(&o, 8); cudaMallocManaged(&c, 8 * 8);
    const int n = 4096;
    chain<<<1, 1>>>(o, c, 1.0000001, 0.9999999, n);
    cudaDeviceSynchronize();
    chain<<<1, 1>>>(o, c, 1.0000001, 0.9999999, n);
    cudaDeviceSynchronize();
    printf("per dependent op (cycles): dadd %.2f dmul %.2f dfma %.2f ddiv %.2f fadd %.2f\n",
           (double)c[0] / n, (double)c[1] / n, (double)c[2] / n, (double)c[3] / n, (double)c[4] / n);
    return 0;
}
