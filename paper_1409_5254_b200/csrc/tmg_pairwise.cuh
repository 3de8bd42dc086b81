// numpy pairwise summation on the GPU, bit-exact with np.sum of a
// contiguous float64 vector (the norm reduction of multigrid.py:459).
#pragma once
#include "tmg_slab.cuh"

namespace tmg {

// ---------------------------------------------------------------------------
// numpy pairwise summation (np.sum, multigrid.py:459), exact for any n.
// Serial form for one thread:
static __device__ __forceinline__ double pw_leaf(const double *a, long long n)
{
    if (n < 8) {
        double res = 0.0;
        for (long long i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    long long i;
    for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
}

// serial pairwise over [0, n) with an explicit stack (no device recursion)
static __device__ double pw_serial(const double *a, long long n)
{
    // depth <= log2(n / 128) + 1; 40 covers any int64 length
    struct Node { long long off, len; double left; int state; };
    Node st[40];
    int sp = 0;
    st[0] = {0, n, 0.0, 0};
    double ret = 0.0;
    while (sp >= 0) {
        Node &nd = st[sp];
        if (nd.len <= 128) {
            ret = pw_leaf(a + nd.off, nd.len);
            --sp;
            continue;
        }
        long long n2 = nd.len / 2;
        n2 -= n2 % 8;
        if (nd.state == 0) {
            nd.state = 1;
            st[sp + 1] = {nd.off, n2, 0.0, 0};
            ++sp;
        } else if (nd.state == 1) {
            nd.left = ret;
            nd.state = 2;
            st[sp + 1] = {nd.off + n2, nd.len - n2, 0.0, 0};
            ++sp;
        } else {
            ret = __dadd_rn(nd.left, ret);
            --sp;
        }
    }
    return ret;
}

// CTA-wide exact pairwise sum; all threads get the result.  `part` has
// blockDim.x doubles of shared scratch; blockDim.x must be a power of two.
static __device__ double block_pairwise(const double *a, long long n, double *part)
{
    const int T = blockDim.x;
    int D = 0;
    while ((1 << D) < T) ++D;
    const int t = threadIdx.x;
    long long off = 0, len = n;
    int d = 0;
    while (d < D && len > 128) {
        long long n2 = len / 2;
        n2 -= n2 % 8;
        if ((t >> (D - 1 - d)) & 1) { off += n2; len -= n2; }
        else len = n2;
        ++d;
    }
    const bool owner = (d == D) || ((t & ((1 << (D - d)) - 1)) == 0);
    if (owner) part[t] = (d == D) ? pw_serial(a + off, len) : pw_leaf(a + off, len);
    __syncthreads();
    if (t == 0) {
        // re-walk the top of the tree, combining owners' partials
        struct Node { long long len; double left; int d, p, state; };
        Node st[24];  // depth <= D + 1 <= 11
        int sp = 0;
        st[0] = {n, 0.0, 0, 0, 0};
        double ret = 0.0;
        while (sp >= 0) {
            Node &nd = st[sp];
            if (nd.d == D || nd.len <= 128) {
                ret = part[nd.p << (D - nd.d)];
                --sp;
                continue;
            }
            long long n2 = nd.len / 2;
            n2 -= n2 % 8;
            if (nd.state == 0) {
                nd.state = 1;
                st[sp + 1] = {n2, 0.0, nd.d + 1, nd.p << 1, 0};
                ++sp;
            } else if (nd.state == 1) {
                nd.left = ret;
                nd.state = 2;
                st[sp + 1] = {nd.len - n2, 0.0, nd.d + 1, (nd.p << 1) | 1, 0};
                ++sp;
            } else {
                ret = __dadd_rn(nd.left, ret);
                --sp;
            }
        }
        part[0] = ret;
    }
    __syncthreads();
    double s = part[0];
    __syncthreads();
    return s;
}

}  // namespace tmg
