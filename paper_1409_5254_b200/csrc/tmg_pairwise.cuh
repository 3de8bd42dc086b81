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

// Fast path for sizes whose numpy recursion halves exactly down to leaves of
// L in (64, 128] (or n itself <= 128 with n % 8 == 0): 8 lanes per leaf run
// the 8 strided accumulators, combine them in numpy's tree, then a shared-
// memory binary tree adds the leaves (left + right at every node).  Same
// association as np.sum, in O(L/8 + log n) steps.  Returns -1 leaf size when
// the structure does not apply.
static __device__ __forceinline__ long long pw_leaf_size(long long n)
{
    long long m = n;
    while (m > 128) {
        if (m % 2 || (m / 2) % 8) return -1;
        m /= 2;
    }
    return (m >= 8 && m % 8 == 0) ? m : -1;
}

static __device__ double block_pairwise_auto(const double *a, long long n, double *part)
{
    const long long L = pw_leaf_size(n);
    const long long nleaf = L > 0 ? n / L : 0;
    if (L <= 0 || nleaf * 8 > (long long)blockDim.x) return block_pairwise(a, n, part);
    const int t = threadIdx.x;
    const int leaf = t >> 3, j = t & 7;
    double r = 0.0;
    if (leaf < nleaf) {
        const double *x = a + leaf * L;
        r = x[j];
        for (long long i = 8 + j; i < L; i += 8) r = __dadd_rn(r, x[i]);
    }
    // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)) within each group of 8 lanes
    double t1 = __dadd_rn(r, __shfl_down_sync(0xffffffffu, r, 1));
    double t2 = __dadd_rn(t1, __shfl_down_sync(0xffffffffu, t1, 2));
    double t3 = __dadd_rn(t2, __shfl_down_sync(0xffffffffu, t2, 4));
    if (j == 0 && leaf < nleaf) part[leaf] = t3;
    __syncthreads();
    for (long long w = 1; w < nleaf; w <<= 1) {
        if ((long long)t * 2 * w + w < nleaf && (long long)t * 2 * w < nleaf)
            part[t * 2 * w] = __dadd_rn(part[t * 2 * w], part[t * 2 * w + w]);
        __syncthreads();
    }
    double s = part[0];
    __syncthreads();
    return s;
}

}  // namespace tmg
