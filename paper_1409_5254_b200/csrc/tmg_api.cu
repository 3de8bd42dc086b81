// C ABI (include/timemg_b200.h) and the cycle/iteration driver.
//
// The driver is the B200 counterpart of the reference's _cycle/_iterate
// (pkg/src/timemg/multigrid.py:263-500): per cycle it enqueues
//   down(l)   for the streaming levels l = 0 .. tl-1   (tmg_stream.cuh)
//   tail(tl)  one CTA per problem for levels tl .. coarsest (tmg_block.cuh)
//   up(l)     for l = tl-1 .. 0, the finest one fused with the residual
//             norm's numpy-pairwise leaf sums
//   finalize  exact tree sum -> sqrt -> stopping rule per problem
// optionally captured once as a CUDA graph and replayed per cycle.  Problems
// of a batch stop independently (per-problem active mask, like B separate
// reference solves).  If the whole problem fits one CTA's shared memory the
// entire solve is one launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>
#include <numeric>

#include "timemg_b200.h"
#include "tmg_launch.cuh"
#include "tmg_norm.cuh"
#include "tmg_slab.cuh"
#include "tmg_stream.cuh"  // StreamArgs / flags / kinds (kernels are instantiated in tmg_inst.cu)

using namespace tmg;

namespace tmg {

void *scan_workspace(size_t bytes, cudaStream_t s, bool *owned)
{
    *owned = false;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone) {
        void *p = nullptr;
        if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) return nullptr;
        *owned = true;
        return p;
    }
    struct Ws {
        void *p = nullptr;
        size_t bytes = 0;
    };
    static std::mutex mu;
    static std::unordered_map<unsigned long long, Ws> per_stream;   // (device, stream)
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    Ws &w = per_stream[((unsigned long long)(uintptr_t)s << 8) ^ (unsigned long long)dev];
    if (w.bytes < bytes) {
        if (w.p) cudaFree(w.p);   // synchronises: no kernel still reads the old buffer
        const size_t want = std::max<size_t>(bytes, 1 << 16);
        if (cudaMalloc(&w.p, want) != cudaSuccess) {
            w.p = nullptr;
            w.bytes = 0;
            return nullptr;
        }
        w.bytes = want;
    }
    return w.p;
}

}  // namespace tmg

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess)                                                           \
            return fail((int)e_, "%s (tmg_api.cu:%d): %s", #x, __LINE__, cudaGetErrorString(e_)); \
    } while (0)

// TMG_SYNC_DEBUG=1: synchronise after every launch (pinpoints a faulting kernel)
bool sync_debug()
{
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TMG_SYNC_DEBUG");
        v = (e && *e && *e != '0') ? 1 : 0;
    }
    return v == 1;
}

// TMG_EVENT_TRACE=1: direct launches with a CUDA event after each kernel;
// solve() prints per-kernel device times (including launch gaps) to stderr
// (or tmg_trace_enable(1); tmg_trace_read() returns the per-kernel totals)
int g_event_trace = -1;
bool event_trace()
{
    if (g_event_trace < 0) {
        const char *e = getenv("TMG_EVENT_TRACE");
        g_event_trace = (e && *e && *e != '0') ? 1 : 0;
    }
    return g_event_trace == 1;
}
std::vector<std::pair<std::string, cudaEvent_t>> g_trace;
bool g_trace_quiet = false;  // tmg_trace_read collects instead of printing
std::string g_trace_text;
void trace_mark(const char *what, cudaStream_t s)
{
    if (!event_trace()) return;
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    g_trace.emplace_back(what, e);
}
void trace_report()
{
    if (!event_trace() || g_trace.size() < 2) return;
    cudaEventSynchronize(g_trace.back().second);
    struct Agg { std::string name; double ms; int count; };
    std::vector<Agg> agg;
    double total = 0;
    for (size_t i = 1; i < g_trace.size(); ++i) {
        float ms = 0;
        cudaEventElapsedTime(&ms, g_trace[i - 1].second, g_trace[i].second);
        total += ms;
        bool found = false;
        for (auto &a : agg)
            if (a.name == g_trace[i].first) { a.ms += ms; a.count += 1; found = true; }
        if (!found) agg.push_back({g_trace[i].first, ms, 1});
    }
    if (g_trace_quiet) {
        char line[256];
        for (auto &a : agg) {
            snprintf(line, sizeof line, "%s\t%d\t%.6f\n", a.name.c_str(), a.count, a.ms);
            g_trace_text += line;
        }
    } else {
        fprintf(stderr, "event-trace total %.3f ms over %zu launches\n", total, g_trace.size() - 1);
        for (auto &a : agg) fprintf(stderr, "event-trace %10.3f ms %5d  %s\n", a.ms, a.count, a.name.c_str());
    }
    for (auto &e : g_trace) cudaEventDestroy(e.second);
    g_trace.clear();
}

#define CK_LAUNCH(what)                                                                  \
    do {                                                                                 \
        CK(cudaGetLastError());                                                          \
        if (sync_debug()) {                                                              \
            cudaError_t e2_ = cudaDeviceSynchronize();                                   \
            if (e2_ != cudaSuccess)                                                      \
                return fail((int)e2_, "%s (tmg_api.cu:%d): %s", what, __LINE__, cudaGetErrorString(e2_)); \
        }                                                                                \
    } while (0)

#define CKR(x)                      \
    do {                            \
        int r_ = (x);               \
        if (r_ != 0) return r_;     \
    } while (0)

bool coupling_is_sparse(const tmg_level_desc &d)
{
    const int nt = d.n_t;
    for (int i = 1; i < nt; ++i)
        for (int j = 0; j < nt; ++j)
            if (d.coupling[i * nt + j] != 0.0) return false;
    return true;
}

template <typename T, int NT> LevelC<T, NT> make_level(const tmg_level_desc &d)
{
    LevelC<T, NT> L;
    memset(&L, 0, sizeof L);
    for (int i = 0; i < NT * NT; ++i) {
        L.A[i] = (T)d.minus_step[i];
        L.C[i] = (T)d.coupling[i];
        L.lu[i] = (T)d.lu[i];
        L.R1[i] = (T)d.r1[i];
        L.R2[i] = (T)d.r2[i];
    }
    L.omega = (T)d.omega;
    for (int i = 0; i < NT; ++i) {
        L.rinv[i] = (T)1 / L.lu[i * NT + i];  // correctly rounded in T (IEEE division)
        for (int j = 0; j < NT; ++j) L.PA[i * NT + j] = L.A[d.perm[i] * NT + j];
    }
    for (int i = 0; i < NT; ++i) {
        L.perm[i] = d.perm[i];
        unsigned m = 0;
        for (int j = 0; j < NT; ++j) m |= (std::signbit(d.coupling[i * NT + j]) ? 1u : 0u) << j;
        L.cneg[i] = m;
    }
    L.has_transfer = d.has_transfer;
    // WK = omega (K+M)^-1 P^T in double: column j is the LU substitution of the
    // permuted unit vector e_j (dg.py:153-168 without the row gather)
    for (int j = 0; j < NT; ++j) {
        double z[NT];
        for (int i = 0; i < NT; ++i) z[i] = i == j ? 1.0 : 0.0;
        for (int i = 1; i < NT; ++i)
            for (int k = 0; k < i; ++k) z[i] -= d.lu[i * NT + k] * z[k];
        for (int i = NT - 1; i >= 0; --i) {
            for (int k = i + 1; k < NT; ++k) z[i] -= d.lu[i * NT + k] * z[k];
            z[i] /= d.lu[i * NT + i];
        }
        for (int i = 0; i < NT; ++i) L.WK[i * NT + j] = (T)(d.omega * z[i]);
    }
    // rank-1 factors of the coupling (outer(eval_start, eval_end), dg.py:236):
    // e = row 0, c_i = N[i, j*] / N[0, j*] (exact for both bases: c = e_0 or +-1)
    int js = 0;
    for (int j = 1; j < NT; ++j)
        if (std::fabs(d.coupling[j]) > std::fabs(d.coupling[js])) js = j;
    double c[NT], e[NT];
    bool ok = d.coupling[js] != 0.0;
    for (int j = 0; j < NT; ++j) e[j] = d.coupling[j];
    for (int i = 0; i < NT; ++i) c[i] = ok ? d.coupling[i * NT + js] / d.coupling[js] : 0.0;
    for (int i = 0; i < NT && ok; ++i)
        for (int j = 0; j < NT; ++j)
            if (std::fabs(c[i] * e[j] - d.coupling[i * NT + j]) > 1e-14 * std::fabs(d.coupling[js])) ok = false;
    // w = LU^-1 c with the level's own factors (dg.py:153-168 order)
    double y[NT];
    for (int i = 0; i < NT; ++i) y[i] = c[d.perm[i]];
    for (int i = 1; i < NT; ++i)
        for (int j = 0; j < i; ++j) y[i] -= d.lu[i * NT + j] * y[j];
    for (int i = NT - 1; i >= 0; --i) {
        for (int j = i + 1; j < NT; ++j) y[i] -= d.lu[i * NT + j] * y[j];
        y[i] /= d.lu[i * NT + i];
    }
    // alpha = e . LU^-1 c, the recurrence's multiplier, in double-double: the
    // scan applies it ~N times, so its rounding must not be systematic at
    // 1e-16 (tmg_scan.cuh)
    auto two_prod = [](double a, double b, double &err) {
        const double p = a * b;
        err = std::fma(a, b, -p);
        return p;
    };
    auto two_sum = [](double a, double b, double &err) {
        const double s = a + b, bb = s - a;
        err = (a - (s - bb)) + (b - bb);
        return s;
    };
    double yh[NT], yl[NT];  // LU^-1 c in double-double
    for (int i = 0; i < NT; ++i) {
        yh[i] = c[d.perm[i]];
        yl[i] = 0.0;
    }
    auto dd_sub_prod = [&](int i, double m, int j) {  // y_i -= m * y_j
        double pe;
        const double p = two_prod(m, yh[j], pe);
        const double pl = pe + m * yl[j];
        double se;
        const double sh = two_sum(yh[i], -p, se);
        const double sl = se + (yl[i] - pl);
        yh[i] = sh + sl;
        yl[i] = sl - (yh[i] - sh);
    };
    for (int i = 1; i < NT; ++i)
        for (int j = 0; j < i; ++j) dd_sub_prod(i, d.lu[i * NT + j], j);
    for (int i = NT - 1; i >= 0; --i) {
        for (int j = i + 1; j < NT; ++j) dd_sub_prod(i, d.lu[i * NT + j], j);
        const double dv = d.lu[i * NT + i];
        const double q = yh[i] / dv;  // (yh + yl) / dv: one correction step
        double pe;
        const double p = two_prod(q, dv, pe);
        const double r = ((yh[i] - p) - pe + yl[i]) / dv;
        yh[i] = q + r;
        yl[i] = r - (yh[i] - q);
    }
    double ah = 0.0, alo = 0.0;
    for (int j = 0; j < NT; ++j) {
        double pe;
        const double p = two_prod(e[j], yh[j], pe);
        double se;
        const double sh = two_sum(ah, p, se);
        alo += se + pe + e[j] * yl[j];
        ah = sh;
    }
    const double al = ah + alo;
    for (int j = 0; j < NT; ++j) {
        L.ce[j] = (T)e[j];
        L.cw[j] = (T)(yh[j] + yl[j]);
    }
    L.calpha = (T)al;
    L.calpha_lo = (ah - (double)L.calpha) + alo;  // calpha + calpha_lo = alpha to ~1e-32
    L.scan_ok = ok ? 1 : 0;
    return L;
}

int check_desc(const tmg_level_desc *d)
{
    if (!d) return fail(TMG_E_ARG, "level descriptor is NULL");
    if (d->n_t < 1 || d->n_t > 4) return fail(TMG_E_UNSUPPORTED, "n_t=%d: GPU kernels support 1..4", d->n_t);
    if (d->n_slabs < 1) return fail(TMG_E_ARG, "n_slabs must be >= 1");
    for (int i = 0; i < d->n_t; ++i)
        if (d->perm[i] < 0 || d->perm[i] >= d->n_t) return fail(TMG_E_ARG, "bad LU permutation");
    return 0;
}

// compile-time LU permutation pattern of a level (PermKind)
int perm_kind(const tmg_level_desc &d)
{
    bool id = true, rot = true;
    for (int i = 0; i < d.n_t; ++i) {
        id &= d.perm[i] == i;
        rot &= d.perm[i] == (i + 1) % d.n_t;
    }
    return id ? P_ID : rot ? P_ROT : P_GEN;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---------------------------------------------------------------------------
// streaming launches

int sm_count()
{
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <typename T, int NT>
int launch_stream(const LevelC<T, NT> &L, const StreamArgs<T> &a, int nu, int kind, int perm, bool sparse,
                  cudaStream_t s)
{
    if (nu < 0 || nu > 4) return fail(TMG_E_UNSUPPORTED, "fused passes support nu <= 4 (got %d)", nu);
    const int rc = stream_launch<T, NT>(L, a, nu, kind, perm, sparse, s);
    if (rc < 0) return fail(TMG_E_UNSUPPORTED, "no stream kernel for nu=%d kind=%d", nu, kind);
    if (rc > 0) return fail(rc, "stream_kernel<nt=%d,nu=%d,kind=%d>: %s", NT, nu, kind,
                            cudaGetErrorString((cudaError_t)rc));
    char what[96];
    snprintf(what, sizeof what, "stream_kernel<nt=%d,nu=%d,kind=%d> n=%lld flags=%d", NT, nu, kind, a.n, a.flags);
    CK_LAUNCH(what);
    trace_mark(what, s);
    return 0;
}

// rows (of w slabs) per warp chunk: enough warps to fill the GPU several
// times over, a multiple of the norm leaf, and long enough to amortise the
// warm-up row
int chunk_rows(long long n, long long batch, int leaf_rows, int w, int stage)
{
    const long long rows = (n + w - 1) / w;
    // TMG_CHUNK_WAVES / TMG_CHUNK_MIN / TMG_CHUNK_MAX: tuning overrides (default 1 wave of
    // 16 resident warps per SM, chunks of 2..64 rows; with the two-level
    // kernels 1 wave is 2 % faster than 2 on config 2 p_t=3, neutral elsewhere)
    static int waves = -1, rmin = -1, rmax = -1;
    if (waves < 0) {
        const char *e = getenv("TMG_CHUNK_WAVES");
        waves = e ? std::max(1, atoi(e)) : 1;
        const char *m = getenv("TMG_CHUNK_MIN");
        rmin = m ? std::max(1, atoi(m)) : 2;
        const char *x = getenv("TMG_CHUNK_MAX");
        rmax = x ? std::max(rmin, atoi(x)) : 64;  // 32-96 measured ~1 % better than 128 on config 3
    }
    const long long target_warps = (long long)sm_count() * 16 * waves;
    // rounded UP: rounded down, 16384 rows over 2368 warps gave 6-row chunks,
    // 2731 of them -- a second, nearly empty wave (config 2's finest pass:
    // 36 -> 27 us with 8-row chunks)
    long long r = (rows * batch + target_warps - 1) / std::max(1LL, target_warps);
    r = std::max((long long)rmin, std::min((long long)rmax, r));
    // a multiple of the ring stage (stage_slabs) and of the norm leaf
    const int g = stage / w;
    const int q = std::lcm(g, std::max(leaf_rows, 1));
    r = ((r + q - 1) / q) * q;
    return (int)std::max<long long>(r, 1);
}

template <typename T, int NT> StreamArgs<T> stream_args(long long n, long long batch, int leaf_rows)
{
    constexpr int w = 32 * slabs_per_lane<T, NT>();
    StreamArgs<T> a;
    memset(&a, 0, sizeof a);
    a.n = n;
    a.batch = (int)batch;
    a.rows_per_chunk = chunk_rows(n, batch, leaf_rows, w, stage_slabs<T, NT>());
    a.chunks = ((n + w - 1) / w + a.rows_per_chunk - 1) / a.rows_per_chunk;
    a.leaf_rows = leaf_rows > 0 ? leaf_rows : 1;
    return a;
}

template <typename T, int NT> bool tma_ok(const StreamArgs<T> &a, bool prolong)
{
    const long long rowbytes = a.n * NT * (long long)sizeof(T);
    if (rowbytes & 15) return false;  // every problem base 16-byte aligned
    if (!aligned16(a.f)) return false;
    if (a.u_in && !aligned16(a.u_in)) return false;
    if (prolong) {
        if (((a.n / 2) * NT * (long long)sizeof(T)) & 15) return false;
        if (!aligned16(a.uc)) return false;
    }
    return true;
}

// numpy pairwise leaf structure of an n-vector: n = m * 2^k with the recursion
// splitting exactly in halves down to leaves of m <= 128 values; the leaf path
// of the streaming kernels needs whole rows of w slabs per leaf
int leaf_rows_for(long long n, int w)
{
    long long m = n;
    while (m > 128) {
        if (m % 2 || (m / 2) % 8) return 0;
        m /= 2;
    }
    if (m % w) return 0;
    return (int)(m / w);
}

// ---------------------------------------------------------------------------
// the plan

struct PlanBase {
    virtual ~PlanBase() {}
    virtual int cycles(const void *f, void *u, int n_cycles, cudaStream_t s) = 0;
    virtual int solve(const void *f, void *u, const double *floor_, double eps, int max_iters,
                      cudaStream_t s) = 0;
    virtual int solve_host(const void *f, const void *u0, void *u_out, const double *floor_, double eps,
                           int max_iters) = 0;
    virtual int stats(int32_t *it, double *norms, int32_t *conv) const = 0;
    virtual int info(int32_t *kpc, int32_t *sl, int32_t *tl) const = 0;
    virtual int solve_host_stream(int nb, const void *const *f, void *const *u, const double *floor_, double eps,
                                  int max_iters, int32_t *it, double *norms, int32_t *conv) = 0;
};

}  // namespace

struct tmg_plan {
    std::unique_ptr<PlanBase> impl;
};

namespace {

template <typename T, int NT, bool SP> struct Plan : PlanBase {
    static constexpr int ROWW = 32 * slabs_per_lane<T, NT>();  // slabs per streaming row
    int depth = 0;
    long long B = 0;
    tmg_plan_opts o{};
    std::vector<long long> n;
    std::vector<LevelC<T, NT>> L;
    std::vector<int> pk;  // LU permutation pattern per level
    LevelC<T, NT> *d_levels = nullptr;
    std::vector<T *> uA, uB, fl, halo;
    T *halo0_alt = nullptr;  // second finest-level halo buffer (K_UP2DOWN alternates them)
    T *fl1_alt = nullptr;    // second level-1 right-hand side (vertical fusion alternates them)
    bool up2 = false;  // up passes recompute the pre-sweeps (nu1 == nu2): no stored pre-smoothed u
    int tl = 0;                 // first tail level
    bool tail_smem = true;
    size_t tail_smem_bytes = 0;
    long long store_elems = 0;
    T *gstore = nullptr;
    TailArgs<T, NT> targ{};
    unsigned long long *d_trace = nullptr;
    // norms
    int leaf_rows0 = 0;
    long long nleaves = 0;
    double *leaves = nullptr, *sqbuf = nullptr;
    ProbState *d_st = nullptr;
    double *d_hist = nullptr, *d_floor = nullptr;
    int *d_active = nullptr, *d_any = nullptr, *h_any = nullptr;
    int hist_stride = 0;
    std::vector<int> h_it, h_conv;
    std::vector<double> h_hist;
    int last_max_iters = 0;
    int kernels_per_cycle = 0;
    // graph cache
    cudaGraphExec_t gexec = nullptr;
    const void *g_f = nullptr;
    void *g_u = nullptr;
    bool g_norm = false;
    double g_eps = 0.0;
    cudaStream_t ps = nullptr;  // private stream: graph capture never touches the caller's
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;

    ~Plan() override
    {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (sexec) cudaGraphExecDestroy(sexec);
        if (ps) cudaStreamDestroy(ps);
        if (ev_in) cudaEventDestroy(ev_in);
        if (ev_out) cudaEventDestroy(ev_out);
        for (auto p : uA) cudaFree(p);
        for (auto p : uB) cudaFree(p);
        for (auto p : fl) cudaFree(p);
        for (auto p : halo) cudaFree(p);
        cudaFree(halo0_alt);
        cudaFree(fl1_alt);
        cudaFree(d_levels);
        if (d_trace) {
            std::vector<unsigned long long> tr(10 * MAXLEV);
            cudaMemcpy(tr.data(), d_trace, sizeof(unsigned long long) * tr.size(), cudaMemcpyDeviceToHost);
            const char *names[10] = {"down", "-", "up", "coarse", "norm", "down.enter", "down.loads",
                                     "down.compute", "down.stores", "down.leave"};
            for (int k = 0; k < 10; ++k)
                for (int l = 0; l < MAXLEV; ++l)
                    if (tr[k * MAXLEV + l]) fprintf(stderr, "tail-trace %s L%d %llu\n", names[k], l, tr[k * MAXLEV + l]);
            cudaFree(d_trace);
        }
        cudaFree(d_fh);
        cudaFree(d_uh);
        if (ev_h2d) cudaEventDestroy(ev_h2d);
        for (cudaStream_t st : {cs_in, cs_out, cs_cmp[0], cs_cmp[1], cs_cmp[2], cs_cmp[3]})
            if (st) cudaStreamDestroy(st);
        cudaFree(gstore);
        cudaFree(leaves);
        cudaFree(sqbuf);
        cudaFree(d_st);
        cudaFree(d_hist);
        cudaFree(d_floor);
        cudaFree(d_active);
        cudaFree(d_any);
        if (h_any) cudaFreeHost(h_any);
        if (hp_floor) cudaFreeHost(hp_floor);
        if (hp_init) cudaFreeHost(hp_init);
        if (hp_st) cudaFreeHost(hp_st);
        if (hp_hist) cudaFreeHost(hp_hist);
        if (ev_done) cudaEventDestroy(ev_done);
        if (ev_small_in) cudaEventDestroy(ev_small_in);
        if (ev_solved) cudaEventDestroy(ev_solved);
    }

    size_t fixed_smem() const { return tail_fixed_smem<T, NT>(depth - tl); }

    // multi: lv holds batch x nl descriptors -- a different operator per
    // problem (same level sizes); only whole-problem-in-one-CTA plans
    int init(const tmg_level_desc *lv, int nl, long long batch, const tmg_plan_opts &opts, bool multi = false)
    {
        depth = nl;
        B = batch;
        o = opts;
        descs.assign(lv, lv + nl);
        if (o.gamma == 0) o.gamma = 1;
        if (o.gamma < 1 || o.gamma > 3)
            return fail(TMG_E_ARG, "gamma (cycle kind) must be 1 (V), 2 (W) or 3 (F), got %d", o.gamma);
        for (int l = 0; l < nl; ++l) {
            n.push_back(lv[l].n_slabs);
            L.push_back(make_level<T, NT>(lv[l]));
        }
        for (int l = 0; l + 1 < nl; ++l)
            if (n[l + 1] != n[l] / 2 || n[l] % 2)
                return fail(TMG_E_ARG, "level %d: %lld slabs does not coarsen to %lld", l, n[l], n[l + 1]);
        CK(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
        if (multi) {
            std::vector<LevelC<T, NT>> all;
            for (long long b = 0; b < batch; ++b)
                for (int l = 0; l < nl; ++l) {
                    if (lv[b * nl + l].n_slabs != n[l] || lv[b * nl + l].n_t != NT)
                        return fail(TMG_E_ARG, "problem %lld level %d: sizes differ from problem 0", b, l);
                    all.push_back(make_level<T, NT>(lv[b * nl + l]));
                }
            CK(cudaMalloc(&d_levels, sizeof(LevelC<T, NT>) * all.size()));
            CK(cudaMemcpy(d_levels, all.data(), sizeof(LevelC<T, NT>) * all.size(), cudaMemcpyHostToDevice));
        } else {
            CK(cudaMalloc(&d_levels, sizeof(LevelC<T, NT>) * nl));
            CK(cudaMemcpy(d_levels, L.data(), sizeof(LevelC<T, NT>) * nl, cudaMemcpyHostToDevice));
        }

        // choose the tail: the longest suffix of small levels that fits in smem
        const size_t smem_cap = 200 * 1024;
        // measured on config 2 (N = 2^20): 1024 (n_t <= 2) and 512 (n_t >= 3) beat 2048 / 1024 by 5-6 %
        long long tail_max = o.tail_max_slabs > 0 ? o.tail_max_slabs : (NT <= 2 ? 1024 : 512);
        auto store_of = [&](int l0) {  // per level u, f and the pre-smoothed iterate
            long long e = 0;
            for (int l = l0; l < nl; ++l) e += 3 * n[l] * NT;
            return e + (e & 1);
        };
        auto smem_of = [&](int l0) {
            return tail_fixed_smem<T, NT>(nl - l0) + sizeof(T) * store_of(l0) +
                   (l0 == 0 ? sizeof(double) * n[0] : 0);
        };
        // small problems (config 1) and per-problem-operator batches run whole
        // in one CTA: one launch per solve
        if (o.tail_max_slabs <= 0 && (multi || n[0] <= (NT <= 2 ? 2048 : 1024)) && smem_of(0) <= smem_cap)
            tail_max = std::max(tail_max, n[0]);
        tl = nl - 1;
        for (int l = nl - 2; l >= 0; --l) {
            if (n[l] <= tail_max && smem_of(l) <= smem_cap) tl = l;
            else break;
        }
        store_elems = store_of(tl);
        tail_smem = smem_of(tl) <= smem_cap;
        tail_smem_bytes = tail_smem ? smem_of(tl) : fixed_smem();
        if (!tail_smem)
            CK(cudaMalloc(&gstore, (sizeof(T) * store_elems + sizeof(double) * (tl == 0 ? n[0] : 0)) * B + 64));
        CK(((cudaError_t)tail_prepare<T, NT>(SP, tail_smem_bytes)));
        for (int l = 0; l < nl; ++l) pk.push_back(perm_kind(lv[l]));

        uA.assign(nl, nullptr);
        uB.assign(nl, nullptr);
        fl.assign(nl, nullptr);
        for (int l = 0; l <= tl && l < nl; ++l) {
            const size_t bytes = sizeof(T) * n[l] * NT * B;
            if (l > 0) {
                CK(cudaMalloc(&uA[l], bytes));
                CK(cudaMalloc(&fl[l], bytes));
            }
            if (l < tl) CK(cudaMalloc(&uB[l], bytes));
        }
        // norm machinery (finest level)
        leaf_rows0 = leaf_rows_for(n[0], ROWW);
        up2 = SP && o.nu1 == o.nu2 && o.nu1 >= 1 && o.nu1 <= 4 && !getenv("TMG_NO_UP2");
        halo.assign(nl, nullptr);
        if (up2) {
            for (int l = 0; l < tl; ++l) {
                StreamArgs<T> a = level_args(l);
                CK(cudaMalloc(&halo[l], sizeof(T) * (size_t)B * a.chunks * ROWW * NT + 16));
                if (l == 0) CK(cudaMalloc(&halo0_alt, sizeof(T) * (size_t)B * a.chunks * ROWW * NT + 16));
            }
            if (tl >= 2 && sizeof(T) == 8 && n[0] % (2 * ROWW) == 0 && pair_rows_ok())
                CK(cudaMalloc(&fl1_alt, sizeof(T) * (size_t)B * n[1] * NT + 16));
        }
        if (leaf_rows0) {
            nleaves = n[0] / ((long long)ROWW * leaf_rows0);
            CK(cudaMalloc(&leaves, sizeof(double) * nleaves * B));
        }
        CK(cudaMalloc(&sqbuf, sizeof(double) * n[0] * B));
        if (getenv("TMG_POISON")) {
            // debug: NaN-fill every scratch buffer so a read-before-write shows
            for (int l = 0; l < tl; ++l)
                if (halo[l]) {
                    StreamArgs<T> a = level_args(l);
                    CK(cudaMemset(halo[l], 0xff, sizeof(T) * (size_t)B * a.chunks * ROWW * NT));
                }
            if (leaves) CK(cudaMemset(leaves, 0xff, sizeof(double) * nleaves * B));
        }
        CK(cudaMalloc(&d_st, sizeof(ProbState) * B));
        CK(cudaMalloc(&d_floor, sizeof(double) * B));
        CK(cudaMalloc(&d_active, sizeof(int) * B));
        CK(cudaMalloc(&d_any, sizeof(int) * 4));
        CK(cudaHostAlloc(&h_any, sizeof(int) * 4, cudaHostAllocDefault));

        targ = TailArgs<T, NT>{};
        targ.levels = d_levels;
        targ.l0 = tl;
        targ.depth = nl;
        long long off = 0;
        for (int l = tl; l < nl; ++l) {
            targ.n[l] = n[l];
            targ.off[l] = off;
            off += 3 * n[l] * NT;
        }
        targ.store_elems = store_elems;
        targ.gstore = gstore;
        targ.in_smem = tail_smem;
        targ.nu1 = o.nu1;
        targ.nu2 = o.nu2;
        targ.gamma = o.gamma;
        targ.dot_variant = o.dot_variant;
        targ.levels_stride = multi ? nl : 0;
        if (multi && tl != 0)
            return fail(TMG_E_UNSUPPORTED, "per-problem operators need the whole problem in one CTA "
                                           "(at most %lld slabs here)", tail_max);
        targ.trace = nullptr;
        if (getenv("TMG_TAIL_TRACE")) {
            CK(cudaMalloc(&d_trace, sizeof(unsigned long long) * 10 * MAXLEV));
            CK(cudaMemset(d_trace, 0, sizeof(unsigned long long) * 10 * MAXLEV));
            targ.trace = d_trace;
        }
        // coarsest solve: serial forward substitution (bitwise) unless asked
        // for the scan, or "auto" and the coarsest level is too long for one thread
        targ.coarse_scan = L[nl - 1].scan_ok && (o.coarse == 1 || (o.coarse == 2 && n[nl - 1] > 16384));
        return 0;
    }

    // one cycle's launches (multigrid.py:263-330 for gamma = 1)
    // chunking of level l, identical for its down and up passes (the halo
    // and the warm-up rows must line up); the finest level follows the norm leaves
    StreamArgs<T> level_args(int l) const
    {
        return stream_args<T, NT>(n[l], B, l == 0 && leaf_rows0 > 0 ? leaf_rows0 : 1);
    }

    // down pass of level l (nu1 sweeps + residual + restriction); with_norm:
    // also the numpy-order norm leaves of its INPUT (finest level, solve mode)
    int enqueue_down(int l, const void *f0, void *u0, bool first_visit, bool with_norm, cudaStream_t s,
                     bool f_by_parity = false)
    {
        const T *fL = l == 0 ? (const T *)f0 : fl[l];
        StreamArgs<T> a = up2 ? level_args(l) : stream_args<T, NT>(n[l], B, with_norm ? leaf_rows0 : 1);
        a.f = fL;
        if (f_by_parity) {  // vertical fusion: level 1's f alternates by cycle parity
            a.f_alt = fl1_alt;
            a.iters = &d_st[0].iters;
            a.iters_stride = (int)(sizeof(ProbState) / sizeof(int));
        }
        const bool zero = (l > 0) && first_visit;
        a.u_in = l == 0 ? (const T *)u0 : (zero ? nullptr : uA[l]);
        a.u_out = up2 ? nullptr : uB[l];
        a.halo = up2 ? halo[l] : nullptr;
        a.fc = fl[l + 1];
        a.active = d_active;
        a.flags = SF_RESTRICT | SF_WRITE_U | (zero ? SF_ZERO_GUESS : 0);
        if (with_norm) {
            a.flags |= SF_NORM_LEAF;
            a.leaf_out = leaves;
        }
        if (tma_ok<T, NT>(a, false)) a.flags |= SF_TMA;
        CKR((launch_stream<T, NT>(L[l], a, o.nu1, with_norm ? K_DOWNNORM : K_DOWN, pk[l], SP, s)));
        ++kernels_per_cycle;
        return 0;
    }

    // coarse-grid correction of level l and its up pass (norm_up: the up pass
    // also produces the norm of its output -- used when the down pass cannot)
    // ckind: this level's cycle (1 V, 2 W, 3 F; 0 = the plan's): a W visits
    // level l+1 twice with W-cycles, an F with an F-cycle then a V-cycle (the
    // oracle's tmo_cycle_rec); the coarsest level is solved once per visit
    static int cycle_visits(int kind) { return kind == 1 ? 1 : 2; }
    static int child_kind(int kind, int visit) { return (kind == 3 && visit > 0) ? 1 : kind; }
    int enqueue_rest(int l, const void *f0, void *u0, bool norm_up, cudaStream_t s, bool first_visit = true,
                     bool fuse_next_down = false, bool skip_up = false, bool child_skip_down = false,
                     int ckind = 0)
    {
        if (ckind == 0) ckind = o.gamma;
        const T *fL = l == 0 ? (const T *)f0 : fl[l];
        const bool pr = !skip_up && pair_up(l, first_visit, ckind);
        if (l + 1 == tl) {
            TailArgs<T, NT> t = targ;
            t.f_in = fl[tl];
            t.u_in = nullptr;
            t.u_out = uA[tl];
            t.full = 0;
            t.n_cycles = (tl == depth - 1) ? 1 : cycle_visits(ckind);
            t.gamma = ckind;
            t.each_kind = 0;
            t.active = d_active;
            CK(((cudaError_t)tail_launch<T, NT>(t, SP, (unsigned)B, tail_smem_bytes, s)));
            CK_LAUNCH("tail_kernel");
            trace_mark("tail_kernel", s);
            ++kernels_per_cycle;
        } else {
            for (int g = 0; g < cycle_visits(ckind); ++g)
                CKR(enqueue_level(l + 1, f0, u0, g == 0, false, s, pr, child_skip_down && g == 0,
                                  child_kind(ckind, g)));
        }
        if (skip_up) return 0;  // this level's up pass runs inside the next finer level's pass
        if (pr) {
            // coarse pair: level l+1's up pass in shared memory feeding level l's
            StreamArgs<T> a = level_args(l);
            a.f = fl[l];
            a.u_out = uA[l];
            a.uc = uA[l + 2];
            a.f1 = fl[l + 1];
            a.active = d_active;
            a.flags = SF_PROLONG | SF_WRITE_U | SF_ZERO_GUESS;
            StreamArgs<T> a1 = a;
            a1.n = n[l + 1];
            const int rc = stream_v_launch<T, NT>(L[l], L[l + 1], a, a1, o.nu2, pk[l], false, s);
            if (rc < 0) return fail(TMG_E_UNSUPPORTED, "coarse pair kernel unavailable");
            if (rc > 0) return fail(rc, "stream_kernel_v pair: %s", cudaGetErrorString((cudaError_t)rc));
            char what[96];
            snprintf(what, sizeof what, "stream_kernel_v pair n=%lld+%lld", n[l], n[l + 1]);
            CK_LAUNCH(what);
            trace_mark(what, s);
            ++kernels_per_cycle;
            return 0;
        }
        if (up2 && (!norm_up || (l == 0 && norm_up2()))) {
            // prolong-add + post-sweeps, the pre-sweeps recomputed from the
            // level's original iterate (read in place; warm-ups from the halo);
            // at the finest level of a solve also the norm leaves of the result
            StreamArgs<T> a = level_args(l);
            const bool zero = (l > 0) && first_visit;
            a.f = fL;
            a.u_in = l == 0 ? (const T *)u0 : (zero ? nullptr : uA[l]);
            a.uc = uA[l + 1];
            a.u_out = l == 0 ? (T *)u0 : uA[l];
            a.halo = halo[l];
            a.active = d_active;
            a.flags = SF_PROLONG | SF_WRITE_U | (zero ? SF_ZERO_GUESS : 0);
            if (norm_up || fuse_next_down) {
                a.flags |= SF_NORM_LEAF;
                a.leaf_out = leaves;
            }
            int kind = norm_up ? K_UP2NORM : K_UP2;
            if (fuse_next_down) {
                // ... and the next cycle's finest down pass on the same rows
                kind = K_UP2DOWN;
                a.flags |= SF_RESTRICT;
                a.fc = fl[1];
                a.halo_alt = halo0_alt;
                a.iters = &d_st[0].iters;
                a.iters_stride = (int)(sizeof(ProbState) / sizeof(int));
            }
            if (tma_ok<T, NT>(a, true)) a.flags |= SF_TMA;
            CKR((launch_stream<T, NT>(L[l], a, o.nu2, kind, pk[l], SP, s)));
            ++kernels_per_cycle;
            return 0;
        }
        const bool leaf = norm_up && leaf_rows0 > 0;
        StreamArgs<T> a = stream_args<T, NT>(n[l], B, leaf ? leaf_rows0 : 1);
        a.f = fL;
        a.u_in = uB[l];
        a.uc = uA[l + 1];
        a.u_out = l == 0 ? (T *)u0 : uA[l];
        a.active = d_active;
        a.flags = SF_PROLONG | SF_WRITE_U;
        if (norm_up) {
            if (leaf) { a.flags |= SF_NORM_LEAF; a.leaf_out = leaves; }
            else { a.flags |= SF_NORM_SQ; a.sq_out = sqbuf; }
        }
        if (tma_ok<T, NT>(a, true)) a.flags |= SF_TMA;
        const int kind = norm_up ? (leaf ? K_UPNORM : K_GENERIC) : K_UP;
        CKR((launch_stream<T, NT>(L[l], a, o.nu2, kind, pk[l], SP, s)));
        ++kernels_per_cycle;
        return 0;
    }

    int enqueue_level(int l, const void *f0, void *u0, bool first_visit, bool norm, cudaStream_t s,
                      bool skip_up = false, bool skip_down = false, int ckind = 0)
    {
        if (up2 && norm && !(l == 0 && norm_up2())) {
            // the up pass cannot produce the norm: take it in a separate pass
            CKR(enqueue_down(l, f0, u0, first_visit, false, s));
            CKR(enqueue_rest(l, f0, u0, false, s, first_visit, false, false, false, ckind));
            return enqueue_norm_pass(f0, u0, s);
        }
        bool dp = false;
        if (!skip_down) {
            dp = pair_down(l, first_visit);
            if (dp) CKR(enqueue_down_pair(l, s, false));  // levels l and l+1
            else CKR(enqueue_down(l, f0, u0, first_visit, false, s));
        }
        return enqueue_rest(l, f0, u0, norm, s, first_visit, false, skip_up, dp, ckind);
    }

    // standalone ||f - L u|| pass at the finest level (r0 / generic sizes)
    int enqueue_norm_pass(const void *f, void *u, cudaStream_t s)
    {
        const bool leaf = leaf_rows0 > 0;
        StreamArgs<T> a = stream_args<T, NT>(n[0], B, leaf ? leaf_rows0 : 1);
        a.f = (const T *)f;
        a.u_in = (const T *)u;
        a.active = d_active;
        a.flags = leaf ? SF_NORM_LEAF : SF_NORM_SQ;
        a.leaf_out = leaves;
        a.sq_out = sqbuf;
        if (tma_ok<T, NT>(a, false)) a.flags |= SF_TMA;
        CKR((launch_stream<T, NT>(L[0], a, 0, K_GENERIC, P_GEN, SP, s)));
        ++kernels_per_cycle;
        return 0;
    }

    // where the stopping norm comes from when it has numpy's leaf structure:
    // the NEXT cycle's finest down pass (K_DOWNNORM: its first sweep's
    // residual, default; one speculative down pass per solve), or the finest
    // up pass (K_UP2NORM: an extra residual of its output; TMG_NORM_UP=1).
    // Measured on config 3: 128.3 vs 131.1 ms per solve, config 2 ~1-2 %.
    bool norm_up2() const { return up2 && leaf_rows0 > 0 && SP && norm_up_env(); }
    bool norm_in() const { return leaf_rows0 > 0 && SP && !norm_up2(); }
    // pairs with one-slab lanes (n_t >= 3 fp64): TMG_PAIR_P1=0 disables
    static bool pair_rows_ok()
    {
        if (ROWW == 64) return true;
        static int v = -1;
        if (v < 0) {
            const char *e = getenv("TMG_PAIR_P1");
            v = (e && *e == '0') ? 0 : 1;
        }
        return v == 1;
    }
    // coarse pairs (level l+1's up pass inside level l's, both from the zero
    // guess; V-cycles only: measured on config 4 F/W with nu = 2 the pairs
    // cost 10-20 % there; TMG_NO_VPAIR=1 disables)
    bool pair_up(int l, bool first_visit, int ckind) const
    {
        static int v = -1;
        if (v < 0) {
            const char *e = getenv("TMG_NO_VPAIR");
            v = (e && *e && *e != '0') ? 0 : 1;
        }
        return v == 1 && up2 && SP && ckind == 1 && o.gamma == 1 && o.nu1 <= 2 && first_visit && l >= 1 && l + 1 < tl && pair_rows_ok() &&
               sizeof(T) == 8 && n[l] % (2 * ROWW) == 0 && pk[l] == pk[l + 1] && aligned16(fl[l]) &&
               aligned16(fl[l + 1]) && aligned16(uA[l]) && aligned16(uA[l + 2]);
    }
    // coarse down pairs (level l's down pass feeding level l+1's through shared
    // memory, both from the zero guess; V-cycles only, see pair_up;
    // TMG_NO_DPAIR=1 disables)
    bool pair_down(int l, bool first_visit) const
    {
        static int v = -1;
        if (v < 0) {
            const char *e = getenv("TMG_NO_DPAIR");
            v = (e && *e && *e != '0') ? 0 : 1;
        }
        return v == 1 && up2 && SP && o.gamma == 1 && o.nu1 <= 2 && first_visit && l >= 1 && l + 1 < tl && pair_rows_ok() &&
               sizeof(T) == 8 && n[l] % (2 * ROWW) == 0 && pk[l] == pk[l + 1] && aligned16(fl[l]) &&
               aligned16(fl[l + 1]) && aligned16(fl[l + 2]) && (l != 1 || !fl1_alt || aligned16(fl1_alt));
    }
    int enqueue_down_pair(int l, cudaStream_t s, bool f_by_parity)
    {
        StreamArgs<T> a = level_args(l);
        a.f = fl[l];
        if (f_by_parity) {
            a.f_alt = fl1_alt;
            a.iters = &d_st[0].iters;
            a.iters_stride = (int)(sizeof(ProbState) / sizeof(int));
        }
        a.fc = fl[l + 1];
        a.active = d_active;
        a.flags = SF_RESTRICT | SF_ZERO_GUESS;
        StreamArgs<T> a1 = a;
        a1.n = n[l + 1];
        a1.fc = fl[l + 2];
        const int rc = stream_d_launch<T, NT>(L[l], L[l + 1], a, a1, o.nu1, pk[l], s);
        if (rc < 0) return fail(TMG_E_UNSUPPORTED, "coarse down pair unavailable");
        if (rc > 0) return fail(rc, "stream_kernel_d: %s", cudaGetErrorString((cudaError_t)rc));
        char what[96];
        snprintf(what, sizeof what, "stream_kernel_d pair n=%lld+%lld", n[l], n[l + 1]);
        CK_LAUNCH(what);
        trace_mark(what, s);
        ++kernels_per_cycle;
        return 0;
    }
    // vertical fusion (level-1 up pass inside the fused finest pass; TMG_NO_VFUSE=1 disables)
    bool vfuse(const void *f, const void *u) const
    {
        static int v = -1;
        if (v < 0) {
            const char *e = getenv("TMG_NO_VFUSE");
            v = (e && *e && *e != '0') ? 0 : 1;
        }
        // one-slab lanes: only in the bandwidth regime (measured: B=16 x 2^22
        // p_t=2 -3.5 %, latency-bound 2^20 +3.5 %)
        const bool big = ROWW == 64 || (long long)B * n[0] >= (1LL << 22);
        return v == 1 && big && fuse_up_down() && fl1_alt && o.gamma == 1 && o.nu1 <= 2 && tl >= 2 && pk[0] == pk[1] &&
               aligned16(f) && aligned16(u) && aligned16(fl[1]) && aligned16(fl1_alt) && aligned16(uA[2]);
    }
    // K_UP2DOWN (default with the up2 scheme; TMG_NO_FUSE=1 keeps the two passes)
    bool fuse_up_down() const
    {
        static int v = -1;
        if (v < 0) {
            const char *e = getenv("TMG_NO_FUSE");
            v = (e && *e && *e != '0') ? 0 : 1;
        }
        return up2 && v == 1 && tl >= 1;
    }
    static bool norm_up_env()
    {
        static int v = -1;
        if (v < 0) {
            const char *e = getenv("TMG_NORM_UP");
            v = (e && *e && *e != '0') ? 1 : 0;
        }
        return v == 1;
    }

    int enqueue_finalize(int mode, double eps, cudaStream_t s, cudaGraphConditionalHandle h = 0,
                         bool use_h = false)
    {
        if (leaf_rows0)
            CK(launch_pdl(finalize_leaves_kernel, dim3((unsigned)B), dim3(1024), 0, s, (const double *)leaves,
                          nleaves, d_st, d_hist, hist_stride, (const double *)d_floor, eps, mode));
        else
            finalize_sq_kernel<<<(unsigned)B, 1024, 0, s>>>(sqbuf, n[0], d_st, d_hist, hist_stride, d_floor,
                                                           eps, mode, nullptr);
        CK_LAUNCH("finalize");
        trace_mark("finalize", s);
        CK(launch_pdl(set_active_kernel, dim3(1), dim3(256), 0, s, (const ProbState *)d_st, d_active, d_any,
                      (int)B, h, use_h ? 1 : 0));
        CK_LAUNCH("set_active");
        trace_mark("set_active", s);
        kernels_per_cycle += 2;
        return 0;
    }

    int enqueue_cycle(const void *f, void *u, bool norm, double eps, cudaStream_t s,
                      cudaGraphConditionalHandle h = 0, bool use_h = false)
    {
        kernels_per_cycle = 0;
        if (norm && norm_in() && vfuse(f, u)) {
            // vertical fusion: level 1's down pass (f_1 by parity), the coarser
            // levels, then ONE finest pass = level-1 up pass + finest up pass +
            // the next cycle's finest down pass
            const bool dp1 = pair_down(1, true);
            if (dp1) CKR(enqueue_down_pair(1, s, true));
            else CKR(enqueue_down(1, f, u, true, false, s, true));
            CKR(enqueue_rest(1, f, u, false, s, true, false, true, dp1));
            StreamArgs<T> a = level_args(0);
            a.f = (const T *)f;
            a.u_in = (const T *)u;
            a.u_out = (T *)u;
            a.uc = uA[2];
            a.f1 = fl[1];
            a.f1_alt = fl1_alt;
            a.halo = halo[0];
            a.halo_alt = halo0_alt;
            a.iters = &d_st[0].iters;
            a.iters_stride = (int)(sizeof(ProbState) / sizeof(int));
            a.active = d_active;
            a.leaf_out = leaves;
            a.flags = SF_PROLONG | SF_WRITE_U | SF_RESTRICT | SF_NORM_LEAF | SF_TMA;
            StreamArgs<T> a1 = a;
            a1.n = n[1];
            a1.flags = SF_PROLONG | SF_WRITE_U | SF_ZERO_GUESS;
            const int rc = stream_v_launch<T, NT>(L[0], L[1], a, a1, o.nu2, pk[0], true, s);
            if (rc < 0) return fail(TMG_E_UNSUPPORTED, "vertical fusion unavailable");
            if (rc > 0) return fail(rc, "stream_kernel_v: %s", cudaGetErrorString((cudaError_t)rc));
            CK_LAUNCH("stream_kernel_v");
            trace_mark("stream_kernel_v (level-1 up + finest up + next finest down)", s);
            ++kernels_per_cycle;
        } else if (norm && norm_in() && fuse_up_down()) {
            // rest of this cycle; its finest up pass fused with the NEXT cycle's
            // finest down pass (whose first sweep yields ||f - L u||)
            CKR(enqueue_rest(0, f, u, false, s, true, true));
        } else if (norm && norm_in()) {
            // rest of this cycle, then the NEXT cycle's finest down pass, whose
            // first sweep yields ||f - L u|| of this cycle's result
            CKR(enqueue_rest(0, f, u, false, s));
            CKR(enqueue_down(0, f, u, true, true, s));
        } else {
            CKR(enqueue_level(0, f, u, true, norm, s));
        }
        if (norm) CKR(enqueue_finalize(1, eps, s, h, use_h));
        return 0;
    }

    // r0 = ||f - L u_init|| and the initial stopping state (multigrid.py:478-481)
    int enqueue_prefix(const void *f, void *u, double eps, cudaStream_t s, cudaGraphConditionalHandle h = 0,
                       bool use_h = false)
    {
        CK(cudaMemsetAsync(d_active, 0xff, sizeof(int) * B, s));
        if (norm_in()) CKR(enqueue_down(0, f, u, true, true, s));  // the first cycle's down pass
        else CKR(enqueue_norm_pass(f, u, s));
        return enqueue_finalize(0, eps, s, h, use_h);
    }

    // the whole solve as one graph: prefix, then a conditional while node
    // whose body is one cycle + finalize + set_active (which sets the condition)
    cudaGraphExec_t sexec = nullptr;
    const void *s_f = nullptr;
    void *s_u = nullptr;
    double s_eps = -1.0;
    int s_hist = -1;

    int build_solve_graph(const void *f, void *u, double eps)
    {
        if (sexec) { cudaGraphExecDestroy(sexec); sexec = nullptr; }
        cudaGraph_t g;
        CK(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
        CK(cudaStreamBeginCaptureToGraph(ps, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_prefix(f, u, eps, ps, h, true);
        cudaGraph_t tmp;
        cudaError_t ce = cudaStreamEndCapture(ps, &tmp);
        if (rc) { cudaGraphDestroy(g); return rc; }
        CK(ce);
        size_t nn = 0;
        CK(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn), leaves_;
        CK(cudaGraphGetNodes(g, nodes.data(), &nn));
        for (auto nd : nodes) {
            size_t nd_out = 0;
            CK(cudaGraphNodeGetDependentNodes(nd, nullptr, &nd_out));
            if (nd_out == 0) leaves_.push_back(nd);
        }
        cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cn;
        CK(cudaGraphAddNode(&cn, g, leaves_.data(), leaves_.size(), &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(ps, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        rc = enqueue_cycle(f, u, true, eps, ps, h, true);
        ce = cudaStreamEndCapture(ps, &tmp);
        if (rc) { cudaGraphDestroy(g); return rc; }
        CK(ce);
        CK(cudaGraphInstantiate(&sexec, g, 0));
        cudaGraphDestroy(g);
        s_f = f; s_u = u; s_eps = eps; s_hist = hist_stride;
        return 0;
    }

    int run_cycle(const void *f, void *u, bool norm, double eps, cudaStream_t s)
    {
        if (!o.use_graph || sync_debug() || event_trace()) return enqueue_cycle(f, u, norm, eps, s);
        if (!gexec || g_f != f || g_u != u || g_norm != norm || g_eps != eps) {
            if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            int rc = enqueue_cycle(f, u, norm, eps, s);
            cudaError_t ce = cudaStreamEndCapture(s, &g);
            if (rc) return rc;
            CK(ce);
            CK(cudaGraphInstantiate(&gexec, g, 0));
            cudaGraphDestroy(g);
            g_f = f; g_u = u; g_norm = norm; g_eps = eps;
        }
        CK(cudaGraphLaunch(gexec, s));
        return 0;
    }

    int enter(cudaStream_t user)
    {
        CK(cudaEventRecord(ev_in, user));
        CK(cudaStreamWaitEvent(ps, ev_in, 0));
        return 0;
    }
    int leave(cudaStream_t user)
    {
        CK(cudaEventRecord(ev_out, ps));
        CK(cudaStreamWaitEvent(user, ev_out, 0));
        return 0;
    }

    int cycles(const void *f, void *u, int nc, cudaStream_t user) override
    {
        CKR(enter(user));
        CKR(cycles_on(f, u, nc, ps));
        return leave(user);
    }
    int solve(const void *f, void *u, const double *floor_, double eps, int max_iters,
              cudaStream_t user) override
    {
        CKR(enter(user));
        CKR(solve_on(f, u, floor_, eps, max_iters, ps));
        return leave(user);
    }

    T *d_fh = nullptr, *d_uh = nullptr;  // device copies for the host-buffer entry point
    cudaEvent_t ev_h2d = nullptr;         // this sub-batch's inputs are on the device
    cudaStream_t cs_in = nullptr, cs_out = nullptr, cs_cmp[4] = {};  // host-buffer pipeline
    std::vector<tmg_level_desc> descs;   // kept to build sub-batch plans
    std::vector<std::unique_ptr<Plan>> subs;

    // host buffers in, solve, host buffer out, this plan's problems only
    int enqueue_host(const T *f, const T *u0, T *u_out, const double *floor_, double eps, int max_iters)
    {
        const size_t bytes = sizeof(T) * n[0] * NT * B;
        if (!d_fh) {
            CK(cudaMalloc(&d_fh, bytes));
            CK(cudaMalloc(&d_uh, bytes));
        }
        if (ev_done) CK(cudaEventSynchronize(ev_done));  // previous chunk's D2H finished
        CK(cudaMemcpyAsync(d_fh, f, bytes, cudaMemcpyHostToDevice, ps));
        if (u0) CK(cudaMemcpyAsync(d_uh, u0, bytes, cudaMemcpyHostToDevice, ps));
        else CK(cudaMemsetAsync(d_uh, 0, bytes, ps));
        CKR(enqueue_solve(d_fh, d_uh, floor_, eps, max_iters, ps));
        CK(cudaMemcpyAsync(u_out, d_uh, bytes, cudaMemcpyDeviceToHost, ps));
        CK(cudaEventRecord(ev_done, ps));
        return 0;
    }

    // one sub-batch of the pipelined host-buffer solve: H2D on cin, solve on
    // cmp (after the H2D), D2H on cout (after the solve); no host waits -- the
    // caller collects this sub-plan's previous sub-batch before reusing it
    int enqueue_host_async(const T *f, const T *u0, T *u_out, const double *floor_, double eps, int max_iters,
                           cudaStream_t cin, cudaStream_t cmp, cudaStream_t cout)
    {
        const size_t bytes = sizeof(T) * n[0] * NT * B;
        if (!d_fh) {
            CK(cudaMalloc(&d_fh, bytes));
            CK(cudaMalloc(&d_uh, bytes));
            CK(cudaEventCreateWithFlags(&ev_h2d, cudaEventDisableTiming));
        }
        CK(cudaMemcpyAsync(d_fh, f, bytes, cudaMemcpyHostToDevice, cin));
        if (u0) CK(cudaMemcpyAsync(d_uh, u0, bytes, cudaMemcpyHostToDevice, cin));
        else CK(cudaMemsetAsync(d_uh, 0, bytes, cin));
        CK(cudaEventRecord(ev_h2d, cin));
        CK(cudaStreamWaitEvent(cmp, ev_h2d, 0));
        // the small floor/stat copies ride on the copy streams (see enqueue_solve);
        // ev_done is recorded on cout after them
        CKR(enqueue_solve(d_fh, d_uh, floor_, eps, max_iters, cmp, cin, cout));
        CK(cudaMemcpyAsync(u_out, d_uh, bytes, cudaMemcpyDeviceToHost, cout));
        CK(cudaEventRecord(ev_done, cout));  // collect() waits for the solution on the host
        return 0;
    }

    // A stream of independent batches, each solved whole (the full-batch
    // graph) from the zero guess, pipelined ACROSS batches: while batch k is
    // solved, batch k+1 is copied in and batch k-1 copied out (copy-in,
    // compute and copy-out streams; three full-batch plans in rotation, each
    // with its own device buffers and graph), so the PCIe traffic hides under
    // the solves and a batch costs max(solve, H2D, D2H) in steady state.
    std::vector<std::unique_ptr<Plan>> ring;
    int solve_host_stream(int nb, const void *const *f, void *const *u, const double *floor_, double eps,
                          int max_iters, int32_t *it, double *norms, int32_t *conv) override
    {
        if (nb < 1) return fail(TMG_E_ARG, "need at least one batch");
        if (ring.empty()) {
            for (int k = 0; k < 3; ++k) {
                auto p = std::make_unique<Plan>();
                CKR(p->init(descs.data(), depth, B, o));
                ring.push_back(std::move(p));
            }
        }
        if (!cs_in) {
            CK(cudaStreamCreateWithFlags(&cs_in, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&cs_out, cudaStreamNonBlocking));
            for (int k = 0; k < 4; ++k) CK(cudaStreamCreateWithFlags(&cs_cmp[k], cudaStreamNonBlocking));
        }
        const int stride = max_iters + 1;
        auto gather = [&](int k) -> int {
            Plan &p = *ring[k % 3];
            CKR(p.collect());
            return p.stats(it ? it + (size_t)k * B : nullptr, norms ? norms + (size_t)k * B * stride : nullptr,
                           conv ? conv + (size_t)k * B : nullptr);
        };
        for (int k = 0; k < nb; ++k) {
            if (k >= 3) CKR(gather(k - 3));
            CKR(ring[k % 3]->enqueue_host_async((const T *)f[k], nullptr, (T *)u[k], floor_ + (size_t)k * B, eps,
                                                 max_iters, cs_in, cs_cmp[0], cs_out));
        }
        for (int k = std::max(0, nb - 3); k < nb; ++k) CKR(gather(k));
        return 0;
    }

    int solve_host(const void *f, const void *u0, void *u_out, const double *floor_, double eps,
                   int max_iters) override
    {
        // Pipelined sub-batches: copy-in and copy-out on their own streams, the
        // solves rotating over three compute streams (so one sub-batch's
        // latency-bound coarse levels overlap another's bandwidth-bound fine
        // levels), 6 sub-plans in rotation; the PCIe traffic of every sub-batch
        // but the first and last hides under the solves.
        // sub-batch count measured on config 3 (B = 64): 4 -> 163 ms, 8 -> 149 ms,
        // 16 -> 145 ms, 32 -> 168 ms per host-buffer solve
        int nch = tl == 0 ? 1 : (B >= 32 && B % 16 == 0) ? 16 : (B >= 16 && B % 8 == 0) ? 8
                : (B >= 8 && B % 4 == 0) ? 4 : 1;
        if (const char *e = getenv("TMG_HOST_CHUNKS")) {  // tuning override (must divide the batch)
            const int k = atoi(e);
            if (k >= 1 && B % k == 0 && tl > 0) nch = k;
        }
        if (nch == 1) {
            CKR(enqueue_host((const T *)f, (const T *)u0, (T *)u_out, floor_, eps, max_iters));
            return collect();
        }
        const long long bc = B / nch;
        static int ncs = -1;  // compute streams (TMG_HOST_STREAMS, 1..4)
        if (ncs < 0) {
            const char *e = getenv("TMG_HOST_STREAMS");
            ncs = e ? std::min(4, std::max(1, atoi(e))) : 3;  // measured: 1 -> 156, 2 -> 122.5, 3 -> 118, 4 -> 119 ms
        }
        const int nsub = std::min(nch, 2 * ncs);
        if ((int)subs.size() != nsub || subs[0]->B != bc) {
            subs.clear();
            for (int k = 0; k < nsub; ++k) {
                auto p = std::make_unique<Plan>();
                CKR(p->init(descs.data(), depth, bc, o));
                subs.push_back(std::move(p));
            }
        }
        if (!cs_in) {
            CK(cudaStreamCreateWithFlags(&cs_in, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&cs_out, cudaStreamNonBlocking));
            for (int k = 0; k < 4; ++k) CK(cudaStreamCreateWithFlags(&cs_cmp[k], cudaStreamNonBlocking));
        }
        const size_t per = (size_t)n[0] * NT * bc;
        last_max_iters = max_iters;
        CKR(ensure_hist(max_iters));
        h_hist.assign((size_t)hist_stride * B, 0.0);
        h_it.assign(B, 0);
        h_conv.assign(B, 0);
        auto gather = [&](int c) -> int {
            Plan &p = *subs[c % nsub];
            CKR(p.collect());
            for (long long b = 0; b < bc; ++b) {
                const long long g = c * bc + b;
                h_it[g] = p.h_it[b];
                h_conv[g] = p.h_conv[b];
                for (int k = 0; k <= max_iters; ++k)
                    h_hist[(size_t)g * hist_stride + k] = p.h_hist[(size_t)b * p.hist_stride + k];
            }
            return 0;
        };
        for (int c = 0; c < nch; ++c) {
            if (c >= nsub) CKR(gather(c - nsub));
            Plan &p = *subs[c % nsub];
            CKR(p.enqueue_host_async((const T *)f + c * per, u0 ? (const T *)u0 + c * per : nullptr,
                                     (T *)u_out + c * per, floor_ + c * bc, eps, max_iters, cs_in,
                                     cs_cmp[c % ncs], cs_out));
        }
        for (int c = std::max(0, nch - nsub); c < nch; ++c) CKR(gather(c));
        return 0;
    }

    int cycles_on(const void *f, void *u, int nc, cudaStream_t s)
    {
        if (tl == 0) {
            TailArgs<T, NT> t = targ;
            t.f_in = (const T *)f;
            t.u_in = (const T *)u;
            t.u_out = (T *)u;
            t.full = 0;
            t.n_cycles = nc;
            t.each_kind = 1;
            t.active = nullptr;
            CK(((cudaError_t)tail_launch<T, NT>(t, SP, (unsigned)B, tail_smem_bytes, s)));
            CK_LAUNCH("tail_kernel");
            return 0;
        }
        CK(cudaMemsetAsync(d_active, 0xff, sizeof(int) * B, s));  // all active (nonzero)
        for (int c = 0; c < nc; ++c) CKR(run_cycle(f, u, false, 0.0, s));
        return 0;
    }

    // pinned staging so a solve can be enqueued without host synchronisation
    double *hp_floor = nullptr;
    ProbState *hp_init = nullptr, *hp_st = nullptr;
    double *hp_hist = nullptr;
    cudaEvent_t ev_done = nullptr;

    int ensure_hist(int max_iters)
    {
        if (!hp_floor) {
            CK(cudaHostAlloc(&hp_floor, sizeof(double) * B, cudaHostAllocDefault));
            CK(cudaHostAlloc(&hp_init, sizeof(ProbState) * B, cudaHostAllocDefault));
            CK(cudaHostAlloc(&hp_st, sizeof(ProbState) * B, cudaHostAllocDefault));
            CK(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
        }
        if (max_iters + 1 > hist_stride) {
            cudaFree(d_hist);
            if (hp_hist) cudaFreeHost(hp_hist);
            hist_stride = max_iters + 1;
            CK(cudaMalloc(&d_hist, sizeof(double) * hist_stride * B));
            CK(cudaHostAlloc(&hp_hist, sizeof(double) * hist_stride * B, cudaHostAllocDefault));
            if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
        }
        return 0;
    }

    // enqueue a whole solve on stream s; the stopping state and the residual
    // histories land in pinned host buffers (collect() reads them)
    // s: the solve's kernels.  s_in / s_out (default s): the small copies of
    // the stopping floors in and the statistics out -- a pipelined caller puts
    // them on its copy streams, so the compute stream holds kernels only and a
    // copy engine busy with another batch's bulk transfer never delays a solve
    cudaEvent_t ev_small_in = nullptr, ev_solved = nullptr;
    int enqueue_solve(const void *f, void *u, const double *floor_, double eps, int max_iters, cudaStream_t s,
                      cudaStream_t s_in = nullptr, cudaStream_t s_out = nullptr)
    {
        if (max_iters < 1) return fail(TMG_E_ARG, "max_iters must be >= 1");
        CKR(ensure_hist(max_iters));
        if (ev_done) CK(cudaEventSynchronize(ev_done));  // the staging buffers are free again
        if (!ev_small_in) {
            CK(cudaEventCreateWithFlags(&ev_small_in, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ev_solved, cudaEventDisableTiming));
        }
        const cudaStream_t si = s_in ? s_in : s, so = s_out ? s_out : s;
        last_max_iters = max_iters;
        memcpy(hp_floor, floor_, sizeof(double) * B);
        for (long long b = 0; b < B; ++b) hp_init[b] = ProbState{0.0, 0, 1, max_iters, 0};
        CK(cudaMemcpyAsync(d_floor, hp_floor, sizeof(double) * B, cudaMemcpyHostToDevice, si));
        CK(cudaMemcpyAsync(d_st, hp_init, sizeof(ProbState) * B, cudaMemcpyHostToDevice, si));
        if (si != s) {
            CK(cudaEventRecord(ev_small_in, si));
            CK(cudaStreamWaitEvent(s, ev_small_in, 0));
        }
        if (tl == 0) {
            TailArgs<T, NT> t = targ;
            t.f_in = (const T *)f;
            t.u_in = (const T *)u;
            t.u_out = (T *)u;
            t.full = 1;
            t.eps = eps;
            t.floor_ = d_floor;
            t.max_iters = max_iters;
            t.hist = d_hist;
            t.st = d_st;
            t.active = nullptr;
            CK(((cudaError_t)tail_launch<T, NT>(t, SP, (unsigned)B, tail_smem_bytes, s)));
            CK_LAUNCH("tail_kernel");
        } else if (o.use_graph && !sync_debug() && !event_trace() && !getenv("TMG_NO_SOLVE_GRAPH")) {
            if (!sexec || s_f != f || s_u != u || s_eps != eps || s_hist != hist_stride)
                CKR(build_solve_graph(f, u, eps));
            CK(cudaGraphLaunch(sexec, s));
        } else {
            trace_mark("start", s);
            CKR(enqueue_prefix(f, u, eps, s));
            CK(cudaMemcpyAsync(h_any, d_any, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            int it = 0;
            while (h_any[0] && it < max_iters) {
                trace_mark("host round trip", s);  // keeps the sync gap out of the next kernel's time
                CKR(run_cycle(f, u, true, eps, s));
                CK(cudaMemcpyAsync(h_any, d_any, sizeof(int), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                ++it;
            }
        }
        if (so != s) {
            CK(cudaEventRecord(ev_solved, s));
            CK(cudaStreamWaitEvent(so, ev_solved, 0));
        }
        CK(cudaMemcpyAsync(hp_st, d_st, sizeof(ProbState) * B, cudaMemcpyDeviceToHost, so));
        CK(cudaMemcpyAsync(hp_hist, d_hist, sizeof(double) * hist_stride * B, cudaMemcpyDeviceToHost, so));
        CK(cudaEventRecord(ev_done, so));
        return 0;
    }

    int collect()
    {
        CK(cudaEventSynchronize(ev_done));
        trace_report();
        h_hist.assign(hp_hist, hp_hist + (size_t)hist_stride * B);
        h_it.resize(B);
        h_conv.resize(B);
        for (long long b = 0; b < B; ++b) {
            h_it[b] = hp_st[b].iters;
            h_conv[b] = hp_st[b].converged;
        }
        return 0;
    }

    int solve_on(const void *f, void *u, const double *floor_, double eps, int max_iters, cudaStream_t s)
    {
        CKR(enqueue_solve(f, u, floor_, eps, max_iters, s));
        return collect();
    }

    int stats(int32_t *it, double *norms, int32_t *conv) const override
    {
        if (h_it.empty()) return fail(TMG_E_ARG, "no solve has run on this plan");
        for (long long b = 0; b < B; ++b) {
            if (it) it[b] = h_it[b];
            if (conv) conv[b] = h_conv[b];
            if (norms)
                for (int k = 0; k <= last_max_iters; ++k)
                    norms[b * (last_max_iters + 1) + k] = k <= h_it[b] ? h_hist[b * hist_stride + k] : 0.0;
        }
        return 0;
    }

    int info(int32_t *kpc, int32_t *sl, int32_t *t) const override
    {
        if (kpc) *kpc = kernels_per_cycle;
        if (sl) *sl = tl;
        if (t) *t = tl;
        return 0;
    }
};

template <typename T, int NT>
int make_plan_sp(std::unique_ptr<PlanBase> &out, const tmg_level_desc *lv, int nl, long long B,
                 const tmg_plan_opts &o, bool multi)
{
    bool sparse = true;
    for (long long b = 0; b < (multi ? B : 1); ++b)
        for (int l = 0; l < nl; ++l) sparse &= coupling_is_sparse(lv[b * nl + l]);
    if (sparse) {
        auto p = std::make_unique<Plan<T, NT, true>>();
        CKR(p->init(lv, nl, B, o, multi));
        out = std::move(p);
    } else {
        auto p = std::make_unique<Plan<T, NT, false>>();
        CKR(p->init(lv, nl, B, o, multi));
        out = std::move(p);
    }
    return 0;
}

template <typename T>
int make_plan_t(std::unique_ptr<PlanBase> &out, const tmg_level_desc *lv, int nl, long long B,
                const tmg_plan_opts &o, bool multi = false)
{
    switch (lv[0].n_t) {
    case 1: return make_plan_sp<T, 1>(out, lv, nl, B, o, multi);
    case 2: return make_plan_sp<T, 2>(out, lv, nl, B, o, multi);
    case 3: return make_plan_sp<T, 3>(out, lv, nl, B, o, multi);
    case 4: return make_plan_sp<T, 4>(out, lv, nl, B, o, multi);
    }
    return fail(TMG_E_UNSUPPORTED, "n_t=%d", lv[0].n_t);
}

// ---------------------------------------------------------------------------
// single-level entry points

enum Op { OP_SWEEP, OP_RESID, OP_DOWN, OP_UP, OP_NORM, OP_SQSUM };

struct OpArgs {
    const void *f, *u_in, *uc;
    void *u_out, *aux;  // aux: r (RESID), f_coarse (DOWN)
    double *sq;
    long long batch;
    int nu;
    const int32_t *active;
    long long skip = 0;  // OP_SQSUM: first slab of the summed range
};

template <typename T, int NT, bool SP>
int run_op(Op op, const tmg_level_desc &d, const OpArgs &x, cudaStream_t s)
{
    const LevelC<T, NT> L = make_level<T, NT>(d);
    const long long n = d.n_slabs;
    StreamArgs<T> a = stream_args<T, NT>(n, x.batch, 1);
    a.f = (const T *)x.f;
    a.u_in = (const T *)x.u_in;
    a.active = x.active;
    switch (op) {
    case OP_SWEEP: {
        if (x.nu == 0) {
            if (x.u_in) CK(cudaMemcpyAsync(x.u_out, x.u_in, sizeof(T) * n * NT * x.batch, cudaMemcpyDeviceToDevice, s));
            else CK(cudaMemsetAsync(x.u_out, 0, sizeof(T) * n * NT * x.batch, s));
            return 0;
        }
        // chains of <= 4 fused sweeps; ping-pong through a scratch buffer
        int left = x.nu;
        const T *src = (const T *)x.u_in;
        T *tmp = nullptr;
        const int passes = (x.nu + 3) / 4;
        if (passes > 1) CK(cudaMallocAsync(&tmp, sizeof(T) * n * NT * x.batch, s));
        // make the last pass land in u_out
        T *bufs[2] = {(T *)x.u_out, tmp};
        int idx = (passes % 2 == 1) ? 0 : 1;
        while (left > 0) {
            const int k = std::min(4, left);
            StreamArgs<T> b = a;
            b.u_in = src;
            b.u_out = bufs[idx];
            b.flags = SF_WRITE_U | (src ? 0 : SF_ZERO_GUESS);
            if (tma_ok<T, NT>(b, false)) b.flags |= SF_TMA;
            CKR((launch_stream<T, NT>(L, b, k, K_GENERIC, P_GEN, SP, s)));
            src = bufs[idx];
            idx ^= 1;
            left -= k;
        }
        if (tmp) CK(cudaFreeAsync(tmp, s));
        return 0;
    }
    case OP_RESID:
        a.r_out = (T *)x.aux;
        a.flags = SF_WRITE_R;
        if (tma_ok<T, NT>(a, false)) a.flags |= SF_TMA;
        return launch_stream<T, NT>(L, a, 0, K_GENERIC, P_GEN, SP, s);
    case OP_DOWN:
        a.u_out = (T *)x.u_out;
        a.fc = (T *)x.aux;
        a.flags = SF_RESTRICT | SF_WRITE_U | (x.u_in ? 0 : SF_ZERO_GUESS);
        if (tma_ok<T, NT>(a, false)) a.flags |= SF_TMA;
        return launch_stream<T, NT>(L, a, x.nu, K_DOWN, perm_kind(d), SP, s);
    case OP_UP:
        a.uc = (const T *)x.uc;
        a.u_out = (T *)x.u_out;
        a.flags = SF_PROLONG | SF_WRITE_U | (x.sq ? SF_NORM_SQ : 0);
        a.sq_out = x.sq;
        if (tma_ok<T, NT>(a, true)) a.flags |= SF_TMA;
        return launch_stream<T, NT>(L, a, x.nu, x.sq ? K_GENERIC : K_UP, perm_kind(d), SP, s);
    case OP_SQSUM:
    case OP_NORM: {
        if (op == OP_SQSUM && (x.skip < 0 || x.skip >= n)) return fail(TMG_E_ARG, "skip must lie in [0, n_slabs)");
        double *sq = nullptr;
        CK(cudaMallocAsync(&sq, sizeof(double) * n * x.batch, s));
        a.sq_out = sq;
        a.flags = SF_NORM_SQ;
        if (tma_ok<T, NT>(a, false)) a.flags |= SF_TMA;
        int rc = launch_stream<T, NT>(L, a, 0, K_GENERIC, P_GEN, SP, s);
        if (!rc && op == OP_SQSUM) {
            range_sum_kernel<<<(unsigned)x.batch, 1024, 0, s>>>(sq, n, x.skip, n - x.skip, (double *)x.aux);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) rc = fail((int)e, "range sum: %s", cudaGetErrorString(e));
        } else if (!rc) {
            finalize_sq_kernel<<<(unsigned)x.batch, 1024, 0, s>>>(sq, n, nullptr, nullptr, 0, nullptr, 0.0, 0,
                                                                (double *)x.aux);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) rc = fail((int)e, "finalize: %s", cudaGetErrorString(e));
        }
        cudaFreeAsync(sq, s);
        return rc;
    }
    }
    return fail(TMG_E_ARG, "bad op");
}

template <typename T>
int run_op_t(Op op, const tmg_level_desc &d, const OpArgs &x, cudaStream_t s)
{
    const bool sp = coupling_is_sparse(d);
#define TMG_CASE(NTV)                                                             \
    case NTV:                                                                     \
        return sp ? run_op<T, NTV, true>(op, d, x, s) : run_op<T, NTV, false>(op, d, x, s);
    switch (d.n_t) {
        TMG_CASE(1)
        TMG_CASE(2)
        TMG_CASE(3)
        TMG_CASE(4)
    }
#undef TMG_CASE
    return fail(TMG_E_UNSUPPORTED, "n_t=%d", d.n_t);
}

int run_op_any(int dtype, Op op, const tmg_level_desc *d, const OpArgs &x, void *stream)
{
    CKR(check_desc(d));
    if (x.batch < 1) return fail(TMG_E_ARG, "batch must be >= 1");
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == TMG_F64) return run_op_t<double>(op, *d, x, s);
    if (dtype == TMG_F32) return run_op_t<float>(op, *d, x, s);
    return fail(TMG_E_ARG, "unknown dtype %d", dtype);
}

template <typename T, int NT, bool SP>
int coarse_op(const tmg_level_desc &d, const void *f, void *u, long long B, int method, int variant,
              cudaStream_t s)
{
    const LevelC<T, NT> L = make_level<T, NT>(d);
    if (method == 1) {
        if (!L.scan_ok) return fail(TMG_E_UNSUPPORTED, "coupling is not rank one: no scan solve");
        CK(((cudaError_t)coarse_scan_launch<T, NT>(L, (const T *)f, (T *)u, d.n_slabs, (int)B, nullptr, s)));
        return 0;
    }
    CK(((cudaError_t)coarse_serial_launch<T, NT>(L, SP, (const T *)f, (T *)u, d.n_slabs, (int)B, variant, nullptr, s)));
    return 0;
}

}  // namespace

// ---------------------------------------------------------------------------
// exported C ABI

extern "C" {

const char *tmg_last_error(void) { return g_err.c_str(); }

int tmg_version(void) { return 100; }

int tmg_device_check(int device)
{
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, device));
    if (p.major < 10) return fail(TMG_E_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a",
                                  device, p.major, p.minor);
    return 0;
}

int tmg_sweep(int dtype, const tmg_level_desc *lev, const void *f, const void *u_in, void *u_out,
              int64_t batch, int nu, const int32_t *active, void *stream)
{
    if (nu < 0) return fail(TMG_E_ARG, "sweep count must be >= 0, got %d", nu);
    if (lev && !(lev->omega > 0.0 && lev->omega < 2.0))
        return fail(TMG_E_ARG, "damping must lie in (0, 2), got %g", lev->omega);
    if (u_in && u_in == u_out) return fail(TMG_E_ARG, "u_in and u_out must not alias");
    OpArgs x{f, u_in, nullptr, u_out, nullptr, nullptr, batch, nu, active};
    return run_op_any(dtype, OP_SWEEP, lev, x, stream);
}

int tmg_residual(int dtype, const tmg_level_desc *lev, const void *f, const void *u, void *r,
                 int64_t batch, void *stream)
{
    OpArgs x{f, u, nullptr, nullptr, r, nullptr, batch, 0, nullptr};
    return run_op_any(dtype, OP_RESID, lev, x, stream);
}

int tmg_down(int dtype, const tmg_level_desc *lev, const void *f, const void *u_in, void *u_out,
             void *f_coarse, int64_t batch, int nu1, const int32_t *active, void *stream)
{
    if (u_in && u_in == u_out) return fail(TMG_E_ARG, "u_in and u_out must not alias");
    OpArgs x{f, u_in, nullptr, u_out, f_coarse, nullptr, batch, nu1, active};
    return run_op_any(dtype, OP_DOWN, lev, x, stream);
}

int tmg_up(int dtype, const tmg_level_desc *lev, const void *f, const void *u_in, const void *u_coarse,
           void *u_out, double *sq_out, int64_t batch, int nu2, const int32_t *active, void *stream)
{
    if (u_in == u_out) return fail(TMG_E_ARG, "u_in and u_out must not alias");
    OpArgs x{f, u_in, u_coarse, u_out, nullptr, sq_out, batch, nu2, active};
    return run_op_any(dtype, OP_UP, lev, x, stream);
}

int tmg_coarse_solve(int dtype, const tmg_level_desc *lev, const void *f, void *u, int64_t batch,
                     int method, int dot_variant, void *stream)
{
    CKR(check_desc(lev));
    if (dot_variant == 0 && lev->n_t > 4) return fail(TMG_E_UNSUPPORTED, "no calibrated dgemv tree for n_t > 4");
    cudaStream_t s = (cudaStream_t)stream;
    const bool sp = coupling_is_sparse(*lev);
#define TMG_CC(T, NTV) \
    case NTV: return sp ? coarse_op<T, NTV, true>(*lev, f, u, batch, method, dot_variant, s) \
                        : coarse_op<T, NTV, false>(*lev, f, u, batch, method, dot_variant, s);
    if (dtype == TMG_F64) {
        switch (lev->n_t) { TMG_CC(double, 1) TMG_CC(double, 2) TMG_CC(double, 3) TMG_CC(double, 4) }
    } else if (dtype == TMG_F32) {
        switch (lev->n_t) { TMG_CC(float, 1) TMG_CC(float, 2) TMG_CC(float, 3) TMG_CC(float, 4) }
    }
#undef TMG_CC
    return fail(TMG_E_ARG, "bad dtype/n_t");
}

int tmg_resid_norm(int dtype, const tmg_level_desc *lev, const void *f, const void *u, double *norms_out,
                   int64_t batch, void *stream)
{
    OpArgs x{f, u, nullptr, nullptr, norms_out, nullptr, batch, 0, nullptr};
    return run_op_any(dtype, OP_NORM, lev, x, stream);
}

int tmg_trace_enable(int on)
{
    g_event_trace = on ? 1 : 0;
    g_trace_quiet = on != 0;
    g_trace_text.clear();
    return 0;
}

int64_t tmg_trace_read(char *buf, int64_t cap)
{
    const int64_t n = (int64_t)g_trace_text.size();
    if (buf && cap > 0) {
        const int64_t k = std::min(n, cap - 1);
        memcpy(buf, g_trace_text.data(), (size_t)k);
        buf[k] = 0;
    }
    g_trace_text.clear();
    return n;
}

int tmg_resid_sqsum(int dtype, const tmg_level_desc *lev, const void *f, const void *u, int64_t skip,
                    double *sums_out, int64_t batch, void *stream)
{
    OpArgs x{f, u, nullptr, nullptr, sums_out, nullptr, batch, 0, nullptr};
    x.skip = skip;
    return run_op_any(dtype, OP_SQSUM, lev, x, stream);
}

int tmg_plan_create(tmg_plan **plan, const tmg_level_desc *levels, int n_levels, int64_t batch,
                    const tmg_plan_opts *opts)
{
    if (!plan || !levels || !opts) return fail(TMG_E_ARG, "NULL argument");
    *plan = nullptr;
    if (n_levels < 2 || n_levels > MAXLEV) return fail(TMG_E_ARG, "need 2..%d levels, got %d", MAXLEV, n_levels);
    if (batch < 1) return fail(TMG_E_ARG, "batch must be >= 1");
    for (int l = 0; l < n_levels; ++l) {
        CKR(check_desc(&levels[l]));
        if (levels[l].n_t != levels[0].n_t) return fail(TMG_E_ARG, "levels disagree on n_t");
    }
    if (opts->nu1 < 0 || opts->nu2 < 0 || opts->nu1 + opts->nu2 < 1)
        return fail(TMG_E_ARG, "need nu1, nu2 >= 0 with nu1 + nu2 >= 1");
    if (opts->nu1 > 4 || opts->nu2 > 4) return fail(TMG_E_UNSUPPORTED, "nu > 4 not supported");
    if (opts->dot_variant == 0 && levels[0].n_t > 4) return fail(TMG_E_UNSUPPORTED, "dgemv tree");
    auto p = std::make_unique<tmg_plan>();
    int rc;
    if (opts->dtype == TMG_F64) rc = make_plan_t<double>(p->impl, levels, n_levels, batch, *opts);
    else if (opts->dtype == TMG_F32) rc = make_plan_t<float>(p->impl, levels, n_levels, batch, *opts);
    else return fail(TMG_E_ARG, "unknown dtype");
    if (rc) return rc;
    *plan = p.release();
    return 0;
}

int tmg_plan_create_multi(tmg_plan **plan, const tmg_level_desc *levels, int n_levels, int64_t batch,
                          const tmg_plan_opts *opts)
{
    if (!plan || !levels || !opts) return fail(TMG_E_ARG, "NULL argument");
    *plan = nullptr;
    if (n_levels < 2 || n_levels > MAXLEV) return fail(TMG_E_ARG, "need 2..%d levels, got %d", MAXLEV, n_levels);
    if (batch < 1) return fail(TMG_E_ARG, "batch must be >= 1");
    for (long long i = 0; i < batch * n_levels; ++i) {
        CKR(check_desc(&levels[i]));
        if (levels[i].n_t != levels[0].n_t) return fail(TMG_E_ARG, "problems disagree on n_t");
    }
    if (opts->nu1 < 0 || opts->nu2 < 0 || opts->nu1 + opts->nu2 < 1)
        return fail(TMG_E_ARG, "need nu1, nu2 >= 0 with nu1 + nu2 >= 1");
    auto p = std::make_unique<tmg_plan>();
    int rc;
    if (opts->dtype == TMG_F64) rc = make_plan_t<double>(p->impl, levels, n_levels, batch, *opts, true);
    else if (opts->dtype == TMG_F32) rc = make_plan_t<float>(p->impl, levels, n_levels, batch, *opts, true);
    else return fail(TMG_E_ARG, "unknown dtype");
    if (rc) return rc;
    *plan = p.release();
    return 0;
}

int tmg_plan_destroy(tmg_plan *plan)
{
    delete plan;
    return 0;
}

int tmg_plan_cycles(tmg_plan *plan, const void *f, void *u, int n_cycles, void *stream)
{
    if (!plan) return fail(TMG_E_ARG, "NULL plan");
    return plan->impl->cycles(f, u, n_cycles, (cudaStream_t)stream);
}

int tmg_plan_solve(tmg_plan *plan, const void *f, void *u, const double *floor_per_problem, double eps,
                   int max_iters, void *stream)
{
    if (!plan) return fail(TMG_E_ARG, "NULL plan");
    if (!(eps > 0.0 && eps < 1.0)) return fail(TMG_E_ARG, "eps must lie in (0, 1)");
    return plan->impl->solve(f, u, floor_per_problem, eps, max_iters, (cudaStream_t)stream);
}

int tmg_plan_solve_host(tmg_plan *plan, const void *f_host, const void *u_init_host, void *u_host,
                        const double *floor_per_problem, double eps, int max_iters)
{
    if (!plan || !f_host || !u_host) return fail(TMG_E_ARG, "NULL argument");
    if (!(eps > 0.0 && eps < 1.0)) return fail(TMG_E_ARG, "eps must lie in (0, 1)");
    return plan->impl->solve_host(f_host, u_init_host, u_host, floor_per_problem, eps, max_iters);
}

int tmg_plan_solve_host_stream(tmg_plan *plan, int n_batches, const void *const *f_hosts, void *const *u_hosts,
                               const double *floor_per_problem, double eps, int max_iters, int32_t *iterations,
                               double *norms, int32_t *converged)
{
    if (!plan || !f_hosts || !u_hosts || !floor_per_problem) return fail(TMG_E_ARG, "NULL argument");
    if (!(eps > 0.0 && eps < 1.0)) return fail(TMG_E_ARG, "eps must lie in (0, 1)");
    if (max_iters < 1) return fail(TMG_E_ARG, "max_iters must be >= 1");
    for (int k = 0; k < n_batches; ++k)
        if (!f_hosts[k] || !u_hosts[k]) return fail(TMG_E_ARG, "batch %d: NULL host buffer", k);
    return plan->impl->solve_host_stream(n_batches, f_hosts, u_hosts, floor_per_problem, eps, max_iters, iterations,
                                         norms, converged);
}

int tmg_plan_stats(const tmg_plan *plan, int32_t *iterations, double *norms, int32_t *converged)
{
    if (!plan) return fail(TMG_E_ARG, "NULL plan");
    return plan->impl->stats(iterations, norms, converged);
}

int tmg_plan_info(const tmg_plan *plan, int32_t *kernels_per_cycle, int32_t *stream_levels,
                  int32_t *tail_level)
{
    if (!plan) return fail(TMG_E_ARG, "NULL plan");
    return plan->impl->info(kernels_per_cycle, stream_levels, tail_level);
}

}  // extern "C"
