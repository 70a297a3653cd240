// C-ABI layer: argument validation, launch planning and host-pointer forms.
// Declarations and conventions: include/osc_b200.h.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <utility>
#include <vector>

#include <cuda.h>  // driver types only: entry points via cudaGetDriverEntryPoint

#include "../../include/osc_b200.h"
#include "osc_kernels.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char *where)
{
    return fail(OSC_CUDA_ERROR, "%s: %s", where, cudaGetErrorString(e));
}

#define OSC_CUDA(call)                                                                      \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return cuda_fail(e_, #call);                                                    \
    } while (0)

// The reference's argument checks: rk4_step's dt (oscillator.py:201-202) and
// integrate's nsteps/stride (oscillator.py:247-250).
int check_run_args(double dt, int64_t nsteps, int64_t stride)
{
    if (!(std::isfinite(dt) && dt > 0.0))
        return fail(OSC_INVALID, "dt must be positive and finite, got %.17g", dt);
    if (nsteps < 1)
        return fail(OSC_INVALID, "nsteps must be >= 1, got %lld", (long long)nsteps);
    if (stride < 1)
        return fail(OSC_INVALID, "stride must be >= 1, got %lld", (long long)stride);
    return OSC_OK;
}

osc::StepConsts consts(double dt)
{
    // Exactly the reference's constants: half_dt = 0.5 * dt (oscillator.py:208)
    // and dt / 6.0 inside combine_value (oscillator.py:174).
    return osc::StepConsts{dt, 0.5 * dt, dt / 6.0};
}

constexpr int64_t kWholeChainMax = 2048;  // 256 threads x 8 cells
constexpr int64_t kWholeChainSteps = 512; // steps per launch in whole-chain mode
constexpr int64_t kSplitChains = 1024;     // whole-chain batches this large run as two halves
// Tiled shape, measured on B200 for s = 2^24 (profiles/r01/README.md): with
// the persistent prefetching kernel, 8 cells x 256 threads and 32-step halos
// beat 8 x 128 at T = 16..24 by 3-8% and 4 x 256 / 4 x 512 by 12-14%.
constexpr int kTileK = 8, kTileThreads = 256;
constexpr int64_t kTile = int64_t(kTileK) * kTileThreads;
constexpr int64_t kDefaultHaloSteps = 32;

void pick_whole(int64_t s, int &K, int &threads)
{
    // Fewest cells per thread that keep the CTA at <= 128 threads, else 256
    // threads of 8 cells.  Measured on B200 for s = 1024 (profiles/r01
    // sweep_C4_*): K=8 x 128 threads beats K=4 x 256 by 8% and K=2 x 512 by 2.4x.
    K = 8;
    for (int k : {1, 2, 4, 8}) {
        if ((s + k - 1) / k <= 128) {
            K = k;
            break;
        }
    }
    const int64_t t = (s + K - 1) / K;
    threads = static_cast<int>(((t + 31) / 32) * 32);
}

// Steps per tiled launch when the caller leaves it to us.  A launch costs
// rounds(T) tile-times of (T + c) steps, where rounds(T) = ceil(tiles(T) /
// CTAs) (one persistent CTA per SM) and c ~ 4 steps covers a tile's load,
// setup and store; per step that is rounds(T) * (T + c) / T.  Deeper halos
// mean fewer launches but narrower owned tiles, so the tile count can cross
// a multiple of the CTA count: for C3 (2^24 cells) T = 31 gives 59 rounds
// instead of 60 (+0.7% measured, profiles/r01/README.md).
int64_t pick_halo_steps(int64_t s, int64_t B, int64_t nsteps)
{
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        sms = 148;            // no device (planning only): B200
        cudaGetLastError();   // do not leave the query's error pending
    }
    constexpr double c = 4.0;
    int64_t best = kDefaultHaloSteps;
    double best_cost = 0.0;
    for (int64_t T : {int64_t(32), int64_t(31), int64_t(30), int64_t(28)}) {
        if (T > nsteps && T != kDefaultHaloSteps)
            continue;
        const int64_t W = kTile - 4 * T;
        const int64_t tiles = B * ((s + W - 1) / W);
        const int64_t rounds = (tiles + sms - 1) / sms;
        const double cost = double(rounds) * (double(T) + c) / double(T);
        if (best_cost == 0.0 || cost < best_cost * (1.0 - 1e-9)) {
            best = T;
            best_cost = cost;
        }
    }
    return best;
}

// Tuning hook (benchmarks only): OSC_TILE="K,threads" / OSC_WHOLE="K,threads"
// override the tiled / whole-chain launch shapes.  Read-only process state.
bool env_shape(const char *name, int &K, int &threads)
{
    const char *e = std::getenv(name);
    int k = 0, t = 0;
    if (!e || std::sscanf(e, "%d,%d", &k, &t) != 2)
        return false;
    if ((k != 1 && k != 2 && k != 4 && k != 8) || t < 32 || t > 1024 || t % 32)
        return false;
    K = k;
    threads = t;
    return true;
}

struct ChainPlan {
    int K = kTileK, threads = kTileThreads;
    int64_t W = 0, H = 0, tiles = 1, per_launch = 0;
};

// Launch plan of osc_rk4_chains: whole chains up to kWholeChainMax cells
// (one CTA per chain, kWholeChainSteps steps per launch), else temporally
// blocked tiles of K x threads cells, H = 2T halo, T steps per launch.
int plan_chain(int64_t s, int64_t B, int64_t nsteps, int64_t halo_steps, ChainPlan &p)
{
    int wk = 0, wt = 0;
    const bool whole_env = env_shape("OSC_WHOLE", wk, wt) && int64_t(wk) * wt >= s;
    if (s <= kWholeChainMax || whole_env) {
        pick_whole(s, p.K, p.threads);
        if (whole_env) {
            p.K = wk;
            p.threads = wt;
        }
        p.W = s;
        p.H = 0;
        p.tiles = 1;
        p.per_launch = kWholeChainSteps;
        return OSC_OK;
    }
    const bool shaped = env_shape("OSC_TILE", p.K, p.threads);
    const int64_t T = halo_steps > 0 ? halo_steps
                                     : (shaped ? kDefaultHaloSteps : pick_halo_steps(s, B, nsteps));
    p.H = 2 * T;
    p.W = int64_t(p.K) * p.threads - 2 * p.H;
    if (p.W < 1)
        return fail(OSC_INVALID, "halo_steps=%lld too deep for a %lld-cell tile", (long long)T,
                    (long long)p.K * p.threads);
    p.tiles = (s + p.W - 1) / p.W;
    p.per_launch = T;
    return OSC_OK;
}

// Keep freed stream-ordered allocations in the device's default pool instead
// of returning them to the driver at every synchronisation (the default
// release threshold is 0), so repeated host-API calls do not re-map memory.
void retain_pool_memory()
{
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev)
        return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done_dev = dev;
}

struct Scratch {
    double *p = nullptr;
    cudaStream_t s = nullptr;
    ~Scratch()
    {
        if (p)
            cudaFreeAsync(p, s);
    }
};

}  // namespace

extern "C" {

int osc_abi_version(void) { return OSC_ABI_VERSION; }

const char *osc_last_error(void) { return g_last_error.c_str(); }

int osc_rk4_batch2(const double *m, const double *C, double *x, double *v, int64_t B, double dt,
                   int64_t nsteps, int64_t stride, double *xs, double *vs, double *es,
                   int64_t *first_bad, uint32_t flags, void *stream)
{
    if (flags & ~uint32_t(OSC_FMA))
        return fail(OSC_INVALID, "unknown flags 0x%x", flags);
    if (int rc = check_run_args(dt, nsteps, stride))
        return rc;
    if (B < 0)
        return fail(OSC_INVALID, "B must be >= 0");
    if (B == 0)
        return OSC_OK;
    if (!m || !C || !x || !v || !first_bad || (!xs) != (!vs))
        return fail(OSC_INVALID, "null buffer");
    cudaError_t e = osc::launch_batch2(m, C, x, v, B, consts(dt), nsteps, stride, xs, vs, es,
                                       first_bad, (flags & OSC_FMA) != 0,
                                       static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "batch2_rk4_kernel");
}

int osc_rk4_batch2_compare(const double *m, const double *C, double *x, double *v, int64_t B,
                           double dt, int64_t nsteps, int64_t stride, const double *ts,
                           const double *sol, double *report, int64_t *first_bad, uint32_t flags,
                           void *stream)
{
    if (flags & ~uint32_t(OSC_FMA))
        return fail(OSC_INVALID, "unknown flags 0x%x", flags);
    if (int rc = check_run_args(dt, nsteps, stride))
        return rc;
    if (B < 0)
        return fail(OSC_INVALID, "B must be >= 0");
    if (B == 0)
        return OSC_OK;
    if (!m || !C || !x || !v || !first_bad || !ts || !sol || !report)
        return fail(OSC_INVALID, "null buffer");
    const osc::CmpArgs cmp{ts, sol, report};
    cudaError_t e = osc::launch_batch2(m, C, x, v, B, consts(dt), nsteps, stride, nullptr, nullptr,
                                       nullptr, first_bad, (flags & OSC_FMA) != 0,
                                       static_cast<cudaStream_t>(stream), &cmp);
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "batch2_rk4_kernel<compare>");
}

int osc_analytic_batch2(const double *m, const double *C, const double *x0, const double *v0,
                        int64_t B, double *sol, void *stream)
{
    if (B < 0)
        return fail(OSC_INVALID, "B must be >= 0");
    if (B == 0)
        return OSC_OK;
    if (!m || !C || !x0 || !v0 || !sol)
        return fail(OSC_INVALID, "null buffer");
    cudaError_t e = osc::launch_modal_batch2(m, C, x0, v0, B, sol,
                                             static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "modal_batch2_kernel");
}

int osc_compare_batch2(const double *sol, const double *xs, const double *ts, int64_t nsamp,
                       int64_t B, double *report, void *stream)
{
    if (B < 0)
        return fail(OSC_INVALID, "B must be >= 0");
    if (nsamp < 1)
        return fail(OSC_INVALID, "empty trajectory");  // modal.py:143-144
    if (B == 0)
        return OSC_OK;
    if (!sol || !xs || !ts || !report)
        return fail(OSC_INVALID, "null buffer");
    cudaError_t e = osc::launch_compare_batch2(sol, xs, ts, nsamp, B, report,
                                               static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "compare_batch2_kernel");
}

int osc_rk4_chains(const double *m, const double *C, double *x, double *v, int64_t B, int64_t s,
                   double dt, int64_t nsteps, int64_t stride, double *xs, double *vs, double *es,
                   int64_t *first_bad, int64_t halo_steps, uint32_t flags, void *stream_)
{
    if (flags & ~uint32_t(OSC_FMA))
        return fail(OSC_INVALID, "unknown flags 0x%x", flags);
    if (int rc = check_run_args(dt, nsteps, stride))
        return rc;
    if (B < 0 || s < 1)
        return fail(OSC_INVALID, "need B >= 0 and s >= 1 (got B=%lld s=%lld)", (long long)B,
                    (long long)s);
    if (B == 0)
        return OSC_OK;
    if (!m || !C || !x || !v || !first_bad || (!xs) != (!vs))
        return fail(OSC_INVALID, "null buffer");
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    const int64_t cells = B * s;
    const size_t bytes = sizeof(double) * static_cast<size_t>(cells);

    osc::SegArgs g{};
    g.m = m;
    g.C = C;
    g.first_bad = first_bad;
    g.n = s;
    g.nbuf = B;
    g.own_lo = 0;
    g.own_hi = s;
    g.k = consts(dt);
    g.fma = (flags & OSC_FMA) != 0;
    ChainPlan plan;
    if (int rc = plan_chain(s, B, nsteps, halo_steps, plan))
        return rc;
    const int K = plan.K, threads = plan.threads;
    const int64_t per_launch = plan.per_launch;
    g.W = plan.W;
    g.H = plan.H;
    g.tiles = plan.tiles;

    OSC_CUDA(cudaMemsetAsync(first_bad, 0, sizeof(int64_t) * B, stream));
    if (xs) {
        OSC_CUDA(cudaMemcpyAsync(xs, x, bytes, cudaMemcpyDeviceToDevice, stream));
        OSC_CUDA(cudaMemcpyAsync(vs, v, bytes, cudaMemcpyDeviceToDevice, stream));
    }
    if (es) {  // energy() of every retained sample, exact sequential sum per chain
        cudaError_t e = osc::launch_energy(m, C, x, v, es, B, s, false, stream);
        if (e != cudaSuccess)
            return cuda_fail(e, "energy_kernel");
    }
    retain_pool_memory();
    Scratch scratch;
    scratch.s = stream;
    OSC_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&scratch.p), 2 * bytes, stream));

    // The time loop over chains [b0, b0 + nb) on stream st.
    auto run_group = [&](int64_t b0, int64_t nb, cudaStream_t st) -> int {
        const int64_t o = b0 * s;
        osc::SegArgs gg = g;
        gg.m = m + o;
        gg.C = C + o;
        gg.first_bad = first_bad + b0;
        gg.nbuf = nb;
        double *cx = x + o, *cv = v + o, *nx = scratch.p + o, *nv = scratch.p + cells + o;
        for (int64_t k0 = 0; k0 < nsteps;) {
            int64_t n = nsteps - k0;
            if (n > per_launch)
                n = per_launch;
            const int64_t next_sample = (k0 / stride + 1) * stride;
            if (next_sample - k0 < n)
                n = next_sample - k0;
            gg.xin = cx;
            gg.vin = cv;
            gg.xout = nx;
            gg.vout = nv;
            gg.nsteps = n;
            gg.step0 = k0;
            const bool sample = xs && (k0 + n) % stride == 0;
            gg.xs = sample ? xs + ((k0 + n) / stride) * cells + o : nullptr;
            gg.vs = sample ? vs + ((k0 + n) / stride) * cells + o : nullptr;
            cudaError_t e = osc::launch_chain(gg, K, threads, st);
            if (e != cudaSuccess)
                return cuda_fail(e, "chain_rk4_kernel");
            if (es && (k0 + n) % stride == 0) {
                e = osc::launch_energy(gg.m, gg.C, nx, nv, es + ((k0 + n) / stride) * B + b0, nb,
                                       s, false, st);
                if (e != cudaSuccess)
                    return cuda_fail(e, "energy_kernel");
            }
            std::swap(cx, nx);
            std::swap(cv, nv);
            k0 += n;
        }
        if (cx != x + o) {
            const size_t gb = sizeof(double) * static_cast<size_t>(nb * s);
            OSC_CUDA(cudaMemcpyAsync(x + o, cx, gb, cudaMemcpyDeviceToDevice, st));
            OSC_CUDA(cudaMemcpyAsync(v + o, cv, gb, cudaMemcpyDeviceToDevice, st));
        }
        return OSC_OK;
    };

    // Whole-chain batches of many waves run as two independent halves on two
    // streams, so that one half's launches fill the other's tail wave
    // (chains are independent: same bytes either way).
    if (!(plan.tiles == 1 && B >= kSplitChains))
        return run_group(0, B, stream);
    cudaStream_t side = nullptr;
    OSC_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    struct SideStream {
        cudaStream_t s;
        ~SideStream() { cudaStreamDestroy(s); }
    } side_guard{side};
    cudaEvent_t fork, join;
    OSC_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    OSC_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    struct Events {
        cudaEvent_t a, b;
        ~Events()
        {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } ev_guard{fork, join};
    OSC_CUDA(cudaEventRecord(fork, stream));
    OSC_CUDA(cudaStreamWaitEvent(side, fork, 0));
    const int64_t half = B / 2;
    int rc = run_group(0, half, stream);
    const int rc2 = run_group(half, B - half, side);
    OSC_CUDA(cudaEventRecord(join, side));
    OSC_CUDA(cudaStreamWaitEvent(stream, join, 0));  // also orders the scratch free
    if (rc == OSC_OK)
        rc = rc2;
    return rc;
}

int osc_chain_plan(int64_t B, int64_t s, int64_t nsteps, int64_t halo_steps, int64_t *plan)
{
    if (B < 1 || s < 1 || nsteps < 1 || !plan)
        return fail(OSC_INVALID, "need B, s, nsteps >= 1 and a plan buffer");
    ChainPlan p;
    if (int rc = plan_chain(s, B, nsteps, halo_steps, p))
        return rc;
    const int64_t launches = (nsteps + p.per_launch - 1) / p.per_launch;
    const int64_t out[7] = {p.K, p.threads, p.per_launch, p.W, p.H, p.tiles, launches};
    for (int i = 0; i < 7; ++i)
        plan[i] = out[i];
    return OSC_OK;
}

int osc_rk4_chain_advance(const double *m, const double *C, const double *xin, const double *vin,
                          double *xout, double *vout, int64_t n, int64_t own_lo, int64_t own_hi,
                          double dt, int64_t nsteps, int64_t step0, int64_t *first_bad,
                          const osc_peer_t *left, const osc_peer_t *right, uint32_t flags,
                          void *stream)
{
    if (flags & ~uint32_t(OSC_FMA))
        return fail(OSC_INVALID, "unknown flags 0x%x", flags);
    if (int rc = check_run_args(dt, nsteps, 1))
        return rc;
    if (n < 1 || own_lo < 0 || own_hi > n || own_lo >= own_hi)
        return fail(OSC_INVALID, "bad shard range [%lld,%lld) of %lld", (long long)own_lo,
                    (long long)own_hi, (long long)n);
    if (!m || !C || !xin || !vin || !xout || !vout || !first_bad)
        return fail(OSC_INVALID, "null buffer");
    osc::SegArgs g{};
    g.m = m;
    g.C = C;
    g.xin = xin;
    g.vin = vin;
    g.xout = xout;
    g.vout = vout;
    g.first_bad = first_bad;
    g.n = n;
    g.nbuf = 1;
    g.own_lo = own_lo;
    g.own_hi = own_hi;
    g.H = 2 * nsteps;
    g.W = kTile - 2 * g.H;
    if (g.W < 1)
        return fail(OSC_INVALID, "nsteps=%lld too deep for a %lld-cell tile", (long long)nsteps,
                    (long long)kTile);
    g.tiles = (own_hi - own_lo + g.W - 1) / g.W;
    g.k = consts(dt);
    g.nsteps = nsteps;
    g.step0 = step0;
    g.fma = (flags & OSC_FMA) != 0;
    const osc_peer_t *peers[2] = {left, right};
    for (int side = 0; side < 2; ++side) {
        const osc_peer_t *p = peers[side];
        if (!p || !p->x)
            continue;
        if (!p->v || p->count < 0 || p->count > own_hi - own_lo)
            return fail(OSC_INVALID, "bad peer ghost descriptor");
        // left neighbour receives our first `count` owned cells, right our last
        const int64_t lo = side == 0 ? own_lo : own_hi - p->count;
        g.peer[side] = osc::PeerGhost{p->x, p->v, p->offset, lo, lo + p->count};
    }
    cudaError_t e = osc::launch_chain(g, kTileK, kTileThreads, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "chain_rk4_kernel");
}

int osc_rowscale(const double *K, const double *m, double *A, int64_t s, void *stream)
{
    if (s < 1 || !K || !m || !A)
        return fail(OSC_INVALID, "bad rowscale arguments");
    cudaError_t e = osc::launch_rowscale(K, m, A, s, s, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "rowscale_kernel");
}

int osc_rk4_dense(const double *A, double *X, double *V, int64_t s, int64_t N, double dt,
                  int64_t nsteps, int64_t *first_bad, void *stream_)
{
    if (int rc = check_run_args(dt, nsteps, 1))
        return rc;
    if (s < 1 || N < 0)
        return fail(OSC_INVALID, "need s >= 1 and N >= 0");
    if (N == 0)
        return OSC_OK;
    if (!A || !X || !V || !first_bad)
        return fail(OSC_INVALID, "null buffer");
    retain_pool_memory();
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    const int64_t sp = osc::dense_pad_s(s), Np = osc::dense_pad_n(N);
    const size_t op = static_cast<size_t>(sp) * 2 * Np, st = static_cast<size_t>(sp) * Np;
    const bool pad_a = sp != s;
    const size_t total = 2 * op + 3 * st + (pad_a ? static_cast<size_t>(sp) * sp : 0);
    Scratch ws;
    ws.s = stream;
    OSC_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&ws.p), total * sizeof(double), stream));
    double *BA = ws.p, *BB = BA + op, *Vp = BB + op, *SX = Vp + st, *SV = SX + st;
    const double *Ause = A;
    if (pad_a) {
        double *Ap = SV + st;
        OSC_CUDA(cudaMemsetAsync(Ap, 0, sizeof(double) * sp * sp, stream));
        OSC_CUDA(cudaMemcpy2DAsync(Ap, sp * sizeof(double), A, s * sizeof(double),
                                   s * sizeof(double), s, cudaMemcpyDeviceToDevice, stream));
        Ause = Ap;
    }
    const osc::StepConsts k = consts(dt);
    OSC_CUDA(cudaMemsetAsync(first_bad, 0, sizeof(int64_t), stream));
    cudaError_t e = osc::launch_dense_pack(X, V, BA, Vp, s, N, sp, Np, k.half_dt, stream);
    if (e != cudaSuccess)
        return cuda_fail(e, "pack_kernel");
    cudaStream_t side = nullptr;
    OSC_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    e = osc::launch_dense_steps(Ause, BA, BB, Vp, SX, SV, first_bad, sp, Np, k, 0, nsteps,
                                stream, side);
    cudaStreamDestroy(side);  // released once its queued work is done
    if (e != cudaSuccess)
        return cuda_fail(e, "dense_rk4_gemm");
    e = osc::launch_dense_unpack(BA, Vp, X, V, s, N, Np, stream);
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "unpack_kernel");
}

int osc_equation_engine(const double *m, const double *C, const double *x0, const double *v0,
                        int64_t s, double dt, int64_t nsteps, int64_t stride, double *xs,
                        double *vs, int64_t *first_bad, int64_t *step_ns, void *stream)
{
    if (int rc = check_run_args(dt, nsteps, stride))
        return rc;
    if (s < 1 || s > 64)
        return fail(OSC_INVALID, "the one-warp equation engine takes 1 <= s <= 64, got %lld",
                    (long long)s);
    if (!m || !C || !x0 || !v0 || !first_bad || !step_ns || (!xs) != (!vs))
        return fail(OSC_INVALID, "null buffer");
    cudaError_t e = osc::launch_equation_engine(m, C, x0, v0, static_cast<int>(s), dt, nsteps,
                                                stride, xs, vs, first_bad, step_ns,
                                                static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "equation_engine_kernel");
}

// ---------------------------------------------------------------------------
// Peer memory for the fused halo exchange: plain allocations (so an exported
// pointer is an allocation base), CUDA IPC handles and interprocess events.
// ---------------------------------------------------------------------------
int osc_device_alloc(uint64_t bytes, void **ptr)
{
    if (!ptr)
        return fail(OSC_INVALID, "null ptr");
    OSC_CUDA(cudaMalloc(ptr, bytes));
    return OSC_OK;
}

int osc_device_free(void *ptr)
{
    OSC_CUDA(cudaFree(ptr));
    return OSC_OK;
}

int osc_ipc_export(const void *ptr, unsigned char *handle64)
{
    cudaIpcMemHandle_t h;
    OSC_CUDA(cudaIpcGetMemHandle(&h, const_cast<void *>(ptr)));
    std::memcpy(handle64, &h, sizeof h);
    return OSC_OK;
}

int osc_ipc_import(const unsigned char *handle64, void **ptr)
{
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof h);
    OSC_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return OSC_OK;
}

int osc_ipc_close(void *ptr)
{
    OSC_CUDA(cudaIpcCloseMemHandle(ptr));
    return OSC_OK;
}

int osc_ipc_event_create(void **event, unsigned char *handle64)
{
    cudaEvent_t ev;
    OSC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventInterprocess));
    cudaIpcEventHandle_t h;
    OSC_CUDA(cudaIpcGetEventHandle(&h, ev));
    std::memcpy(handle64, &h, sizeof h);
    *event = ev;
    return OSC_OK;
}

int osc_ipc_event_open(const unsigned char *handle64, void **event)
{
    cudaIpcEventHandle_t h;
    std::memcpy(&h, handle64, sizeof h);
    cudaEvent_t ev;
    OSC_CUDA(cudaIpcOpenEventHandle(&ev, h));
    *event = ev;
    return OSC_OK;
}

int osc_event_record(void *event, void *stream)
{
    OSC_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(event), static_cast<cudaStream_t>(stream)));
    return OSC_OK;
}

int osc_stream_wait_event(void *stream, void *event)
{
    OSC_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream),
                                 static_cast<cudaEvent_t>(event), 0));
    return OSC_OK;
}

int osc_event_destroy(void *event)
{
    OSC_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(event)));
    return OSC_OK;
}

int osc_derivative(const double *m, const double *C, const double *x, double *dvel, int64_t B,
                   int64_t s, int cell_major, void *stream)
{
    if (B < 0 || s < 1)
        return fail(OSC_INVALID, "need B >= 0 and s >= 1");
    cudaError_t e = osc::launch_derivative(m, C, x, dvel, B, s, cell_major != 0,
                                           static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "derivative_kernel");
}

int osc_energy(const double *m, const double *C, const double *x, const double *v, double *out,
               int64_t B, int64_t s, int cell_major, void *stream)
{
    if (B < 0 || s < 1)
        return fail(OSC_INVALID, "need B >= 0 and s >= 1");
    cudaError_t e = osc::launch_energy(m, C, x, v, out, B, s, cell_major != 0,
                                       static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "energy_kernel");
}

int osc_check_division(int64_t n, uint64_t seed, int mode, uint64_t *mismatches, void *stream_)
{
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    unsigned long long *d = nullptr;
    OSC_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&d), sizeof *d, stream));
    OSC_CUDA(cudaMemsetAsync(d, 0, sizeof *d, stream));
    cudaError_t e = osc::launch_check_division(n, seed, mode, d, stream);
    if (e != cudaSuccess)
        return cuda_fail(e, "check_division_kernel");
    unsigned long long h = 0;
    OSC_CUDA(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, stream));
    OSC_CUDA(cudaFreeAsync(d, stream));
    OSC_CUDA(cudaStreamSynchronize(stream));
    *mismatches = h;
    return OSC_OK;
}

int osc_bench_fp64(int64_t iters, int mode, double *sink, int64_t *lane_ops, void *stream)
{
    if (iters < 1 || !sink || !lane_ops)
        return fail(OSC_INVALID, "bad fp64 bench arguments");
    cudaError_t e = osc::launch_fp64_peak(iters, mode, sink, lane_ops,
                                          static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "fp64_peak_kernel");
}

// ---------------------------------------------------------------------------
// Host-pointer forms: the end-to-end path a CPU caller (the reference's own
// Python objects via ctypes) uses.  One cudaMemcpyAsync per buffer.
// ---------------------------------------------------------------------------

namespace {

// Host-pointer form of a batched run.  The batch is cut into chunks that are
// pipelined over a few streams: chunk c's H2D copy, kernels and D2H copy are
// ordered on stream c % S, so copies of one chunk overlap the compute of
// another and consecutive chunks' kernels fill each other's tail waves.
// Sampled runs use a single chunk (their [nsamp][...] layout spans the batch).
int host_run(bool chains, const double *m, const double *C, double *x, double *v, int64_t B,
             int64_t s, double dt, int64_t nsteps, int64_t stride, double *xs, double *vs,
             int64_t *first_bad)
{
    if (int rc = check_run_args(dt, nsteps, stride))
        return rc;
    if (B < 0 || s < 1)
        return fail(OSC_INVALID, "need B >= 0 and s >= 1");
    if (B == 0)
        return OSC_OK;
    if (!m || !C || !x || !v || !first_bad || (!xs) != (!vs))
        return fail(OSC_INVALID, "null buffer");
    retain_pool_memory();
    const size_t cells = static_cast<size_t>(B * s);
    const size_t bytes = cells * sizeof(double);
    const size_t nsamp = xs ? static_cast<size_t>(1 + nsteps / stride) : 0;

    // Chunking, so that only the first chunk's H2D and the last one's D2H are
    // exposed: >= 2 MB of state per chunk, at most 8 chunks; 2-DOF chunks
    // keep >= 148*1024 systems so each launch keeps K1's throughput shape.
    int64_t nchunk = 1;
    if (!xs && B > 1)
        nchunk = std::max<int64_t>(1, std::min<int64_t>({8, B, (int64_t)(bytes >> 21)}));
    if (!chains)
        nchunk = std::max<int64_t>(1, std::min<int64_t>(nchunk, B / (148 * 1024)));
    const int nstream = static_cast<int>(std::min<int64_t>(nchunk, 3));
    cudaStream_t streams[3] = {nullptr, nullptr, nullptr};
    for (int i = 0; i < nstream; ++i)
        OSC_CUDA(cudaStreamCreateWithFlags(&streams[i], cudaStreamNonBlocking));
    struct Cleanup {
        cudaStream_t *st;
        int n;
        void *mem = nullptr;
        ~Cleanup()
        {
            for (int i = 0; i < n; ++i)
                cudaStreamSynchronize(st[i]);  // every stream is done with mem
            if (mem)
                cudaFreeAsync(mem, st[0]);
            for (int i = 0; i < n; ++i) {
                cudaStreamSynchronize(st[i]);
                cudaStreamDestroy(st[i]);
            }
        }
    } cleanup{streams, nstream};

    const size_t total = 4 * bytes + B * sizeof(int64_t) + 2 * nsamp * bytes + 16;
    OSC_CUDA(cudaMallocAsync(&cleanup.mem, total, streams[0]));
    cudaEvent_t ready;
    OSC_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    OSC_CUDA(cudaEventRecord(ready, streams[0]));
    for (int i = 1; i < nstream; ++i)
        OSC_CUDA(cudaStreamWaitEvent(streams[i], ready, 0));
    cudaEventDestroy(ready);

    double *dm = static_cast<double *>(cleanup.mem), *dC = dm + cells, *dx = dC + cells,
           *dv = dx + cells;
    int64_t *dfb = reinterpret_cast<int64_t *>(dv + cells);
    double *dxs = xs ? reinterpret_cast<double *>(dfb + B) : nullptr;
    double *dvs = xs ? dxs + nsamp * cells : nullptr;
    unsigned long long *dworst = reinterpret_cast<unsigned long long *>(
        reinterpret_cast<double *>(dfb + B) + 2 * nsamp * cells);
    const auto H2D = cudaMemcpyHostToDevice;
    const auto D2H = cudaMemcpyDeviceToHost;

    for (int64_t c = 0; c < nchunk; ++c) {
        cudaStream_t st = streams[c % nstream];
        const int64_t b0 = B * c / nchunk, b1 = B * (c + 1) / nchunk, nb = b1 - b0;
        int rc;
        if (chains) {
            // [B][s]: a chunk of chains is one contiguous block per array
            const size_t o = static_cast<size_t>(b0 * s), n = static_cast<size_t>(nb * s) * 8;
            OSC_CUDA(cudaMemcpyAsync(dm + o, m + o, n, H2D, st));
            OSC_CUDA(cudaMemcpyAsync(dC + o, C + o, n, H2D, st));
            OSC_CUDA(cudaMemcpyAsync(dx + o, x + o, n, H2D, st));
            OSC_CUDA(cudaMemcpyAsync(dv + o, v + o, n, H2D, st));
            rc = osc_rk4_chains(dm + o, dC + o, dx + o, dv + o, nb, s, dt, nsteps, stride, dxs,
                                dvs, nullptr, dfb + b0, 0, 0, st);
            if (rc != OSC_OK)
                return rc;
            OSC_CUDA(cudaMemcpyAsync(x + o, dx + o, n, D2H, st));
            OSC_CUDA(cudaMemcpyAsync(v + o, dv + o, n, D2H, st));
        } else {
            // [2][B]: the chunk is packed as its own [2][nb] block on the device
            const size_t o = static_cast<size_t>(2 * b0), n = static_cast<size_t>(nb) * 8;
            const double *hs[4] = {m, C, x, v};
            double *ds[4] = {dm, dC, dx, dv};
            for (int a = 0; a < 4; ++a)
                for (int r = 0; r < 2; ++r)
                    OSC_CUDA(cudaMemcpyAsync(ds[a] + o + r * nb, hs[a] + r * B + b0, n, H2D, st));
            rc = osc_rk4_batch2(dm + o, dC + o, dx + o, dv + o, nb, dt, nsteps, stride, dxs, dvs,
                                nullptr, dfb + b0, 0, st);
            if (rc != OSC_OK)
                return rc;
            for (int r = 0; r < 2; ++r) {
                OSC_CUDA(cudaMemcpyAsync(x + r * B + b0, dx + o + r * nb, n, D2H, st));
                OSC_CUDA(cudaMemcpyAsync(v + r * B + b0, dv + o + r * nb, n, D2H, st));
            }
        }
        OSC_CUDA(cudaMemcpyAsync(first_bad + b0, dfb + b0, nb * sizeof(int64_t), D2H, st));
    }
    if (xs) {
        OSC_CUDA(cudaMemcpyAsync(xs, dxs, nsamp * bytes, D2H, streams[0]));
        OSC_CUDA(cudaMemcpyAsync(vs, dvs, nsamp * bytes, D2H, streams[0]));
    }
    // earliest divergence, reduced on the device once every chunk is done
    for (int i = 1; i < nstream; ++i) {
        cudaEvent_t done;
        OSC_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        OSC_CUDA(cudaEventRecord(done, streams[i]));
        OSC_CUDA(cudaStreamWaitEvent(streams[0], done, 0));
        cudaEventDestroy(done);
    }
    OSC_CUDA(osc::launch_first_bad(dfb, B, dworst, streams[0]));
    unsigned long long worst[2];
    OSC_CUDA(cudaMemcpyAsync(worst, dworst, sizeof worst, D2H, streams[0]));
    for (int i = 0; i < nstream; ++i)
        OSC_CUDA(cudaStreamSynchronize(streams[i]));
    if (worst[0] != ~0ull)
        return fail(OSC_NONFINITE, "integration diverged at step %lld (system %lld)",
                    (long long)worst[0], (long long)worst[1]);
    return OSC_OK;
}

}  // namespace

int osc_rk4_batch2_host(const double *m, const double *C, double *x, double *v, int64_t B,
                        double dt, int64_t nsteps, int64_t stride, double *xs, double *vs,
                        int64_t *first_bad)
{
    return host_run(false, m, C, x, v, B, 2, dt, nsteps, stride, xs, vs, first_bad);
}

int osc_rk4_chains_host(const double *m, const double *C, double *x, double *v, int64_t B,
                        int64_t s, double dt, int64_t nsteps, int64_t stride, double *xs,
                        double *vs, int64_t *first_bad)
{
    return host_run(true, m, C, x, v, B, s, dt, nsteps, stride, xs, vs, first_bad);
}

// ---------------------------------------------------------------------------
// Stream-ordered 64-bit counters (cross-process ordering in the GPU front-end)
// ---------------------------------------------------------------------------
namespace {

using StreamValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

// Driver entry points resolved through the runtime, so the library does not
// link libcuda (it must load on machines without a driver for the CPU tests).
StreamValueFn driver_fn(const char *name)
{
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return reinterpret_cast<StreamValueFn>(p);
}

}  // namespace

int osc_stream_write_u64(void *stream, void *addr, uint64_t value)
{
    static const StreamValueFn f = driver_fn("cuStreamWriteValue64");
    if (!addr)
        return fail(OSC_INVALID, "null counter");
    if (!f)
        return fail(OSC_CUDA_ERROR, "cuStreamWriteValue64 is not available");
    // default flags: a system-scope fence orders all prior work of the stream
    // (the kernel's peer stores included) before the store
    const CUresult r = f(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr), value,
                         CU_STREAM_WRITE_VALUE_DEFAULT);
    return r == CUDA_SUCCESS ? OSC_OK
                             : fail(OSC_CUDA_ERROR, "cuStreamWriteValue64 failed (%d)", int(r));
}

int osc_stream_wait_u64(void *stream, const void *addr, uint64_t value)
{
    static const StreamValueFn f = driver_fn("cuStreamWaitValue64");
    static int flush = -1;  // does the device take CU_STREAM_WAIT_VALUE_FLUSH?
    if (!addr)
        return fail(OSC_INVALID, "null counter");
    if (!f)
        return fail(OSC_CUDA_ERROR, "cuStreamWaitValue64 is not available");
    const CUstream st = static_cast<CUstream>(stream);
    const CUdeviceptr a = reinterpret_cast<CUdeviceptr>(addr);
    if (flush != 0) {
        // GEQ + flush of outstanding remote (peer) writes into this device
        const CUresult r = f(st, a, value, CU_STREAM_WAIT_VALUE_GEQ | CU_STREAM_WAIT_VALUE_FLUSH);
        if (r == CUDA_SUCCESS) {
            flush = 1;
            return OSC_OK;
        }
        if (flush == 1)
            return fail(OSC_CUDA_ERROR, "cuStreamWaitValue64 failed (%d)", int(r));
        flush = 0;  // not supported here: plain GEQ (the writer's fence orders its stores)
    }
    const CUresult r = f(st, a, value, CU_STREAM_WAIT_VALUE_GEQ);
    return r == CUDA_SUCCESS ? OSC_OK
                             : fail(OSC_CUDA_ERROR, "cuStreamWaitValue64 failed (%d)", int(r));
}

// ---------------------------------------------------------------------------
// One chain sharded over the GPUs of this process, fused halo exchange.
// ---------------------------------------------------------------------------
namespace {

struct ShardRes {
    int dev = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    double *m = nullptr, *C = nullptr, *x = nullptr, *v = nullptr, *x2 = nullptr, *v2 = nullptr;
    int64_t *fb = nullptr;
    int64_t blo = 0, n = 0, own_lo = 0, own_hi = 0;
};

struct ShardSet {
    std::vector<ShardRes> sh;
    ~ShardSet()
    {
        for (auto &r : sh) {
            cudaSetDevice(r.dev);
            if (r.st)
                cudaStreamSynchronize(r.st);
        }
        for (auto &r : sh) {
            cudaSetDevice(r.dev);
            for (void *p : {(void *)r.m, (void *)r.C, (void *)r.x, (void *)r.v, (void *)r.x2,
                            (void *)r.v2, (void *)r.fb})
                if (p)
                    cudaFree(p);
            for (auto e : r.ev)
                if (e)
                    cudaEventDestroy(e);
            if (r.st)
                cudaStreamDestroy(r.st);
        }
    }
};

}  // namespace

int osc_rk4_chain_sharded(int ngpu, const int *devs, const double *m, const double *C, double *x,
                          double *v, int64_t s, double dt, int64_t nsteps, int64_t halo_steps,
                          int64_t *first_bad, uint32_t flags)
{
    if (flags & ~uint32_t(OSC_FMA))
        return fail(OSC_INVALID, "unknown flags 0x%x", flags);
    if (int rc = check_run_args(dt, nsteps, 1))
        return rc;
    if (ngpu < 1 || !devs)
        return fail(OSC_INVALID, "need ngpu >= 1 devices");
    if (s < 1 || !m || !C || !x || !v || !first_bad)
        return fail(OSC_INVALID, "need s >= 1 and non-null buffers");
    const int64_t T = halo_steps > 0 ? halo_steps : kDefaultHaloSteps;
    const int64_t g = 2 * T;  // ghost cells per interior side (dependency radius 2/step)
    if (4 + 2 * g >= kTile)
        return fail(OSC_INVALID, "halo_steps=%lld too deep for a %lld-cell tile", (long long)T,
                    (long long)kTile);
    int count = 0;
    OSC_CUDA(cudaGetDeviceCount(&count));
    for (int i = 0; i < ngpu; ++i)
        if (devs[i] < 0 || devs[i] >= count)
            return fail(OSC_INVALID, "device %d out of range (%d devices)", devs[i], count);
    if (ngpu > 1 && s / ngpu < g)
        return fail(OSC_INVALID, "shards of %lld cells are narrower than the %lld-cell ghost zone",
                    (long long)(s / ngpu), (long long)g);
    int prev = 0;
    cudaGetDevice(&prev);
    struct Restore {
        int d;
        ~Restore() { cudaSetDevice(d); }
    } restore{prev};

    ShardSet set;
    set.sh.resize(ngpu);
    const size_t D = sizeof(double);
    for (int i = 0; i < ngpu; ++i) {
        ShardRes &r = set.sh[i];
        r.dev = devs[i];
        const int64_t lo = s * i / ngpu, hi = s * (i + 1) / ngpu;
        r.blo = i > 0 ? lo - g : 0;
        const int64_t bhi = i + 1 < ngpu ? hi + g : s;
        r.n = bhi - r.blo;
        r.own_lo = lo - r.blo;
        r.own_hi = hi - r.blo;
        OSC_CUDA(cudaSetDevice(r.dev));
        OSC_CUDA(cudaStreamCreateWithFlags(&r.st, cudaStreamNonBlocking));
        for (auto &e : r.ev)
            OSC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (double **p : {&r.m, &r.C, &r.x, &r.v, &r.x2, &r.v2})
            OSC_CUDA(cudaMalloc(reinterpret_cast<void **>(p), r.n * D));
        OSC_CUDA(cudaMalloc(reinterpret_cast<void **>(&r.fb), sizeof(int64_t)));
        OSC_CUDA(cudaMemsetAsync(r.fb, 0, sizeof(int64_t), r.st));
        OSC_CUDA(cudaMemcpyAsync(r.m, m + r.blo, r.n * D, cudaMemcpyHostToDevice, r.st));
        OSC_CUDA(cudaMemcpyAsync(r.C, C + r.blo, r.n * D, cudaMemcpyHostToDevice, r.st));
        OSC_CUDA(cudaMemcpyAsync(r.x, x + r.blo, r.n * D, cudaMemcpyHostToDevice, r.st));
        OSC_CUDA(cudaMemcpyAsync(r.v, v + r.blo, r.n * D, cudaMemcpyHostToDevice, r.st));
        // the ghost zones of both ping-pong buffers start as the same input
        OSC_CUDA(cudaMemcpyAsync(r.x2, x + r.blo, r.n * D, cudaMemcpyHostToDevice, r.st));
        OSC_CUDA(cudaMemcpyAsync(r.v2, v + r.blo, r.n * D, cudaMemcpyHostToDevice, r.st));
        OSC_CUDA(cudaEventRecord(r.ev[1], r.st));  // "period -1" done: the uploads
    }
    // neighbours on other devices store into each other's memory over NVLink
    for (int i = 0; i + 1 < ngpu; ++i) {
        const int a = set.sh[i].dev, b = set.sh[i + 1].dev;
        if (a == b)
            continue;
        for (auto [p, q] : {std::pair<int, int>{a, b}, std::pair<int, int>{b, a}}) {
            int ok = 0;
            OSC_CUDA(cudaDeviceCanAccessPeer(&ok, p, q));
            if (!ok)
                return fail(OSC_CUDA_ERROR, "device %d cannot access device %d (no P2P)", p, q);
            OSC_CUDA(cudaSetDevice(p));
            const cudaError_t e = cudaDeviceEnablePeerAccess(q, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled)
                cudaGetLastError();
            else if (e != cudaSuccess)
                return cuda_fail(e, "cudaDeviceEnablePeerAccess");
        }
    }

    for (int64_t k = 0, p = 0; k < nsteps; ++p) {
        const int64_t n = std::min(T, nsteps - k);
        for (int i = 0; i < ngpu; ++i) {
            ShardRes &r = set.sh[i];
            OSC_CUDA(cudaSetDevice(r.dev));
            // our period p writes the neighbours' next-input ghosts, which
            // their period p-1 produced the buffer for and finished reading
            for (int j : {i - 1, i + 1})
                if (j >= 0 && j < ngpu)
                    OSC_CUDA(cudaStreamWaitEvent(r.st, set.sh[j].ev[(p + 1) % 2], 0));
            osc_peer_t left{}, right{};
            if (i > 0) {
                const ShardRes &l = set.sh[i - 1];
                left = osc_peer_t{l.x2, l.v2, r.blo - l.blo, g};
            }
            if (i + 1 < ngpu) {
                const ShardRes &q = set.sh[i + 1];
                right = osc_peer_t{q.x2, q.v2, r.blo - q.blo, g};
            }
            if (int rc = osc_rk4_chain_advance(r.m, r.C, r.x, r.v, r.x2, r.v2, r.n, r.own_lo,
                                               r.own_hi, dt, n, k, r.fb,
                                               i > 0 ? &left : nullptr,
                                               i + 1 < ngpu ? &right : nullptr, flags, r.st))
                return rc;
            OSC_CUDA(cudaEventRecord(r.ev[p % 2], r.st));
        }
        for (auto &r : set.sh) {
            std::swap(r.x, r.x2);
            std::swap(r.v, r.v2);
        }
        k += n;
    }
    int64_t worst = 0;
    for (int i = 0; i < ngpu; ++i) {
        ShardRes &r = set.sh[i];
        OSC_CUDA(cudaSetDevice(r.dev));
        for (int j : {i - 1, i + 1})  // no neighbour still stores into our buffers
            if (j >= 0 && j < ngpu) {
                OSC_CUDA(cudaStreamWaitEvent(r.st, set.sh[j].ev[0], 0));
                OSC_CUDA(cudaStreamWaitEvent(r.st, set.sh[j].ev[1], 0));
            }
        const int64_t len = r.own_hi - r.own_lo;
        OSC_CUDA(cudaMemcpyAsync(x + r.blo + r.own_lo, r.x + r.own_lo, len * D,
                                 cudaMemcpyDeviceToHost, r.st));
        OSC_CUDA(cudaMemcpyAsync(v + r.blo + r.own_lo, r.v + r.own_lo, len * D,
                                 cudaMemcpyDeviceToHost, r.st));
        int64_t fb = 0;
        OSC_CUDA(cudaMemcpyAsync(&fb, r.fb, sizeof fb, cudaMemcpyDeviceToHost, r.st));
        OSC_CUDA(cudaStreamSynchronize(r.st));
        if (fb > 0 && (worst == 0 || fb < worst))
            worst = fb;
    }
    *first_bad = worst;
    if (worst)
        return fail(OSC_NONFINITE, "integration diverged at step %lld", (long long)worst);
    return OSC_OK;
}

}  // extern "C"
