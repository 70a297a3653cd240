// Internal helpers shared by the C-ABI translation units (capi*.cu): the
// per-thread last error, argument checks the reference makes, the chain
// launch plan, stream-ordered scratch.  Not part of the public ABI
// (include/osc_b200.h is).
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <utility>
#include <vector>

#include "../../include/osc_b200.h"
#include "osc_kernels.h"

namespace osc_capi {

inline thread_local std::string g_last_error;  // one per thread, shared by every capi_*.cu
// The offending parameter of the calling thread's last error, when it was a
// parameter-rule violation (osc_last_invalid_parameter); which = -1 otherwise.
inline thread_local int g_bad_param_which = -1;
inline thread_local int64_t g_bad_param_index = -1;

inline int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
inline int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    g_bad_param_which = -1;
    g_bad_param_index = -1;
    return code;
}

inline int cuda_fail(cudaError_t e, const char *where)
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
inline int check_run_args(double dt, int64_t nsteps, int64_t stride)
{
    if (!(std::isfinite(dt) && dt > 0.0))
        return fail(OSC_INVALID, "dt must be positive and finite, got %.17g", dt);
    if (nsteps < 1)
        return fail(OSC_INVALID, "nsteps must be >= 1, got %lld", (long long)nsteps);
    if (stride < 1)
        return fail(OSC_INVALID, "stride must be >= 1, got %lld", (long long)stride);
    return OSC_OK;
}

// Flags every integrate entry point accepts (osc_rk4_chain_advance also
// takes the tile subsets).
constexpr uint32_t kRunFlags = OSC_FMA | OSC_TRUSTED;
constexpr uint32_t kAdvanceFlags = kRunFlags | OSC_TILES_INTERIOR | OSC_TILES_EDGES;

// How a flat parameter index maps to (system, cell) for the error message:
// CellMajor = [s][B] (the batched 2-DOF SoA [2][B]: coordinate i / B of
// system i % B), Chains = [B][s] (cell i % s of chain i / s).
enum class ParamLayout { Flat, CellMajor, Chains };

// One device pass of OscillatorSystem's rule (oscillator.py:75-80) over n
// masses and n spring rates; bad[0] / bad[1] = the smallest offending mass /
// spring index, -1 if none.  Synchronises `stream`.
inline int scan_params(const double *m, const double *C, int64_t n, cudaStream_t stream,
                       int64_t bad[2])
{
    bad[0] = bad[1] = -1;
    if (n <= 0)
        return OSC_OK;
    unsigned long long *d = nullptr;
    OSC_CUDA(osc::scratch_alloc(reinterpret_cast<void **>(&d), 2 * sizeof *d, stream));
    unsigned long long h[2] = {~0ull, ~0ull};
    cudaError_t e = osc::launch_param_check(m, C, n, d, stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, stream);
    cudaFreeAsync(d, stream);
    if (e == cudaSuccess)
        e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess)
        return cuda_fail(e, "param_check_kernel");
    for (int w = 0; w < 2; ++w)
        bad[w] = h[w] == ~0ull ? -1 : static_cast<int64_t>(h[w]);
    return OSC_OK;
}

// OSC_INVALID naming parameter `which` (0 masses, 1 springs) at flat index
// gi with value val; recorded for osc_last_invalid_parameter.
inline int param_fail(int which, int64_t gi, double val, ParamLayout layout, int64_t B,
                      int64_t s)
{
    const char *label = which ? "springs" : "masses";
    if (layout == ParamLayout::CellMajor)
        fail(OSC_INVALID, "%s[%lld] = %.17g; must be positive and finite (system %lld)", label,
             (long long)(gi / B), val, (long long)(gi % B));
    else if (layout == ParamLayout::Chains)
        fail(OSC_INVALID, "%s[%lld] = %.17g; must be positive and finite (chain %lld)", label,
             (long long)(gi % s), val, (long long)(gi / s));
    else
        fail(OSC_INVALID, "%s[%lld] = %.17g; must be positive and finite", label,
             (long long)gi, val);
    g_bad_param_which = which;
    g_bad_param_index = gi;
    return OSC_INVALID;
}

// Host-side twin for the host-pointer entry points: once the device pass has
// found an offender, the exact first one in the caller's own layout (masses
// before springs, lowest index) is located in the caller's host arrays.
inline int host_param_fail(const double *m, const double *C, int64_t n, ParamLayout layout,
                           int64_t B = 0, int64_t s = 0)
{
    for (int w = 0; w < 2; ++w) {
        const double *a = w ? C : m;
        for (int64_t i = 0; i < n; ++i)
            if (!(a[i] > 0.0 && a[i] <= DBL_MAX))
                return param_fail(w, i, a[i], layout, B, s);
    }
    return fail(OSC_CUDA_ERROR, "parameter check: device and host copies disagree");
}

// The check every entry point taking device m, C makes before integrating:
// one coalesced pass, then a synchronisation of `stream` so the call returns
// OSC_INVALID before enqueuing any work.  Masses are checked before springs,
// lowest index first -- the reference's order for one system.
inline int check_params(const double *m, const double *C, int64_t n, cudaStream_t stream,
                        ParamLayout layout = ParamLayout::Flat, int64_t B = 0, int64_t s = 0)
{
    int64_t bad[2];
    if (int rc = scan_params(m, C, n, stream, bad))
        return rc;
    const int which = bad[0] >= 0 ? 0 : (bad[1] >= 0 ? 1 : -1);
    if (which < 0)
        return OSC_OK;
    double val = 0.0;
    OSC_CUDA(cudaMemcpyAsync(&val, (which ? C : m) + bad[which], sizeof val,
                             cudaMemcpyDeviceToHost, stream));
    OSC_CUDA(cudaStreamSynchronize(stream));
    return param_fail(which, bad[which], val, layout, B, s);
}

inline osc::StepConsts consts(double dt)
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

inline void pick_whole(int64_t s, int &K, int &threads)
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
inline int64_t pick_halo_steps(int64_t s, int64_t B, int64_t nsteps)
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
inline bool env_shape(const char *name, int &K, int &threads)
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
inline int plan_chain(int64_t s, int64_t B, int64_t nsteps, int64_t halo_steps, ChainPlan &p)
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
        if (const char *e = std::getenv("OSC_WHOLE_STEPS"))  // benchmarking knob
            p.per_launch = std::max<int64_t>(1, std::atoll(e));
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

// The edge-tile sets of a sharded launch (osc::EdgeSync::nedge): how many
// leading tiles read the left ghost zone or store into the left neighbour,
// and how many trailing tiles do so on the right.  Tile geometry as the
// kernels compute it (k_chain.cu tile_geom / chain_rk4_kernel): owned
// [own_lo + t*W, +W), input from own_start - H (clamped at 0; slid left to
// end at the buffer end when the tile fits the buffer).  Both sets are
// contiguous because own_start grows with t.
inline void edge_sets(const osc::SegArgs &g, int64_t TILE, int64_t nedge[2])
{
    auto input = [&](int64_t t, int64_t &L, int64_t &end, int64_t &os, int64_t &oe) {
        os = g.own_lo + t * g.W;
        oe = std::min(os + g.W, g.own_hi);
        L = std::max<int64_t>(0, os - g.H);
        if (TILE <= g.n && L + TILE > g.n)
            L = g.n - TILE;
        end = std::min(L + TILE, g.n);
    };
    auto involved = [&](int64_t t, int side) {
        int64_t L, end, os, oe;
        input(t, L, end, os, oe);
        const osc::PeerGhost &p = g.peer[side];
        const bool writes = p.x && os < p.hi && oe > p.lo;
        const bool reads = side == 0 ? L < g.own_lo : end > g.own_hi;
        return writes || reads;
    };
    nedge[0] = nedge[1] = 0;
    for (int side = 0; side < 2; ++side) {
        if (side == 0 ? g.own_lo == 0 : g.own_hi == g.n)
            continue;  // no ghost zone on this side: a true chain end
        auto tile_at = [&](int64_t i) { return side == 0 ? i : g.tiles - 1 - i; };
        // the run of involved tiles from this side's end (own_start grows with
        // the tile, so the involvement of ordinary tiles ends with the run) ...
        int64_t k = 0;
        while (k < g.tiles && involved(tile_at(k), side))
            ++k;
        // ... except on tiny shards, where the slid last tile or a padded
        // first tile can reach the far ghost zone: then every tile counts
        for (int64_t i = std::max(k, g.tiles - 2); i < g.tiles; ++i)
            if (involved(tile_at(i), side))
                k = g.tiles;
        nedge[side] = k;
    }
}

// osc_rk4_batch2 with a shape hint (capi.cu): shares_gpu = the caller runs
// several batches side by side.
int batch2_entry(const double *m, const double *C, double *x, double *v, int64_t B, double dt,
                 int64_t nsteps, int64_t stride, double *xs, double *vs, double *es,
                 int64_t *first_bad, uint32_t flags, void *stream, bool shares_gpu);

struct Scratch {
    double *p = nullptr;
    cudaStream_t s = nullptr;
    ~Scratch()
    {
        if (p)
            cudaFreeAsync(p, s);
    }
};

}  // namespace osc_capi
