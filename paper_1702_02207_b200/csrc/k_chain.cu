// K2/K3 chain_rk4: wall-anchored spring chains (BASELINE configs 2-3).
//
// Restates rk4_step (oscillator.py:194-231) for a chain of n cells, spring i
// joining cell i to cell i-1, spring 0 to the wall, the last cell free
// (oscillator.py:3-5, 152-164).  One CTA owns a TILE of blockDim*K
// contiguous cells, K per thread, all in registers; the four stage
// evaluations of a step exchange one neighbour position per thread edge
// (each thread's {first, last} position in a double-buffered shared-memory
// slot, one __syncthreads -- the on-chip form of the reference engine's
// per-stage StageBarrier, parallel.py:174-255).  Exact runs divide in two
// operations warp by warp (div2_chain_consts table; osc_device.cuh).
//
// Two launch shapes use the same kernel:
//   * whole-chain (K2, config 3): the tile is the whole chain (H = 0), so
//     both ends are the true wall / free end.
//   * temporally blocked (K3, config 2): tiles own W cells plus an H = 2T
//     halo each side and advance T steps per launch.  A step's dependency
//     radius is 2 cells of x and v, so after T steps the owned
//     cells are exact; tile edges that are not chain ends are treated as a
//     wall / free end, and the garbage this creates never reaches the owned
//     cells.  Ping-pong buffers: each launch reads (xin,vin) and writes only
//     owned cells of (xout,vout).
//
// Forces: f_i = C_i*d_i with d_i = x_i - x_{i-1} (d_0 = x_0 - 0.0 == x_0);
//   a_i = (f_{i+1} - f_i)/m_i, last cell a = (-f_i)/m_i.  This is the
//   reference's RN(RN(-C_i*left) + RN(C_{i+1}*(x_{i+1}-x_i)))/m_i term for
//   term, since (-C)*d == -(C*d) exactly and IEEE addition commutes.
#include "osc_device.cuh"
#include "osc_kernels.h"

#include <algorithm>
#include <atomic>
#include <cstdlib>

namespace osc {
namespace {

constexpr int kMaxDevices = 64;
#ifndef OSC_PERSIST_BUFS
#define OSC_PERSIST_BUFS 3
#endif
constexpr int kPersistBufs = OSC_PERSIST_BUFS;  // tile buffers of the persistent kernel (see there)
static_assert(kPersistBufs == 2 || kPersistBufs == 3, "2 or 3 tile buffers");

template <int K>
struct Tile {
    double C[K];
    Divisor md[K];
    double Cn;     // spring of the first cell of the next thread
    int lastj;     // index of the tile's last cell if this thread owns it, else -1
    int validn;    // cells of this thread inside the tile (pad variant)
    bool first;    // this thread's cell 0 is the tile's first cell (wall side)
    bool last;     // this thread's cell K-1 is the tile's last cell (free side)
    int pr_off;    // byte offset in a stage's slot row of the value read as the right neighbour
};

// Thread-edge exchange slots, double-buffered by stage parity (compile-time:
// a step has four stages, so parity restarts at 0 every step).  Slot t + 1
// holds thread t's {first, last} stage position; slot 0 stays {0.0, 0.0}:
// the tile's first cell then reads x_{-1} = 0.0 and d_0 = x_0 - 0.0 == x_0
// exactly (also for x_0 = -0.0), with no select.  One 16-byte store, one
// barrier and two 8-byte loads per stage replace the warp shuffles plus the
// per-warp edge slots of round 1 (the chain kernels are issue-bound: ncu
// shows their time proportional to instructions issued; 8 -> 3 exchange
// instructions per stage).
template <int NT>
struct Edges {
    double2 v[2][NT + 2];
};

// acceleration_at for the K cells of this thread at positions p.  kPad: the
// tile extends past the buffer end, so cells >= validn are padding whose
// numerators are replaced by 1.0 (they never feed a real cell: the last real
// cell has no right neighbour) to keep them off the slow division path.
template <int K, bool kPad, Arith A, int B, int NT>
__device__ __forceinline__ void accel(const Tile<K> &t, const double (&p)[K], double (&a)[K],
                                      Edges<NT> &e, bool &ok)
{
    e.v[B][threadIdx.x + 1] = make_double2(p[0], p[K - 1]);
    __syncthreads();
    const double pl = e.v[B][threadIdx.x].y;      // left neighbour's last, or the 0.0 slot
    // right neighbour's first position; the last thread reads its own last
    // one (t.pr_off), so that with t.Cn = -0.0 its fr is exactly -0.0 and
    // the free end's numerator (-0.0) - f needs no select (see below)
    const double pr = *reinterpret_cast<const double *>(
        reinterpret_cast<const char *>(&e.v[B][0]) + t.pr_off);
    double f[K];
    f[0] = mul(t.C[0], sub(p[0], pl));
#pragma unroll
    for (int j = 1; j < K; ++j)
        f[j] = mul(t.C[j], sub(p[j], p[j - 1]));
    const double fr = mul(t.Cn, sub(pr, p[K - 1]));
    // Fast2C: the significand tests accumulate in their own flag, merged once
    // per stage, so they form a chain of their own beside the quotient tests
    // instead of doubling the length of one serial predicate chain.
    bool okb = true;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        double num;
        // The free end's numerator -f is formed as (-0.0) - f: bit for bit
        // -f (also for f = +-0), selected as an operand so no separate
        // negation is issued.
        if constexpr (kPad) {
            const double fnext = (j + 1 < K) ? f[j + 1] : fr;
            num = sub((j == t.lastj) ? -0.0 : fnext, f[j]);
            num = (j < t.validn) ? num : 1.0;
        } else if (j + 1 < K) {
            num = sub(f[j + 1], f[j]);
        } else if constexpr (A == Arith::Exact) {
            num = sub(t.last ? -0.0 : fr, f[j]);
        } else {
            // The last thread's fr = (-0.0)*(p - p) is -0.0 for a finite p,
            // so this is (-0.0) - f bit for bit.  A non-finite p makes the
            // cell non-finite in the reference too: the chunk is replayed
            // with the literal select above.
            num = sub(fr, f[j]);
        }
        if constexpr (A == Arith::Fast2C)
            a[j] = div2c_fast2(num, t.md[j], ok, okb);
        else
            a[j] = qdiv<A>(num, t.md[j], ok);
    }
    if constexpr (A == Arith::Fast2C)
        ok &= okb;
}

// A buffer whose divergence was recorded in an EARLIER launch (first_bad <=
// step0) is skipped: integrate has raised, its state is unspecified.  A step
// recorded during this launch by another tile must not skip this one, which
// may hold an earlier step of the same launch (tiles run in any order).
__device__ __forceinline__ bool diverged_before(const SegArgs &g, int64_t buf)
{
    const int64_t fb = g.first_bad[buf];
    return fb != 0 && fb <= g.step0;
}

// ---------------------------------------------------------------------------
// Edge-tile ordering with the neighbouring shards (EdgeSync, the fused
// exchange of the multi-process peer transport).  Only the tiles next to a
// ghost zone depend on a neighbour: they read ghosts the neighbour's previous
// period stored into our buffer and store our boundary cells into the buffer
// the neighbour reads next.  So the interior tiles run first without any
// ordering, and each edge tile's thread 0 waits -- bounded, on the device --
// until the neighbour's edge counter shows its previous period's edge done;
// the last edge tile of a side then posts ours.  In steady state the wait is
// already satisfied when an edge tile comes up; a neighbour that stops
// making progress turns into a timeout record instead of a hang.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p)
{
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Position `it` of a buffer's tile walk -> tile index: with edge sync the
// interior tiles first, then the left-edge set, then the right-edge set.
__device__ __forceinline__ int64_t tile_order(const SegArgs &g, int64_t it)
{
    if (!g.ordered)
        return it;
    const int64_t a = g.nedge[0], b = g.nedge[1];
    const int64_t rs = max(a, g.tiles - b);  // first tile of the right set
    const int64_t nint = rs - a;              // interior tiles (>= 0)
    if (it < nint)
        return a + it;
    const int64_t j = it - nint;
    return j < a ? j : rs + (j - a);
}

// Bit 0: the tile involves the left neighbour, bit 1: the right one.
__device__ __forceinline__ int edge_sides(const SegArgs &g, int64_t tile)
{
    if (!g.sync.ctr)
        return 0;
    return (tile < g.nedge[0] ? 1 : 0) | (tile >= g.tiles - g.nedge[1] ? 2 : 0);
}

// Thread 0, before an edge tile touches its inputs: wait until each involved
// neighbour's counter reaches `period`.  After timeout_ns the first waiter
// records {1, period, side, value seen} in ctr[4..7]; from then on nobody
// waits (the launch drains, its results are garbage, the host raises).
__device__ void edge_wait(const EdgeSync &s, int sides)
{
    for (int side = 0; side < 2; ++side) {
        const uint64_t *r = s.ready[side];
        if (!((sides >> side) & 1) || !r)
            continue;
        uint64_t t0 = 0;
        for (uint32_t spin = 0;; ++spin) {
            const uint64_t c = ld_acquire_sys(r);
            if (static_cast<int64_t>(c - s.period) >= 0)
                break;
            if (*reinterpret_cast<volatile uint64_t *>(&s.ctr[4]) != 0)
                break;  // a wait has already timed out: drain
            const uint64_t now = globaltimer_ns();
            if (spin == 0) {
                t0 = now;
            } else if (static_cast<int64_t>(now - t0) > s.timeout_ns) {
                auto *flag = reinterpret_cast<unsigned long long *>(&s.ctr[4]);
                if (atomicCAS(flag, 0ull, 1ull) == 0ull) {
                    s.ctr[5] = s.period;
                    s.ctr[6] = static_cast<uint64_t>(side);
                    s.ctr[7] = c;
                    __threadfence_system();
                }
                break;
            }
            __nanosleep(128);
        }
    }
    // the bulk (async-proxy) reads that follow must see the peers' stores
    asm volatile("fence.proxy.async;" ::: "memory");
}

// Thread 0, after every thread of an edge tile has stored (and fenced) its
// cells: count the tile; the last edge tile of a side resets the tally for
// the next launch and posts period + 1.
__device__ void edge_done(const SegArgs &g, int sides)
{
    const EdgeSync &s = g.sync;
    for (int side = 0; side < 2; ++side) {
        if (!((sides >> side) & 1) || g.nedge[side] == 0)
            continue;
        unsigned long long old;
        asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;"
                     : "=l"(old)
                     : "l"(&s.ctr[2 + side])
                     : "memory");
        if (static_cast<int64_t>(old) + 1 == g.nedge[side]) {
            s.ctr[2 + side] = 0;  // the next launch is stream-ordered after this one
            __threadfence_system();
            st_release_sys(&s.ctr[side], s.period + 1);
        }
    }
}

// Zero every slot (sentinels included); callers then __syncthreads().
template <int NT>
__device__ __forceinline__ void edges_init(Edges<NT> &e)
{
    for (int i = threadIdx.x; i < 2 * (NT + 2); i += blockDim.x)
        (&e.v[0][0])[i] = make_double2(0.0, 0.0);
}

// One classical RK4 step (oscillator.py:208-231) of the thread's K cells.
template <int K, bool kPad, Arith A, int NT>
__device__ __forceinline__ void step(const Tile<K> &t, double (&x)[K], double (&v)[K],
                                     const StepConsts &k, Edges<NT> &e, bool &ok)
{
    double a[K], yp[K], yv[K], sx[K], sv[K];
    if constexpr (A != Arith::Exact && A != Arith::Fma) {
#pragma unroll
        for (int j = 0; j < K; ++j)
            ok &= velocity_small(v[j]);  // add_twice_fused's condition
    }
    accel<K, kPad, A, 0>(t, x, a, e, ok);  // k1
#pragma unroll
    for (int j = 0; j < K; ++j) {
        sx[j] = v[j];
        sv[j] = a[j];
        yp[j] = stage<A>(x[j], k.half_dt, v[j]);
        yv[j] = stage<A>(v[j], k.half_dt, a[j]);
    }
    accel<K, kPad, A, 1>(t, yp, a, e, ok);  // k2
#pragma unroll
    for (int j = 0; j < K; ++j) {
        sx[j] = add_twice_fused<A>(sx[j], yv[j]);
        sv[j] = add_twice<A>(sv[j], a[j]);
        yp[j] = stage<A>(x[j], k.half_dt, yv[j]);
        yv[j] = stage<A>(v[j], k.half_dt, a[j]);
    }
    accel<K, kPad, A, 0>(t, yp, a, e, ok);  // k3
#pragma unroll
    for (int j = 0; j < K; ++j) {
        sx[j] = add_twice_fused<A>(sx[j], yv[j]);
        sv[j] = add_twice<A>(sv[j], a[j]);
        yp[j] = stage<A>(x[j], k.dt, yv[j]);
        yv[j] = stage<A>(v[j], k.dt, a[j]);
    }
    accel<K, kPad, A, 1>(t, yp, a, e, ok);  // k4
#pragma unroll
    for (int j = 0; j < K; ++j) {
        sx[j] = add(sx[j], yv[j]);
        sv[j] = add(sv[j], a[j]);
        x[j] = stage<A>(x[j], k.dt6, sx[j]);
        v[j] = stage<A>(v[j], k.dt6, sv[j]);
    }
}

// Does owned range [lo, hi) store anything into a neighbour's ghost zone?
// Uniform per tile: the per-cell range tests below run only where it does
// (the edge tiles of a sharded run), not in every tile of every launch.
__device__ __forceinline__ bool touches_peer(const SegArgs &g, int64_t lo, int64_t hi)
{
    return (g.peer[0].x && lo < g.peer[0].hi && hi > g.peer[0].lo) ||
           (g.peer[1].x && lo < g.peer[1].hi && hi > g.peer[1].lo);
}

// Neighbour ghost copies of an owned cell c (the fused exchange of the peer
// transport): straight into the neighbour's next-input buffer.
__device__ __forceinline__ void store_peers(const SegArgs &g, int64_t c, double x, double v)
{
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        const PeerGhost &p = g.peer[side];
        if (p.x && c >= p.lo && c < p.hi) {
            p.x[c + p.offset] = x;
            p.v[c + p.offset] = v;
        }
    }
}

template <int K>
__device__ __forceinline__ void load_state(const SegArgs &g, int64_t base, int64_t c0,
                                           int64_t cend, double (&x)[K], double (&v)[K])
{
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int64_t c = c0 + j;
        x[j] = c < cend ? g.xin[base + c] : 0.0;
        v[j] = c < cend ? g.vin[base + c] : 0.0;
    }
}

template <int K>
__device__ __forceinline__ bool owned_bad(const double (&x)[K], const double (&v)[K], int64_t c0,
                                          int64_t own_start, int64_t own_end)
{
    bool bad = false;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int64_t c = c0 + j;
        if (c >= own_start && c < own_end)
            bad |= !(finite(x[j]) & finite(v[j]));
    }
    return bad;
}

// Register budget: K cells x ~10 live doubles per thread.
template <int K>
constexpr int max_threads() { return K <= 1 ? 1024 : K <= 4 ? 512 : 256; }

// K * kMaxT = 1024 (K = 8 x 128 threads -- C4 -- or K = 4 x 256): two CTAs
// per SM promised to ptxas, which then keeps the single-test division's
// loop free of rematerialised indices; these builds divide with div_fastq
// (one FSETP per division).  The wider builds keep div_fast
// (profiles/r01/README.md).
// kD2: the two-operation division from the SegArgs table (non-padded
// tiles; see chain_tiles_persistent for the warp-by-warp choice).
template <int K, bool kPad, bool kFma, int kMaxT = max_threads<K>(), bool kD2 = false>
__global__ void __launch_bounds__(kMaxT, (K >= 4 && K * kMaxT == 1024) ? 2 : 1)
    chain_rk4_kernel(SegArgs g)
{
    static_assert(!(kD2 && (kPad || kFma)), "two-operation build: exact, unpadded tiles");
    constexpr bool kQ = K * kMaxT == 1024 && K >= 4;
    __shared__ Edges<kMaxT> edges;
    __shared__ int s_skip;
    const int64_t nw = walk_tiles(g);
    const int64_t buf_id = blockIdx.x / nw;
    const int64_t tile = tile_order(g, g.walk0 + blockIdx.x % nw);
    const int sides = edge_sides(g, tile);
    // One read, broadcast: another CTA may record a divergence at any time,
    // and the exit must be uniform across this CTA's barriers.
    edges_init(edges);
    if (threadIdx.x == 0) {
        s_skip = diverged_before(g, buf_id);
        if (sides && !s_skip)
            edge_wait(g.sync, sides);
    }
    __syncthreads();
    if (s_skip) {
        if (threadIdx.x == 0 && sides)
            edge_done(g, sides);  // nothing stored, but the neighbours must not stall
        return;  // already diverged: state is unspecified, as integrate raised
    }

    const int64_t TILE = static_cast<int64_t>(blockDim.x) * K;
    const int64_t own_start = g.own_lo + tile * g.W;
    const int64_t own_end = min(own_start + g.W, g.own_hi);
    int64_t L = max(static_cast<int64_t>(0), own_start - g.H);
    if (!kPad && L + TILE > g.n)
        L = g.n - TILE;  // slide the last tile left so it ends at the buffer end: no padding
    const int64_t cend = min(L + TILE, g.n);  // one past the tile's last cell
    const int64_t base = buf_id * g.n;
    const int64_t c0 = L + static_cast<int64_t>(threadIdx.x) * K;

    Tile<K> t;
    t.first = threadIdx.x == 0;
    t.last = threadIdx.x == blockDim.x - 1;
    t.pr_off = t.last ? static_cast<int>((threadIdx.x + 1) * sizeof(double2) + sizeof(double))
                      : static_cast<int>((threadIdx.x + 2) * sizeof(double2));
    const int64_t lastc = cend - 1;
    t.lastj = (lastc >= c0 && lastc < c0 + K) ? static_cast<int>(lastc - c0) : -1;
    t.validn = static_cast<int>(max(static_cast<int64_t>(0), min(static_cast<int64_t>(K),
                                                                 cend - c0)));
    bool ok0 = true;
    int d2 = 0;  // kD2: 2 = untested two-operation loop, 1 = tested, 0 = exact replay only
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int64_t c = c0 + j;
        t.C[j] = c < cend ? g.C[base + c] : 1.0;
        if constexpr (!kD2) {
            t.md[j] = make_divisor(c < cend ? g.m[base + c] : 1.0);
            ok0 &= (kQ && !kFma) ? divisor_range_ok(t.md[j]) : divisor_fast_ok(t.md[j]);
        }
    }
    if constexpr (kD2) {
        bool elig = true, clean = true;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const int64_t c = base + c0 + j;
            const uint64_t w = g.bad[c];
            t.md[j] = Divisor{0.0, g.zh[c], g.zl[c], static_cast<uint32_t>(w)};
            elig &= t.md[j].y != 0.0;
            clean &= (w & kDiv2Clean) != 0;
        }
        if (__syncthreads_and(elig))
            d2 = __all_sync(kFull, clean) ? 2 : 1;
        else
            ok0 = false;  // a divisor outside the two-operation range: exact replay
    }
    t.Cn = (c0 + K < cend) ? g.C[base + c0 + K] : (t.last ? -0.0 : 1.0);

    double x[K], v[K];
    load_state<K>(g, base, c0, cend, x, v);
    bool ok = ok0 && fused_dt_ok(g.k.half_dt);
    if constexpr (kD2) {
        if (d2 == 2) {
            for (int64_t s = 0; s < g.nsteps; ++s)
                step<K, false, Arith::Fast2>(t, x, v, g.k, edges, ok);
        } else if (d2 == 1) {
            for (int64_t s = 0; s < g.nsteps; ++s)
                step<K, false, Arith::Fast2C>(t, x, v, g.k, edges, ok);
        }
    } else {
        for (int64_t s = 0; s < g.nsteps; ++s)
            step<K, kPad, kFma ? Arith::Fma : (kQ ? Arith::FastQ : Arith::Fast)>(t, x, v, g.k,
                                                                                 edges, ok);
    }

    if (__syncthreads_or(!ok || owned_bad<K>(x, v, c0, own_start, own_end))) {
        // A division left nvcc's fast path, or a value went non-finite:
        // replay the launch from the untouched input with IEEE division,
        // checking every step, to keep exact values and find the exact first
        // bad step of the owned cells (NonFiniteStateError.step,
        // oscillator.py:255-260).
        load_state<K>(g, base, c0, cend, x, v);
        if constexpr (kD2) {  // the replay divides by the masses themselves
#pragma unroll
            for (int j = 0; j < K; ++j)
                t.md[j].b = g.m[base + c0 + j];
        }
        for (int64_t s = 0; s < g.nsteps; ++s) {
            step<K, kPad, kFma ? Arith::Fma : Arith::Exact>(t, x, v, g.k, edges, ok);
            if (__syncthreads_or(owned_bad<K>(x, v, c0, own_start, own_end))) {
                if (threadIdx.x == 0)
                    record_bad(&g.first_bad[buf_id], g.step0 + s + 1);
                break;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int64_t c = c0 + j;
        if (c >= own_start && c < own_end) {
            g.xout[base + c] = x[j];
            g.vout[base + c] = v[j];
            if (g.xs) {
                g.xs[base + c] = x[j];
                g.vs[base + c] = v[j];
            }
        }
    }
    if (touches_peer(g, own_start, own_end)) {
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const int64_t c = c0 + j;
            if (c >= own_start && c < own_end)
                store_peers(g, c, x[j], v[j]);
        }
    }
    if (sides) {
        __threadfence_system();  // our peer stores, before the post
        __syncthreads();
        if (threadIdx.x == 0)
            edge_done(g, sides);
    }
}

// ---------------------------------------------------------------------------
// Persistent tiled form (K3 for long chains): each CTA walks a strided list
// of tiles and prefetches the NEXT tile's m, C, x, v into a second shared-
// memory buffer with bulk async copies (cp.async.bulk, TMA engine, mbarrier
// completion) while it integrates the current one, so the per-tile HBM load
// latency overlaps compute.  The tile input stays in shared memory until the
// tile is finished, which is what the exact replay reloads from.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p)
{
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity)
{
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Bulk copy shared -> global (TMA engine, bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, unsigned bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}

// A thread's K contiguous cells of one tile array in shared memory, moved as
// 16-byte chunks in a lane-rotated order: at instruction j lane L touches
// chunk (j + rot) % (K/2), rot = (L >> 1) % (K/2).  Plain ascending order puts
// 16 lanes of a warp on one 16-byte bank group (the cells of a thread are 64
// bytes apart lane to lane): 4x the wavefronts of a conflict-free access
// (ncu: "L1 Wavefronts Shared Excessive" 3/4 of every tile load and store).
// The rotation is undone with selects, two stages for K = 8.
template <int K>
__device__ __forceinline__ int chunk_rot()
{
    return static_cast<int>((threadIdx.x >> 1) & (K / 2 - 1));
}

template <int K>
__device__ __forceinline__ void lds_cells(const double *p, double (&out)[K])
{
    static_assert(K == 8 || K == 4, "rotated tile access for K = 4 or 8");
    constexpr int NC = K / 2;
    const int rot = chunk_rot<K>();
    const double2 *q = reinterpret_cast<const double2 *>(p);
    double2 c[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j)
        c[j] = q[(j + rot) & (NC - 1)];  // c[j] = chunk (j + rot)
#pragma unroll
    for (int b = 1; b < NC; b <<= 1) {  // chunk k = c[(k - rot) % NC]
        double2 t[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k)
            t[k] = (rot & b) ? c[(k - b) & (NC - 1)] : c[k];
#pragma unroll
        for (int k = 0; k < NC; ++k)
            c[k] = t[k];
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        out[2 * k] = c[k].x;
        out[2 * k + 1] = c[k].y;
    }
}

template <int K>
__device__ __forceinline__ void sts_cells(double *p, const double (&in)[K])
{
    constexpr int NC = K / 2;
    const int rot = chunk_rot<K>();
    double2 c[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k)
        c[k] = make_double2(in[2 * k], in[2 * k + 1]);
#pragma unroll
    for (int b = 1; b < NC; b <<= 1) {  // c[j] = chunk (j + rot)
        double2 t[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k)
            t[k] = (rot & b) ? c[(k + b) & (NC - 1)] : c[k];
#pragma unroll
        for (int k = 0; k < NC; ++k)
            c[k] = t[k];
    }
    double2 *q = reinterpret_cast<double2 *>(p);
#pragma unroll
    for (int j = 0; j < NC; ++j)
        q[(j + rot) & (NC - 1)] = c[j];
}

struct TileGeom {
    int64_t buf_id, base, L, own_start, own_end;
    int sides;  // edge-sync sides of the tile (edge_sides)
};

__device__ __forceinline__ TileGeom tile_geom(const SegArgs &g, int64_t it, int64_t TILE)
{
    TileGeom tg;
    // one buffer (every tiled run but batches of long chains): no 64-bit
    // division in the tile transition
    const int64_t nw = walk_tiles(g);
    tg.buf_id = g.nbuf == 1 ? 0 : it / nw;
    const int64_t tile = tile_order(g, g.walk0 + (g.nbuf == 1 ? it : it % nw));
    tg.sides = edge_sides(g, tile);
    tg.own_start = g.own_lo + tile * g.W;
    tg.own_end = min(tg.own_start + g.W, g.own_hi);
    tg.L = max(static_cast<int64_t>(0), tg.own_start - g.H);
    if (tg.L + TILE > g.n)
        tg.L = g.n - TILE;
    tg.base = tg.buf_id * g.n;
    return tg;
}

// Shared-memory layout of one tile buffer, in doubles of TILE cells:
//   three-operation division: [m | C | x | v]
//   checked two-operation division (kD2): [zh | C | x | v | zl | bad]
template <bool kD2>
__host__ __device__ constexpr int64_t tile_slots() { return kD2 ? 6 : 4; }
template <bool kD2>
__host__ __device__ constexpr int persist_bufs() { return kD2 ? 2 : kPersistBufs; }

template <int K, int NT, bool kD2>
__device__ __forceinline__ void issue_tile(const SegArgs &g, int64_t it, double *dst,
                                           uint64_t *bar)
{
    constexpr int64_t TILE = int64_t(NT) * K;
    constexpr unsigned bytes = TILE * sizeof(double);
    const TileGeom tg = tile_geom(g, it, TILE);
    if (tg.sides)  // an edge tile reads ghosts the neighbour stores: wait for them
        edge_wait(g.sync, tg.sides);
    const int64_t o = tg.base + tg.L;
    mbar_expect_tx(bar, tile_slots<kD2>() * bytes);
    bulk_g2s(dst, (kD2 ? g.zh : g.m) + o, bytes, bar);
    bulk_g2s(dst + TILE, g.C + o, bytes, bar);
    bulk_g2s(dst + 2 * TILE, g.xin + o, bytes, bar);
    bulk_g2s(dst + 3 * TILE, g.vin + o, bytes, bar);
    if constexpr (kD2) {
        bulk_g2s(dst + 4 * TILE, g.zl + o, bytes, bar);
        bulk_g2s(dst + 5 * TILE, g.bad + o, bytes, bar);
    }
}

template <int K, int NT, bool kFma, bool kD2>
__global__ void __launch_bounds__(NT, (NT * K <= 1024 ? 2 : 1)) chain_tiles_persistent(SegArgs g)
{
    constexpr int64_t TILE = int64_t(NT) * K;
    constexpr int kBufs = persist_bufs<kD2>();
    constexpr int64_t kStride = tile_slots<kD2>() * TILE;  // doubles per tile buffer
    // kBufs x [m | C | x | v] x TILE (kD2: [zh | C | x | v | zl | bad], two buffers).  Three buffers: tile i computes
    // in buffer i % 3 while tile i + 1's inputs sit loaded in the next one and
    // tile i - 1's results still drain from the third by bulk store, so the
    // refill at the end of tile i (tile i + 2, into the buffer tile i - 1
    // used) waits for a store issued a whole tile earlier, not for the one it
    // just issued.
    extern __shared__ __align__(128) double tbuf[];
    __shared__ Edges<NT> edges;
    __shared__ __align__(8) uint64_t bars[kBufs];
    __shared__ int s_skip;

    const int64_t ntiles = walk_tiles(g) * g.nbuf;
    edges_init(edges);
    if (threadIdx.x == 0) {
        for (int b = 0; b < kBufs; ++b)
            mbar_init(&bars[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int b = 0; b < 2; ++b) {
            const int64_t it = blockIdx.x + int64_t(b) * gridDim.x;
            if (it < ntiles)
                issue_tile<K, NT, kD2>(g, it, tbuf + b * kStride, &bars[b]);
        }
        // one buffer: the skip decision is launch-invariant (diverged_before
        // reads the state at launch start), so it is read once, not per tile
        // behind a barrier every warp waits at
        if (g.nbuf == 1)
            s_skip = diverged_before(g, 0);
    }
    __syncthreads();
    const bool skip_once = g.nbuf == 1 && s_skip != 0;

    Tile<K> t;
    t.first = threadIdx.x == 0;
    t.last = threadIdx.x == NT - 1;
    t.pr_off = t.last ? static_cast<int>((threadIdx.x + 1) * sizeof(double2) + sizeof(double))
                      : static_cast<int>((threadIdx.x + 2) * sizeof(double2));
    t.lastj = -1;
    t.validn = K;
    const int cl = threadIdx.x * K;  // first cell of this thread within the tile
    int i = 0, b = 0, use = 0;  // b = i % kBufs, use = i / kBufs
    for (int64_t it = blockIdx.x; it < ntiles; it += gridDim.x, ++i) {
        double *sm = tbuf + b * kStride;
        mbar_wait(&bars[b], use & 1);
        const TileGeom tg = tile_geom(g, it, TILE);
        const int64_t c0 = tg.L + cl;
        bool skip = skip_once;
        if (g.nbuf > 1) {
            if (threadIdx.x == 0)  // uniform skip decision (see chain_rk4_kernel)
                s_skip = diverged_before(g, tg.buf_id);
            __syncthreads();
            skip = s_skip != 0;
        }
        if (!skip) {
            bool ok = fused_dt_ok(g.k.half_dt);
            // kD2: 2 = this warp divides in two operations without tests (all
            // its divisors have a class), 1 = with the wrong-quotient tests,
            // 0 = a divisor of the tile is not eligible: straight to the
            // exact replay (masses outside [2^-100, 2^101); none in C3)
            int d2 = 0;
            if constexpr (kD2) {
                double zh[K], zl[K];
                lds_cells<K>(sm + cl, zh);
                bool elig = true;
#pragma unroll
                for (int j = 0; j < K; ++j)
                    elig &= zh[j] != 0.0;
                if (__syncthreads_and(elig)) {
                    lds_cells<K>(sm + 4 * TILE + cl, zl);
                    const uint64_t *bw = reinterpret_cast<const uint64_t *>(sm + 5 * TILE) + cl;
                    bool clean = true;
#pragma unroll
                    for (int j = 0; j < K; ++j) {
                        const uint64_t w = bw[j];
                        t.md[j] = Divisor{0.0, zh[j], zl[j], static_cast<uint32_t>(w)};
                        clean &= (w & kDiv2Clean) != 0;
                    }
d2 = __all_sync(kFull, clean) ? 2 : 1;
                } else {
                    ok = false;
                }
            } else {
                double mj[K];
                lds_cells<K>(sm + cl, mj);
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    t.md[j] = make_divisor(mj[j]);
                    ok &= kFma ? divisor_fast_ok(t.md[j]) : divisor_range_ok(t.md[j]);
                }
            }
            lds_cells<K>(sm + TILE + cl, t.C);
            t.Cn = (cl + K < TILE) ? sm[TILE + cl + K] : -0.0;  // -0.0: the free end (accel)
            double x[K], v[K];
            lds_cells<K>(sm + 2 * TILE + cl, x);
            lds_cells<K>(sm + 3 * TILE + cl, v);
            // single-test division here (div_fastq): -5% instructions, C3
            // +1.1%; the whole-chain kernel keeps div_fast, whose schedule
            // ptxas handles better (profiles/r01/README.md)
            if constexpr (kD2) {
                // warp-uniform choice; both loops pass the same barriers
                if (d2 == 2) {
                    for (int64_t s = 0; s < g.nsteps; ++s)
                        step<K, false, Arith::Fast2>(t, x, v, g.k, edges, ok);
                } else if (d2 == 1) {
                    for (int64_t s = 0; s < g.nsteps; ++s)
                        step<K, false, Arith::Fast2C>(t, x, v, g.k, edges, ok);
                }
            } else {
                for (int64_t s = 0; s < g.nsteps; ++s)
                    step<K, false, kFma ? Arith::Fma : Arith::FastQ>(t, x, v, g.k, edges, ok);
            }
            if (__syncthreads_or(!ok || owned_bad<K>(x, v, c0, tg.own_start, tg.own_end))) {
                // exact replay from the tile input still in shared memory
                lds_cells<K>(sm + 2 * TILE + cl, x);
                lds_cells<K>(sm + 3 * TILE + cl, v);
                if (kD2) {  // the masses are not in the tile buffer
#pragma unroll
                    for (int j = 0; j < K; ++j)
                        t.md[j].b = g.m[tg.base + c0 + j];
                }
                for (int64_t s = 0; s < g.nsteps; ++s) {
                    step<K, false, kFma ? Arith::Fma : Arith::Exact>(t, x, v, g.k, edges, ok);
                    if (__syncthreads_or(owned_bad<K>(x, v, c0, tg.own_start, tg.own_end))) {
                        if (threadIdx.x == 0)
                            record_bad(&g.first_bad[tg.buf_id], g.step0 + s + 1);
                        break;
                    }
                }
            }
            // The tile input is no longer needed: the results go into its x/v
            // slots and leave as one bulk copy per array (TMA store) instead
            // of 16 strided 8-byte stores per thread.
            sts_cells<K>(sm + 2 * TILE + cl, x);
            sts_cells<K>(sm + 3 * TILE + cl, v);
            if (touches_peer(g, tg.own_start, tg.own_end)) {
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    const int64_t c = c0 + j;
                    if (c >= tg.own_start && c < tg.own_end)
                        store_peers(g, c, x[j], v[j]);
                }
            }
            if (tg.sides)
                __threadfence_system();  // our peer stores, before the post
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncthreads();  // every thread is done with buffer b; the results are in it
        const bool stored = !skip;
        if (threadIdx.x == 0) {
            if (tg.sides)  // post before waiting for the next tile (no wait cycle)
                edge_done(g, tg.sides);
            if (stored) {
                const int64_t o = tg.own_start - tg.L;
                const unsigned bytes = static_cast<unsigned>(tg.own_end - tg.own_start) * 8u;
                const int64_t go = tg.base + tg.own_start;
                bulk_s2g(g.xout + go, sm + 2 * TILE + o, bytes);
                bulk_s2g(g.vout + go, sm + 3 * TILE + o, bytes);
                if (g.xs) {
                    bulk_s2g(g.xs + go, sm + 2 * TILE + o, bytes);
                    bulk_s2g(g.vs + go, sm + 3 * TILE + o, bytes);
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            const int64_t nx = it + 2 * int64_t(gridDim.x);
            if (nx < ntiles) {
                // tile i + 2 goes into the buffer tile i - 1 used: its store
                // group must have finished reading it (the group just
                // committed for tile i may stay in flight)
                if (stored && kBufs == 3)
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                else
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                const int nb = kBufs == 2 ? b : (b == 0 ? kBufs - 1 : b - 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue_tile<K, NT, kD2>(g, nx, tbuf + nb * kStride, &bars[nb]);
            }
        }
        if (++b == kBufs) {
            b = 0;
            ++use;
        }
    }
    if (threadIdx.x == 0)
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // writes performed
}

template <int K, int NT, bool kD2>
constexpr size_t persist_smem()
{
    return persist_bufs<kD2>() * tile_slots<kD2>() * size_t(K) * NT * sizeof(double);
}

// Resident CTAs of a persistent kernel on device `dev` (SMs x CTAs per SM),
// computed once per kernel and device: the attribute call and the occupancy
// query cost more host time than a short sharded period's launch itself.
template <int K, int NT, bool kFma, bool kD2>
int64_t persistent_ctas(int dev)
{
    static std::atomic<int64_t> cache[kMaxDevices];  // one per kernel instantiation
    if (dev >= 0 && dev < kMaxDevices) {
        const int64_t c = cache[dev].load(std::memory_order_relaxed);
        if (c > 0)
            return c;
    }
    auto kern = chain_tiles_persistent<K, NT, kFma, kD2>;
    int sms = 148, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(persist_smem<K, NT, kD2>()));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, persist_smem<K, NT, kD2>());
    const int64_t c = int64_t(sms) * std::max(per_sm, 1);
    if (dev >= 0 && dev < kMaxDevices)
        cache[dev].store(c, std::memory_order_relaxed);
    return c;
}

template <int K, int NT, bool kFma, bool kD2>
cudaError_t launch_persistent_as(const SegArgs &g, cudaStream_t stream)
{
    int dev = 0;
    cudaGetDevice(&dev);
    const int64_t ctas = persistent_ctas<K, NT, kFma, kD2>(dev);
    const int64_t ntiles = walk_tiles(g) * g.nbuf;
    const int64_t grid = std::min<int64_t>(ntiles, ctas);
    chain_tiles_persistent<K, NT, kFma, kD2>
        <<<static_cast<unsigned>(grid), NT, persist_smem<K, NT, kD2>(), stream>>>(g);
    return cudaGetLastError();
}

template <int K, int NT>
cudaError_t launch_persistent(const SegArgs &g, cudaStream_t stream)
{
    if (g.fma)
        return launch_persistent_as<K, NT, true, false>(g, stream);
    // the checked two-operation build for the default tile shape only
    if constexpr (K == 8 && NT == 256) {
        if (g.zh)
            return launch_persistent_as<K, NT, false, true>(g, stream);
    }
    return launch_persistent_as<K, NT, false, false>(g, stream);
}

template <int K>
cudaError_t launch_k(const SegArgs &g, int threads, cudaStream_t stream)
{
    if (threads > max_threads<K>() || threads % 32)
        return cudaErrorInvalidConfiguration;
    const int64_t blocks = walk_tiles(g) * g.nbuf;
    const int64_t TILE = int64_t(threads) * K;
    const unsigned nb = static_cast<unsigned>(blocks);
    // Padding is needed only when a tile is longer than the whole buffer.
    constexpr int kT2 = 1024 / K;  // two CTAs of <= 1024 cells per SM
    if (K >= 4 && threads <= kT2) {
        if (TILE > g.n)
            (g.fma ? chain_rk4_kernel<K, true, true, kT2> : chain_rk4_kernel<K, true, false, kT2>)
                <<<nb, threads, 0, stream>>>(g);
        else if (K == 8 && g.zh && !g.fma)  // the two-operation build (C4's shape)
            chain_rk4_kernel<K, false, false, kT2, true><<<nb, threads, 0, stream>>>(g);
        else
            (g.fma ? chain_rk4_kernel<K, false, true, kT2> : chain_rk4_kernel<K, false, false, kT2>)
                <<<nb, threads, 0, stream>>>(g);
        return cudaGetLastError();
    }
    if (TILE > g.n)
        (g.fma ? chain_rk4_kernel<K, true, true> : chain_rk4_kernel<K, true, false>)
            <<<nb, threads, 0, stream>>>(g);
    else
        (g.fma ? chain_rk4_kernel<K, false, true> : chain_rk4_kernel<K, false, false>)
            <<<nb, threads, 0, stream>>>(g);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_chain(const SegArgs &g, int K, int threads, cudaStream_t stream)
{
    // Tiled runs of the default shape go through the persistent prefetching
    // kernel when the bulk copies are 16-byte aligned: even cell offsets AND
    // 16-byte aligned base pointers (a caller may pass any 8-byte aligned
    // view, e.g. a tensor with an odd storage offset); otherwise the plain
    // tiled kernel, same bytes.
    const int64_t TILE = int64_t(threads) * K;
    const bool tiled = g.H > 0 || g.tiles > 1;
    auto a16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    const bool aligned = (g.n % 2 == 0) && (g.own_lo % 2 == 0) && (g.own_hi % 2 == 0) &&
                         (g.W % 2 == 0) && (g.H % 2 == 0) && g.n >= TILE && a16(g.m) &&
                         a16(g.C) && a16(g.xin) && a16(g.vin) && a16(g.xout) && a16(g.vout) &&
                         (!g.xs || (a16(g.xs) && a16(g.vs))) &&
                         (!g.zh || (a16(g.zh) && a16(g.zl) && a16(g.bad)));
    static const bool disable = std::getenv("OSC_NO_PERSIST") != nullptr;
    if (tiled && aligned && !disable) {
        if (K == 8 && threads == 128)
            return launch_persistent<8, 128>(g, stream);
        if (K == 8 && threads == 256)
            return launch_persistent<8, 256>(g, stream);
        if (K == 4 && threads == 256)
            return launch_persistent<4, 256>(g, stream);
        if (K == 4 && threads == 512)
            return launch_persistent<4, 512>(g, stream);
    }
    switch (K) {
    case 1: return launch_k<1>(g, threads, stream);
    case 2: return launch_k<2>(g, threads, stream);
    case 4: return launch_k<4>(g, threads, stream);
    case 8: return launch_k<8>(g, threads, stream);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace osc
