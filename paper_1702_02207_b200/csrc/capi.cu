// C-ABI layer: argument validation and the device-pointer entry points.
// Declarations and conventions: include/osc_b200.h; host-pointer forms in
// capi_host.cu, peer memory / multi-GPU in capi_peer.cu.
#include "capi_internal.h"

using namespace osc_capi;

extern "C" {

int osc_abi_version(void) { return OSC_ABI_VERSION; }

const char *osc_last_error(void) { return g_last_error.c_str(); }

int osc_rk4_batch2(const double *m, const double *C, double *x, double *v, int64_t B, double dt,
                   int64_t nsteps, int64_t stride, double *xs, double *vs, double *es,
                   int64_t *first_bad, uint32_t flags, void *stream)
{
    return osc_capi::batch2_entry(m, C, x, v, B, dt, nsteps, stride, xs, vs, es, first_bad,
                                  flags, stream, false);
}

}  // extern "C"

// osc_rk4_batch2 proper; shares_gpu: the caller runs several batches side
// by side (the host pipeline's chunks), so K1 keeps its throughput shape
// even for a small batch.
int osc_capi::batch2_entry(const double *m, const double *C, double *x, double *v, int64_t B,
                           double dt, int64_t nsteps, int64_t stride, double *xs, double *vs,
                           double *es, int64_t *first_bad, uint32_t flags, void *stream,
                           bool shares_gpu)
{
    if (flags & ~kRunFlags)
        return fail(OSC_INVALID, "unknown flags 0x%x", flags);
    if (int rc = check_run_args(dt, nsteps, stride))
        return rc;
    if (B < 0)
        return fail(OSC_INVALID, "B must be >= 0");
    if (B == 0)
        return OSC_OK;
    if (!m || !C || !x || !v || !first_bad || (!xs) != (!vs))
        return fail(OSC_INVALID, "null buffer");
    if (!(flags & OSC_TRUSTED))
        if (int rc = check_params(m, C, 2 * B, static_cast<cudaStream_t>(stream),
                                  ParamLayout::CellMajor, B))
            return rc;
    cudaError_t e = osc::launch_batch2(m, C, x, v, B, consts(dt), nsteps, stride, xs, vs, es,
                                       first_bad, (flags & OSC_FMA) != 0,
                                       static_cast<cudaStream_t>(stream), nullptr, shares_gpu);
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "batch2_rk4_kernel");
}

extern "C" {

int osc_rk4_batch2_compare(const double *m, const double *C, double *x, double *v, int64_t B,
                           double dt, int64_t nsteps, int64_t stride, const double *ts,
                           const double *sol, double *report, int64_t *first_bad, uint32_t flags,
                           void *stream)
{
    if (flags & ~kRunFlags)
        return fail(OSC_INVALID, "unknown flags 0x%x", flags);
    if (int rc = check_run_args(dt, nsteps, stride))
        return rc;
    if (B < 0)
        return fail(OSC_INVALID, "B must be >= 0");
    if (B == 0)
        return OSC_OK;
    if (!m || !C || !x || !v || !first_bad || !ts || !sol || !report)
        return fail(OSC_INVALID, "null buffer");
    if (!(flags & OSC_TRUSTED))
        if (int rc = check_params(m, C, 2 * B, static_cast<cudaStream_t>(stream),
                                  ParamLayout::CellMajor, B))
            return rc;
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
    if (int rc = check_params(m, C, 2 * B, static_cast<cudaStream_t>(stream),
                              ParamLayout::CellMajor, B))
        return rc;
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
    if (flags & ~kRunFlags)
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
    if (!(flags & OSC_TRUSTED))
        if (int rc = check_params(m, C, cells, stream, ParamLayout::Chains, B, s))
            return rc;

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
    Scratch scratch;
    scratch.s = stream;
    // The default tile shape and the whole-chain 8-cell builds divide in two
    // operations where a warp's divisors allow it (div2_chain_consts): one
    // table pass over the masses first.  OSC_DIV2=0 keeps three operations
    // (A/B timing).
    const char *d2env = std::getenv("OSC_DIV2");
    // (tiled: the persistent 8 x 256 tiles; whole chains: 8 cells x <= 128
    // threads without padding -- the builds that read the table)
    const bool tiled = plan.tiles > 1 || plan.H > 0;
    const bool d2 = !g.fma && K == kTileK && !(d2env && d2env[0] == '0') &&
                    (tiled ? threads == kTileThreads : (threads <= 128 && threads * K <= s));
    OSC_CUDA(osc::scratch_alloc(reinterpret_cast<void **>(&scratch.p), (d2 ? 5 : 2) * bytes,
                                stream));
    if (d2) {
        double *zh = scratch.p + 2 * cells;
        g.zh = zh;
        g.zl = zh + cells;
        g.bad = reinterpret_cast<const uint64_t *>(zh + 2 * cells);
        cudaError_t e = osc::launch_div2c_table(m, cells, zh, zh + cells,
                                                reinterpret_cast<uint64_t *>(zh + 2 * cells),
                                                stream);
        if (e != cudaSuccess)
            return cuda_fail(e, "div2c_table_kernel");
    }

    // The time loop over chains [b0, b0 + nb) on stream st.
    auto run_group = [&](int64_t b0, int64_t nb, cudaStream_t st) -> int {
        const int64_t o = b0 * s;
        osc::SegArgs gg = g;
        gg.m = m + o;
        gg.C = C + o;
        if (g.zh) {
            gg.zh = g.zh + o;
            gg.zl = g.zl + o;
            gg.bad = g.bad + o;
        }
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
                          const osc_peer_t *left, const osc_peer_t *right,
                          const osc_edge_sync_t *sync, uint32_t flags, void *stream)
{
    return osc_rk4_chain_advance_div2(m, C, xin, vin, xout, vout, n, own_lo, own_hi, dt, nsteps,
                                      step0, first_bad, left, right, sync, nullptr, flags,
                                      stream);
}

int osc_rk4_chain_advance_div2(const double *m, const double *C, const double *xin,
                               const double *vin, double *xout, double *vout, int64_t n,
                               int64_t own_lo, int64_t own_hi, double dt, int64_t nsteps,
                               int64_t step0, int64_t *first_bad, const osc_peer_t *left,
                               const osc_peer_t *right, const osc_edge_sync_t *sync,
                               const double *div2, uint32_t flags, void *stream)
{
    if (flags & ~kAdvanceFlags)
        return fail(OSC_INVALID, "unknown flags 0x%x", flags);
    const uint32_t subset = flags & (OSC_TILES_INTERIOR | OSC_TILES_EDGES);
    if (subset == (OSC_TILES_INTERIOR | OSC_TILES_EDGES))
        return fail(OSC_INVALID, "OSC_TILES_INTERIOR and OSC_TILES_EDGES are exclusive");
    if (int rc = check_run_args(dt, nsteps, 1))
        return rc;
    if (n < 1 || own_lo < 0 || own_hi > n || own_lo >= own_hi)
        return fail(OSC_INVALID, "bad shard range [%lld,%lld) of %lld", (long long)own_lo,
                    (long long)own_hi, (long long)n);
    if (!m || !C || !xin || !vin || !xout || !vout || !first_bad)
        return fail(OSC_INVALID, "null buffer");
    if (!(flags & OSC_TRUSTED))
        if (int rc = check_params(m, C, n, static_cast<cudaStream_t>(stream)))
            return rc;
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
    if (div2 && !g.fma) {
        g.zh = div2;
        g.zl = div2 + n;
        g.bad = reinterpret_cast<const uint64_t *>(div2 + 2 * n);
    }
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
    if (sync) {
        if (!sync->counters || sync->timeout_ns < 0)
            return fail(OSC_INVALID, "bad edge sync descriptor");
        if (subset)
            return fail(OSC_INVALID, "edge sync orders whole launches: no tile subset");
        g.sync.ready[0] = sync->ready[0];
        g.sync.ready[1] = sync->ready[1];
        g.sync.ctr = sync->counters;
        g.sync.period = sync->period;
        g.sync.timeout_ns = sync->timeout_ns;
    }
    if (sync || subset) {
        g.ordered = true;
        edge_sets(g, kTileK * kTileThreads, g.nedge);
        const int64_t rs = std::max(g.nedge[0], g.tiles - g.nedge[1]);
        const int64_t nint = rs - g.nedge[0];  // interior tiles, walked first
        if (subset == OSC_TILES_INTERIOR) {
            g.walk0 = 0;
            g.nwalk = nint;
        } else if (subset == OSC_TILES_EDGES) {
            g.walk0 = nint;
            g.nwalk = g.tiles - nint;
        }
        if (subset && g.nwalk == 0)
            return OSC_OK;  // an empty subset: nothing to launch
    }
    cudaError_t e = osc::launch_chain(g, kTileK, kTileThreads, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "chain_rk4_kernel");
}

int osc_edge_sync_status(const uint64_t *counters, uint64_t *record, void *stream)
{
    if (!counters || !record)
        return fail(OSC_INVALID, "null buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    OSC_CUDA(cudaMemcpyAsync(record, counters + 4, 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                             st));
    OSC_CUDA(cudaStreamSynchronize(st));
    if (record[0] == 0)
        return OSC_OK;
    return fail(OSC_CUDA_ERROR,
                "edge sync timed out: period %llu waited for the %s neighbour's counter to reach "
                "%llu, saw %llu",
                (unsigned long long)record[1], record[2] ? "right" : "left",
                (unsigned long long)record[1], (unsigned long long)record[3]);
}

int osc_rowscale(const double *K, const double *m, double *A, int64_t s, void *stream)
{
    if (s < 1 || !K || !m || !A)
        return fail(OSC_INVALID, "bad rowscale arguments");
    if (int rc = check_params(m, m, s, static_cast<cudaStream_t>(stream)))  // masses only
        return rc;
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
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    const int64_t sp = osc::dense_pad_s(s), Np = osc::dense_pad_n(N);
    const size_t op = static_cast<size_t>(sp) * 2 * Np, st = static_cast<size_t>(sp) * Np;
    const bool pad_a = sp != s;
    const size_t total = 2 * op + 3 * st + (pad_a ? static_cast<size_t>(sp) * sp : 0);
    Scratch ws;
    ws.s = stream;
    OSC_CUDA(osc::scratch_alloc(reinterpret_cast<void **>(&ws.p), total * sizeof(double), stream));
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
    if (int rc = check_params(m, C, s, static_cast<cudaStream_t>(stream)))
        return rc;
    cudaError_t e = osc::launch_equation_engine(m, C, x0, v0, static_cast<int>(s), dt, nsteps,
                                                stride, xs, vs, first_bad, step_ns,
                                                static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "equation_engine_kernel");
}

int osc_derivative(const double *m, const double *C, const double *x, double *dvel, int64_t B,
                   int64_t s, int cell_major, void *stream)
{
    if (B < 0 || s < 1)
        return fail(OSC_INVALID, "need B >= 0 and s >= 1");
    if (B == 0)
        return OSC_OK;
    if (!m || !C || !x)
        return fail(OSC_INVALID, "null buffer");
    if (int rc = check_params(m, C, B * s, static_cast<cudaStream_t>(stream),
                              cell_major ? ParamLayout::CellMajor : ParamLayout::Chains, B, s))
        return rc;
    cudaError_t e = osc::launch_derivative(m, C, x, dvel, B, s, cell_major != 0,
                                           static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "derivative_kernel");
}

int osc_energy(const double *m, const double *C, const double *x, const double *v, double *out,
               int64_t B, int64_t s, int cell_major, void *stream)
{
    if (B < 0 || s < 1)
        return fail(OSC_INVALID, "need B >= 0 and s >= 1");
    if (B == 0)
        return OSC_OK;
    if (!m || !C || !x)
        return fail(OSC_INVALID, "null buffer");
    if (int rc = check_params(m, C, B * s, static_cast<cudaStream_t>(stream),
                              cell_major ? ParamLayout::CellMajor : ParamLayout::Chains, B, s))
        return rc;
    cudaError_t e = osc::launch_energy(m, C, x, v, out, B, s, cell_major != 0,
                                       static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "energy_kernel");
}

int osc_validate_parameters(const double *m, const double *C, int64_t n, int64_t *bad,
                            void *stream)
{
    if (bad)
        *bad = -1;
    if (n < 0 || (n > 0 && (!m || !C)))
        return fail(OSC_INVALID, "osc_validate_parameters: n < 0 or null buffer");
    const int rc = check_params(m, C, n, static_cast<cudaStream_t>(stream));
    if (rc == OSC_INVALID && bad && g_bad_param_which >= 0)
        *bad = g_bad_param_index;
    return rc;
}

int osc_last_invalid_parameter(int *which, int64_t *index)
{
    if (g_bad_param_which < 0)
        return 0;
    if (which)
        *which = g_bad_param_which;
    if (index)
        *index = g_bad_param_index;
    return 1;
}

int osc_div2_classify(const double *b, int64_t n, uint8_t *pass, void *stream)
{
    if (n < 0 || (n > 0 && (!b || !pass)))
        return fail(OSC_INVALID, "osc_div2_classify: n < 0 or null buffer");
    cudaError_t e = osc::launch_div2_classify(b, n, pass, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "div2_classify_kernel");
}

int osc_div2c_table(const double *b, int64_t n, double *zh, double *zl, uint64_t *bad,
                    void *stream)
{
    if (n < 0 || (n > 0 && (!b || !zh || !zl || !bad)))
        return fail(OSC_INVALID, "osc_div2c_table: n < 0 or null buffer");
    cudaError_t e = osc::launch_div2c_table(b, n, zh, zl, bad, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? OSC_OK : cuda_fail(e, "div2c_table_kernel");
}

int osc_check_division(int64_t n, uint64_t seed, int mode, uint64_t *mismatches, void *stream_)
{
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    unsigned long long *d = nullptr;
    OSC_CUDA(osc::scratch_alloc(reinterpret_cast<void **>(&d), sizeof *d, stream));
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

}  // extern "C"
