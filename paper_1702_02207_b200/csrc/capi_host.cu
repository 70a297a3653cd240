// Host-pointer forms of the batched entry points (synchronous; pinned or
// pageable buffers): chunked, multi-stream pipelines over capi.cu's
// device-pointer entry points.
#include "capi_internal.h"

using namespace osc_capi;

// ---------------------------------------------------------------------------
// Host-pointer forms: the end-to-end path a CPU caller (the reference's own
// Python objects via ctypes) uses.  One cudaMemcpyAsync per buffer.
// ---------------------------------------------------------------------------

namespace {

// Per-thread, per-device resources of the host-pointer forms, created once
// and reused: the pipeline's streams (creating and destroying three streams
// cost more than a small run itself) and a pinned staging buffer through
// which small calls move all their inputs in ONE host-to-device copy and
// all their outputs in ONE device-to-host copy.
struct HostCtx {
    int dev = -1;
    cudaStream_t st[4] = {nullptr, nullptr, nullptr, nullptr};  // [3]: parameter uploads
    unsigned char *pin = nullptr;
    size_t pin_cap = 0;
    unsigned char *dmem = nullptr;  // the staged calls' device block, grown as needed
    size_t dmem_cap = 0;

    ~HostCtx()
    {
        // thread exit; errors (runtime already unloading) are ignored
        if (dev < 0)
            return;
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
        for (auto s : st)
            if (s)
                cudaStreamDestroy(s);
        if (pin)
            cudaFreeHost(pin);
        if (dmem)
            cudaFree(dmem);
        cudaSetDevice(prev);
        cudaGetLastError();
    }
};

constexpr size_t kStagedMax = size_t(8) << 20;  // calls moving <= 8 MB go through staging

int host_ctx(HostCtx *&out)
{
    static thread_local std::vector<HostCtx> ctx;
    int dev = 0;
    OSC_CUDA(cudaGetDevice(&dev));
    if (ctx.size() <= static_cast<size_t>(dev))
        ctx.resize(dev + 1);
    HostCtx &c = ctx[dev];
    if (c.dev < 0) {
        // Chunk streams in descending priority (chunk c runs on stream c % 3):
        // the GPU finishes chunk 0 first, so its results copy back while later
        // chunks compute, and the lower-priority chunks fill the earlier ones'
        // tail waves.  The parameter / result-copy stream gets the highest.
        int lo = 0, hi = 0;  // numerically: lo = least, hi = greatest priority
        OSC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        const int step = (lo - hi) >= 2 ? 1 : 0;
        const int p[4] = {hi + 0 * step, hi + 1 * step, hi + 2 * step, hi};
        for (int i = 0; i < 4; ++i)
            OSC_CUDA(cudaStreamCreateWithPriority(&c.st[i], cudaStreamNonBlocking,
                                                  std::min(p[i], lo)));
        c.dev = dev;
    }
    out = &c;
    return OSC_OK;
}

int device_block(HostCtx &c, size_t bytes, unsigned char *&p)
{
    if (c.dmem_cap < bytes) {
        if (c.dmem) {
            OSC_CUDA(cudaStreamSynchronize(c.st[0]));  // the block's last user is done
            OSC_CUDA(cudaFree(c.dmem));
        }
        c.dmem = nullptr;
        c.dmem_cap = 0;
        const size_t cap = std::max<size_t>(bytes, size_t(1) << 16);
        OSC_CUDA(cudaMalloc(reinterpret_cast<void **>(&c.dmem), cap));
        c.dmem_cap = cap;
    }
    p = c.dmem;
    return OSC_OK;
}

int staging(HostCtx &c, size_t bytes, unsigned char *&p)
{
    if (c.pin_cap < bytes) {
        if (c.pin)
            OSC_CUDA(cudaFreeHost(c.pin));
        c.pin = nullptr;
        c.pin_cap = 0;
        const size_t cap = std::max<size_t>(bytes, size_t(1) << 16);
        OSC_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&c.pin), cap, cudaHostAllocDefault));
        c.pin_cap = cap;
    }
    p = c.pin;
    return OSC_OK;
}

// A small host-pointer call, as one round trip through the pinned staging
// buffer: the inputs go up in one copy (with the check record's two slots
// pre-set to ~0, so no memset), the parameter rule is checked ON THE DEVICE
// in the same stream as the work -- fused into the work's own kernel where
// it supports it (`fused`), else one param_check launch -- the outputs and
// the check record come back in one copy, and only then is anything written
// to the caller's buffers: an invalid system returns OSC_INVALID with the
// caller's outputs untouched.  Device block and stream are cached per thread.
//
// Layout (device block and staging alike, all 8-byte slots):
//   [ inputs (in_slots) | badp[2] | outputs (out_slots) ]
// `work(d, st, badp)` enqueues the computation given the device block; when
// `fused` it applies the parameter rule to m = d + m_off, C = d + C_off itself.
template <class Work>
int staged_call(size_t in_slots, size_t out_slots, size_t m_off, size_t C_off, int64_t nparam,
                const std::vector<std::pair<const void *, size_t>> &ins,
                const std::vector<std::pair<void *, size_t>> &outs, Work work,
                const double *hm, const double *hC, ParamLayout layout, int64_t B, int64_t s,
                bool fused = false)
{
    HostCtx *c = nullptr;
    if (int rc = host_ctx(c))
        return rc;
    cudaStream_t st = c->st[0];
    const size_t slots = in_slots + 2 + out_slots;
    unsigned char *pin = nullptr, *dmem = nullptr;
    if (int rc = staging(*c, slots * 8, pin))
        return rc;
    if (int rc = device_block(*c, slots * 8, dmem))
        return rc;
    size_t off = 0;
    for (auto &[p, n] : ins) {
        std::memcpy(pin + off, p, n);
        off += n;
    }
    std::memset(pin + in_slots * 8, 0xff, 16);  // the check record: "no offender"
    OSC_CUDA(cudaMemcpyAsync(dmem, pin, (in_slots + 2) * 8, cudaMemcpyHostToDevice, st));
    double *d = reinterpret_cast<double *>(dmem);
    auto *badp = reinterpret_cast<unsigned long long *>(d + in_slots);
    if (!fused && nparam > 0)
        OSC_CUDA(osc::launch_param_check(d + m_off, d + C_off, nparam, badp, st, false));
    if (int rc = work(d, st, badp))
        return rc;
    OSC_CUDA(cudaMemcpyAsync(pin + in_slots * 8, d + in_slots, (out_slots + 2) * 8,
                             cudaMemcpyDeviceToHost, st));
    OSC_CUDA(cudaStreamSynchronize(st));
    unsigned long long bad[2];
    std::memcpy(bad, pin + in_slots * 8, sizeof bad);
    if (bad[0] != ~0ull || bad[1] != ~0ull)  // the first offender in the caller's layout
        return host_param_fail(hm, hC, nparam, layout, B, s);
    off = (in_slots + 2) * 8;
    for (auto &[p, n] : outs) {
        if (p)
            std::memcpy(p, pin + off, n);
        off += n;
    }
    return OSC_OK;
}

// Host-pointer form of a batched run.  Small runs are one staged round trip
// (staged_call).  Large ones are cut into chunks that are pipelined over
// three streams: chunk c's H2D copy, kernels and D2H copy are ordered on
// stream c % S, so copies of one chunk overlap the compute of another and
// consecutive chunks' kernels fill each other's tail waves.  Sampled runs use
// a single chunk (their [nsamp][...] layout spans the batch).
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
    const size_t cells = static_cast<size_t>(B * s);
    const size_t bytes = cells * sizeof(double);
    const size_t nsamp = xs ? static_cast<size_t>(1 + nsteps / stride) : 0;
    const ParamLayout layout = chains ? ParamLayout::Chains : ParamLayout::CellMajor;

    // -- small: one staged round trip --------------------------------------
    // inputs [m | C | x | v], outputs [x | v | first_bad | worst[2] | xs | vs]
    const size_t out_slots = 2 * cells + B + 2 + 2 * nsamp * cells;
    if ((4 * cells + out_slots) * 8 <= kStagedMax) {
        unsigned long long worst[2] = {~0ull, ~0ull};
        const size_t sb = nsamp * bytes;
        auto work = [&](double *d, cudaStream_t st, unsigned long long *) -> int {
            double *dm = d, *dC = d + cells, *dx = d + 2 * cells;  // x, v adjacent
            double *o = d + 4 * cells + 2;  // the output slots (after the check record)
            OSC_CUDA(cudaMemcpyAsync(o, dx, 2 * bytes, cudaMemcpyDeviceToDevice, st));
            double *ox = o, *ov = o + cells;
            int64_t *fb = reinterpret_cast<int64_t *>(o + 2 * cells);
            auto *dw = reinterpret_cast<unsigned long long *>(o + 2 * cells + B);
            double *dxs = xs ? o + 2 * cells + B + 2 : nullptr;
            double *dvs = xs ? dxs + nsamp * cells : nullptr;
            int rc = chains ? osc_rk4_chains(dm, dC, ox, ov, B, s, dt, nsteps, stride, dxs, dvs,
                                             nullptr, fb, 0, OSC_TRUSTED, st)
                            : osc_rk4_batch2(dm, dC, ox, ov, B, dt, nsteps, stride, dxs, dvs,
                                             nullptr, fb, OSC_TRUSTED, st);
            if (rc != OSC_OK)
                return rc;
            OSC_CUDA(osc::launch_first_bad(fb, B, dw, st));
            return OSC_OK;
        };
        const int rc = staged_call(
            4 * cells, out_slots, 0, cells, static_cast<int64_t>(cells),
            {{m, bytes}, {C, bytes}, {x, bytes}, {v, bytes}},
            {{x, bytes}, {v, bytes}, {first_bad, B * sizeof(int64_t)}, {worst, sizeof worst},
             {xs, sb}, {vs, sb}},
            work, m, C, layout, B, s);
        if (rc != OSC_OK)
            return rc;
        if (worst[0] != ~0ull)
            return fail(OSC_NONFINITE, "integration diverged at step %lld (system %lld)",
                        (long long)worst[0], (long long)worst[1]);
        return OSC_OK;
    }

    // -- large: chunked multi-stream pipeline ---------------------------------
    // Chunking, so that only the first chunk's H2D and the last one's D2H are
    // exposed: >= 2 MB of state per chunk, at most 8 chunks, 2-DOF chunks of
    // >= 148*1024 systems; chunks share the GPU, so K1 keeps its two-systems-
    // per-thread shape for them (batch2_entry's shares_gpu).
    int64_t nchunk = 1;
    if (!xs && B > 1)
        nchunk = std::max<int64_t>(1, std::min<int64_t>({8, B, (int64_t)(bytes >> 21)}));
    if (!chains)
        // at most 4: measured for C2 (scripts/e2e_chunks.py, profiles/r02):
        // 2-4 and 8 chunks 49.8-49.9 ms, 6 chunks 53.8 ms
        nchunk = std::max<int64_t>(1, std::min<int64_t>({nchunk, int64_t(4), B / (148 * 1024)}));
    if (const char *e = std::getenv("OSC_HOST_CHUNKS")) {  // benchmarking knob
        const long long n = std::atoll(e);
        if (!xs && n >= 1 && n <= 64)
            nchunk = std::min<int64_t>(n, B);
    }
    // 2-DOF batches: three chunks, a small first one (its H2D is the only
    // exposed upload; it computes while the big one's inputs land), a big one,
    // and a small last one (its D2H is the only exposed download; its kernels
    // fill the big chunk's tail).  Small chunks of B/16 systems, rounded to
    // whole 512-system CTAs of K1: C2 end to end 50.2 -> 48.7 ms against a
    // 48.1 ms device step (scripts/gpu_e2e_edge.sh, profiles/r02/README.md;
    // B/20, B/24, B/40 -- not whole CTAs -- and B/64 measured slower).
    // OSC_HOST_EDGE=k: small chunks of B/k (benchmarking knob; 0 = equal).
    int64_t edge = 0;
    if (!chains && nchunk >= 2 && !std::getenv("OSC_HOST_CHUNKS")) {
        int64_t k = 16;
        if (const char *e = std::getenv("OSC_HOST_EDGE"))
            k = std::atoll(e);
        const int64_t cta = 2 * 256;  // systems per K1 CTA (batch2_entry's shape)
        if (k >= 3 && B / k >= 148 * 128) {
            nchunk = 3;
            edge = std::max<int64_t>(cta, B / k / cta * cta);
        }
    }
    auto bound = [&](int64_t c) -> int64_t {  // first system of chunk c (c = nchunk: B)
        if (edge)
            return c == 0 ? 0 : c == 1 ? edge : c == 2 ? B - edge : B;
        return B * c / nchunk;
    };
    const int nstream = static_cast<int>(std::min<int64_t>(nchunk, 3));
    HostCtx *ctx = nullptr;
    if (int rc = host_ctx(ctx))
        return rc;
    cudaStream_t *streams = ctx->st;
    struct Cleanup {
        cudaStream_t *st;
        int n;
        void *mem = nullptr;
        ~Cleanup()
        {
            for (int i = 0; i < n; ++i)
                cudaStreamSynchronize(st[i]);  // every stream is done with mem
            cudaStreamSynchronize(st[3]);      // the parameter / result-copy stream
            if (mem) {
                cudaFreeAsync(mem, st[0]);
                cudaStreamSynchronize(st[0]);
            }
        }
    } cleanup{streams, nstream};

    const size_t total = 4 * bytes + B * sizeof(int64_t) + 2 * nsamp * bytes + 16;
    OSC_CUDA(osc::scratch_alloc(&cleanup.mem, total, streams[0]));
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

    // The parameter rule without giving up the overlap: chunk by chunk, m and
    // C go up on the parameter stream, the chunk's state on its own stream
    // (after its m, C: an event), then its kernels -- so the copy engine sees
    // m0 C0 x0 v0 m1 ... and chunk 0 starts computing at once.  After the
    // last m, C the parameter stream checks all of them in one device pass.
    // The host waits for that check (it ends ~1 ms in, chunk 0 computes for
    // ~50/nchunk ms) and only then enqueues the device-to-host copies: an
    // invalid call returns OSC_INVALID with the caller's buffers untouched
    // (the reference rejects it at construction, oscillator.py:66-80).
    cudaStream_t pst = ctx->st[3];
    struct Events {
        std::vector<cudaEvent_t> ev;
        ~Events()
        {
            for (auto e : ev)
                cudaEventDestroy(e);
        }
    } evs;
    evs.ev.resize(2 * nchunk + 1, nullptr);  // [c]: m, C of chunk c up; [nchunk + 1 + c]: its kernels done
    for (auto &e : evs.ev)
        OSC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    OSC_CUDA(cudaEventRecord(evs.ev[nchunk], streams[0]));  // scratch allocated
    OSC_CUDA(cudaStreamWaitEvent(pst, evs.ev[nchunk], 0));
    for (int64_t c = 0; c < nchunk; ++c) {
        cudaStream_t st = streams[c % nstream];
        const int64_t b0 = bound(c), b1 = bound(c + 1), nb = b1 - b0;
        if (chains) {
            const size_t o = static_cast<size_t>(b0 * s), n = static_cast<size_t>(nb * s) * 8;
            OSC_CUDA(cudaMemcpyAsync(dm + o, m + o, n, H2D, pst));
            OSC_CUDA(cudaMemcpyAsync(dC + o, C + o, n, H2D, pst));
            OSC_CUDA(cudaEventRecord(evs.ev[c], pst));
            OSC_CUDA(cudaStreamWaitEvent(st, evs.ev[c], 0));
            OSC_CUDA(cudaMemcpyAsync(dx + o, x + o, n, H2D, st));
            OSC_CUDA(cudaMemcpyAsync(dv + o, v + o, n, H2D, st));
            if (int rc = osc_rk4_chains(dm + o, dC + o, dx + o, dv + o, nb, s, dt, nsteps,
                                        stride, dxs, dvs, nullptr, dfb + b0, 0, OSC_TRUSTED, st))
                return rc;
            OSC_CUDA(cudaEventRecord(evs.ev[nchunk + 1 + c], st));
        } else {
            // [2][B]: the chunk is packed as its own [2][nb] block on the device
            const size_t o = static_cast<size_t>(2 * b0), n = static_cast<size_t>(nb) * 8;
            for (int r = 0; r < 2; ++r) {
                OSC_CUDA(cudaMemcpyAsync(dm + o + r * nb, m + r * B + b0, n, H2D, pst));
                OSC_CUDA(cudaMemcpyAsync(dC + o + r * nb, C + r * B + b0, n, H2D, pst));
            }
            OSC_CUDA(cudaEventRecord(evs.ev[c], pst));
            OSC_CUDA(cudaStreamWaitEvent(st, evs.ev[c], 0));
            const double *hs[2] = {x, v};
            double *ds[2] = {dx, dv};
            for (int a = 0; a < 2; ++a)
                for (int r = 0; r < 2; ++r)
                    OSC_CUDA(cudaMemcpyAsync(ds[a] + o + r * nb, hs[a] + r * B + b0, n, H2D, st));
            if (int rc = batch2_entry(dm + o, dC + o, dx + o, dv + o, nb, dt, nsteps, stride,
                                      dxs, dvs, nullptr, dfb + b0, OSC_TRUSTED, st,
                                      nchunk > 1))
                return rc;
            OSC_CUDA(cudaEventRecord(evs.ev[nchunk + 1 + c], st));
        }
    }
    {
        int64_t bad[2];
        if (int rc = scan_params(dm, dC, static_cast<int64_t>(cells), pst, bad))
            return rc;  // (synchronises the parameter stream only)
        if (bad[0] >= 0 || bad[1] >= 0)  // the first offender in the caller's layout
            return host_param_fail(m, C, static_cast<int64_t>(cells), layout, B, s);
    }
    // results leave on the (now idle) parameter stream, each chunk as soon as
    // its kernels are done -- not behind the later chunks queued on its stream
    for (int64_t c = 0; c < nchunk; ++c) {
        cudaStream_t st = pst;
        OSC_CUDA(cudaStreamWaitEvent(st, evs.ev[nchunk + 1 + c], 0));
        const int64_t b0 = bound(c), b1 = bound(c + 1), nb = b1 - b0;
        if (chains) {
            const size_t o = static_cast<size_t>(b0 * s), n = static_cast<size_t>(nb * s) * 8;
            OSC_CUDA(cudaMemcpyAsync(x + o, dx + o, n, D2H, st));
            OSC_CUDA(cudaMemcpyAsync(v + o, dv + o, n, D2H, st));
        } else {
            const size_t o = static_cast<size_t>(2 * b0), n = static_cast<size_t>(nb) * 8;
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
    OSC_CUDA(cudaStreamSynchronize(pst));  // the result copies
    if (worst[0] != ~0ull)
        return fail(OSC_NONFINITE, "integration diverged at step %lld (system %lld)",
                    (long long)worst[0], (long long)worst[1]);
    return OSC_OK;
}

}  // namespace

extern "C" {

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

int osc_derivative_host(const double *m, const double *C, const double *x, double *dvel,
                        int64_t B, int64_t s, int cell_major)
{
    if (B < 0 || s < 1)
        return fail(OSC_INVALID, "need B >= 0 and s >= 1");
    if (B == 0)
        return OSC_OK;
    if (!m || !C || !x || !dvel)
        return fail(OSC_INVALID, "null buffer");
    const size_t cells = static_cast<size_t>(B * s), bytes = cells * sizeof(double);
    auto work = [&](double *d, cudaStream_t st, unsigned long long *bad) -> int {
        OSC_CUDA(osc::launch_derivative(d, d + cells, d + 2 * cells, d + 3 * cells + 2, B, s,
                                        cell_major != 0, st, bad));
        return OSC_OK;
    };
    return staged_call(3 * cells, cells, 0, cells, static_cast<int64_t>(cells),
                       {{m, bytes}, {C, bytes}, {x, bytes}}, {{dvel, bytes}}, work, m, C,
                       cell_major ? ParamLayout::CellMajor : ParamLayout::Chains, B, s, true);
}

int osc_energy_host(const double *m, const double *C, const double *x, const double *v,
                    double *out, int64_t B, int64_t s, int cell_major)
{
    if (B < 0 || s < 1)
        return fail(OSC_INVALID, "need B >= 0 and s >= 1");
    if (B == 0)
        return OSC_OK;
    if (!m || !C || !x || !v || !out)
        return fail(OSC_INVALID, "null buffer");
    const size_t cells = static_cast<size_t>(B * s), bytes = cells * sizeof(double);
    auto work = [&](double *d, cudaStream_t st, unsigned long long *bad) -> int {
        OSC_CUDA(osc::launch_energy(d, d + cells, d + 2 * cells, d + 3 * cells,
                                    d + 4 * cells + 2, B, s, cell_major != 0, st, bad));
        return OSC_OK;
    };
    return staged_call(4 * cells, static_cast<size_t>(B), 0, cells, static_cast<int64_t>(cells),
                       {{m, bytes}, {C, bytes}, {x, bytes}, {v, bytes}},
                       {{out, B * sizeof(double)}}, work, m, C,
                       cell_major ? ParamLayout::CellMajor : ParamLayout::Chains, B, s, true);
}

}  // extern "C"
