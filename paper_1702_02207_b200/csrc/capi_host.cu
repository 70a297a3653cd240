// Host-pointer forms of the batched entry points (synchronous; pinned or
// pageable buffers): chunked, multi-stream pipelines over capi.cu's
// device-pointer entry points.
#include "capi_internal.h"

using namespace osc_capi;

extern "C" {

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
    if (const char *e = std::getenv("OSC_HOST_CHUNKS")) {  // benchmarking knob
        const long long n = std::atoll(e);
        if (!xs && n >= 1 && n <= 64)
            nchunk = std::min<int64_t>(n, B);
    }
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

}  // extern "C"
