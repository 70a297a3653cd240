// Peer memory and multi-GPU entry points: device allocations and CUDA IPC
// handles/events, stream-ordered counters, and one chain sharded over the
// GPUs of a process with the fused halo exchange.
#include <cuda.h>  // driver types only: entry points via cudaGetDriverEntryPoint

#include "capi_internal.h"

#include <cstdlib>

using namespace osc_capi;

extern "C" {

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
// One shard's period loop of the multi-process fused exchange.
// ---------------------------------------------------------------------------
int osc_rk4_shard_run(osc_shard_t *sh, double dt, int64_t nsteps, int64_t halo_steps,
                      int64_t step0, uint32_t flags, void *stream)
{
    if (!sh)
        return fail(OSC_INVALID, "null shard");
    if (int rc = check_run_args(dt, nsteps, 1))
        return rc;
    if (halo_steps < 1 || sh->ghost < 0)
        return fail(OSC_INVALID, "halo_steps must be >= 1");
    const int64_t T = halo_steps;
    for (int64_t k = 0; k < nsteps;) {
        const int64_t n = std::min(T, nsteps - k);
        const int b = static_cast<int>(sh->sync.period & 1), nb = b ^ 1;
        osc_peer_t peer[2] = {};
        for (int side = 0; side < 2; ++side)
            if (sh->nx[side][nb])
                peer[side] = osc_peer_t{sh->nx[side][nb], sh->nv[side][nb], sh->offset[side],
                                        sh->ghost};
        if (int rc = osc_rk4_chain_advance_div2(sh->m, sh->C, sh->x[b], sh->v[b], sh->x[nb],
                                                sh->v[nb], sh->n, sh->own_lo, sh->own_hi, dt, n,
                                                step0 + k, sh->first_bad,
                                                peer[0].x ? &peer[0] : nullptr,
                                                peer[1].x ? &peer[1] : nullptr, &sh->sync,
                                                sh->div2, flags | OSC_TRUSTED, stream))
            return rc;
        ++sh->sync.period;
        k += n;
    }
    return OSC_OK;
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
    double *div2 = nullptr;  // the shard's two-operation division table (3n words)
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
                            (void *)r.v2, (void *)r.fb, (void *)r.div2})
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
    if (flags & ~kRunFlags)
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
    // the parameter rule (oscillator.py:66-80), one device pass per shard;
    // the exact first offender is then located in the caller's arrays
    if (!(flags & OSC_TRUSTED)) {
        bool any = false;
        for (auto &r : set.sh) {
            OSC_CUDA(cudaSetDevice(r.dev));
            int64_t bad[2];
            if (int rc = scan_params(r.m, r.C, r.n, r.st, bad))
                return rc;
            any = any || bad[0] >= 0 || bad[1] >= 0;
        }
        if (any)
            return host_param_fail(m, C, s, ParamLayout::Flat);
    }
    flags |= OSC_TRUSTED;  // per-period launches below skip the check
    if (!(flags & OSC_FMA)) {  // each shard's two-operation division table, once
        const char *d2env = std::getenv("OSC_DIV2");
        if (!(d2env && d2env[0] == '0'))
            for (auto &r : set.sh) {
                OSC_CUDA(cudaSetDevice(r.dev));
                OSC_CUDA(cudaMalloc(reinterpret_cast<void **>(&r.div2), 3 * r.n * D));
                if (int rc = osc_div2c_table(r.m, r.n, r.div2, r.div2 + r.n,
                                             reinterpret_cast<uint64_t *>(r.div2 + 2 * r.n),
                                             r.st))
                    return rc;
            }
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
            if (int rc = osc_rk4_chain_advance_div2(r.m, r.C, r.x, r.v, r.x2, r.v2, r.n,
                                                    r.own_lo, r.own_hi, dt, n, k, r.fb,
                                                    i > 0 ? &left : nullptr,
                                                    i + 1 < ngpu ? &right : nullptr, nullptr,
                                                    r.div2, flags, r.st))
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
