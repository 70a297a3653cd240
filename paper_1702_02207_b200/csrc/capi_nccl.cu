// The NCCL transport's period loop in native code (one process per GPU).
//
// Per period (T steps) of a chain shard: the interior tiles -- those that
// read no ghost cell -- run on the caller's stream while, on a side stream
// that waited for the previous period only, the ghost zones of the current
// buffer are refreshed by NCCL point-to-point transfers with the two
// neighbouring ranks (x and v, `ghost` cells each way: the halo exchange of
// SURVEY 8(e), ncclGroupStart; ncclSend/ncclRecv; ncclGroupEnd) and then ONE
// launch covers the edge tiles of both sides; the caller's stream waits for
// the side stream before the next period.  The same schedule as
// sharded.ShardedChain.run's NCCL transport, without a Python round trip per
// period.  Counterpart of the reference's per-stage publish/snapshot of the
// shared phase (parallel.py:136-155); bytes equal a single-GPU run.
//
// libnccl.so.2 is not linked: it is opened at the first call (the process
// that owns the communicator has it loaded already, e.g. through torch).
#include "capi_internal.h"

#include <dlfcn.h>

#include <algorithm>
#include <mutex>

using namespace osc_capi;

namespace {

// The few NCCL entry points used, by their C signatures (nccl.h): ncclComm_t
// is an opaque pointer, ncclDataType_t / ncclResult_t are ints.
constexpr int kNcclFloat64 = 8;  // ncclFloat64
using GroupFn = int (*)();
using P2PFn = int (*)(void *, size_t, int, int, void *, cudaStream_t);
using ErrFn = const char *(*)(int);

struct Nccl {
    GroupFn group_start = nullptr, group_end = nullptr;
    P2PFn send = nullptr, recv = nullptr;
    ErrFn error = nullptr;
    const char *why = "not loaded";
};

const Nccl &nccl()
{
    static Nccl api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = "libnccl.so.2 not found";
            return;
        }
        api.group_start = reinterpret_cast<GroupFn>(dlsym(h, "ncclGroupStart"));
        api.group_end = reinterpret_cast<GroupFn>(dlsym(h, "ncclGroupEnd"));
        api.send = reinterpret_cast<P2PFn>(dlsym(h, "ncclSend"));
        api.recv = reinterpret_cast<P2PFn>(dlsym(h, "ncclRecv"));
        api.error = reinterpret_cast<ErrFn>(dlsym(h, "ncclGetErrorString"));
        if (!api.group_start || !api.group_end || !api.send || !api.recv || !api.error)
            api.why = "libnccl.so.2 lacks ncclGroupStart/ncclSend/ncclRecv";
        else
            api.why = nullptr;
    });
    return api;
}

struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
    ~SideStream()  // no synchronisation: released once their work is done
    {
        if (ready)
            cudaEventDestroy(ready);
        if (done)
            cudaEventDestroy(done);
        if (s)
            cudaStreamDestroy(s);
    }
};

// The ghost refresh of buffer (x, v) with the neighbours, as one NCCL group.
int exchange(const Nccl &api, void *comm, int rank, int nranks, double *x, double *v,
             int64_t own_lo, int64_t own_hi, int64_t g, cudaStream_t st)
{
    if (int e = api.group_start())
        return fail(OSC_CUDA_ERROR, "ncclGroupStart: %s", api.error(e));
    int e = 0;
    const size_t n = static_cast<size_t>(g);
    if (rank > 0) {  // our first g owned cells out, the left neighbour's last g into our ghosts
        for (double *a : {x, v}) {
            if (!e)
                e = api.send(a + own_lo, n, kNcclFloat64, rank - 1, comm, st);
            if (!e)
                e = api.recv(a + own_lo - g, n, kNcclFloat64, rank - 1, comm, st);
        }
    }
    if (rank + 1 < nranks) {
        for (double *a : {x, v}) {
            if (!e)
                e = api.send(a + own_hi - g, n, kNcclFloat64, rank + 1, comm, st);
            if (!e)
                e = api.recv(a + own_hi, n, kNcclFloat64, rank + 1, comm, st);
        }
    }
    const int e2 = api.group_end();
    if (e || e2)
        return fail(OSC_CUDA_ERROR, "NCCL halo exchange: %s", api.error(e ? e : e2));
    return OSC_OK;
}

}  // namespace

extern "C" {

int osc_rk4_shard_run_nccl(osc_shard_t *sh, void *comm, int rank, int nranks, double dt,
                           int64_t nsteps, int64_t halo_steps, int64_t step0, uint32_t flags,
                           void *stream_)
{
    if (!sh)
        return fail(OSC_INVALID, "null shard");
    if (flags & ~kRunFlags)
        return fail(OSC_INVALID, "unknown flags 0x%x", flags);
    if (int rc = check_run_args(dt, nsteps, 1))
        return rc;
    if (halo_steps < 1 || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(OSC_INVALID, "need halo_steps >= 1 and 0 <= rank < nranks");
    const int64_t g = sh->ghost;
    if ((rank > 0 && sh->own_lo < g) || (rank + 1 < nranks && sh->own_hi + g > sh->n) ||
        (nranks > 1 && (g < 2 * halo_steps || g > sh->own_hi - sh->own_lo)))
        return fail(OSC_INVALID, "ghost zones of %lld cells do not fit the shard (T=%lld)",
                    (long long)g, (long long)halo_steps);
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    const bool multi = nranks > 1;
    const Nccl *api = nullptr;
    SideStream side;
    if (multi) {
        if (!comm)
            return fail(OSC_INVALID, "null NCCL communicator");
        api = &nccl();
        if (api->why)
            return fail(OSC_CUDA_ERROR, "%s", api->why);
        OSC_CUDA(cudaStreamCreateWithFlags(&side.s, cudaStreamNonBlocking));
        OSC_CUDA(cudaEventCreateWithFlags(&side.ready, cudaEventDisableTiming));
        OSC_CUDA(cudaEventCreateWithFlags(&side.done, cudaEventDisableTiming));
    }
    flags |= OSC_TRUSTED;  // validated once per shard (osc_validate_parameters)
    for (int64_t k = 0; k < nsteps;) {
        const int64_t n = std::min(halo_steps, nsteps - k);
        const int b = static_cast<int>(sh->sync.period & 1), nb = b ^ 1;
        auto advance = [&](uint32_t subset, cudaStream_t st) {
            return osc_rk4_chain_advance_div2(sh->m, sh->C, sh->x[b], sh->v[b], sh->x[nb],
                                              sh->v[nb], sh->n, sh->own_lo, sh->own_hi, dt, n,
                                              step0 + k, sh->first_bad, nullptr, nullptr,
                                              nullptr, sh->div2, flags | subset, st);
        };
        if (!multi) {
            if (int rc = advance(0, stream))
                return rc;
        } else {
            OSC_CUDA(cudaEventRecord(side.ready, stream));  // the previous period is done
            if (int rc = advance(OSC_TILES_INTERIOR, stream))
                return rc;
            OSC_CUDA(cudaStreamWaitEvent(side.s, side.ready, 0));
            if (int rc = exchange(*api, comm, rank, nranks, sh->x[b], sh->v[b], sh->own_lo,
                                  sh->own_hi, g, side.s))
                return rc;
            if (int rc = advance(OSC_TILES_EDGES, side.s))
                return rc;
            OSC_CUDA(cudaEventRecord(side.done, side.s));
            OSC_CUDA(cudaStreamWaitEvent(stream, side.done, 0));
        }
        ++sh->sync.period;
        k += n;
    }
    return OSC_OK;
}

}  // extern "C"
