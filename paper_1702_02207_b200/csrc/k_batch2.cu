// K1 batch2_rk4: millions of independent 2-DOF systems (BASELINE configs 0-1).
//
// Restates rk4_step + integrate (oscillator.py:194-263) for s = 2, one system
// per thread, the whole time loop register-resident: a system's 8 doubles are
// read from HBM once and its final state written once, so the kernel is
// bound by FP64 issue, not by the 48 B/DOF-step one-step-per-round-trip
// roofline.  Layout is SoA [2][B]: coordinate 0 of every system,
// then coordinate 1, so a warp's loads/stores are 256 B runs.  Divisions by
// the masses take two operations (div2s, osc_device.cuh) in every warp
// whose systems' masses all have a div2 class: a classify kernel and a
// stable cub partition put those systems first (Div2Plan).
//
// acceleration_at for s = 2 (oscillator.py:160-164), with d1 = x1 - x0:
//   i=0: left = x0 - 0.0 (== x0 exactly), a = (-C0)*x0, a += C1*d1, a /= m0
//   i=1: left = d1, a = (-C1)*d1 (no right neighbour), a /= m1
// (-C)*d == -(C*d) exactly under round-to-nearest, so f1 = C1*d1 is shared.
#include "k_batch2_impl.cuh"

#include <cstdio>
#include <cstdlib>

#include <cub/device/device_partition.cuh>
#include <thrust/iterator/counting_iterator.h>

namespace osc {

cudaError_t launch_batch2(const double *m, const double *C, double *x, double *v, int64_t B,
                          StepConsts k, int64_t nsteps, int64_t stride, double *xs, double *vs,
                          double *es, int64_t *first_bad, bool fma, cudaStream_t stream,
                          const CmpArgs *cmp, bool wide)
{
    // Launch shape: NS systems per thread x threads per CTA.  OSC_B2="NS,threads"
    // overrides it for benchmarking (read-only process state).
    int ns = kBatch2NS, threads = kBatch2Threads;
    // Fewer systems than ~2048 per SM (the per-rank slices of C2 at 4 and 8
    // GPUs: 2^18, 2^17): one system per thread in 128-thread CTAs -- many
    // small CTAs, no partly filled last wave.  Measured on B200
    // (scripts/k1_split_sweep.py, profiles/r02/k1_split.txt): 2^18 systems
    // 3.64e11 -> 4.07e11 DOF-steps/s, 2^17 3.49e11 -> 3.95e11; 2^19 and 2^20
    // keep NS=2 x 256.  C1 (a single latency-bound system) stays below.
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (B < int64_t(sms) * 2048 && !(wide && B >= int64_t(sms) * 256)) {
        ns = 1;
        threads = 128;
    }
    if (B <= int64_t(sms) * 32)
        threads = 32;  // at most one warp per SM anyway: the latency build
    if (const char *e = std::getenv("OSC_B2")) {
        int a = 0, b = 0;
        if (std::sscanf(e, "%d,%d", &a, &b) == 2 && (a == 1 || a == 2 || a == 4) && b >= 32 &&
            b <= 256 && b % 32 == 0) {
            ns = a;
            threads = b;
        }
    }
    // Two-operation division (div2_classify): classify every system, then
    // list the passing ones first.  OSC_DIV2=0 disables it (A/B timing); the
    // FMA mode keeps its own x*(1/m).
    Div2Plan plan{nullptr, nullptr};
    void *scratch = nullptr;
    const char *d2 = std::getenv("OSC_DIV2");
    if (!fma && B > 0 && !(d2 && d2[0] == '0')) {
        const thrust::counting_iterator<int64_t> ids(0);
        size_t temp = 0;
        cudaError_t e = cub::DevicePartition::Flagged(
            nullptr, temp, ids, static_cast<const uint8_t *>(nullptr),
            static_cast<int64_t *>(nullptr), static_cast<int64_t *>(nullptr), B, stream);
        if (e != cudaSuccess)
            return e;
        const size_t off_cls = size_t(B + 1) * sizeof(int64_t);  // mcls [2][B], sys [B]
        const size_t off_tmp = (off_cls + 3 * size_t(B) + 255) & ~size_t(255);
        if ((e = scratch_alloc(&scratch, off_tmp + temp, stream)) != cudaSuccess)
            return e;
        char *p = static_cast<char *>(scratch);
        int64_t *order = reinterpret_cast<int64_t *>(p);
        uint8_t *mcls = reinterpret_cast<uint8_t *>(p + off_cls), *sys = mcls + 2 * B;
        const int64_t want = (B + 255) / 256;
        const unsigned grid = static_cast<unsigned>(want < int64_t(sms) * 32 ? want : int64_t(sms) * 32);
        batch2_classify_kernel<<<grid, 256, 0, stream>>>(m, B, mcls, sys);
        e = cudaGetLastError();
        if (e == cudaSuccess)
            e = cub::DevicePartition::Flagged(p + off_tmp, temp, ids, sys, order, order + B, B,
                                              stream);
        if (e != cudaSuccess) {
            cudaFreeAsync(scratch, stream);
            return e;
        }
        plan = Div2Plan{order, mcls};
    }
    cudaError_t e;
    switch (ns) {
    case 1: e = launch_ns<1>(m, C, x, v, B, k, nsteps, stride, xs, vs, es, first_bad, threads, fma, stream, cmp, plan);
        break;
    default:  // 2 or 4 systems per thread: the throughput builds' own translation unit
        e = launch_batch2_wide(ns, m, C, x, v, B, k, nsteps, stride, xs, vs, es, first_bad, threads,
                               fma, stream, cmp, plan);
    }
    if (scratch) {
        const cudaError_t f = cudaFreeAsync(scratch, stream);
        if (e == cudaSuccess)
            e = f;
    }
    return e;
}

}  // namespace osc
