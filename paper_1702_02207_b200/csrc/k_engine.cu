// The paper's thread-per-equation engine on one warp.
//
// The reference's run_parallel (parallel.py:395-573) gives each of the 2s
// first-order equations to a worker thread; workers exchange stage values
// through double-banked shared cells (SharedPhase, parallel.py:100-166) and
// meet at a StageBarrier five times per step (parallel.py:473-520).  Here the
// workers are the lanes of one warp (equation j -> lane j % 32), the banks are
// two shared-memory arrays and the barrier is __syncwarp.  Every lane applies
// the same helpers in the same order (acceleration_at, stage_value,
// combine_value, oscillator.py:152-174), so the trajectory is bit-identical
// to integrate(), as the reference engine's is (parallel.py:11-14).  Lane 0
// stamps %globaltimer around every step: the per-step latency whose
// distribution the paper studies (section 4), on a GPU SM.
#include "osc_device.cuh"
#include "osc_kernels.h"

namespace osc {
namespace {

constexpr int kMaxEq = 128;  // 2s <= 128: s <= 64, at most 4 equations per lane

__device__ __forceinline__ uint64_t globaltimer()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// acceleration_at (oscillator.py:160-164) reading positions from a bank.
__device__ __forceinline__ double accel_at(const double *m, const double *C, const double *pos,
                                           int i, int s)
{
    const double left = sub(pos[i], i > 0 ? pos[i - 1] : 0.0);
    double a = mul(-C[i], left);
    if (i + 1 < s)
        a = add(a, mul(C[i + 1], sub(pos[i + 1], pos[i])));
    return __ddiv_rn(a, m[i]);
}

__device__ __forceinline__ double combine(double base, double dt, double k1, double k2,
                                          double k3, double k4)
{
    // base + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)   (oscillator.py:174)
    return add(base, mul(__ddiv_rn(dt, 6.0),
                         add(add(add(k1, mul(2.0, k2)), mul(2.0, k3)), k4)));
}

__global__ void __launch_bounds__(32) equation_engine_kernel(
    const double *__restrict__ m, const double *__restrict__ C, const double *__restrict__ x0,
    const double *__restrict__ v0, int s, double dt, int64_t nsteps, int64_t stride,
    double *__restrict__ xs, double *__restrict__ vs, int64_t *__restrict__ first_bad,
    int64_t *__restrict__ step_ns)
{
    __shared__ double bank_a[kMaxEq], bank_b[kMaxEq];
    __shared__ double sm[kMaxEq / 2], sC[kMaxEq / 2];
    const int lane = threadIdx.x;
    const int neq = 2 * s;
    for (int j = lane; j < s; j += 32) {
        sm[j] = m[j];
        sC[j] = C[j];
    }
    for (int j = lane; j < neq; j += 32)
        bank_a[j] = j < s ? x0[j] : v0[j - s];
    __syncwarp();
    constexpr int E = kMaxEq / 32;
    double y0[E], k1[E], k2[E], k3[E];
    const double half_dt = 0.5 * dt;
    // slope of equation j at a snapshot: dx_j = v_j, dv_i = acceleration_at
    const auto slope = [&](const double *snap, int j) {
        return j < s ? snap[s + j] : accel_at(sm, sC, snap, j - s, s);
    };
    if (xs) {
        for (int j = lane; j < neq; j += 32)
            (j < s ? xs[j] : vs[j - s]) = bank_a[j];
    }
    int64_t bad = 0;
    for (int64_t step = 0; step < nsteps && !bad; ++step) {
        const uint64_t t0 = globaltimer();
        // Stage 1: derivative at the committed state (bank A) -> bank B.
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = lane + 32 * e;
            if (j < neq) {
                y0[e] = bank_a[j];
                k1[e] = slope(bank_a, j);
                bank_b[j] = add(y0[e], mul(half_dt, k1[e]));
            }
        }
        __syncwarp();
        // Stage 2: midpoint estimate (bank B) -> bank A (no lane reads A now).
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = lane + 32 * e;
            if (j < neq) {
                k2[e] = slope(bank_b, j);
                bank_a[j] = add(y0[e], mul(half_dt, k2[e]));
            }
        }
        __syncwarp();
        // Stage 3: refined midpoint (bank A) -> bank B.
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = lane + 32 * e;
            if (j < neq) {
                k3[e] = slope(bank_a, j);
                bank_b[j] = add(y0[e], mul(dt, k3[e]));
            }
        }
        __syncwarp();
        // Stage 4 and the combination -> bank A.
        double k4[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = lane + 32 * e;
            if (j < neq)
                k4[e] = slope(bank_b, j);
        }
        __syncwarp();
        bool nonfinite = false;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = lane + 32 * e;
            if (j < neq) {
                const double val = combine(y0[e], dt, k1[e], k2[e], k3[e], k4[e]);
                nonfinite |= !finite(val);
                bank_a[j] = val;
            }
        }
        __syncwarp();
        if (__any_sync(kFull, nonfinite))
            bad = step + 1;  // NonFiniteStateError.step (parallel.py:511-515)
        else if (xs && (step + 1) % stride == 0) {
            const int64_t o = ((step + 1) / stride) * s;
            for (int j = lane; j < neq; j += 32)
                (j < s ? xs[o + j] : vs[o + j - s]) = bank_a[j];
        }
        if (lane == 0)
            step_ns[step] = static_cast<int64_t>(globaltimer() - t0);
    }
    if (lane == 0)
        *first_bad = bad;
}

}  // namespace

cudaError_t launch_equation_engine(const double *m, const double *C, const double *x0,
                                   const double *v0, int s, double dt, int64_t nsteps,
                                   int64_t stride, double *xs, double *vs, int64_t *first_bad,
                                   int64_t *step_ns, cudaStream_t stream)
{
    if (2 * s > kMaxEq)
        return cudaErrorInvalidValue;
    equation_engine_kernel<<<1, 32, 0, stream>>>(m, C, x0, v0, s, dt, nsteps, stride, xs, vs,
                                                 first_bad, step_ns);
    return cudaGetLastError();
}

}  // namespace osc
