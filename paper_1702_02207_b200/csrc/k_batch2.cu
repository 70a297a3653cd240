// K1 batch2_rk4: millions of independent 2-DOF systems (BASELINE configs 0-1).
//
// Restates rk4_step + integrate (oscillator.py:194-263) for s = 2, one system
// per thread, the whole time loop register-resident: a system's 8 doubles are
// read from HBM once and its final state written once, so the kernel is
// bound by FP64 issue, not by the 48 B/DOF-step one-step-per-round-trip
// roofline.  Layout is SoA [2][B]: coordinate 0 of every system,
// then coordinate 1, so every load/store of a warp is one 256 B run.
//
// acceleration_at for s = 2 (oscillator.py:160-164), with d1 = x1 - x0:
//   i=0: left = x0 - 0.0 (== x0 exactly), a = (-C0)*x0, a += C1*d1, a /= m0
//   i=1: left = d1, a = (-C1)*d1 (no right neighbour), a /= m1
// (-C)*d == -(C*d) exactly under round-to-nearest, so f1 = C1*d1 is shared.
#include "osc_device.cuh"
#include "osc_kernels.h"

namespace osc {
namespace {

struct Sys2 {
    double x0, x1, v0, v1;
};

template <bool kExact>
__device__ __forceinline__ void accel2(double p0, double p1, double C0, double C1,
                                       const Divisor &m0, const Divisor &m1, double &a0,
                                       double &a1, bool &ok)
{
    const double d1 = sub(p1, p0);
    const double f1 = mul(C1, d1);
    const double g0 = mul(-C0, p0);
    a0 = qdiv<kExact>(add(g0, f1), m0, ok);
    a1 = qdiv<kExact>(-f1, m1, ok);
}

// One classical RK4 step (oscillator.py:208-231).  The combination sums are
// accumulated left to right exactly as combine_value's
// ((k1 + 2k2) + 2k3) + k4; 2.0*k is exact.
template <bool kExact>
__device__ __forceinline__ void step2(Sys2 &s, double C0, double C1, const Divisor &m0,
                                      const Divisor &m1, const StepConsts &k, bool &ok)
{
    double a0, a1;
    // k1 at the step start; position slopes are the velocities.
    accel2<kExact>(s.x0, s.x1, C0, C1, m0, m1, a0, a1, ok);
    double sx0 = s.v0, sx1 = s.v1, sv0 = a0, sv1 = a1;
    double yv0 = add(s.v0, mul(k.half_dt, a0));
    double yv1 = add(s.v1, mul(k.half_dt, a1));
    double yp0 = add(s.x0, mul(k.half_dt, s.v0));
    double yp1 = add(s.x1, mul(k.half_dt, s.v1));
    // k2 at the midpoint; y2v doubles as the k2 position slope.
    accel2<kExact>(yp0, yp1, C0, C1, m0, m1, a0, a1, ok);
    sx0 = add(sx0, mul(2.0, yv0));
    sx1 = add(sx1, mul(2.0, yv1));
    sv0 = add(sv0, mul(2.0, a0));
    sv1 = add(sv1, mul(2.0, a1));
    yp0 = add(s.x0, mul(k.half_dt, yv0));
    yp1 = add(s.x1, mul(k.half_dt, yv1));
    yv0 = add(s.v0, mul(k.half_dt, a0));
    yv1 = add(s.v1, mul(k.half_dt, a1));
    // k3 at the refined midpoint.
    accel2<kExact>(yp0, yp1, C0, C1, m0, m1, a0, a1, ok);
    sx0 = add(sx0, mul(2.0, yv0));
    sx1 = add(sx1, mul(2.0, yv1));
    sv0 = add(sv0, mul(2.0, a0));
    sv1 = add(sv1, mul(2.0, a1));
    yp0 = add(s.x0, mul(k.dt, yv0));
    yp1 = add(s.x1, mul(k.dt, yv1));
    yv0 = add(s.v0, mul(k.dt, a0));
    yv1 = add(s.v1, mul(k.dt, a1));
    // k4 at the endpoint, then the weighted combination.
    accel2<kExact>(yp0, yp1, C0, C1, m0, m1, a0, a1, ok);
    sx0 = add(sx0, yv0);
    sx1 = add(sx1, yv1);
    sv0 = add(sv0, a0);
    sv1 = add(sv1, a1);
    s.x0 = add(s.x0, mul(k.dt6, sx0));
    s.x1 = add(s.x1, mul(k.dt6, sx1));
    s.v0 = add(s.v0, mul(k.dt6, sv0));
    s.v1 = add(s.v1, mul(k.dt6, sv1));
}

__device__ __forceinline__ bool finite2(const Sys2 &s)
{
    return finite(s.x0) & finite(s.x1) & finite(s.v0) & finite(s.v1);
}

constexpr int kChunk = 64;  // steps between divergence checks

__global__ void __launch_bounds__(256)
batch2_rk4_kernel(const double *__restrict__ m, const double *__restrict__ C,
                  double *__restrict__ x, double *__restrict__ v, int64_t B,
                  StepConsts k, int64_t nsteps, int64_t stride, double *__restrict__ xs,
                  double *__restrict__ vs, int64_t *__restrict__ first_bad)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= B)
        return;
    const Divisor m0 = make_divisor(m[i]), m1 = make_divisor(m[B + i]);
    const double C0 = C[i], C1 = C[B + i];
    Sys2 s{x[i], x[B + i], v[i], v[B + i]};
    if (xs) {
        xs[i] = s.x0;
        xs[B + i] = s.x1;
        vs[i] = s.v0;
        vs[B + i] = s.v1;
    }
    const bool ok0 = divisor_fast_ok(m0) & divisor_fast_ok(m1);
    int64_t bad = 0;
    int64_t kstep = 0;
    while (kstep < nsteps) {
        const int64_t next_sample = (kstep / stride + 1) * stride;
        int64_t n = nsteps - kstep;
        if (next_sample - kstep < n)
            n = next_sample - kstep;
        if (n > kChunk)
            n = kChunk;
        const Sys2 saved = s;
        bool ok = ok0;
        for (int j = 0; j < n; ++j)
            step2<false>(s, C0, C1, m0, m1, k, ok);
        if (!(ok & finite2(s))) {
            // A division left nvcc's fast path or a value went non-finite:
            // replay the chunk with IEEE division, checking every step.
            // Non-finite values are absorbing under + - * /, so the first
            // non-finite step is integrate's NonFiniteStateError.step
            // (oscillator.py:255-260).
            s = saved;
            for (int j = 0; j < n; ++j) {
                step2<true>(s, C0, C1, m0, m1, k, ok);
                if (!finite2(s)) {
                    bad = kstep + j + 1;
                    break;
                }
            }
            if (bad)
                break;
        }
        kstep += n;
        if (xs && kstep % stride == 0) {
            const int64_t o = (kstep / stride) * 2 * B;
            xs[o + i] = s.x0;
            xs[o + B + i] = s.x1;
            vs[o + i] = s.v0;
            vs[o + B + i] = s.v1;
        }
    }
    x[i] = s.x0;
    x[B + i] = s.x1;
    v[i] = s.v0;
    v[B + i] = s.v1;
    first_bad[i] = bad;
}

}  // namespace

cudaError_t launch_batch2(const double *m, const double *C, double *x, double *v, int64_t B,
                          StepConsts k, int64_t nsteps, int64_t stride, double *xs, double *vs,
                          int64_t *first_bad, cudaStream_t stream)
{
    const int threads = 256;
    const int64_t blocks = (B + threads - 1) / threads;
    batch2_rk4_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
        m, C, x, v, B, k, nsteps, stride, xs, vs, first_bad);
    return cudaGetLastError();
}

}  // namespace osc
