// K1's kernel template and its launcher, shared by the two translation units
// that instantiate it: k_batch2.cu (the one-system builds: C1's latency launch
// and the 128-thread build of small batches) and k_batch2_wide.cu (the
// two- and four-systems-per-thread throughput builds, C2).  Two units because
// the throughput loops schedule best at ptxas register-usage level 2 (C2
// 47.62 -> 47.29 ms) while the one-system builds lose with it (C1 93.8 ->
// 101.5 ns/step): build.py's PER_SOURCE_FLAGS gives the option to the wide
// unit only.
#pragma once
#include "osc_device.cuh"
#include "osc_kernels.h"
#include "osc_modal.cuh"

#include <cstdint>

namespace osc {

// Launch order of the systems for the two-operation division: mcls [2][B]
// holds the div2_classify class of every mass, sys[i] != 0 when both masses
// of system i have one; order lists those systems first (ascending), so all
// but one boundary warp are uniform.  order == nullptr: identity order,
// three-operation division everywhere.
struct Div2Plan {
    const int64_t *order;
    const uint8_t *mcls;
};

// ns = 2 or 4 systems per thread (k_batch2_wide.cu).
cudaError_t launch_batch2_wide(int ns, const double *m, const double *C, double *x, double *v,
                               int64_t B, StepConsts k, int64_t nsteps, int64_t stride,
                               double *xs, double *vs, double *es, int64_t *first_bad,
                               int threads, bool fma, cudaStream_t stream, const CmpArgs *cmp,
                               Div2Plan plan);

namespace {


// Range tests of the two-operation loops: on the step's START state only
// (Arith::Fast2S, state_range_ok: 6 FSETPs per system-step, none on the step's
// dependency chain; osc_device.cuh has the argument).  C2 48.14 -> 47.76 ms,
// C1 96.0 -> 93.8 ns/step (profiles/r02/README.md).  kVT (the three-operation
// loop of the one-system builds): one start-velocity test per step for the
// fused position sums (add_twice_fused) instead of a test per sum.

// Default launch shape (profiles/r01 sweep).
constexpr int kBatch2NS = 2, kBatch2Threads = 256;

struct Sys2 {
    double x0, x1, v0, v1;
};

template <Arith A>
__device__ __forceinline__ void accel2(double p0, double p1, double C0, double C1,
                                       const Divisor &m0, const Divisor &m1, double &a0,
                                       double &a1, bool &ok)
{
    const double d1 = sub(p1, p0);
    const double f1 = mul(C1, d1);
    const double num0 = (A == Arith::Fma) ? __fma_rn(-C0, p0, f1) : add(mul(-C0, p0), f1);
    a0 = qdiv<A>(num0, m0, ok);
    if constexpr (A == Arith::Fast2S) {
        // Untested quotients must be right for a ZERO numerator too.  f1 = +0
        // when p1 == p0 (never -0: a stage position x + c*y of a nonzero x is
        // never -0, so d1 is not either), and (-f1)/m1 is then -0; but
        // RN((-0)*zh + RN((-0)*zl)) is +0 when zl < 0.  So the quotient is
        // negated instead of the numerator: RN(f1*zh + RN(f1*zl)) = +0 for
        // either sign of zl, and -(f1/m1) == (-f1)/m1 bit for bit otherwise.
        // The negation folds into the operand modifiers of the uses.  (num0 =
        // RN((-C0 p0) + f1) is +0 when it is zero; +0/m0 = +0 either way.)
        a1 = -div2s(f1, m1);
    } else {
        a1 = qdiv_neg<A>(f1, m1, ok);
    }
}

// One classical RK4 step (oscillator.py:208-231).  The combination sums are
// accumulated left to right exactly as combine_value's
// ((k1 + 2k2) + 2k3) + k4; 2.0*k is exact.
template <Arith A, bool kVT = false>
__device__ __forceinline__ void step2(Sys2 &s, double C0, double C1, const Divisor &m0,
                                      const Divisor &m1, const StepConsts &k, bool &ok)
{
    double a0, a1;
    // add_twice_fused's condition (osc_device.cuh): the start velocities,
    // once per step, instead of a test per fused position sum
    // Fast2S: the range of the step's START state replaces every per-quotient
    // and per-sum test of the step (div2s, osc_device.cuh)
    constexpr bool kState = A == Arith::Fast2S;
    constexpr bool kFused = (kVT || kState) && A != Arith::Exact && A != Arith::Fma;
    if constexpr (kState)
        ok &= state_range_ok(s.x0, s.v0) & state_range_ok(s.x1, s.v1);
    else if constexpr (kFused)
        ok &= velocity_small(s.v0) & velocity_small(s.v1);
    // k1 at the step start; position slopes are the velocities.
    accel2<A>(s.x0, s.x1, C0, C1, m0, m1, a0, a1, ok);
    double sx0 = s.v0, sx1 = s.v1, sv0 = a0, sv1 = a1;
    double yv0 = stage<A>(s.v0, k.half_dt, a0);
    double yv1 = stage<A>(s.v1, k.half_dt, a1);
    double yp0 = stage<A>(s.x0, k.half_dt, s.v0);
    double yp1 = stage<A>(s.x1, k.half_dt, s.v1);
    // k2 at the midpoint; y2v doubles as the k2 position slope.
    accel2<A>(yp0, yp1, C0, C1, m0, m1, a0, a1, ok);
    sx0 = kFused ? add_twice_fused<A>(sx0, yv0) : add_twice_checked<A>(sx0, yv0, ok);
    sx1 = kFused ? add_twice_fused<A>(sx1, yv1) : add_twice_checked<A>(sx1, yv1, ok);
    sv0 = add_twice<A>(sv0, a0);
    sv1 = add_twice<A>(sv1, a1);
    yp0 = stage<A>(s.x0, k.half_dt, yv0);
    yp1 = stage<A>(s.x1, k.half_dt, yv1);
    yv0 = stage<A>(s.v0, k.half_dt, a0);
    yv1 = stage<A>(s.v1, k.half_dt, a1);
    // k3 at the refined midpoint.
    accel2<A>(yp0, yp1, C0, C1, m0, m1, a0, a1, ok);
    sx0 = kFused ? add_twice_fused<A>(sx0, yv0) : add_twice_checked<A>(sx0, yv0, ok);
    sx1 = kFused ? add_twice_fused<A>(sx1, yv1) : add_twice_checked<A>(sx1, yv1, ok);
    sv0 = add_twice<A>(sv0, a0);
    sv1 = add_twice<A>(sv1, a1);
    yp0 = stage<A>(s.x0, k.dt, yv0);
    yp1 = stage<A>(s.x1, k.dt, yv1);
    yv0 = stage<A>(s.v0, k.dt, a0);
    yv1 = stage<A>(s.v1, k.dt, a1);
    // k4 at the endpoint, then the weighted combination.
    accel2<A>(yp0, yp1, C0, C1, m0, m1, a0, a1, ok);
    sx0 = add(sx0, yv0);
    sx1 = add(sx1, yv1);
    sv0 = add(sv0, a0);
    sv1 = add(sv1, a1);
    s.x0 = stage<A>(s.x0, k.dt6, sx0);
    s.x1 = stage<A>(s.x1, k.dt6, sx1);
    s.v0 = stage<A>(s.v0, k.dt6, sv0);
    s.v1 = stage<A>(s.v1, k.dt6, sv1);
}

// energy() (oscillator.py:266-276) of one 2-DOF system, in the reference's
// order: total += 0.5*m*v*v; total += 0.5*C*ext*ext, cell by cell.
__device__ __forceinline__ double energy2(const Sys2 &s, double m0, double m1, double C0,
                                          double C1)
{
    double total = 0.0;
    total = add(total, mul(mul(mul(0.5, m0), s.v0), s.v0));
    total = add(total, mul(mul(mul(0.5, C0), s.x0), s.x0));  // ext = x0 - 0.0 == x0
    total = add(total, mul(mul(mul(0.5, m1), s.v1), s.v1));
    const double e1 = sub(s.x1, s.x0);
    total = add(total, mul(mul(mul(0.5, C1), e1), e1));
    return total;
}

__device__ __forceinline__ bool finite2(const Sys2 &s)
{
    return finite(s.x0) & finite(s.x1) & finite(s.v0) & finite(s.v1);
}

#ifndef OSC_B2_CHUNK
#define OSC_B2_CHUNK 512  // measured: C2 47.31 / 47.21 / 47.16 / 47.13 / 47.13 ms, C1 93.8 / 91.5 / 90.5 / 90.1 / 90.1 ns per step at 64 / 128 / 256 / 512 / 1024
#endif
constexpr int kChunk = OSC_B2_CHUNK;  // steps between divergence checks
#ifndef OSC_B2_UNROLL
#define OSC_B2_UNROLL 2  // steps per hot-loop iteration (variant builds: scripts/build_variants.py); 2 measured best with the state-range tests (47.62 ms vs 47.78 at 4, 47.97 at 3, 48.14 at 1)
#endif
constexpr int kUnroll = OSC_B2_UNROLL;
#ifndef OSC_NS1_STATE
#define OSC_NS1_STATE 1  // one-system builds: 0 numerator tests, 1 state tests, 2 state tests in the 128-thread build only
#endif

__global__ void batch2_classify_kernel(const double *__restrict__ m, int64_t B,
                                       uint8_t *__restrict__ mcls, uint8_t *__restrict__ sys)
{
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < B;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double zh, zl;
        const int a = div2_classify(m[i], zh, zl);
        const int b = div2_classify(m[B + i], zh, zl);
        mcls[i] = static_cast<uint8_t>(a);
        mcls[B + i] = static_cast<uint8_t>(b);
        sys[i] = a != 0 && b != 0;
    }
}

// NS systems per thread, interleaved for instruction-level parallelism:
// slot j of thread t in block b is g = b*NS*blockDim + j*blockDim + t and
// holds system order[g] (g itself without a plan).  The partition is stable,
// so a warp's systems stay one contiguous 256 B run except where unclassed
// systems were moved out; loads and stores happen once per run.  Slots past
// B duplicate the last one and are never stored.  kCmp: also accumulate
// compare() against the analytic solution at every retained sample (when
// cmp.sol is set).
template <int NS, bool kFma, bool kCmp = false, int kMaxThreads = 256>
__global__ void __launch_bounds__(kMaxThreads, (NS == 2 && kMaxThreads == 256) ? 2 : 1)
batch2_rk4_kernel(const double *__restrict__ m, const double *__restrict__ C,
                  double *__restrict__ x, double *__restrict__ v, int64_t B,
                  StepConsts k, int64_t nsteps, int64_t stride, double *__restrict__ xs,
                  double *__restrict__ vs, double *__restrict__ es,
                  int64_t *__restrict__ first_bad, Div2Plan plan, CmpArgs cmp = CmpArgs{})
{
    // Two-operation loop: range tests on the step's start state (Fast2S) or,
    // in the builds OSC_NS1_STATE leaves out, on each numerator (Fast2A).
    constexpr bool kStateTests = NS > 1 || (OSC_NS1_STATE == 1) ||
                                 (OSC_NS1_STATE == 2 && kMaxThreads == 128);
    const int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x * NS + threadIdx.x;
    int64_t idx[NS];
    bool live[NS];
    // Divisor words of both masses: (b, y) for the three-operation division,
    // (zh, zl) for the two-operation one.  A warp runs the two-operation
    // division only when every one of its systems passed div2_classify
    // (plan.order groups those systems); its exact replay re-reads b.
    double u0[NS], w0[NS], u1[NS], w1[NS];
    double C0[NS], C1[NS];
    Sys2 s[NS];
    bool ok0 = true;
    bool two = !kFma && plan.order != nullptr;
#pragma unroll
    for (int j = 0; j < NS; ++j) {
        const int64_t gi = base + static_cast<int64_t>(j) * blockDim.x;
        live[j] = gi < B;
        const int64_t g = live[j] ? gi : B - 1;
        idx[j] = plan.order ? plan.order[g] : g;
        const int64_t i = idx[j];
        two &= plan.order ? (plan.mcls[i] != 0) & (plan.mcls[B + i] != 0) : false;
        C0[j] = C[i];
        C1[j] = C[B + i];
        if constexpr (kStateTests)  // the state-tested loop's spring range (div2s)
            two &= spring_range_ok(C0[j]) & spring_range_ok(C1[j]);
        s[j] = Sys2{x[i], x[B + i], v[i], v[B + i]};
        if (xs && live[j]) {
            xs[i] = s[j].x0;
            xs[B + i] = s[j].x1;
            vs[i] = s[j].v0;
            vs[B + i] = s[j].v1;
        }
        if (es && live[j])
            es[i] = energy2(s[j], m[i], m[B + i], C0[j], C1[j]);
    }
    two = __all_sync(kFull, two);
#pragma unroll
    for (int j = 0; j < NS; ++j) {
        const int64_t i = idx[j];
        if (two) {
            div2_consts(m[i], plan.mcls[i], u0[j], w0[j]);
            div2_consts(m[B + i], plan.mcls[B + i], u1[j], w1[j]);
        } else {
            const Divisor d0 = make_divisor(m[i]), d1 = make_divisor(m[B + i]);
            u0[j] = d0.b, w0[j] = d0.y, u1[j] = d1.b, w1[j] = d1.y;
            ok0 &= divisor_fast_ok(d0) & divisor_fast_ok(d1);
        }
    }
    ErrAcc acc[kCmp ? NS : 1];
    if constexpr (kCmp) {
        if (cmp.sol) {
#pragma unroll
            for (int j = 0; j < NS; ++j)
                acc[j].add_sample(load_modal(cmp.sol, B, idx[j]), cmp.ts[0], s[j].x0, s[j].x1);
        }
    }
    int64_t bad[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j)
        bad[j] = 0;
    bool exact_only = false;  // set once a system of this thread diverged
    int64_t kstep = 0;
    while (kstep < nsteps) {
        const int64_t next_sample = (kstep / stride + 1) * stride;
        int64_t n = nsteps - kstep;
        if (next_sample - kstep < n)
            n = next_sample - kstep;
        if (n > kChunk)
            n = kChunk;
        Sys2 saved[NS];
#pragma unroll
        for (int j = 0; j < NS; ++j)
            saved[j] = s[j];
        bool ok = ok0 & !exact_only & ((NS > 1 && !two) || fused_dt_ok(k.half_dt));
        static_assert(kStateTests || NS == 1, "NS > 1 relies on the state tests' half_dt bound");
        if (ok) {
            // Throughput builds unroll OSC_B2_UNROLL steps per iteration (loop control was
            // ~1% of the stall samples; +1.2% on C2).  The latency build (NS=1)
            // keeps one step per iteration: its schedule gets longer unrolled.
            if (!kFma && two) {
#pragma unroll(NS > 1 ? kUnroll : 1)
                for (int t = 0; t < n; ++t) {
#pragma unroll
                    for (int j = 0; j < NS; ++j)
                        step2<kStateTests ? Arith::Fast2S : Arith::Fast2A, NS == 1>(
                            s[j], C0[j], C1[j], Divisor{0.0, u0[j], w0[j]},
                            Divisor{0.0, u1[j], w1[j]}, k, ok);
                }
            } else {
#pragma unroll(NS > 1 ? kUnroll : 1)
                for (int t = 0; t < n; ++t) {
#pragma unroll
                    for (int j = 0; j < NS; ++j)
                        step2<kFma ? Arith::Fma : Arith::Fast, NS == 1>(
                            s[j], C0[j], C1[j], Divisor{u0[j], w0[j], 0.0},
                            Divisor{u1[j], w1[j], 0.0}, k, ok);
                }
            }
#pragma unroll
            for (int j = 0; j < NS; ++j)
                ok &= finite2(s[j]);
        }
        if (!ok) {
            // A division left the fast path's range or a value went
            // non-finite: replay the chunk with IEEE division, checking every
            // step.  Non-finite values are absorbing under + - * /, so the
            // first non-finite step of each system is integrate's
            // NonFiniteStateError.step (oscillator.py:255-260).
#pragma unroll
            for (int j = 0; j < NS; ++j)
                s[j] = saved[j];
            Divisor e0[NS], e1[NS];
#pragma unroll
            for (int j = 0; j < NS; ++j) {
                e0[j] = Divisor{two ? m[idx[j]] : u0[j], w0[j], 0.0};
                e1[j] = Divisor{two ? m[B + idx[j]] : u1[j], w1[j], 0.0};
            }
            for (int t = 0; t < n; ++t) {
#pragma unroll
                for (int j = 0; j < NS; ++j) {
                    step2<kFma ? Arith::Fma : Arith::Exact>(s[j], C0[j], C1[j], e0[j], e1[j], k, ok);
                    if (bad[j] == 0 && !finite2(s[j])) {
                        bad[j] = kstep + t + 1;
                        exact_only = true;
                    }
                }
            }
        }
        kstep += n;
        if ((xs || es) && kstep % stride == 0) {
            const int64_t o = (kstep / stride) * 2 * B;
#pragma unroll
            for (int j = 0; j < NS; ++j) {
                if (live[j] && bad[j] == 0) {
                    const int64_t i = idx[j];
                    if (xs) {
                        xs[o + i] = s[j].x0;
                        xs[o + B + i] = s[j].x1;
                        vs[o + i] = s[j].v0;
                        vs[o + B + i] = s[j].v1;
                    }
                    if (es)
                        es[(kstep / stride) * B + i] = energy2(s[j], m[i], m[B + i], C0[j], C1[j]);
                }
            }
        }
        if constexpr (kCmp) {
            if (cmp.sol && kstep % stride == 0) {
#pragma unroll
                for (int j = 0; j < NS; ++j)
                    if (bad[j] == 0)
                        acc[j].add_sample(load_modal(cmp.sol, B, idx[j]), cmp.ts[kstep / stride],
                                          s[j].x0, s[j].x1);
            }
        }
        bool all_bad = true;
#pragma unroll
        for (int j = 0; j < NS; ++j)
            all_bad &= (bad[j] != 0) | !live[j];
        if (all_bad)
            break;
    }
#pragma unroll
    for (int j = 0; j < NS; ++j) {
        if (live[j]) {
            const int64_t i = idx[j];
            x[i] = s[j].x0;
            x[B + i] = s[j].x1;
            v[i] = s[j].v0;
            v[B + i] = s[j].v1;
            first_bad[i] = bad[j];
            if constexpr (kCmp) {
                const double nan = __longlong_as_double(0x7ff8000000000000ll);
                if (cmp.sol) {
                cmp.out[i] = bad[j] ? nan : acc[j].max_err;
                cmp.out[B + i] = bad[j] ? nan : acc[j].rmse();
                cmp.out[2 * B + i] = bad[j] ? nan : acc[j].at_time;
                }
            }
        }
    }
}

template <int NS>
cudaError_t launch_ns(const double *m, const double *C, double *x, double *v, int64_t B,
                      StepConsts k, int64_t nsteps, int64_t stride, double *xs, double *vs,
                      double *es, int64_t *first_bad, int threads, bool fma,
                      cudaStream_t stream, const CmpArgs *cmp, Div2Plan plan)
{
    const int64_t per_block = int64_t(threads) * NS;
    const unsigned blocks = static_cast<unsigned>((B + per_block - 1) / per_block);
    if constexpr (NS == 1) {
        if (!cmp && !fma && threads == 32) {
        // Latency path (few systems, e.g. C1).  The time loop is the same
        // 113 instructions in every build, but ptxas schedules the serial step
        // of the compare build (its compare switched off: null CmpArgs) ~4%
        // shorter than the others (profiles/r01/c1_latency.md).
            batch2_rk4_kernel<1, false, true><<<blocks, threads, 0, stream>>>(
                m, C, x, v, B, k, nsteps, stride, xs, vs, es, first_bad, plan, CmpArgs{});
            return cudaGetLastError();
        }
    }
    if (cmp) {
        if (fma)
            batch2_rk4_kernel<NS, true, true><<<blocks, threads, 0, stream>>>(
                m, C, x, v, B, k, nsteps, stride, xs, vs, es, first_bad, plan, *cmp);
        else
            batch2_rk4_kernel<NS, false, true><<<blocks, threads, 0, stream>>>(
                m, C, x, v, B, k, nsteps, stride, xs, vs, es, first_bad, plan, *cmp);
    } else if (fma)
        batch2_rk4_kernel<NS, true><<<blocks, threads, 0, stream>>>(
            m, C, x, v, B, k, nsteps, stride, xs, vs, es, first_bad, plan);
    else
        batch2_rk4_kernel<NS, false><<<blocks, threads, 0, stream>>>(
            m, C, x, v, B, k, nsteps, stride, xs, vs, es, first_bad, plan);
    return cudaGetLastError();
}

}  // namespace
}  // namespace osc
