// Off-loop operations of the drop-in API and the division self-test.
//
//   derivative  oscillator.py:184-191  (dvel = acceleration_at per cell)
//   energy      oscillator.py:266-276  (sequential index-order sum, exact)
#include "osc_device.cuh"
#include "osc_kernels.h"

#include <algorithm>
#include <mutex>
#include <cfloat>

namespace osc {
namespace {

// Cells of chain b are at x[b*chain_stride + i*cell_stride]: [B][s] uses
// (s, 1); the batched 2-DOF SoA layout [2][B] uses (1, B).
// bad (may be null): the parameter rule fused in (param_check_kernel's
// out[2] contract, flat indices into m / C) -- every cell is one thread's.
__device__ __forceinline__ void check_cell(const double *m, const double *C, int64_t c,
                                           unsigned long long *bad)
{
    if (!bad)
        return;
    const double a = m[c], b = C[c];
    if (!(a > 0.0 && a <= DBL_MAX))
        atomicMin(&bad[0], static_cast<unsigned long long>(c));
    if (!(b > 0.0 && b <= DBL_MAX))
        atomicMin(&bad[1], static_cast<unsigned long long>(c));
}

__global__ void derivative_kernel(const double *__restrict__ m, const double *__restrict__ C,
                                  const double *__restrict__ x, double *__restrict__ dvel,
                                  int64_t B, int64_t s, int64_t chain_stride,
                                  int64_t cell_stride, unsigned long long *bad)
{
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= B * s)
        return;
    const int64_t b = gid / s, i = gid % s;
    const int64_t o = b * chain_stride;
    check_cell(m, C, o + i * cell_stride, bad);
    const auto at = [&](const double *p, int64_t j) { return p[o + j * cell_stride]; };
    // acceleration_at, oscillator.py:160-164, literally.
    const double left = sub(at(x, i), i > 0 ? at(x, i - 1) : 0.0);
    double a = mul(-at(C, i), left);
    if (i + 1 < s)
        a = add(a, mul(at(C, i + 1), sub(at(x, i + 1), at(x, i))));
    dvel[o + i * cell_stride] = __ddiv_rn(a, at(m, i));
}

__global__ void energy_kernel(const double *__restrict__ m, const double *__restrict__ C,
                              const double *__restrict__ x, const double *__restrict__ v,
                              double *__restrict__ out, int64_t B, int64_t s,
                              int64_t chain_stride, int64_t cell_stride,
                              unsigned long long *bad)
{
    const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= B)
        return;
    const int64_t o = b * chain_stride;
    double total = 0.0;
    double prev = 0.0;
    for (int64_t i = 0; i < s; ++i) {
        const int64_t c = o + i * cell_stride;
        check_cell(m, C, c, bad);
        const double vi = v[c], xi = x[c];
        total = add(total, mul(mul(mul(0.5, m[c]), vi), vi));
        const double ext = sub(xi, prev);  // pos[i] - (pos[i-1] if i > 0 else 0.0)
        total = add(total, mul(mul(mul(0.5, C[c]), ext), ext));
        prev = xi;
    }
    out[b] = total;
}

__device__ __forceinline__ uint64_t splitmix(uint64_t z)
{
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// Compare div(a, make_divisor(b)) with __ddiv_rn(a, b) bit for bit.
//   mode 0: b in [0.5, 2) (the configs' masses), a any bit pattern
//   mode 1: b any positive finite double (normal or subnormal), a any pattern
//   mode 2: b in [0.5, 2), |a| in [2^-40, 2^40) (physical accelerations)
//   mode 3: the two-operation division (div2_fast) as mode 2, divisors that
//           pass div2_classify only
//   mode 4: div2_fast on numerators next to quotient midpoints (see below)
//   mode 5: div_fastq with its flag (divisor_range_ok, quotient_fast_ok), b any
//           positive double, a any pattern
//   mode 6: the checked two-operation division (div2c_fast, div2_checked_consts
//           -- the chain kernels' Fast2C) with its flag, b and a as mode 5
//   mode 7: div2c_fast on mode 4's midpoint-aimed numerators
//   mode 8: as mode 7, but counts the WRONG two-operation quotients that the
//           flag caught (evidence that the aimed numerators hit the failing
//           significands the check exists for)
//   mode 9: the UNTESTED two-operation quotient (div2s, K1's state-tested
//           loop) on mode 4's midpoint-aimed numerators over the whole range
//           the state tests admit: |a| in [2^-557, 2^725) or a = +0, classed
//           b in [2^-100, 2^101); every pair counts
__global__ void check_division_kernel(int64_t n, uint64_t seed, int mode,
                                      unsigned long long *mismatches)
{
    unsigned long long bad = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r1 = splitmix(seed ^ (2 * static_cast<uint64_t>(i)));
        const uint64_t r2 = splitmix(seed ^ (2 * static_cast<uint64_t>(i) + 1));
        const uint64_t mant_b = r2 & 0x000fffffffffffffull;
        uint64_t bb;
        if (mode == 1 || ((mode == 5 || mode == 6) && ((r1 >> 11) & 1))) {
            uint64_t e = (r2 >> 52) & 0x7ff;
            if (e == 0x7ff)
                e = 0x7fe;
            bb = (e << 52) | mant_b;  // includes subnormals, never zero below
            if (bb == 0)
                bb = 1;
        } else {
            bb = ((r2 >> 63) ? 0x3fe0000000000000ull : 0x3ff0000000000000ull) | mant_b;
        }
        uint64_t ab = r1;
        if (mode == 2 || mode == 3) {
            const uint64_t e = 1023 - 40 + ((r1 >> 52) % 80);
            ab = (r1 & 0x800fffffffffffffull) | (e << 52);
        } else if ((r1 & 0xff) == 0) {
            ab = r1 & 0x8000000000000000ull;  // inject signed zeros
        }
        if (mode == 5) {
            // div_fastq (the tiled chain loop's division) with its flag:
            // any numerator pattern, any positive divisor; a pair counts when
            // both tests pass and the bits differ from div.rn.f64.
            const double a = __longlong_as_double(static_cast<long long>(ab));
            const double b = __longlong_as_double(static_cast<long long>(bb));
            const Divisor d = make_divisor(b);
            bool ok = divisor_range_ok(d);
            const double got = div_fastq(a, d, ok);
            if (ok && __double_as_longlong(got) != __double_as_longlong(__ddiv_rn(a, b)))
                ++bad;
            continue;
        }
        if (mode == 6) {
            const double a = __longlong_as_double(static_cast<long long>(ab));
            const double b = __longlong_as_double(static_cast<long long>(bb));
            double zh, zl;
            uint64_t w;
            if (!div2_checked_consts(b, zh, zl, w))
                continue;
            bool ok = true;
            const double got = div2c_fast(a, Divisor{b, zh, zl, static_cast<uint32_t>(w)}, ok);
            if (ok && __double_as_longlong(got) != __double_as_longlong(__ddiv_rn(a, b)))
                ++bad;
            continue;
        }
        if (mode >= 3) {
            // The two-operation division (div2_fast) on divisors that pass
            // div2_classify; mode 4 aims every numerator at a rounding
            // midpoint of the quotient: A 2^sh - B M = k for a random small
            // k and binade (sh = 53: a/b >= 1, sh = 54: a/b < 1), and scales
            // a and b by random powers of two inside the admissible ranges.
            double b0 = __longlong_as_double(static_cast<long long>(bb));
            if (mode == 4 || mode >= 7) {
                const bool wide = mode == 9;
                const uint64_t B = mant_b | (1ull << 52);
                const uint64_t Bo = B >> (__ffsll(static_cast<long long>(B)) - 1);
                const int sh = (r1 & 1) ? 53 : 54;
                const int ak = 1 + static_cast<int>((r1 >> 1) % 64);
                const uint64_t lo = sh == 53 ? B : (1ull << 52), hi = sh == 53 ? (1ull << 53) : B;
                uint64_t A = r1 >> 12 | (1ull << 52);  // a random significand when unsolvable
                if (Bo == B && lo < hi) {
                    A = (static_cast<uint64_t>(ak) * inv_pow2_mod(sh, B)) % B;
                    if ((r1 >> 7) & 1)
                        A = (B - A) % B;
                    if (A < lo)
                        A += ((lo - A + B - 1) / B) * B;
                    if (A >= hi)
                        A = r1 >> 12 | (1ull << 52);
                }
                // a in [2^-400, 2^401), b in [2^-90, 2^91); mode 9: [2^-557, 2^725), [2^-100, 2^101)
                const int ea = wide ? static_cast<int>((r1 >> 20) % 1282) - 557
                                    : static_cast<int>((r1 >> 20) % 801) - 400;
                const int eb = wide ? static_cast<int>((r2 >> 53) % 201) - 100
                                    : static_cast<int>((r2 >> 53) % 181) - 90;
                ab = ((r1 >> 8) & 1ull) << 63 | (uint64_t(1023 + ea) << 52) |
                     (A & 0x000fffffffffffffull);
                b0 = __longlong_as_double(static_cast<long long>(
                    (uint64_t(1023 + eb) << 52) | mant_b));
                if (wide && ((r2 >> 40) & 0xff) == 0)
                    ab = 0;  // +0: the only zero numerator the state-tested loop divides
            }
            if (mode == 7 || mode == 8) {
                double zh, zl;
                uint64_t w;
                if (!div2_checked_consts(b0, zh, zl, w))
                    continue;
                const double a = __longlong_as_double(static_cast<long long>(ab));
                bool ok = true;
                const double got =
                    div2c_fast(a, Divisor{b0, zh, zl, static_cast<uint32_t>(w)}, ok);
                const bool wrong =
                    __double_as_longlong(got) != __double_as_longlong(__ddiv_rn(a, b0));
                if (mode == 7 ? (ok && wrong) : (!ok && wrong))
                    ++bad;
                continue;
            }
            double zh, zl;
            const int cls = div2_classify(b0, zh, zl);
            if (!cls)
                continue;
            double zh2, zl2;
            div2_consts(b0, cls, zh2, zl2);
            const double a = __longlong_as_double(static_cast<long long>(ab));
            if (mode == 9) {
                const double got = div2s(a, Divisor{b0, zh2, zl2});
                if (__double_as_longlong(got) != __double_as_longlong(__ddiv_rn(a, b0)))
                    ++bad;
                continue;
            }
            bool ok = true, ok_a = true;
            const double got = div2_fast(a, Divisor{b0, zh2, zl2}, ok);
            div2a_fast(a, Divisor{b0, zh2, zl2}, ok_a);  // same quotient, numerator test
            const double want = __ddiv_rn(a, b0);
            // a counted pair: either form's range test passed and the bits
            // differ, or the two constant computations disagree
            if (((ok || ok_a) && __double_as_longlong(got) != __double_as_longlong(want)) ||
                __double_as_longlong(zh) != __double_as_longlong(zh2) ||
                __double_as_longlong(zl) != __double_as_longlong(zl2))
                ++bad;
            continue;
        }
        const double a = __longlong_as_double(static_cast<long long>(ab));
        const double b = __longlong_as_double(static_cast<long long>(bb));
        const double got = div(a, make_divisor(b));
        const double want = __ddiv_rn(a, b);
        const bool both_nan = (got != got) && (want != want);
        if (!both_nan && __double_as_longlong(got) != __double_as_longlong(want))
            ++bad;
    }
    if (bad)
        atomicAdd(mismatches, bad);
}

// FP64 issue-rate microbenchmark: 8 independent DFMA (mode 0) or DADD
// (mode 1) chains per thread.  Gives the measured DP-pipe peak the compute
// roofline of K1/K2 is quoted against (MEASURED_PEAKS.json has no FP64).
// One thread, one dependent chain: cycles per DFMA (mode 4), DADD (5) or
// DMUL (6), measured with clock64 around the chain (sink[0] = cycles).
__global__ void fp64_latency_kernel(int64_t iters, int mode, double *sink)
{
    double a = 1.0 + 1e-3 * threadIdx.x;
    const double b = 0.999999, c = 1e-7;
    const long long t0 = clock64();
    if (mode == 4) {
        for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                a = __fma_rn(a, b, c);
        }
    } else if (mode == 5) {
        for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                a = __dadd_rn(a, c);
        }
    } else {
        for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                a = __dmul_rn(a, b);
        }
    }
    const long long t1 = clock64();
    sink[0] = static_cast<double>(t1 - t0);
    sink[1] = a;
}

__global__ void fp64_peak_kernel(int64_t iters, int mode, double *sink)
{
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        a[j] = 1.0 + 1e-3 * (threadIdx.x + j);
    const double b = 0.999999, c = 1e-7;
    if (mode == 0) {
        for (int64_t i = 0; i < iters; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                a[j] = __fma_rn(a[j], b, c);
    } else {
        for (int64_t i = 0; i < iters; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                a[j] = __dadd_rn(a[j], c);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        s += a[j];
    if (s == 12345.678)
        sink[threadIdx.x] = s;
}

// FP64 tensor-core issue rate: 8 independent DMMA.8x8x4 accumulators per
// warp (mma.sync m8n8k4 f64; tcgen05 has no f64 kind on sm_100a).  mode 3
// interleaves 8 DFMA chains to see whether DMMA and DFMA share a pipe.
__global__ void dmma_peak_kernel(int64_t iters, int mode, double *sink)
{
    double acc[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        acc[j][0] = acc[j][1] = 0.0;
    const double a = 1.0 + 1e-3 * threadIdx.x, b = 0.5;
    double f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        f[j] = 1.0 + j;
    for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[j][0]), "+d"(acc[j][1])
                         : "d"(a), "d"(b));
        if (mode == 3) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                f[j] = __fma_rn(f[j], 0.999999, 1e-7);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        s += acc[j][0] + acc[j][1] + f[j];
    if (s == 12345.678)
        sink[threadIdx.x] = s;
}

// Earliest divergence over a batch: out[0] = min positive first_bad (or
// ~0 if none), out[1] = the smallest index holding it.  Two atomic passes;
// out must be preset to {~0, ~0}.
__global__ void first_bad_step_kernel(const int64_t *__restrict__ fb, int64_t B,
                                      unsigned long long *out)
{
    unsigned long long best = ~0ull;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < B;
         i += int64_t(gridDim.x) * blockDim.x)
        if (fb[i] > 0)
            best = min(best, static_cast<unsigned long long>(fb[i]));
    for (int o = 16; o > 0; o >>= 1)
        best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0 && best != ~0ull)
        atomicMin(&out[0], best);
}

__global__ void first_bad_index_kernel(const int64_t *__restrict__ fb, int64_t B,
                                       unsigned long long *out)
{
    const unsigned long long step = out[0];
    if (step == ~0ull)
        return;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < B;
         i += int64_t(gridDim.x) * blockDim.x)
        if (static_cast<unsigned long long>(fb[i]) == step)
            atomicMin(&out[1], static_cast<unsigned long long>(i));
}

}  // namespace

// OscillatorSystem's parameter rule (oscillator.py:75-80) over n masses and
// n spring rates: out[0] / out[1] = the smallest index of a mass / spring
// rate that is not positive and finite (NaN, +-Inf, <= 0, -0.0), ~0 if none.
// One coalesced pass; atomics only on offenders.
__global__ void param_check_kernel(const double *__restrict__ m, const double *__restrict__ C,
                                   int64_t n, unsigned long long *out)
{
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double a = m[i], b = C[i];
        if (!(a > 0.0 && a <= DBL_MAX))
            atomicMin(&out[0], static_cast<unsigned long long>(i));
        if (!(b > 0.0 && b <= DBL_MAX))
            atomicMin(&out[1], static_cast<unsigned long long>(i));
    }
}

// Stream-ordered scratch from a memory pool the library owns, one per device:
// its release threshold keeps freed blocks for the next call (no re-mapping
// per call), and -- unlike raising the threshold of the device's DEFAULT pool
// (round 1) -- it changes nothing for the host application's own
// cudaMallocAsync users.
cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t stream)
{
    constexpr int kMaxDev = 64;
    static cudaMemPool_t pools[kMaxDev] = {};
    static std::mutex mu;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess)
        return e;
    if (dev < 0 || dev >= kMaxDev)
        return cudaMallocAsync(p, bytes, stream);
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (!pools[dev]) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.handleTypes = cudaMemHandleTypeNone;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            if ((e = cudaMemPoolCreate(&pools[dev], &props)) != cudaSuccess)
                return e;
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
        }
        pool = pools[dev];
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, stream);
}

cudaError_t launch_param_check(const double *m, const double *C, int64_t n,
                               unsigned long long *out, cudaStream_t stream, bool init)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>(int64_t(sms) * 8, (n + 255) / 256)));
    if (init) {
        cudaError_t e = cudaMemsetAsync(out, 0xff, 2 * sizeof(unsigned long long), stream);
        if (e != cudaSuccess)
            return e;
    }
    if (n > 0)
        param_check_kernel<<<grid, 256, 0, stream>>>(m, C, n, out);
    return cudaGetLastError();
}

cudaError_t launch_first_bad(const int64_t *fb, int64_t B, unsigned long long *out,
                             cudaStream_t stream)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = static_cast<unsigned>(
        std::max<int64_t>(1, std::min<int64_t>(int64_t(sms) * 4, (B + 255) / 256)));
    cudaError_t e = cudaMemsetAsync(out, 0xff, 2 * sizeof(unsigned long long), stream);
    if (e != cudaSuccess)
        return e;
    first_bad_step_kernel<<<grid, 256, 0, stream>>>(fb, B, out);
    first_bad_index_kernel<<<grid, 256, 0, stream>>>(fb, B, out);
    return cudaGetLastError();
}

cudaError_t launch_fp64_peak(int64_t iters, int mode, double *sink, int64_t *lanes_ops,
                             cudaStream_t stream)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 4, threads = 512;
    if (mode >= 4) {  // latency: returned count = dependent ops of the one thread
        fp64_latency_kernel<<<1, 1, 0, stream>>>(iters, mode, sink);
        *lanes_ops = iters * 16;
        return cudaGetLastError();
    }
    if (mode >= 2) {
        // returned count = flops: 512 per DMMA.8x8x4 per warp (+ 2 per DFMA lane in mode 3)
        dmma_peak_kernel<<<blocks, threads, 0, stream>>>(iters, mode, sink);
        const int64_t warps = int64_t(blocks) * threads / 32;
        *lanes_ops = warps * iters * 8 * 512 + (mode == 3 ? int64_t(blocks) * threads * iters * 16 : 0);
        return cudaGetLastError();
    }
    fp64_peak_kernel<<<blocks, threads, 0, stream>>>(iters, mode, sink);
    *lanes_ops = int64_t(blocks) * threads * iters * 8;
    return cudaGetLastError();
}

cudaError_t launch_derivative(const double *m, const double *C, const double *x, double *dvel,
                              int64_t B, int64_t s, bool cell_major, cudaStream_t stream,
                              unsigned long long *bad)
{
    const int64_t total = B * s;
    if (total == 0)
        return cudaSuccess;
    const int threads = 256;
    derivative_kernel<<<static_cast<unsigned>((total + threads - 1) / threads), threads, 0,
                        stream>>>(m, C, x, dvel, B, s, cell_major ? 1 : s, cell_major ? B : 1, bad);
    return cudaGetLastError();
}

cudaError_t launch_energy(const double *m, const double *C, const double *x, const double *v,
                          double *out, int64_t B, int64_t s, bool cell_major,
                          cudaStream_t stream, unsigned long long *bad)
{
    if (B == 0)
        return cudaSuccess;
    const int threads = 128;
    energy_kernel<<<static_cast<unsigned>((B + threads - 1) / threads), threads, 0, stream>>>(
        m, C, x, v, out, B, s, cell_major ? 1 : s, cell_major ? B : 1, bad);
    return cudaGetLastError();
}

__global__ void div2_classify_kernel(const double *__restrict__ b, int64_t n,
                                     uint8_t *__restrict__ pass)
{
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double zh, zl;
        pass[i] = static_cast<uint8_t>(div2_classify(b[i], zh, zl));
    }
}

cudaError_t launch_div2_classify(const double *b, int64_t n, uint8_t *pass, cudaStream_t stream)
{
    if (n <= 0)
        return cudaSuccess;
    const int64_t want = (n + 255) / 256;
    div2_classify_kernel<<<static_cast<unsigned>(want < 148 * 16 ? want : 148 * 16), 256, 0,
                           stream>>>(b, n, pass);
    return cudaGetLastError();
}

__global__ void div2c_table_kernel(const double *__restrict__ b, int64_t n, double *__restrict__ zh,
                                   double *__restrict__ zl, uint64_t *__restrict__ bad)
{
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double h, l;
        uint64_t w;
        div2_chain_consts(b[i], h, l, w);
        zh[i] = h;
        zl[i] = l;
        bad[i] = w;
    }
}

cudaError_t launch_div2c_table(const double *b, int64_t n, double *zh, double *zl, uint64_t *bad,
                               cudaStream_t stream)
{
    if (n <= 0)
        return cudaSuccess;
    const int64_t want = (n + 255) / 256;
    div2c_table_kernel<<<static_cast<unsigned>(want < 148 * 16 ? want : 148 * 16), 256, 0,
                         stream>>>(b, n, zh, zl, bad);
    return cudaGetLastError();
}

cudaError_t launch_check_division(int64_t n, uint64_t seed, int mode,
                                  unsigned long long *mismatches, cudaStream_t stream)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    check_division_kernel<<<sms * 8, 256, 0, stream>>>(n, seed, mode, mismatches);
    return cudaGetLastError();
}

}  // namespace osc
