// K5 dense_rk4: the dense general-(M,K) path (BASELINE configs[4]).
//
// M x'' + K x = 0 with A = M^-1 K precomputed (osc_rowscale), advancing N
// independent trajectories (columns of X, V) with rk4_step's stage structure
// (oscillator.py:208-231) where acceleration_at becomes a = -(A y).  The
// reference keeps only the chain; the oracle is the
// restatement oracle.dense_rk4 plus the eigen-analytic solution.
//
// The four stage GEMMs of a step form two independent pairs:
//   k1 = -A x            k2 = -A (x + h v)          (need only the step start)
//   k3 = -A (x + h y2v)  k4 = -A (x + dt y3v)       (need k1 resp. k2 only)
// with y2v = v + h k1, y3v = v + h k2.  So one step is TWO GEMMs of
// [s x s] x [s x 2N]:  [k1|k2] = -A [x|y2]  and  [k3|k4] = -A [y3|y4],
// each with the RK4 elementwise work fused into its epilogue.
//
// Operand layout: BA / BB are [s][2N] with columns blocked by TB = 16
// trajectories: block cb holds columns (x of trajectories 16cb..16cb+15 | y2
// of the same), so one 32-column CTA tile owns both halves of its 16
// trajectories and the epilogue is local.  x itself lives in BA's first
// halves.
//
// GEMM: FP64 tensor cores through mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4;
// tcgen05 has no f64 kind on sm_100a -- ptxas rejects kind::f64).
#include "osc_device.cuh"
#include "osc_kernels.h"

#include <cstdio>
#include <cstdlib>

namespace osc {
namespace {

// CTA tile 64 x 32 (16 trajectories x both halves), 4 warps of 32 x 16 (8
// DMMA accumulators each), BK = 16, 4-stage cp.async pipeline, 48 KB of
// shared memory -> 4 CTAs (16 warps) per SM and 4096 CTAs per GEMM at
// s = 4096, N = 1024: 6.92 waves of 592, 98.8% wave efficiency.  (The same
// tiling cuBLAS picks for this shape, cutlass d884gemm_64x32_16x4.)
constexpr int BM = 64, BN = 32, BK = 16, STAGES = 4, THREADS = 128;
constexpr int TB = BN / 2;  // trajectories per operand block
constexpr size_t kStageDoubles = size_t(BM) * BK + size_t(BK) * BN;
constexpr size_t kSmemBytes = STAGES * kStageDoubles * sizeof(double);
static_assert(size_t(BM) * (BN + 1) <= STAGES * kStageDoubles, "epilogue staging fits");

// XOR swizzle of 16-byte chunks so that each half-warp phase of a 64-bit
// fragment load (4 rows x 4 consecutive doubles) hits 32 distinct banks
// without padding: chunk q of row r lives at q ^ 2*(r % 4).
__device__ __forceinline__ int swz_a(int r, int k)  // A tile [BM][BK]
{
    return r * BK + ((((k >> 1) ^ ((r & 3) << 1))) << 1) + (k & 1);
}
__device__ __forceinline__ int swz_b(int k, int n)  // B tile [BK][BN]
{
    return k * BN + ((((n >> 1) ^ ((k & 3) << 1))) << 1) + (n & 1);
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

struct DenseArgs {
    const double *A;   // [s][s] row-major, A = M^-1 K
    const double *Bop; // [s][2N] blocked operand of this GEMM
    double *BA;        // [s][2N]  (x | y2) blocks of TB trajectories
    double *BB;        // [s][2N]  (y3 | y4) blocks
    double *V;         // [s][N]
    double *SX, *SV;   // [s][N] partial combination sums
    int64_t *first_bad;
    int64_t s, N;      // padded sizes: s % 64 == 0, N % TB == 0
    StepConsts k;
    int64_t step;      // 1-based step index (divergence tag)
    int64_t nt0, ntc;  // column tiles [nt0, nt0 + ntc) of this launch (independent trajectories)
};

// Per-thread cp.async plan: the global source of each 16-byte chunk this
// thread copies (advanced by one slab per issue) and its swizzled smem slot.
struct LoadPlan {
    static constexpr int NA = (BM * BK / 2) / THREADS, NB = (BK * BN / 2) / THREADS;
    const double *a[NA];
    const double *b[NB];
    int sa[NA], sb[NB];
    int64_t b_step;  // doubles between consecutive B slabs (BK rows of Bop)

    __device__ __forceinline__ LoadPlan(const DenseArgs &g, int64_t m0, int64_t n0)
    {
        const int tid = threadIdx.x;
        const int64_t ld2 = 2 * g.N;
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            const int c = tid + i * THREADS, r = c / (BK / 2), q = c % (BK / 2);
            a[i] = g.A + (m0 + r) * g.s + 2 * q;
            sa[i] = swz_a(r, 2 * q);
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const int c = tid + i * THREADS, r = c / (BN / 2), q = c % (BN / 2);
            b[i] = g.Bop + r * ld2 + n0 + 2 * q;
            sb[i] = swz_b(r, 2 * q);
        }
        b_step = BK * ld2;
    }

    // Issue the next slab into stage buffer st and advance the sources.
    __device__ __forceinline__ void issue(double *stage)
    {
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            cp_async16(stage + sa[i], a[i]);
            a[i] += BK;
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            cp_async16(stage + BM * BK + sb[i], b[i]);
            b[i] += b_step;
        }
    }
};

template <int kStage>
__global__ void __launch_bounds__(THREADS, 4) dense_rk4_gemm(DenseArgs g)
{
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;  // 2 x 2 warps of 32 x 16
    const int64_t m0 = static_cast<int64_t>(blockIdx.x / g.ntc) * BM;
    const int64_t n0 = (g.nt0 + static_cast<int64_t>(blockIdx.x % g.ntc)) * BN;
    const int64_t KT = g.s / BK;

    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
            acc[i][j][0] = acc[i][j][1] = 0.0;

    LoadPlan plan(g, m0, n0);
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < KT)
            plan.issue(smem + st * kStageDoubles);
        cp_commit();
    }
    const int ar = lane >> 2, ac = lane & 3;  // fragment coordinates
    // Fragment offsets within a stage (loop-invariant, hoisted): A rows
    // wm*32 + 8i + ar at k = 4q + ac; B row 4q + ac, cols wn*16 + 8j + ar.
    const auto offa = [&](int q, int i) { return swz_a(wm * 32 + i * 8 + ar, 4 * q + ac); };
    const auto offb = [&](int q, int j) {
        return BM * BK + swz_b(4 * q + ac, wn * 16 + j * 8 + ar);
    };
    for (int64_t kt = 0; kt < KT; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        if (kt + STAGES - 1 < KT)
            plan.issue(smem + ((kt + STAGES - 1) % STAGES) * kStageDoubles);
        cp_commit();
        const double *sb = smem + (kt % STAGES) * kStageDoubles;
        // double-buffered fragments: load k-step kk+4 while kk's DMMAs issue
        double af[2][4], bf[2][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
            af[0][i] = sb[offa(0, i)];
#pragma unroll
        for (int j = 0; j < 2; ++j)
            bf[0][j] = sb[offb(0, j)];
#pragma unroll
        for (int q = 0; q < BK / 4; ++q) {
            const int cur = q & 1;
            if (q + 1 < BK / 4) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    af[cur ^ 1][i] = sb[offa(q + 1, i)];
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    bf[cur ^ 1][j] = sb[offb(q + 1, j)];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    dmma(acc[i][j], af[cur][i], bf[cur][j]);
        }
    }
    cp_wait<0>();
    __syncthreads();

    // Stage the 64 x 32 accumulator tile through shared memory so each
    // thread sees both halves (stage j and j+1) of its trajectories.
    double *sC = smem;
    constexpr int CS = BN + 1;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int r = wm * 32 + i * 8 + ar;
            const int c = wn * 16 + j * 8 + 2 * ac;
            sC[r * CS + c] = acc[i][j][0];
            sC[r * CS + c + 1] = acc[i][j][1];
        }
    __syncthreads();

    const int64_t cb = n0 / BN;  // trajectory block
    if constexpr (kStage == 2) {
        // benchmark-only: plain GEMM store (no RK4 epilogue), to separate the
        // main loop's efficiency from the fused epilogue's cost
        for (int e = tid; e < BM * BN; e += THREADS) {
            const int r = e / BN, c = e % BN;
            g.BB[(m0 + r) * 2 * g.N + n0 + c] = sC[r * CS + c];
        }
        return;
    }
    const double h = g.k.half_dt, dt = g.k.dt, dt6 = g.k.dt6;
    const int64_t ld2 = 2 * g.N;
    bool bad = false;
    for (int e = tid; e < BM * TB; e += THREADS) {
        const int r = e / TB, c = e % TB;
        const int64_t gr = m0 + r;
        const int64_t n = cb * TB + c;               // trajectory
        const int64_t ix = gr * ld2 + cb * BN + c;   // its first-half column
        const double p = -sC[r * CS + c];            // k1 (stage 0) or k3 (stage 1)
        const double q = -sC[r * CS + c + TB];       // k2 or k4
        const double x = g.BA[ix];
        const double v = g.V[gr * g.N + n];
        if constexpr (kStage == 0) {
            // [k1|k2]: y2v = v + h k1, y3v = v + h k2, y3p = x + h y2v, y4p = x + dt y3v
            const double y2v = add(v, mul(h, p));
            const double y3v = add(v, mul(h, q));
            g.BB[ix] = add(x, mul(h, y2v));
            g.BB[ix + TB] = add(x, mul(dt, y3v));
            g.SX[gr * g.N + n] = add(add(v, mul(2.0, y2v)), mul(2.0, y3v));
            g.SV[gr * g.N + n] = add(p, mul(2.0, q));
        } else {
            // [k3|k4]: y4v = v + dt k3; combine_value for x and v (oscillator.py:227-228)
            const double y4v = add(v, mul(dt, p));
            const double sx = add(g.SX[gr * g.N + n], y4v);
            const double sv = add(add(g.SV[gr * g.N + n], mul(2.0, p)), q);
            const double xn = add(x, mul(dt6, sx));
            const double vn = add(v, mul(dt6, sv));
            g.BA[ix] = xn;
            g.V[gr * g.N + n] = vn;
            g.BA[ix + TB] = add(xn, mul(h, vn));  // y2p of the next step
            bad |= !(finite(xn) & finite(vn));
        }
    }
    if (kStage == 1 && __syncthreads_or(bad) && tid == 0)
        record_bad(g.first_bad, g.step);
}

// A = K / m[:, None] (exact IEEE division per element), padded to sp x sp.
__global__ void rowscale_kernel(const double *__restrict__ K, const double *__restrict__ m,
                                double *__restrict__ A, int64_t s, int64_t sp)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= sp * sp)
        return;
    const int64_t r = i / sp, c = i % sp;
    A[i] = (r < s && c < s) ? __ddiv_rn(K[r * s + c], m[r]) : 0.0;
}

// Pack X, V [s][N] into the blocked operand BA (x | x + h v) and a padded V.
__global__ void pack_kernel(const double *__restrict__ X, const double *__restrict__ V0,
                            double *__restrict__ BA, double *__restrict__ Vp, int64_t s,
                            int64_t N, int64_t sp, int64_t Np, double h)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= sp * Np)
        return;
    const int64_t r = i / Np, n = i % Np;
    const bool in = r < s && n < N;
    const double x = in ? X[r * N + n] : 0.0, v = in ? V0[r * N + n] : 0.0;
    const int64_t ix = r * 2 * Np + (n / TB) * BN + (n % TB);
    BA[ix] = x;
    BA[ix + TB] = add(x, mul(h, v));
    Vp[r * Np + n] = v;
}

__global__ void unpack_kernel(const double *__restrict__ BA, const double *__restrict__ Vp,
                              double *__restrict__ X, double *__restrict__ V, int64_t s,
                              int64_t N, int64_t Np)
{
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= s * N)
        return;
    const int64_t r = i / N, n = i % N;
    X[i] = BA[r * 2 * Np + (n / TB) * BN + (n % TB)];
    V[i] = Vp[r * Np + n];
}

}  // namespace

int64_t dense_pad_s(int64_t s) { return (s + BM - 1) / BM * BM; }  // also a multiple of BK
int64_t dense_pad_n(int64_t n) { return (n + TB - 1) / TB * TB; }

cudaError_t launch_rowscale(const double *K, const double *m, double *A, int64_t s, int64_t sp,
                            cudaStream_t stream)
{
    const int64_t total = sp * sp;
    rowscale_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(K, m, A, s,
                                                                                      sp);
    return cudaGetLastError();
}

// Integrate nsteps with the padded workspace already holding the packed state.
cudaError_t launch_dense_steps(const double *A, double *BA, double *BB, double *Vp, double *SX,
                               double *SV, int64_t *first_bad, int64_t sp, int64_t Np,
                               StepConsts k, int64_t step0, int64_t nsteps, cudaStream_t stream,
                               cudaStream_t side)
{
    DenseArgs g{};
    g.A = A;
    g.BA = BA;
    g.BB = BB;
    g.V = Vp;
    g.SX = SX;
    g.SV = SV;
    g.first_bad = first_bad;
    g.s = sp;
    g.N = Np;
    g.k = k;
    cudaFuncSetAttribute(dense_rk4_gemm<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kSmemBytes));
    cudaFuncSetAttribute(dense_rk4_gemm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kSmemBytes));
    const int64_t ntn = (2 * Np) / BN;  // column tiles
    if (std::getenv("OSC_DENSE_RAW")) {  // benchmark-only: GEMMs without the RK4 epilogue
        cudaFuncSetAttribute(dense_rk4_gemm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kSmemBytes));
        g.nt0 = 0;
        g.ntc = ntn;
        const unsigned blocks = static_cast<unsigned>((sp / BM) * ntn);
        for (int64_t t = 0; t < 2 * nsteps; ++t) {
            g.Bop = BA;
            dense_rk4_gemm<2><<<blocks, THREADS, kSmemBytes, stream>>>(g);
        }
        return cudaGetLastError();
    }
    // Trajectories (column blocks) are independent, so wide batches run as two
    // halves of column tiles on two streams: each half's launches fill the
    // other's tail wave (4096 CTAs = 6.92 waves of 592 at C5).  Same bytes.
    const int nhalf = (side && ntn >= 16) ? 2 : 1;
    cudaStream_t streams[2] = {stream, side};
    int64_t begin[2] = {0, ntn / 2}, count[2] = {ntn, ntn - ntn / 2};
    if (nhalf == 2)
        count[0] = ntn / 2;
    cudaEvent_t fork = nullptr, join = nullptr;
    if (nhalf == 2) {
        cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
        cudaEventRecord(fork, stream);
        cudaStreamWaitEvent(side, fork, 0);
    }
    for (int h = 0; h < nhalf; ++h) {
        g.nt0 = begin[h];
        g.ntc = count[h];
        const unsigned blocks = static_cast<unsigned>((sp / BM) * g.ntc);
        for (int64_t t = 0; t < nsteps; ++t) {
            g.step = step0 + t + 1;
            g.Bop = BA;
            dense_rk4_gemm<0><<<blocks, THREADS, kSmemBytes, streams[h]>>>(g);
            g.Bop = BB;
            dense_rk4_gemm<1><<<blocks, THREADS, kSmemBytes, streams[h]>>>(g);
        }
    }
    if (nhalf == 2) {
        cudaEventRecord(join, side);
        cudaStreamWaitEvent(stream, join, 0);
        cudaEventDestroy(fork);
        cudaEventDestroy(join);
    }
    return cudaGetLastError();
}

cudaError_t launch_dense_pack(const double *X, const double *V0, double *BA, double *Vp,
                              int64_t s, int64_t N, int64_t sp, int64_t Np, double h,
                              cudaStream_t stream)
{
    const int64_t total = sp * Np;
    pack_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(X, V0, BA, Vp, s,
                                                                                 N, sp, Np, h);
    return cudaGetLastError();
}

cudaError_t launch_dense_unpack(const double *BA, const double *Vp, double *X, double *V,
                                int64_t s, int64_t N, int64_t Np, cudaStream_t stream)
{
    const int64_t total = s * N;
    unpack_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(BA, Vp, X, V,
                                                                                   s, N, Np);
    return cudaGetLastError();
}

}  // namespace osc
