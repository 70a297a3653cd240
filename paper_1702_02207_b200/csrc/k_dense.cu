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
// Layout (trajectory-major, so that TMA boxes and the epilogue are
// contiguous): the operands BA / BB are [2N][s] -- operand column j is a
// row of s doubles -- with columns blocked by TB = 16 trajectories: block cb
// holds rows (x of trajectories 16cb..16cb+15 | y2 of the same), so one
// 32-column CTA tile owns both halves of its 16 trajectories and the epilogue
// is local.  V and the partial sums SX, SV are [N][s].
//
// Tiles move by TMA (cp.async.bulk.tensor.2d, 128-byte swizzle, mbarrier
// completion): one elected thread issues the A box [64 rows][16 k] and the B
// box [32 cols][16 k] of a k-slab, STAGES slabs ahead.  The 128-byte swizzle
// (16-byte chunk c of a 128-byte row r stored at c ^ (r % 8)) makes the DMMA
// fragment loads conflict-free: a warp's 32 doubles hit 16 distinct 8-byte
// bank slots, two wavefronts, the minimum for 256 bytes.
//
// GEMM: FP64 tensor cores through mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4;
// tcgen05 has no f64 kind on sm_100a -- ptxas rejects kind::f64).
#include <cuda.h>  // CUtensorMap (the encoder is resolved at run time)

#include "osc_device.cuh"
#include "osc_kernels.h"

#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace osc {
namespace {

// CTA tile 64 x 32 (16 trajectories x both halves), 4 warps of 32 x 16 (8
// DMMA accumulators each), BK = 16, 4 TMA stages of 12 KB -> 4 CTAs (16
// warps) per SM and 4096 CTAs per GEMM at s = 4096, N = 1024: 6.92 waves of
// 592, 98.8% wave efficiency.  (The tiling cuBLAS picks for this shape,
// cutlass d884gemm_64x32_16x4.)
constexpr int BM = 64, BN = 32, BK = 16, STAGES = 4, THREADS = 128;
constexpr int TB = BN / 2;  // trajectories per operand block
constexpr size_t kStageDoubles = size_t(BM) * BK + size_t(BK) * BN;
constexpr uint32_t kStageBytes = uint32_t(kStageDoubles * sizeof(double));
// + 1 KB: the 128-byte swizzle needs 1024-byte aligned stage bases
constexpr size_t kSmemBytes = STAGES * kStageDoubles * sizeof(double) + 1024;
static_assert(size_t(BM) * (BN + 1) <= STAGES * kStageDoubles, "epilogue staging fits");
static_assert(BK * sizeof(double) == 128, "one k-slab row is one 128-byte swizzle row");

// Element (row, k) of a TMA tile of 128-byte rows (BK doubles) under the
// 128-byte swizzle: 16-byte chunk k/2 of row `row` sits at chunk
// (k/2) ^ (row % 8).
__device__ __forceinline__ int swz128(int row, int k)
{
    return row * BK + ((((k >> 1) ^ (row & 7))) << 1) + (k & 1);
}

// Fragment row order within an 8-row group: lane group a (= lane / 4) of an
// m8n8k4 fragment takes tile row perm8(a) = 2(a % 4) + a / 4.  A 64-bit
// shared load is served per half-warp (a = 0..3 or 4..7): with the rows
// {0,2,4,6} (resp. {1,3,5,7}) the swizzle XOR (row % 8) moves the two 16-byte
// chunks a fragment row reads to 8 distinct chunks -- conflict-free -- where
// rows {0,1,2,3} would pair them up (2-way conflicts, ncu: 2x wavefronts).
// The accumulator rows / columns follow the same order (epilogue staging).
__device__ __forceinline__ int perm8(int a) { return ((a & 3) << 1) | (a >> 2); }

__device__ __forceinline__ unsigned smem_addr(const void *p)
{
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity)
{
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// One 2-D TMA box (coordinates: inner k, then the row) into shared memory.
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int k, int row,
                                            uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(k), "r"(row), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

struct DenseArgs {
    double *BA;        // [2N][s]  (x | y2) blocks of TB trajectories
    double *BB;        // [2N][s]  (y3 | y4) blocks
    double *V;         // [N][s]
    double *SX, *SV;   // [N][s] partial combination sums
    int64_t *first_bad;
    int64_t s, N;      // padded sizes: s % 64 == 0, N % TB == 0
    StepConsts k;
    int64_t step;      // 1-based step index (divergence tag)
    int64_t nt0, ntc;  // column tiles [nt0, nt0 + ntc) of this launch (independent trajectories)
};

// tmA: A [s][s] (box 16 k x 64 rows); tmB: this GEMM's operand [2N][s]
// (box 16 k x 32 columns).  Both 128-byte swizzled.
template <int kStage>
__global__ void __launch_bounds__(THREADS, 4)
    dense_rk4_gemm(const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB, DenseArgs g)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // stage bases 1024-byte aligned (the swizzle pattern repeats every 1 KB)
    double *smem = reinterpret_cast<double *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[STAGES];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;  // 2 x 2 warps of 32 x 16
    const int m0 = static_cast<int>(blockIdx.x / g.ntc) * BM;
    const int n0 = static_cast<int>(g.nt0 + blockIdx.x % g.ntc) * BN;
    const int KT = static_cast<int>(g.s / BK);

    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
            acc[i][j][0] = acc[i][j][1] = 0.0;

    // slab kt -> stage kt % STAGES: A box at (k = kt*BK, row m0), B box at
    // (k = kt*BK, column n0); one thread issues, the mbarrier counts bytes
    auto issue = [&](int kt) {
        double *st = smem + (kt % STAGES) * kStageDoubles;
        uint64_t *bar = &full[kt % STAGES];
        mbar_expect_tx(bar, kStageBytes);
        tma_load_2d(st, &tmA, kt * BK, m0, bar);
        tma_load_2d(st + BM * BK, &tmB, kt * BK, n0, bar);
    };
    if (tid == 0) {
        for (int st = 0; st < STAGES; ++st)
            mbar_init(&full[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int st = 0; st < STAGES - 1 && st < KT; ++st)
            issue(st);
    }
    __syncthreads();

    const int ar = lane >> 2, ac = lane & 3;  // fragment coordinates
    const int pr = perm8(ar);
    // Fragment offsets within a stage: A rows wm*32 + 8i + perm8(ar) at
    // k = 4q + ac; B columns wn*16 + 8j + perm8(ar) (rows of the [cols][k]
    // box) at k = 4q + ac.
    const auto offa = [&](int q, int i) { return swz128(wm * 32 + i * 8 + pr, 4 * q + ac); };
    const auto offb = [&](int q, int j) {
        return BM * BK + swz128(wn * 16 + j * 8 + pr, 4 * q + ac);
    };
    for (int kt = 0; kt < KT; ++kt) {
        mbar_wait(&full[kt % STAGES], (kt / STAGES) & 1);
        // every warp is done with slab kt - 1, whose stage the next issue refills
        __syncthreads();
        if (tid == 0 && kt + STAGES - 1 < KT) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(kt + STAGES - 1);
        }
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
    __syncthreads();  // every warp is done with the last slab: reuse the buffers

    // Stage the 64 x 32 accumulator tile through shared memory so each
    // thread sees both halves (stage j and j+1) of its trajectories.
    double *sC = smem;
    constexpr int CS = BN + 1;
    // accumulator (row ar, columns 2ac, 2ac + 1) of each 8 x 8 block is tile
    // row perm8(ar), tile columns perm8(2ac), perm8(2ac + 1)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int r = wm * 32 + i * 8 + pr;
            const int c = wn * 16 + j * 8;
            sC[r * CS + c + perm8(2 * ac)] = acc[i][j][0];
            sC[r * CS + c + perm8(2 * ac + 1)] = acc[i][j][1];
        }
    __syncthreads();

    const int64_t cb = n0 / BN;  // trajectory block
    const int64_t s = g.s;
    if constexpr (kStage == 2) {
        // benchmark-only: plain GEMM store (no RK4 epilogue), to separate the
        // main loop's efficiency from the fused epilogue's cost
        for (int e = tid; e < BM * BN; e += THREADS) {
            const int r = e % BM, c = e / BM;
            g.BB[(n0 + c) * s + m0 + r] = sC[r * CS + c];
        }
        return;
    }
    const double h = g.k.half_dt, dt = g.k.dt, dt6 = g.k.dt6;
    bool bad = false;
    // consecutive threads take consecutive rows: every global access below is
    // a contiguous run of the trajectory-major arrays
    for (int e = tid; e < BM * TB; e += THREADS) {
        const int r = e % BM, c = e / BM;
        const int64_t gr = m0 + r;
        const int64_t n = cb * TB + c;                   // trajectory
        const int64_t ix = (cb * BN + c) * s + gr;       // its first-half operand row
        const int64_t iy = ix + TB * s;                  // its second-half row
        const int64_t iv = n * s + gr;
        const double p = -sC[r * CS + c];                // k1 (stage 0) or k3 (stage 1)
        const double q = -sC[r * CS + c + TB];           // k2 or k4
        const double x = g.BA[ix];
        const double v = g.V[iv];
        if constexpr (kStage == 0) {
            // [k1|k2]: y2v = v + h k1, y3v = v + h k2, y3p = x + h y2v, y4p = x + dt y3v
            const double y2v = add(v, mul(h, p));
            const double y3v = add(v, mul(h, q));
            g.BB[ix] = add(x, mul(h, y2v));
            g.BB[iy] = add(x, mul(dt, y3v));
            g.SX[iv] = add(add(v, mul(2.0, y2v)), mul(2.0, y3v));
            g.SV[iv] = add(p, mul(2.0, q));
        } else {
            // [k3|k4]: y4v = v + dt k3; combine_value for x and v (oscillator.py:227-228)
            const double y4v = add(v, mul(dt, p));
            const double sx = add(g.SX[iv], y4v);
            const double sv = add(add(g.SV[iv], mul(2.0, p)), q);
            const double xn = add(x, mul(dt6, sx));
            const double vn = add(v, mul(dt6, sv));
            g.BA[ix] = xn;
            g.V[iv] = vn;
            g.BA[iy] = add(xn, mul(h, vn));  // y2p of the next step
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

// Pack X, V [s][N] into the blocked, trajectory-major operand BA (x | x + h v)
// and V [Np][sp]: a 32 x 32 shared-memory transpose per block (coalesced on
// both sides); padding rows / trajectories are zero.
__global__ void pack_kernel(const double *__restrict__ X, const double *__restrict__ V0,
                            double *__restrict__ BA, double *__restrict__ Vp, int64_t s,
                            int64_t N, int64_t sp, int64_t Np, double h)
{
    __shared__ double tx[32][33], tv[32][33];
    const int64_t r0 = int64_t(blockIdx.y) * 32, n0 = int64_t(blockIdx.x) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {  // read rows r0+i, cols n0+tx
        const int64_t r = r0 + i, n = n0 + threadIdx.x;
        const bool in = r < s && n < N;
        tx[i][threadIdx.x] = in ? X[r * N + n] : 0.0;
        tv[i][threadIdx.x] = in ? V0[r * N + n] : 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {  // write trajectory n0+i, rows r0+tx
        const int64_t n = n0 + i, r = r0 + threadIdx.x;
        if (n >= Np || r >= sp)
            continue;
        const double x = tx[threadIdx.x][i], v = tv[threadIdx.x][i];
        const int64_t row = (n / TB) * BN + (n % TB);
        BA[row * sp + r] = x;
        BA[(row + TB) * sp + r] = add(x, mul(h, v));
        Vp[n * sp + r] = v;
    }
}

__global__ void unpack_kernel(const double *__restrict__ BA, const double *__restrict__ Vp,
                              double *__restrict__ X, double *__restrict__ V, int64_t s,
                              int64_t N, int64_t sp)
{
    __shared__ double tx[32][33], tv[32][33];
    const int64_t r0 = int64_t(blockIdx.y) * 32, n0 = int64_t(blockIdx.x) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {  // read trajectory n0+i, rows r0+tx
        const int64_t n = n0 + i, r = r0 + threadIdx.x;
        if (n < N && r < s) {
            tx[i][threadIdx.x] = BA[((n / TB) * BN + (n % TB)) * sp + r];
            tv[i][threadIdx.x] = Vp[n * sp + r];
        }
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {  // write row r0+i, cols n0+tx
        const int64_t r = r0 + i, n = n0 + threadIdx.x;
        if (r < s && n < N) {
            X[r * N + n] = tx[threadIdx.x][i];
            V[r * N + n] = tv[threadIdx.x][i];
        }
    }
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

namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                   const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                   const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled through the runtime's driver entry point (the
// library does not link libcuda: it must load where there is no driver).
EncodeTiledFn encode_tiled()
{
    static EncodeTiledFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            p = nullptr;
        }
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// A row-major [rows][cols] fp64 matrix viewed as 2-D tiles of box_cols x
// box_rows, 128-byte swizzled (box_cols * 8 == 128).
cudaError_t tile_map(CUtensorMap *map, const double *base, int64_t rows, int64_t cols,
                     uint32_t box_rows)
{
    EncodeTiledFn enc = encode_tiled();
    if (!enc)
        return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * sizeof(double)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base),
                           dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace

// Integrate nsteps with the padded workspace already holding the packed state.
cudaError_t launch_dense_steps(const double *A, double *BA, double *BB, double *Vp, double *SX,
                               double *SV, int64_t *first_bad, int64_t sp, int64_t Np,
                               StepConsts k, int64_t step0, int64_t nsteps, cudaStream_t stream,
                               cudaStream_t side)
{
    DenseArgs g{};
    g.BA = BA;
    g.BB = BB;
    g.V = Vp;
    g.SX = SX;
    g.SV = SV;
    g.first_bad = first_bad;
    g.s = sp;
    g.N = Np;
    g.k = k;
    CUtensorMap tmA, tmBA, tmBB;
    cudaError_t e;
    if ((e = tile_map(&tmA, A, sp, sp, BM)) != cudaSuccess ||
        (e = tile_map(&tmBA, BA, 2 * Np, sp, BN)) != cudaSuccess ||
        (e = tile_map(&tmBB, BB, 2 * Np, sp, BN)) != cudaSuccess)
        return e;
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
        for (int64_t t = 0; t < 2 * nsteps; ++t)
            dense_rk4_gemm<2><<<blocks, THREADS, kSmemBytes, stream>>>(tmA, tmBA, g);
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
    for (int hh = 0; hh < nhalf; ++hh) {
        g.nt0 = begin[hh];
        g.ntc = count[hh];
        const unsigned blocks = static_cast<unsigned>((sp / BM) * g.ntc);
        for (int64_t t = 0; t < nsteps; ++t) {
            g.step = step0 + t + 1;
            dense_rk4_gemm<0><<<blocks, THREADS, kSmemBytes, streams[hh]>>>(tmA, tmBA, g);
            dense_rk4_gemm<1><<<blocks, THREADS, kSmemBytes, streams[hh]>>>(tmA, tmBB, g);
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
    const dim3 grid(static_cast<unsigned>((Np + 31) / 32), static_cast<unsigned>((sp + 31) / 32));
    pack_kernel<<<grid, dim3(32, 8), 0, stream>>>(X, V0, BA, Vp, s, N, sp, Np, h);
    return cudaGetLastError();
}

cudaError_t launch_dense_unpack(const double *BA, const double *Vp, double *X, double *V,
                                int64_t s, int64_t N, int64_t sp, cudaStream_t stream)
{
    const dim3 grid(static_cast<unsigned>((N + 31) / 32), static_cast<unsigned>((s + 31) / 32));
    unpack_kernel<<<grid, dim3(32, 8), 0, stream>>>(BA, Vp, X, V, s, N, sp);
    return cudaGetLastError();
}

}  // namespace osc
