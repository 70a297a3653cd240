// Internal launch interface between the C-ABI layer (capi*.cu) and kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "osc_device.cuh"

namespace osc {

// A neighbouring shard's next-input buffers (peer memory over NVLink, or a
// local buffer): owned cells [lo, hi) of this shard are also stored at
// x[c + offset], v[c + offset] -- the neighbour's ghost zone.
struct PeerGhost {
    double *x, *v;
    int64_t offset, lo, hi;
};

// In-kernel ordering of a shard's edge tiles with its neighbouring shards
// (the multi-process fused exchange; include/osc_b200.h osc_edge_sync_t):
// the edge tiles (SegArgs::nedge) run LAST, wait (bounded) until the
// neighbour's edge counter reaches `period` before touching anything, and
// the last of them on a side posts period + 1 into our counter for that side.
struct EdgeSync {
    const uint64_t *ready[2];  // neighbours' edge counters facing us (peer memory)
    uint64_t *ctr;             // ours: [0],[1] edge done; [2],[3] tallies; [4..7] timeout record
    uint64_t period;
    int64_t timeout_ns;
};

// One launch of the chain kernel over nbuf buffers of n cells each.
struct SegArgs {
    const double *m, *C;     // [nbuf][n]
    const double *xin, *vin; // [nbuf][n] state at step0
    double *xout, *vout;     // [nbuf][n] owned cells written after nsteps
    double *xs, *vs;         // optional copy of the owned cells (a sample slot)
    int64_t *first_bad;      // [nbuf], 0 = finite so far
    int64_t n, nbuf;
    int64_t own_lo, own_hi;  // owned cell range of every buffer
    int64_t W, H;            // owned cells per tile, halo cells per side
    int64_t tiles;           // tiles per buffer
    StepConsts k;
    int64_t nsteps, step0;
    bool fma;                // OSC_FMA mode (not bit-identical)
    PeerGhost peer[2];       // left / right neighbour ghost targets (x == nullptr: none)
    EdgeSync sync;           // sync.ctr == nullptr: no in-kernel ordering (stream/event order)
    // Tile walk of a sharded buffer (nbuf == 1).  ordered: positions are
    // mapped interior tiles first, then the left edge set [0, nedge[0]),
    // then the right edge set [tiles - nedge[1], tiles) -- the tiles that
    // read a ghost zone or store into a neighbour.  The launch covers walk
    // positions [walk0, walk0 + nwalk) (nwalk == 0: all tiles), which is how
    // the interior and the edges run as two launches on two streams.
    bool ordered;
    int64_t nedge[2];
    int64_t walk0, nwalk;
    // Checked two-operation division (div2_checked_consts) of every cell,
    // [nbuf][n] like m; zh == 0 marks an ineligible divisor, bad holds the
    // tested low word in 8-byte slots (bulk-copy alignment).  Null: the
    // three-operation division.
    const double *zh, *zl;
    const uint64_t *bad;
};

// Tiles one buffer's launch walks.
__host__ __device__ inline int64_t walk_tiles(const SegArgs &g)
{
    return g.nwalk ? g.nwalk : g.tiles;
}

// Fused compare (modal.py:141-162) at every retained sample of K1: ts are
// the samples' time labels, sol the [8][B] analytic solutions, out the
// [3][B] ErrorReport fields (max_err, rmse, at_time; NaN if diverged).
struct CmpArgs {
    const double *ts;
    const double *sol;
    double *out;
};

// wide: keep the two-systems-per-thread throughput shape for small batches
// too (set when several batches share the GPU side by side).
cudaError_t launch_batch2(const double *m, const double *C, double *x, double *v, int64_t B,
                          StepConsts k, int64_t nsteps, int64_t stride, double *xs, double *vs,
                          double *es, int64_t *first_bad, bool fma, cudaStream_t stream,
                          const CmpArgs *cmp = nullptr, bool wide = false);

cudaError_t launch_modal_batch2(const double *m, const double *C, const double *x0,
                                const double *v0, int64_t B, double *sol, cudaStream_t stream);

cudaError_t launch_compare_batch2(const double *sol, const double *xs, const double *ts,
                                  int64_t nsamp, int64_t B, double *out, cudaStream_t stream);

cudaError_t launch_chain(const SegArgs &g, int K, int threads, cudaStream_t stream);

// cell_major: [s][B] layout (the batched 2-DOF SoA); else [B][s].  bad (may
// be null, else pre-set to ~0): the parameter rule fused into the same launch
// (launch_param_check's out[2] contract).
cudaError_t launch_derivative(const double *m, const double *C, const double *x, double *dvel,
                              int64_t B, int64_t s, bool cell_major, cudaStream_t stream,
                              unsigned long long *bad = nullptr);

cudaError_t launch_energy(const double *m, const double *C, const double *x, const double *v,
                          double *out, int64_t B, int64_t s, bool cell_major,
                          cudaStream_t stream, unsigned long long *bad = nullptr);

// Earliest divergence of a batch on the device: out[0] = min positive step,
// out[1] = its smallest index (both ~0 when nothing diverged).
cudaError_t launch_first_bad(const int64_t *fb, int64_t B, unsigned long long *out,
                             cudaStream_t stream);

// Stream-ordered scratch from the library's own per-device memory pool
// (freed with cudaFreeAsync); the device's default pool is left untouched.
cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t stream);

// Parameter rule of OscillatorSystem (oscillator.py:75-80): out[0] / out[1]
// = smallest index of an invalid mass / spring rate (~0 when none).
// init = false: out[] is already ~0 (staged host calls upload it).
cudaError_t launch_param_check(const double *m, const double *C, int64_t n,
                               unsigned long long *out, cudaStream_t stream, bool init = true);

// zh, zl, bad of div2_checked_consts for n divisors (SegArgs::zh/zl/bad).
cudaError_t launch_div2c_table(const double *b, int64_t n, double *zh, double *zl, uint64_t *bad,
                               cudaStream_t stream);

cudaError_t launch_div2_classify(const double *b, int64_t n, uint8_t *pass, cudaStream_t stream);

cudaError_t launch_check_division(int64_t n, uint64_t seed, int mode,
                                  unsigned long long *mismatches, cudaStream_t stream);

cudaError_t launch_fp64_peak(int64_t iters, int mode, double *sink, int64_t *lanes_ops,
                             cudaStream_t stream);

// K5 dense path (k_dense.cu): padded sizes s -> multiple of 128, N -> of 32.
int64_t dense_pad_s(int64_t s);
int64_t dense_pad_n(int64_t n);
cudaError_t launch_rowscale(const double *K, const double *m, double *A, int64_t s, int64_t sp,
                            cudaStream_t stream);
cudaError_t launch_dense_pack(const double *X, const double *V0, double *BA, double *Vp,
                              int64_t s, int64_t N, int64_t sp, int64_t Np, double h,
                              cudaStream_t stream);
cudaError_t launch_dense_steps(const double *A, double *BA, double *BB, double *Vp, double *SX,
                               double *SV, int64_t *first_bad, int64_t sp, int64_t Np,
                               StepConsts k, int64_t step0, int64_t nsteps, cudaStream_t stream,
                               cudaStream_t side = nullptr);
cudaError_t launch_dense_unpack(const double *BA, const double *Vp, double *X, double *V,
                                int64_t s, int64_t N, int64_t Np, cudaStream_t stream);

cudaError_t launch_equation_engine(const double *m, const double *C, const double *x0,
                                   const double *v0, int s, double dt, int64_t nsteps,
                                   int64_t stride, double *xs, double *vs, int64_t *first_bad,
                                   int64_t *step_ns, cudaStream_t stream);

}  // namespace osc
