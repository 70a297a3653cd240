/*
 * osc_b200.h -- C ABI of the B200-native RK4 oscillator integrator.
 *
 * This is the drop-in boundary for the reference's hot path
 *   integrate(system, state0, dt, nsteps, stride)  oscbench/oscillator.py:234-263
 *   rk4_step(system, state, dt)                     oscbench/oscillator.py:194-231
 * The reference is a pure-Python package with no FFI of its own;
 * INTEGRATION.md shows the ctypes binding a maintainer would add to it and
 * paper_1702_02207_b200/_native.py is that binding.
 *
 * Conventions
 *   - extern "C", plain pointers and sizes; no C++ exception crosses the ABI.
 *   - Status codes: OSC_OK, OSC_NONFINITE (host API only: some system
 *     diverged, see first_bad), OSC_INVALID (bad argument -- the reference's
 *     ValueError: dt not finite/positive (oscillator.py:201-202), nsteps < 1 or
 *     stride < 1 (:247-250)), OSC_CUDA_ERROR.  osc_last_error() returns the
 *     calling thread's last message.
 *   - Device API: all pointers are device pointers, work is enqueued on
 *     `stream` (a cudaStream_t; NULL = legacy default stream) and the call
 *     returns without synchronising.  Host API (*_host): host pointers,
 *     synchronous, host<->device copies inside.
 *   - first_bad[b] receives the 1-based step at which system/chain b first
 *     produced a NaN or infinity (NonFiniteStateError.step,
 *     oscillator.py:255-260), or 0.  After divergence the final state of that
 *     system is unspecified (the reference raises instead of returning it);
 *     samples before the bad step are exact.
 *   - Samples: xs/vs (may be NULL) receive the initial state plus every
 *     stride-th state, 1 + nsteps/stride slots of the state layout -- the
 *     reference Trajectory's retention rule (oscillator.py:252, 261-262).
 *     Time labels are not produced on the device: the host accumulates
 *     t += dt exactly as the reference does (oscillator.py:231).
 *   - Energies: es (may be NULL) receives energy() (oscillator.py:266-276)
 *     of every retained sample, [1 + nsteps/stride][B], computed on the
 *     device in the reference's sequential order (bit-identical) -- the
 *     drift diagnostic without copying trajectories back.
 *   - All arithmetic is IEEE binary64 in the reference's operation order:
 *     results are byte-identical to oscbench.integrate.
 */
#ifndef OSC_B200_H
#define OSC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OSC_OK 0
#define OSC_NONFINITE 1
#define OSC_INVALID 2
#define OSC_CUDA_ERROR 3

#define OSC_ABI_VERSION 11

/* flags: OSC_FMA selects the opt-in FMA mode -- a*b+c contracted and x/m
 * computed as x*(1/m).  Roughly half the FP64 instructions, NOT bit-identical
 * to the reference (measured tolerance in DESIGN.md / tests/test_gpu_fma.py).
 * 0 = the default, byte-identical arithmetic. */
#define OSC_FMA 1u
/* flags: OSC_TRUSTED -- the caller has already validated m and C (e.g. with
 * osc_validate_parameters) and the entry point skips its own check.  Needed
 * when the call is captured into a CUDA graph (the check synchronises the
 * stream) and for per-period calls of a sharded run. */
#define OSC_TRUSTED 2u
/* flags (osc_rk4_chain_advance only): launch a subset of the shard's tiles.
 * OSC_TILES_EDGES = the tiles that read a ghost zone or store into a
 * neighbour (next to each ghost zone), OSC_TILES_INTERIOR = all the others;
 * the two launches together equal one plain launch byte for byte (same tile
 * geometry).  The NCCL transport runs the interior while the ghost exchange
 * is in flight, then one launch covering both edges on the exchange's
 * stream, concurrent with the interior's tail. */
#define OSC_TILES_INTERIOR 4u
#define OSC_TILES_EDGES 8u

int osc_abi_version(void);
const char *osc_last_error(void);

/* Parameter rule of the reference's OscillatorSystem (oscillator.py:66-80):
 * every mass and spring rate must be positive and finite.  Every entry point
 * that takes masses m and spring rates C (unless given OSC_TRUSTED) checks
 * it on the device before integrating -- one pass over m and C, then a
 * synchronisation of `stream`, so the call returns OSC_INVALID instead of
 * enqueuing work -- and reports the first offender (masses before springs,
 * lowest index first: the reference's order for one system).  After such an
 * OSC_INVALID, osc_last_invalid_parameter returns 1 with which = 0 (masses)
 * or 1 (springs) and *index = the flat element index into that array (for
 * host entry points, into the caller's array); otherwise it returns 0.
 * osc_validate_parameters runs the check alone over n device elements:
 * OSC_OK, or OSC_INVALID with *bad (may be NULL) = the flat index. */
int osc_validate_parameters(const double *m, const double *C, int64_t n, int64_t *bad,
                            void *stream);
int osc_last_invalid_parameter(int *which, int64_t *index);

/* Scratch memory: entry points that need it allocate it stream-ordered from a
 * memory pool the library owns (one per device, created on first use, which
 * keeps freed blocks for the next call).  The device's default pool -- the
 * host application's cudaMallocAsync -- is not touched. */

/* Batched independent 2-DOF systems (paper eq. 2), SoA layout [2][B]:
 * m, C, x, v hold coordinate 0 of all B systems, then coordinate 1.
 * Replaces integrate() for s = 2 (oscillator.py:234-263).
 * xs/vs: [1 + nsteps/stride][2][B].  first_bad: [B]. */
int osc_rk4_batch2(const double *m, const double *C, double *x, double *v, int64_t B,
                   double dt, int64_t nsteps, int64_t stride, double *xs, double *vs,
                   double *es, int64_t *first_bad, uint32_t flags, void *stream);

/* Numeric-vs-analytic validation of 2-DOF batches on the device (the
 * reference's modal.py, batched).  Solution records are SoA [8][B] in the
 * order omega1, omega2, r1, r2, a1c, a1s, a2c, a2s (Analytic2DOF,
 * modal.py:44-62); reports are [3][B]: max_abs_error, rmse, at_time
 * (ErrorReport, modal.py:65-71).
 * osc_analytic_batch2: analytic_solution (modal.py:98-120) per system;
 *   bit-identical to the reference for equal parameters (m0 == m1, C0 == C1),
 *   the same modal construction for the general 2x2 pencil otherwise.
 *   Parameters are not validated here (callers validate as
 *   OscillatorSystem does).
 * osc_compare_batch2: compare (modal.py:141-162) of nsamp retained samples,
 *   xs [nsamp][2][B] with time labels ts [nsamp]; OSC_INVALID if nsamp < 1.
 * osc_rk4_batch2_compare: osc_rk4_batch2 with compare() accumulated in the
 *   time loop at every retained sample (ts: the 1 + nsteps/stride labels)
 *   and no samples written; a diverged system's report is NaN.
 * eval_analytic's cos/sin are CUDA's (<= 2 ulp), so reports match the
 * reference to a tolerance, not bit for bit. */
int osc_analytic_batch2(const double *m, const double *C, const double *x0, const double *v0,
                        int64_t B, double *sol, void *stream);
int osc_compare_batch2(const double *sol, const double *xs, const double *ts, int64_t nsamp,
                       int64_t B, double *report, void *stream);
int osc_rk4_batch2_compare(const double *m, const double *C, double *x, double *v, int64_t B,
                           double dt, int64_t nsteps, int64_t stride, const double *ts,
                           const double *sol, double *report, int64_t *first_bad, uint32_t flags,
                           void *stream);

/* B independent wall-anchored chains of s cells, layout [B][s]
 * (spring i joins cell i to cell i-1, spring 0 to the wall, last cell free;
 * oscillator.py:3-5, 152-164).  Chains up to 2048 cells run one CTA per chain
 * for the whole run; longer chains use temporally blocked tiles of
 * halo_steps steps per launch (0 = default 32).
 * Replaces integrate() (oscillator.py:234-263).
 * xs/vs: [1 + nsteps/stride][B][s].  first_bad: [B]. */
int osc_rk4_chains(const double *m, const double *C, double *x, double *v, int64_t B,
                   int64_t s, double dt, int64_t nsteps, int64_t stride, double *xs, double *vs,
                   double *es, int64_t *first_bad, int64_t halo_steps, uint32_t flags,
                   void *stream);

/* The launch plan osc_rk4_chains uses for B chains of s cells and nsteps
 * steps (halo_steps as there; 0 = chosen here): plan[7] = {cells per thread,
 * threads per CTA, steps per launch, owned cells per tile, halo cells per
 * side, tiles per chain, launches without sampling}.  No device work. */
int osc_chain_plan(int64_t B, int64_t s, int64_t nsteps, int64_t halo_steps, int64_t *plan);

/* A neighbouring shard's next-input buffers for the fused halo exchange:
 * `count` boundary cells of ours (our first `count` owned cells for the left
 * neighbour, our last `count` for the right one) are stored, by the same
 * kernel that computes them, at x[c + offset] / v[c + offset], c being our
 * buffer index -- peer memory over NVLink (CUDA IPC) or a local buffer. */
typedef struct {
    double *x, *v;
    int64_t offset;
    int64_t count;
} osc_peer_t;

/* In-kernel ordering of a shard's launches with its neighbours (the fused
 * exchange between processes, one per GPU).  Only the tiles next to a ghost
 * zone depend on a neighbour; with a sync descriptor they run after the
 * interior tiles, and before one touches its inputs its CTA waits ON THE
 * DEVICE until the neighbour's edge counter facing us has reached `period`
 * (the neighbour's previous period stored our ghosts and finished reading the
 * buffer we are about to store into); the last edge tile of a side then
 * posts period + 1 into our counter for that side.  No host involvement and
 * no stream-level wait per period.
 *   ready[0] / ready[1]: the left / right neighbour's counter facing us (its
 *     counters[1] / counters[0]), mapped peer memory; NULL = no neighbour.
 *   counters: ours, 8 x uint64 device memory zeroed before the first launch:
 *     [0] / [1] our left / right edge done through period q (= q + 1),
 *     [2] / [3] internal tallies, [4..7] the timeout record
 *     {flag, period, side (0 left, 1 right), counter value seen}.
 *   period: q, counted over all launches since the counters were zeroed.
 *   timeout_ns: bound of every wait.  On expiry the record is written, no
 *     later wait (this launch or any other on these counters) blocks, the
 *     launch completes -- its results are garbage -- and the caller reads
 *     the record (osc_edge_sync_status) and fails instead of hanging. */
typedef struct {
    const uint64_t *ready[2];
    uint64_t *counters;
    uint64_t period;
    int64_t timeout_ns;
} osc_edge_sync_t;

/* Copy the timeout record of `counters` to record[4] (host) after the
 * stream's work is done: returns OSC_OK if no wait timed out, else
 * OSC_CUDA_ERROR with osc_last_error() naming the period, the side and the
 * counter value seen. */
int osc_edge_sync_status(const uint64_t *counters, uint64_t *record, void *stream);

/* One temporally blocked launch over a chain shard buffer of n cells, used by
 * the multi-GPU driver: cells [own_lo, own_hi) are advanced nsteps steps from
 * (xin, vin) into (xout, vout); the cells outside are ghosts of the
 * neighbouring shards.  Buffer cell 0 is treated as wall-adjacent and cell
 * n-1 as the free end, which is exact at the true chain ends and, elsewhere,
 * harmless as long as each ghost zone is at least 2*nsteps cells wide.
 * left/right (may be NULL): write our boundary cells straight into the
 * neighbours' next-input ghost zones (no separate exchange).
 * sync (may be NULL): order the edge tiles with the neighbours on the device
 * (osc_edge_sync_t); NULL = the caller orders launches (streams / events).
 * first_bad: [1], updated to the minimum bad step (global step0 + j). */
int osc_rk4_chain_advance(const double *m, const double *C, const double *xin,
                          const double *vin, double *xout, double *vout, int64_t n,
                          int64_t own_lo, int64_t own_hi, double dt, int64_t nsteps,
                          int64_t step0, int64_t *first_bad, const osc_peer_t *left,
                          const osc_peer_t *right, const osc_edge_sync_t *sync, uint32_t flags,
                          void *stream);

/* osc_rk4_chain_advance with the shard's two-operation division table
 * (div2: NULL, or 3n 8-byte words [zh | zl | bad] filled by osc_div2c_table
 * over the same m -- zh = div2, zl = div2 + n, bad = (uint64_t *)(div2 +
 * 2n)): the tile kernel then divides in two operations warp by warp, as
 * osc_rk4_chains does by itself.  Same bytes either way. */
int osc_rk4_chain_advance_div2(const double *m, const double *C, const double *xin,
                               const double *vin, double *xout, double *vout, int64_t n,
                               int64_t own_lo, int64_t own_hi, double dt, int64_t nsteps,
                               int64_t step0, int64_t *first_bad, const osc_peer_t *left,
                               const osc_peer_t *right, const osc_edge_sync_t *sync,
                               const double *div2, uint32_t flags, void *stream);

/* One shard of a chain in the multi-process fused exchange (one process per
 * GPU): the period loop of osc_rk4_chain_advance launches in native code, so
 * a run of P periods costs P kernel launches of host time and nothing else.
 * Period q (sync.period, counted over all runs) reads our buffer q % 2,
 * writes our owned cells into buffer (q + 1) % 2 and our first / last `ghost`
 * owned cells into the left / right neighbour's buffer (q + 1) % 2 at cell
 * c + offset[side]; its edge tiles are ordered with the neighbours on the
 * device (osc_edge_sync_t).  x[b], v[b]: our buffer b (n cells, ghosts
 * included); nx[side][b], nv[side][b]: the neighbour's buffer b, mapped peer
 * memory (NULL for a chain end).  On return sync.period has advanced by the
 * number of periods enqueued; the state is in buffer sync.period % 2.
 * Asynchronous (stream-ordered); parameters are not re-validated (validate
 * the shard once: osc_validate_parameters).  first_bad: [1] device. */
typedef struct {
    const double *m, *C;
    double *x[2], *v[2];
    double *nx[2][2], *nv[2][2];
    int64_t n, own_lo, own_hi;
    int64_t offset[2];
    int64_t ghost;
    int64_t *first_bad;
    osc_edge_sync_t sync;
    const double *div2; /* NULL or the shard's table (osc_rk4_chain_advance_div2) */
} osc_shard_t;

int osc_rk4_shard_run(osc_shard_t *shard, double dt, int64_t nsteps, int64_t halo_steps,
                      int64_t step0, uint32_t flags, void *stream);

/* The NCCL transport's period loop (one process per GPU, the library
 * baseline beside the fused peer exchange): per period of halo_steps steps
 * the interior tiles run on `stream` while, on an internal side stream that
 * waited for the previous period, our current buffer's ghost zones are
 * refreshed from the neighbours (ranks rank-1 and rank+1 of `comm`, an
 * ncclComm_t -- e.g. torch's ProcessGroupNCCL._comm_ptr(); ncclSend/ncclRecv
 * of `ghost` cells of x and v each way in one NCCL group) and one launch
 * covers the edge tiles; `stream` then waits for the side stream.  Uses the
 * shard's m, C, x[2], v[2], n, own_lo, own_hi, ghost (>= 2*halo_steps),
 * first_bad, div2 and sync.period (buffer parity, advanced per period); the
 * peer fields are unused.  nranks == 1: plain launches, comm may be NULL.
 * libnccl.so.2 is opened at the first multi-rank call (not linked).
 * Asynchronous (stream-ordered); parameters are not re-validated. */
int osc_rk4_shard_run_nccl(osc_shard_t *shard, void *comm, int rank, int nranks, double dt,
                           int64_t nsteps, int64_t halo_steps, int64_t step0, uint32_t flags,
                           void *stream);

/* Stream-ordered 64-bit counters, for ordering work across processes
 * without host synchronisation: osc_stream_write_u64 stores value at addr
 * once all prior work of stream is done (preceded by a system-scope fence, so
 * a kernel's peer-memory stores are visible first); osc_stream_wait_u64 holds
 * later work of stream until (int64_t)(*addr - value) >= 0.  The wait is
 * done by the GPU front-end -- no kernel spins.  addr: device memory of this
 * process or a peer's, mapped with osc_ipc_import. */
int osc_stream_write_u64(void *stream, void *addr, uint64_t value);
int osc_stream_wait_u64(void *stream, const void *addr, uint64_t value);

/* One chain of s cells sharded over the GPUs of THIS process (devs[ngpu],
 * ids may repeat), host buffers m, C, x, v [s] (x, v updated in place),
 * byte-identical to osc_rk4_chains for any ngpu.  Contiguous shards with
 * 2*halo_steps ghost cells per interior side (0 = default 32); every
 * halo_steps steps each shard's tile kernel stores its boundary cells
 * straight into its neighbours' next-input ghost zones (peer memory over
 * NVLink, peer access enabled here) -- the fused exchange of
 * osc_rk4_chain_advance, ordered by cross-device events only.  The
 * single-process counterpart of the one-process-per-GPU driver
 * (paper_1702_02207_b200/sharded.py).  Synchronous.  first_bad: [1]. */
int osc_rk4_chain_sharded(int ngpu, const int *devs, const double *m, const double *C, double *x,
                          double *v, int64_t s, double dt, int64_t nsteps, int64_t halo_steps,
                          int64_t *first_bad, uint32_t flags);

/* Dense general system M x'' + K x = 0 (BASELINE configs[4]; outside the
 * reference).  osc_rowscale: A = K / m[:, None] (IEEE division
 * per element), A [s][s] row-major.  osc_rk4_dense: N trajectories, X, V
 * [s][N] row-major (one trajectory per column) advanced in place nsteps
 * classical RK4 steps with acceleration -(A y) (rk4_step's stage structure,
 * oscillator.py:208-231), each step as two FP64 tensor-core GEMMs
 * [s x s] x [s x 2N] with the RK4 elementwise work fused into the epilogue.
 * Not bit-identical to a CPU BLAS (summation order); deterministic run to
 * run.  first_bad: [1], first step with a non-finite entry, or 0. */
int osc_rowscale(const double *K, const double *m, double *A, int64_t s, void *stream);
int osc_rk4_dense(const double *A, double *X, double *V, int64_t s, int64_t N, double dt,
                  int64_t nsteps, int64_t *first_bad, void *stream);

/* The paper's thread-per-equation engine (run_parallel, parallel.py:395-573)
 * on one warp: lane j % 32 owns first-order equation j, shared-memory double
 * banks stand in for SharedPhase and __syncwarp for StageBarrier.  Bit-
 * identical trajectory to integrate(); step_ns[nsteps] receives the
 * %globaltimer duration of every step (the per-step latency the paper
 * studies).  1 <= s <= 64.  xs/vs: [1 + nsteps/stride][s]; first_bad: [1]. */
int osc_equation_engine(const double *m, const double *C, const double *x0, const double *v0,
                        int64_t s, double dt, int64_t nsteps, int64_t stride, double *xs,
                        double *vs, int64_t *first_bad, int64_t *step_ns, void *stream);

/* Peer memory for the fused halo exchange between processes (one per GPU):
 * plain device allocations whose CUDA IPC handles (64 bytes) are exchanged
 * out of band, mapped by the neighbours (NVLink peer access), and
 * interprocess events that order a neighbour's launch after ours. */
int osc_device_alloc(uint64_t bytes, void **ptr);
int osc_device_free(void *ptr);
int osc_ipc_export(const void *ptr, unsigned char *handle64);
int osc_ipc_import(const unsigned char *handle64, void **ptr);
int osc_ipc_close(void *ptr);
int osc_ipc_event_create(void **event, unsigned char *handle64);
int osc_ipc_event_open(const unsigned char *handle64, void **event);
int osc_event_record(void *event, void *stream);
int osc_stream_wait_event(void *stream, void *event);
int osc_event_destroy(void *event);

/* derivative() (oscillator.py:184-191): dvel[b][i] = acceleration_at(...).
 * cell_major != 0 selects the [s][B] layout (batched 2-DOF SoA). */
int osc_derivative(const double *m, const double *C, const double *x, double *dvel, int64_t B,
                   int64_t s, int cell_major, void *stream);

/* energy() (oscillator.py:266-276), exact sequential index-order sum per chain. */
int osc_energy(const double *m, const double *C, const double *x, const double *v, double *out,
               int64_t B, int64_t s, int cell_major, void *stream);

/* Self-test of the hoisted-reciprocal division against IEEE div.rn.f64 on n
 * random operand pairs (mode 0: masses in [0.5,2), any numerator; 1: any
 * positive divisor; 2: physical ranges; 3: the two-operation division of
 * osc_rk4_batch2 on physical ranges; 4: the same on numerators next to
 * quotient rounding midpoints; 5: the loops' three-operation division with
 * its flag, any operands; 6 / 7: the chain kernels' checked two-operation
 * division with its tests, any operands / midpoint-aimed numerators; 8: as
 * 7 but counting the WRONG two-operation quotients the tests caught; 9: the
 * untested two-operation quotient of osc_rk4_batch2's state-tested loop on
 * midpoint-aimed numerators over the whole range its state tests admit).
 * Synchronous; *mismatches (host) receives the number of pairs whose bits
 * differ (mode 8: the number caught). */
int osc_check_division(int64_t n, uint64_t seed, int mode, uint64_t *mismatches, void *stream);

/* pass[i] = the class of b[i] for the two-operation division q = RN(a*zh +
 * RN(a*zl)) (zh = RN(1/b), zl = RN(1/b - zh); Brisebarre-Muller-Raina,
 * osc_device.cuh): 1 = correctly rounded for every numerator the kernels
 * feed it, 2 / 3 = the same with zl moved one ulp toward +inf / -inf, 0 =
 * none.  osc_rk4_batch2 runs the systems whose two masses have a class with
 * it (the tiled chain kernels use the checked form, osc_div2c_table).
 * Device buffers;
 * enqueued on `stream`.  Not part of the reference interface (diagnostic). */
int osc_div2_classify(const double *b, int64_t n, uint8_t *pass, void *stream);

/* The chain kernels' two-operation division table (osc_device.cuh
 * div2_chain_consts), one entry per divisor b[i]: a divisor with a class (as
 * osc_div2_classify; 99.95% of random masses) gets that class's zh[i] =
 * RN(1/b), zl[i] and bad[i] = 2^63 | 0x9e3779b9 ("clean": its quotients need
 * no test).  Any other divisor gets the class-1 constants and bad[i] = the
 * fraction bits of the one wrong value RN(a*zh + RN(a*zl)) can take instead
 * of RN(a/b) (one failing numerator significand at most); the kernels
 * replay a chunk with IEEE division whenever a quotient's low 32 bits equal
 * bad[i]'s.  zh[i] = 0 marks a divisor that is not eligible (outside
 * [2^-100, 2^101), or two failing significands): its tile takes the exact
 * replay.  A warp whose divisors are all clean runs the untested loop.
 * osc_rk4_chains computes this table itself.  Device buffers; enqueued on
 * `stream`.  Not part of the reference interface (diagnostic). */
int osc_div2c_table(const double *b, int64_t n, double *zh, double *zl, uint64_t *bad,
                    void *stream);

/* FP64 pipe microbenchmark (roofline denominator; not part of the hot path):
 * enqueues one launch of 8 independent DFMA (mode 0) or DADD (mode 1)
 * chains per thread -- *lane_ops (host) = DP lane-instructions executed -- or
 * of 8 independent DMMA.8x8x4 chains per warp (mode 2; mode 3 adds 8 DFMA
 * chains per thread) -- *lane_ops = flops executed.  Modes 4/5/6: ONE
 * thread running a dependent DFMA/DADD/DMUL chain, sink[0] = its clock64
 * cycles, *lane_ops = the chain length (latency, not throughput).
 * sink: device scratch of >= 512 doubles. */
int osc_bench_fp64(int64_t iters, int mode, double *sink, int64_t *lane_ops, void *stream);

/* Host-pointer convenience forms: synchronous, copies inside, return
 * OSC_NONFINITE when any system diverged.  The parameter rule is checked on
 * the device before anything is written back: OSC_INVALID leaves x, v, xs,
 * vs and first_bad untouched.  Small calls (<= 8 MB of data) are one round
 * trip -- one host-to-device and one device-to-host copy through a pinned
 * per-thread staging buffer, streams reused per thread -- which is the
 * latency a drop-in caller stepping one small system sees; large ones are a
 * chunked three-stream pipeline. */
int osc_rk4_batch2_host(const double *m, const double *C, double *x, double *v, int64_t B,
                        double dt, int64_t nsteps, int64_t stride, double *xs, double *vs,
                        int64_t *first_bad);
int osc_rk4_chains_host(const double *m, const double *C, double *x, double *v, int64_t B,
                        int64_t s, double dt, int64_t nsteps, int64_t stride, double *xs,
                        double *vs, int64_t *first_bad);
/* derivative() / energy() of host arrays (layouts as osc_derivative /
 * osc_energy), one staged round trip each. */
int osc_derivative_host(const double *m, const double *C, const double *x, double *dvel,
                        int64_t B, int64_t s, int cell_major);
int osc_energy_host(const double *m, const double *C, const double *x, const double *v,
                    double *out, int64_t B, int64_t s, int cell_major);

#ifdef __cplusplus
}
#endif

#endif /* OSC_B200_H */
