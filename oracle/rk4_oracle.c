/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the RK4 hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  The product path (the CUDA kernels in
 * paper_1702_02207_b200/csrc) never links or calls it.
 *
 * A plain-C restatement of the reference integrator
 *   /root/reference/pkg/src/oscbench/oscillator.py
 * for batches of wall-anchored chains.  Every arithmetic operation is one IEEE
 * binary64 operation in round-to-nearest, in the order the reference performs
 * it; the build uses -ffp-contract=off so no a*b+c is fused.  With that the
 * output is byte-identical to oscbench.integrate (pinned in tests/test_oracle.py
 * against tests/golden/, which were produced by the reference itself).
 *
 *   acceleration_at   oscillator.py:152-164
 *   stage_value       oscillator.py:167-169   base + coeff*slope
 *   combine_value     oscillator.py:172-174   base + (dt/6)*(((k1+2k2)+2k3)+k4)
 *   rk4_step          oscillator.py:194-231
 *   integrate         oscillator.py:234-263   (stride sampling, first bad step)
 *   PhaseState check  oscillator.py:107-109   (NaN/Inf -> NonFiniteStateError)
 *   energy            oscillator.py:266-276
 *
 * Layout: chains are [B][s] row-major, samples [nsamp][B][s].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* acceleration_at (oscillator.py:152-164) for every cell of one chain.
 *   left = x_i - (x_{i-1} if i>0 else 0.0)         (160)
 *   a    = -C_i * left                               (161)
 *   if i+1 < s: a += C_{i+1} * (x_{i+1} - x_i)       (162-163)
 *   return a / m_i                                   (164)
 * Written literally (no sharing of C_i*d_i between neighbours) so the
 * restatement reads line-for-line against the reference. */
static void accel(const double *m, const double *C, const double *x, double *a,
                  int64_t lo, int64_t hi, int64_t s)
{
    for (int64_t i = lo; i < hi; ++i) {
        double left = x[i] - (i > 0 ? x[i - 1] : 0.0);
        double acc = -C[i] * left;
        if (i + 1 < s)
            acc += C[i + 1] * (x[i + 1] - x[i]);
        a[i] = acc / m[i];
    }
}

static inline double stage_value(double base, double coeff, double slope)
{
    return base + coeff * slope; /* oscillator.py:169 */
}

static inline double combine_value(double base, double dt, double k1, double k2,
                                   double k3, double k4)
{
    return base + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4); /* :174 */
}

static inline int finite_all(const double *p, const double *q, int64_t n)
{
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(p[i]) || !isfinite(q[i]))
            return 0;
    return 1;
}

/* Scratch for one chain: k1v..k4v, y2p..y4p, y2v..y4v (11 vectors of s). */
typedef struct {
    double *k1, *k2, *k3, *k4, *y2p, *y3p, *y4p, *y2v, *y3v, *y4v, *np, *nv;
} scratch_t;

static int scratch_alloc(scratch_t *w, int64_t s)
{
    double *base = (double *)malloc(sizeof(double) * (size_t)s * 12);
    if (!base)
        return -1;
    double **f[12] = {&w->k1, &w->k2, &w->k3, &w->k4, &w->y2p, &w->y3p,
                      &w->y4p, &w->y2v, &w->y3v, &w->y4v, &w->np, &w->nv};
    for (int j = 0; j < 12; ++j)
        *f[j] = base + (size_t)j * s;
    return 0;
}

/* rk4_step (oscillator.py:194-231) on cells [lo,hi) of one chain; the caller
 * brackets each phase with a barrier when cells are split across threads.
 * Phase p in 0..4 corresponds to the blocks at lines 211-213, 216-218,
 * 221-223, 226 and 227-228. */
static void step_phase(int p, const double *m, const double *C, const double *pos,
                       const double *vel, scratch_t *w, double dt, int64_t lo,
                       int64_t hi, int64_t s)
{
    const double half_dt = 0.5 * dt; /* :208 */
    switch (p) {
    case 0:
        accel(m, C, pos, w->k1, lo, hi, s);
        for (int64_t i = lo; i < hi; ++i) {
            w->y2p[i] = stage_value(pos[i], half_dt, vel[i]);
            w->y2v[i] = stage_value(vel[i], half_dt, w->k1[i]);
        }
        break;
    case 1:
        accel(m, C, w->y2p, w->k2, lo, hi, s);
        for (int64_t i = lo; i < hi; ++i) {
            w->y3p[i] = stage_value(pos[i], half_dt, w->y2v[i]);
            w->y3v[i] = stage_value(vel[i], half_dt, w->k2[i]);
        }
        break;
    case 2:
        accel(m, C, w->y3p, w->k3, lo, hi, s);
        for (int64_t i = lo; i < hi; ++i) {
            w->y4p[i] = stage_value(pos[i], dt, w->y3v[i]);
            w->y4v[i] = stage_value(vel[i], dt, w->k3[i]);
        }
        break;
    case 3:
        accel(m, C, w->y4p, w->k4, lo, hi, s);
        for (int64_t i = lo; i < hi; ++i) {
            w->np[i] = combine_value(pos[i], dt, vel[i], w->y2v[i], w->y3v[i], w->y4v[i]);
            w->nv[i] = combine_value(vel[i], dt, w->k1[i], w->k2[i], w->k3[i], w->k4[i]);
        }
        break;
    }
}

/* integrate (oscillator.py:234-263) for one chain held in x/v (in/out).
 * Samples k = stride, 2*stride, ... are written to xs/vs[(k/stride)*rowstride].
 * Returns the 1-based first non-finite step or 0. */
static int64_t integrate_chain(const double *m, const double *C, double *x, double *v,
                               int64_t s, double dt, int64_t nsteps, int64_t stride,
                               double *xs, double *vs, int64_t rowstride, scratch_t *w)
{
    if (xs) {
        memcpy(xs, x, sizeof(double) * (size_t)s);
        memcpy(vs, v, sizeof(double) * (size_t)s);
    }
    for (int64_t k = 0; k < nsteps; ++k) {
        for (int p = 0; p < 4; ++p)
            step_phase(p, m, C, x, v, w, dt, 0, s, s);
        memcpy(x, w->np, sizeof(double) * (size_t)s);
        memcpy(v, w->nv, sizeof(double) * (size_t)s);
        if (!finite_all(x, v, s))
            return k + 1; /* :255-260 */
        if ((k + 1) % stride == 0 && xs) {
            int64_t j = (k + 1) / stride;
            memcpy(xs + j * rowstride, x, sizeof(double) * (size_t)s);
            memcpy(vs + j * rowstride, v, sizeof(double) * (size_t)s);
        }
    }
    return 0;
}

/* Batch of B independent chains of s cells, [B][s].  xs/vs may be NULL
 * (no sampling); otherwise [1 + nsteps/stride][B][s].  first_bad[B].
 * Returns 0, 1 if any chain diverged, -1 on allocation failure. */
int oracle_rk4_chains(const double *m, const double *C, double *x, double *v,
                      int64_t B, int64_t s, double dt, int64_t nsteps, int64_t stride,
                      double *xs, double *vs, int64_t *first_bad, int nthreads)
{
    int any = 0, err = 0;
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#pragma omp parallel reduction(| : any, err)
#endif
    {
        scratch_t w;
        if (scratch_alloc(&w, s) != 0) {
            err = 1;
        } else {
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
            for (int64_t b = 0; b < B; ++b) {
                int64_t o = b * s;
                int64_t fb = integrate_chain(m + o, C + o, x + o, v + o, s, dt, nsteps,
                                             stride, xs ? xs + o : NULL,
                                             vs ? vs + o : NULL, B * s, &w);
                first_bad[b] = fb;
                any |= (fb != 0);
            }
            free(w.k1);
        }
    }
    return err ? -1 : any;
}

/* One long chain with its cells split across threads inside every phase
 * (the paper's thread-per-equation decomposition with a barrier per phase,
 * PAPER.md section 4 / parallel.py:476-520).  Each phase is elementwise over
 * cells, so the split does not change any result bit. */
int oracle_rk4_chain_mt(const double *m, const double *C, double *x, double *v,
                        int64_t s, double dt, int64_t nsteps, int64_t *first_bad,
                        int nthreads)
{
    scratch_t w;
    if (scratch_alloc(&w, s) != 0)
        return -1;
    int64_t fb = 0;
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        int nt = 1, t = 0;
#ifdef _OPENMP
        nt = omp_get_num_threads();
        t = omp_get_thread_num();
#endif
        int64_t lo = s * t / nt, hi = s * (t + 1) / nt;
        for (int64_t k = 0; k < nsteps; ++k) {
            for (int p = 0; p < 4; ++p) {
                step_phase(p, m, C, x, v, &w, dt, lo, hi, s);
#ifdef _OPENMP
#pragma omp barrier
#endif
            }
            int bad = 0;
            for (int64_t i = lo; i < hi; ++i) {
                x[i] = w.np[i];
                v[i] = w.nv[i];
                bad |= !isfinite(x[i]) || !isfinite(v[i]);
            }
            if (bad) {
#ifdef _OPENMP
#pragma omp critical
#endif
                if (fb == 0 || fb > k + 1)
                    fb = k + 1;
            }
#ifdef _OPENMP
#pragma omp barrier
#endif
            if (fb != 0)
                break;
#ifdef _OPENMP
#pragma omp barrier
#endif
        }
    }
    free(w.k1);
    *first_bad = fb;
    return fb != 0;
}

/* energy (oscillator.py:266-276), sequential sum in index order, per chain. */
void oracle_energy(const double *m, const double *C, const double *x, const double *v,
                   int64_t B, int64_t s, double *out)
{
    for (int64_t b = 0; b < B; ++b) {
        const double *mm = m + b * s, *cc = C + b * s, *xx = x + b * s, *vv = v + b * s;
        double total = 0.0;
        for (int64_t i = 0; i < s; ++i) {
            total += 0.5 * mm[i] * vv[i] * vv[i];
            double ext = xx[i] - (i > 0 ? xx[i - 1] : 0.0);
            total += 0.5 * cc[i] * ext * ext;
        }
        out[b] = total;
    }
}

/* derivative (oscillator.py:184-191): dvel per cell, [B][s]. */
void oracle_derivative(const double *m, const double *C, const double *x, int64_t B,
                       int64_t s, double *dvel)
{
    for (int64_t b = 0; b < B; ++b)
        accel(m + b * s, C + b * s, x + b * s, dvel + b * s, 0, s, s);
}

/* Batched 2-DOF systems in the product's SoA layout [2][B] (BASELINE
 * configs 0-1): the same restatement, unrolled for s = 2 and run one system
 * at a time with its state in registers -- the fastest honest CPU form of
 * the reference algorithm, used as the timed CPU baseline.  Static blocks of
 * systems per thread (no false sharing).  No sampling; first_bad[B]. */
int oracle_rk4_batch2(const double *m, const double *C, double *x, double *v, int64_t B,
                      double dt, int64_t nsteps, int64_t *first_bad, int nthreads)
{
    const double half_dt = 0.5 * dt, dt6 = dt / 6.0;
    int any = 0;
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static) reduction(| : any)
#endif
    for (int64_t i = 0; i < B; ++i) {
        const double m0 = m[i], m1 = m[B + i], C0 = C[i], C1 = C[B + i];
        double x0 = x[i], x1 = x[B + i], v0 = v[i], v1 = v[B + i];
        int64_t bad = 0;
        for (int64_t k = 0; k < nsteps; ++k) {
            /* acceleration_at (oscillator.py:160-164) for i = 0, 1 */
#define ACC(p0, p1, a0, a1)                                   \
    do {                                                      \
        double l0 = (p0) - 0.0, l1 = (p1) - (p0);             \
        double t0 = -C0 * l0;                                 \
        t0 += C1 * ((p1) - (p0));                             \
        a0 = t0 / m0;                                         \
        a1 = (-C1 * l1) / m1;                                 \
    } while (0)
            double k10, k11, k20, k21, k30, k31, k40, k41;
            ACC(x0, x1, k10, k11);
            double y2p0 = x0 + half_dt * v0, y2p1 = x1 + half_dt * v1;
            double y2v0 = v0 + half_dt * k10, y2v1 = v1 + half_dt * k11;
            ACC(y2p0, y2p1, k20, k21);
            double y3p0 = x0 + half_dt * y2v0, y3p1 = x1 + half_dt * y2v1;
            double y3v0 = v0 + half_dt * k20, y3v1 = v1 + half_dt * k21;
            ACC(y3p0, y3p1, k30, k31);
            double y4p0 = x0 + dt * y3v0, y4p1 = x1 + dt * y3v1;
            double y4v0 = v0 + dt * k30, y4v1 = v1 + dt * k31;
            ACC(y4p0, y4p1, k40, k41);
#undef ACC
            double nx0 = x0 + dt6 * (v0 + 2.0 * y2v0 + 2.0 * y3v0 + y4v0);
            double nx1 = x1 + dt6 * (v1 + 2.0 * y2v1 + 2.0 * y3v1 + y4v1);
            double nv0 = v0 + dt6 * (k10 + 2.0 * k20 + 2.0 * k30 + k40);
            double nv1 = v1 + dt6 * (k11 + 2.0 * k21 + 2.0 * k31 + k41);
            x0 = nx0; x1 = nx1; v0 = nv0; v1 = nv1;
            if (!isfinite(x0) || !isfinite(x1) || !isfinite(v0) || !isfinite(v1)) {
                bad = k + 1;
                break;
            }
        }
        x[i] = x0; x[B + i] = x1; v[i] = v0; v[B + i] = v1;
        first_bad[i] = bad;
        any |= bad != 0;
    }
    return any;
}
