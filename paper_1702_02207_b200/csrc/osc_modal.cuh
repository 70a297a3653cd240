// Closed-form two-mode solution of a 2-DOF chain and the numeric-vs-analytic
// error report, on the device (validate at scale without a D2H
// copy of full trajectories).
//
// Equal parameters (m0 == m1, C0 == C1) restate modal.py operation for
// operation, so the coefficients are the reference's bits (sqrt and / are
// IEEE-exact on both sides):
//   characteristic_frequencies  modal.py:76-82   w = sqrt(c*(3 +- sqrt5)/(2m))
//   mode_ratios                 modal.py:85-95   r = 2 - m*(w*w)/c
//   analytic_solution           modal.py:98-120  two closed-form 2x2 solves
// Unequal parameters (outside modal.py, whose docstring leaves them to
// "RK4 plus energy diagnostics") use the same modal structure for the pencil
// K - w^2 M with K = [[C0 + C1, -C1], [-C1, C1]], M = diag(m0, m1): the roots
// of m0 m1 L^2 - (m0 C1 + m1 (C0 + C1)) L + C0 C1 = 0, fast root first, the
// slow one as c/(a L1) (no cancellation), ratios r = x1/x0 from row 1.
//   eval_analytic  modal.py:123-129 and compare  modal.py:141-162 keep the
// reference's order (sequential sum of squares, strict > for the maximum);
// only cos/sin differ from glibc in the last bits (CUDA: <= 2 ulp).
#pragma once

#include "osc_device.cuh"

namespace osc {

// Field order of a solution record (struct-of-arrays [8][B] in memory).
enum ModalField { kW1, kW2, kR1, kR2, kA1c, kA1s, kA2c, kA2s, kModalFields };

struct Modal2 {
    double f[kModalFields];
};

__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

__device__ inline Modal2 analytic2(double m0, double m1, double C0, double C1, double x0,
                                   double x1, double v0, double v1)
{
    double w1, w2, r1, r2;
    if (m0 == m1 && C0 == C1) {
        const double sqrt5 = dsqrt(5.0);  // _SQRT5, modal.py:40
        const double m = m0, c = C0;
        w1 = dsqrt(ddiv(mul(c, add(3.0, sqrt5)), mul(2.0, m)));
        w2 = dsqrt(ddiv(mul(c, sub(3.0, sqrt5)), mul(2.0, m)));
        r1 = sub(2.0, ddiv(mul(m, mul(w1, w1)), c));
        r2 = sub(2.0, ddiv(mul(m, mul(w2, w2)), c));
    } else {
        const double a = mul(m0, m1);
        const double b = add(mul(m0, C1), mul(m1, add(C0, C1)));
        const double c = mul(C0, C1);
        const double disc = sub(mul(b, b), mul(4.0, mul(a, c)));
        const double q = add(b, dsqrt(disc > 0.0 ? disc : 0.0));
        const double L1 = ddiv(q, mul(2.0, a));
        const double L2 = ddiv(mul(2.0, c), q);
        w1 = dsqrt(L1);
        w2 = dsqrt(L2);
        r1 = ddiv(C1, sub(C1, mul(L1, m1)));
        r2 = ddiv(C1, sub(C1, mul(L2, m1)));
    }
    const double det = sub(r2, r1);
    const double a1c = ddiv(sub(mul(r2, x0), x1), det);
    const double a2c = ddiv(sub(x1, mul(r1, x0)), det);
    const double u1 = ddiv(sub(mul(r2, v0), v1), det);
    const double u2 = ddiv(sub(v1, mul(r1, v0)), det);
    return Modal2{{w1, w2, r1, r2, a1c, ddiv(u1, w1), a2c, ddiv(u2, w2)}};
}

// eval_analytic (modal.py:123-129): exact positions at time t.
__device__ __forceinline__ void eval2(const Modal2 &s, double t, double &xa0, double &xa1)
{
    double s1, c1, s2, c2;
    sincos(mul(s.f[kW1], t), &s1, &c1);
    sincos(mul(s.f[kW2], t), &s2, &c2);
    const double mode1 = add(mul(s.f[kA1c], c1), mul(s.f[kA1s], s1));
    const double mode2 = add(mul(s.f[kA2c], c2), mul(s.f[kA2s], s2));
    xa0 = add(mode1, mode2);
    xa1 = add(mul(s.f[kR1], mode1), mul(s.f[kR2], mode2));
}

// compare's running state (modal.py:146-162): max_err starts at -1.0.
struct ErrAcc {
    double max_err = -1.0, sum_sq = 0.0, at_time = 0.0;
    int64_t count = 0;

    __device__ __forceinline__ void add_sample(const Modal2 &s, double t, double x0, double x1)
    {
        double xa0, xa1;
        eval2(s, t, xa0, xa1);
        one(fabs(sub(x0, xa0)), t);
        one(fabs(sub(x1, xa1)), t);
    }
    __device__ __forceinline__ void one(double err, double t)
    {
        sum_sq = add(sum_sq, mul(err, err));
        ++count;
        if (err > max_err) {
            max_err = err;
            at_time = t;
        }
    }
    // ErrorReport(max_err, sqrt(sum_sq / count), at_time)
    __device__ __forceinline__ double rmse() const
    {
        return dsqrt(ddiv(sum_sq, static_cast<double>(count)));
    }
};

__device__ __forceinline__ Modal2 load_modal(const double *sol, int64_t B, int64_t i)
{
    Modal2 s;
#pragma unroll
    for (int f = 0; f < kModalFields; ++f)
        s.f[f] = sol[f * B + i];
    return s;
}

}  // namespace osc
