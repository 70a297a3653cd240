"""CPU checks of the two-operation division's theory (exact rationals).

The batched 2-DOF kernel divides by each mass with q = RN(a*zh + RN(a*zl))
when both masses of a system pass div2_classify (osc_device.cuh).  Its
correctness argument: the two-operation quotient can only differ from
RN(a/b) when a/b is within 2^-106 (relative) of a rounding midpoint, and the
classifier tests every numerator significand where that can happen.  These
tests check the argument itself on random divisors: numerators aimed at
midpoints from much further out (|k| <= 12) only ever fail where the argument
says they can (a/b < 1, |k| = 1), and never for a divisor the classifier
passes.  tests/test_gpu_parity.py checks the device classifier against this
model and the device quotient against div.rn.f64.
"""

import random

import div2_model as dm


def test_failures_only_where_the_bound_allows():
    rng = random.Random(20240607)
    seen = 0
    for _ in range(1500):
        b = rng.uniform(1.0, 2.0)
        B, _ = dm.significand(b)
        bs = B / 2 ** 52
        zh, zl = dm.consts(bs)
        passes = dm.classify(b)
        for sh, k, A in dm.candidates(b, kmax53=12, kmax54=12):
            x = A / 2 ** 52
            if dm.div2(x, zh, zl) != x / bs:
                seen += 1
                assert sh == 54 and abs(k) == 1, (b, sh, k, A)
                assert not passes, (b, sh, k, A)
    assert seen > 0  # the adversarial numerators do find the failing divisors


def test_random_numerators_on_passing_divisors():
    rng = random.Random(7)
    n = 0
    for _ in range(300):
        b = rng.uniform(0.5, 2.0)
        if not dm.classify(b):
            continue
        zh, zl = dm.consts(b)
        for _ in range(100):
            a = rng.uniform(-4.0, 4.0) * 2.0 ** rng.randint(-40, 40)
            assert dm.div2(a, zh, zl) == a / b, (a, b)
            n += 1
    assert n > 25_000


def test_pass_fraction_and_edges():
    rng = random.Random(3)
    frac = sum(dm.classify(rng.uniform(0.5, 2.0)) for _ in range(3000)) / 3000
    assert 0.97 < frac < 0.999, frac
    for b in (1.0, 0.5, 2.0, 2.0 ** 100, 2.0 ** -100):
        assert dm.classify(b)
    for b in (2.0 ** 101, 2.0 ** -101, 0.0, -1.0, float("inf")):
        assert not dm.classify(b)
