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
        cls = dm.classify(b)
        for sh, k, A in dm.candidates(b, kmax53=12, kmax54=12):
            x = A / 2 ** 52
            if dm.div2(x, zh, zl) != x / bs:
                seen += 1
                assert sh == 54 and abs(k) == 1, (b, sh, k, A)
                assert cls != 1, (b, sh, k, A)
    assert seen > 0  # the adversarial numerators do find the failing divisors


def test_moved_zl_fails_only_inside_the_tested_superset():
    """Classes 2/3 (zl moved one ulp): |S - a/b| < 2^-105, so failures need
    |k| = 1 (a/b >= 1) or |k| <= 3 (a/b < 1); the classifier tests |k| <= 2
    resp. 4.  Aim numerators from |k| <= 12 at every moved form."""
    rng = random.Random(99)
    for _ in range(800):
        b = rng.uniform(1.0, 2.0)
        B, _ = dm.significand(b)
        bs = B / 2 ** 52
        zh, zl = dm.consts(bs)
        for cls in (2, 3):
            z = dm.class_zl(zl, cls)
            for sh, k, A in dm.candidates(b, kmax53=12, kmax54=12):
                x = A / 2 ** 52
                if dm.div2(x, zh, z) != x / bs:
                    assert (sh == 53 and abs(k) <= 2) or (sh == 54 and abs(k) <= 4), (b, cls, k)


def test_random_numerators_on_passing_divisors():
    rng = random.Random(7)
    n = 0
    for _ in range(300):
        b = rng.uniform(0.5, 2.0)
        cls = dm.classify(b)
        if not cls:
            continue
        zh, zl = dm.consts(b)
        zl = dm.class_zl(zl, cls)
        for _ in range(100):
            a = rng.uniform(-4.0, 4.0) * 2.0 ** rng.randint(-40, 40)
            assert dm.div2(a, zh, zl) == a / b, (a, b)
            n += 1
    assert n > 25_000


def test_pass_fraction_and_edges():
    rng = random.Random(3)
    cls = [dm.classify(rng.uniform(0.5, 2.0)) for _ in range(20000)]
    first = cls.count(1) / len(cls)
    assert 0.98 < first < 0.995, first  # zl itself
    assert cls.count(0) < 30  # ~0.05% left after the moved forms
    assert cls.count(2) > 50 and cls.count(3) > 50
    for b in (1.0, 0.5, 2.0, 2.0 ** 100, 2.0 ** -100):
        assert dm.classify(b) == 1
    for b in (2.0 ** 101, 2.0 ** -101, 0.0, -1.0, float("inf")):
        assert not dm.classify(b)


def _device_enumeration(B):
    """The division-free candidate walk of div2_classify (osc_device.cuh),
    restated: trailing zeros v, odd part Bo, 2^-(sh-v) mod Bo from Newton's
    inverse of Bo mod 2^64, multiples by repeated addition."""
    def inv_pow2_mod(n, Bo):
        u = Bo
        for _ in range(5):
            u = (u * (2 - Bo * u)) % 2 ** 64
        return (Bo * ((-u) % 2 ** n) + 1) >> n

    out = []
    v = (B & -B).bit_length() - 1
    if v > 2:
        return out
    Bo = B >> v
    inv53 = inv_pow2_mod(53 - v, Bo)
    inv54 = (inv53 + Bo) >> 1 if inv53 & 1 else inv53 >> 1
    for inv, kmax, lo, hi in ((inv53, 2, B, 2 ** 53), (inv54, 4, 2 ** 52, B)):
        mk = 0
        for _ in range(kmax >> v):
            mk = mk + inv - Bo if mk + inv >= Bo else mk + inv
            for A in (mk, Bo - mk if mk else 0):
                while A < lo:
                    A += Bo
                while A < hi:
                    out.append(A)
                    A += Bo
    return sorted(out)


def test_device_candidate_walk_equals_gcd_solution():
    rng = random.Random(1)
    for i in range(8000):
        B = rng.randrange(2 ** 52, 2 ** 53)
        B = (B | 1, B & ~1, B & ~3, B & ~7)[i % 4] | (1 << 52)
        want = sorted(A for _, _, A in dm.candidates(B / 2 ** 52))
        assert _device_enumeration(B) == want, B


# ---------------------------------------------------------------------------
# The checked form of the chain kernels (div2_checked_consts / div2c_fast):
# class-1 constants for every divisor, and a per-division test of the one
# significand that can round wrongly.
# ---------------------------------------------------------------------------

def test_checked_form_fails_only_at_the_stored_significand():
    """Numerators aimed at midpoints from |k| <= 12: a wrong two-operation
    quotient only ever comes from the one failing significand and equals the
    stored wrong quotient, so the kernels' low-word test catches every one."""
    rng = random.Random(20261020)
    caught = 0
    for _ in range(1500):
        b = rng.uniform(1.0, 2.0)
        cc = dm.checked_consts(b)
        assert cc is not None, b
        zh, zl, bad = cc
        for sh, k, A in dm.candidates(b, kmax53=12, kmax54=12):
            x = A / 2 ** 52
            q = dm.div2(x, zh, zl)
            if q != x / b:
                assert dm.fraction_bits(q) == bad, (b, sh, k, A)
                assert (bad & 0xFFFFFFFF) != dm.NO_BAD
                caught += 1
    assert caught > 5  # the aimed numerators do hit failing significands


def test_checked_form_eligibility_and_scaling():
    rng = random.Random(4)
    n_fail = n_inel = 0
    for _ in range(20000):
        b = rng.uniform(0.5, 2.0)
        cc = dm.checked_consts(b)
        if cc is None:
            n_inel += 1
            continue
        n_fail += (cc[2] & 0xFFFFFFFF) != dm.NO_BAD
    assert n_inel == 0  # every random mass is eligible (two failures: none seen)
    assert 0.005 < n_fail / 20000 < 0.03  # ~1.2% carry one failing significand
    for b in (1.0, 0.5, 2.0, 2.0 ** 100, 2.0 ** -100):
        assert dm.checked_consts(b)[1:] == (0.0, dm.NO_BAD)
    for b in (2.0 ** 101, 2.0 ** -101, 0.0, -1.0, float("inf")):
        assert dm.checked_consts(b) is None
    # scaled divisors, numerators in many binades: exact, or flagged -- also
    # the failing significand itself, scaled (the wrong quotient scales too)
    for _ in range(300):
        b = rng.uniform(0.5, 2.0) * 2.0 ** rng.randint(-90, 90)
        zh, zl, bad = dm.checked_consts(b)
        B, _ = dm.significand(b)
        bs = B / 2 ** 52
        hs, ls = dm.consts(bs)
        fails = [A for _, _, A in dm.candidates(b) if dm.div2(A / 2 ** 52, hs, ls) != (A / 2 ** 52) / bs]
        nums = [rng.uniform(-4.0, 4.0) * 2.0 ** rng.randint(-40, 40) for _ in range(50)]
        nums += [A / 2 ** 52 * 2.0 ** rng.randint(-40, 40) * rng.choice((1, -1)) for A in fails]
        for a in nums:
            q = dm.div2(a, zh, zl)
            if (dm.fraction_bits(q) & 0xFFFFFFFF) != (bad & 0xFFFFFFFF):
                assert q == a / b, (a, b)
            elif a in nums[50:]:
                assert q != a / b  # the failing numerator really is caught


def test_chain_table_entries():
    """div2_chain_consts: classed divisors keep their class constants and need
    no test; the rest carry the checked form's wrong quotient."""
    rng = random.Random(8)
    kinds = {"clean": 0, "checked": 0}
    for _ in range(6000):
        b = rng.uniform(0.5, 2.0)
        zh, zl, bad = dm.chain_consts(b)
        cls = dm.classify(b)
        if cls:
            assert bad == dm.CLEAN | dm.NO_BAD
            assert (zh, zl) == (dm.consts(b)[0], dm.class_zl(dm.consts(b)[1], cls))
            kinds["clean"] += 1
        else:
            assert not bad & dm.CLEAN and (zh, zl, bad) == dm.checked_consts(b)
            kinds["checked"] += 1
    assert kinds["checked"] < 20 and kinds["clean"] > 5900
