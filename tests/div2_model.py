"""Exact-rational model of the two-operation division (test infrastructure).

q = RN(a*zh + RN(a*zl)), zh = RN(1/b), zl = RN(1/b - zh) (Brisebarre,
Muller, Raina 2004), restated with ``fractions.Fraction`` so every rounding is
exact: Python's float(Fraction) and float ``*``/``/`` are correctly rounded.
``classify`` mirrors div2_classify (paper_1702_02207_b200/csrc/osc_device.cuh):
class 1 (zl), 2 (zl one ulp toward +inf) or 3 (toward -inf) is the first
whose two-operation quotient is correct on every significand A with
A*2^sh = k (mod B), |k| <= 2 (sh = 53, a/b >= 1) and |k| <= 4 (sh = 54,
a/b < 1); 0 = none.
"""

from __future__ import annotations

import math
import struct
from fractions import Fraction


def consts(b: float):
    zh = 1.0 / b
    zl = float(Fraction(1) / Fraction(b) - Fraction(zh))
    return zh, zl


def div2(a: float, zh: float, zl: float) -> float:
    return float(Fraction(a) * Fraction(zh) + Fraction(a * zl))


def significand(b: float):
    m, e = math.frexp(b)  # b = m 2^e, m in [0.5, 1)
    return int(m * 2 ** 53), e - 1


def solutions(B: int, sh: int, k: int, lo: int, hi: int):
    """Significands A in [lo, hi) with A 2^sh - B M = k for some integer M."""
    g = math.gcd(B, 2 ** sh)
    if k % g:
        return []
    Bo, kk = B // g, k // g
    if Bo == 1:
        return []
    A = (kk * pow(2 ** sh // g, -1, Bo)) % Bo
    if A < lo:
        A += -(-(lo - A) // Bo) * Bo
    return list(range(A, hi, Bo))


def candidates(b: float, kmax53: int = 2, kmax54: int = 4):
    B, _ = significand(b)
    out = []
    for sh, kmax, lo, hi in ((53, kmax53, B, 2 ** 53), (54, kmax54, 2 ** 52, B)):
        for k in range(-kmax, kmax + 1):
            if k:
                out += [(sh, k, A) for A in solutions(B, sh, k, lo, hi)]
    return out


def class_zl(zl: float, cls: int) -> float:
    return zl if cls == 1 else math.nextafter(zl, math.inf if cls == 2 else -math.inf)


def classify(b: float) -> int:
    if not (2.0 ** -100 <= b < 2.0 ** 101):
        return 0
    B, _ = significand(b)
    bs = B / 2 ** 52
    zh, zl = consts(bs)
    if B == 2 ** 52:
        return 1
    cands = candidates(b)
    for cls in (1, 2, 3):
        z = class_zl(zl, cls)
        if abs(z) < 2.0 ** -80 * zh:
            continue
        if all(div2(A / 2 ** 52, zh, z) == (A / 2 ** 52) / bs for _, _, A in cands):
            return cls
    return 0


NO_BAD = 0x9E3779B9  # kDiv2NoBad: the tested low word of a divisor with no failure


def checked_consts(b: float):
    """div2_checked_consts (osc_device.cuh), the chain kernels' checked
    two-operation division: (zh, zl, bad) with class-1 constants in b's own
    binade and ``bad`` the fraction bits of the wrong two-operation quotient
    of the one failing candidate significand (NO_BAD when none), or None when
    b is not eligible (outside [2^-100, 2^101), |zl| < 2^-80 zh, or two
    failures)."""
    if not (2.0 ** -100 <= b < 2.0 ** 101):
        return None
    B, e = significand(b)
    bs = B / 2 ** 52
    zh, zl = consts(bs)
    scale = 2.0 ** -e
    if B == 2 ** 52:
        return zh * scale, 0.0, NO_BAD
    if abs(zl) < 2.0 ** -80 * zh:
        return None
    fails = [A for _, _, A in candidates(b) if div2(A / 2 ** 52, zh, zl) != (A / 2 ** 52) / bs]
    if len(fails) > 1:
        return None
    bad = fraction_bits(div2(fails[0] / 2 ** 52, zh, zl)) if fails else NO_BAD
    return zh * scale, zl * scale, bad


def fraction_bits(a: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", a))[0] & (2 ** 52 - 1)


CLEAN = 1 << 63  # kDiv2Clean: a divisor whose quotients need no test


def chain_consts(b: float):
    """div2_chain_consts (osc_device.cuh), the chain kernels' table entry: a
    divisor with a class gets that class's constants and ``CLEAN | NO_BAD``;
    any other divisor the checked form's (checked_consts), or None."""
    cls = classify(b)
    if cls:
        zh, zl = consts(b)
        return zh, class_zl(zl, cls), CLEAN | NO_BAD
    return checked_consts(b)
