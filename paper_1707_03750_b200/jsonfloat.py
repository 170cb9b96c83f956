"""Byte-exact rendering of doubles the way the reference's JSON library dumps them.

summary_to_json(...).dump(2) (report.hpp:121-185, 304) prints number_float values with the
Grisu2 digit generator (Loitsch 2010, "Printing Floating-Point Numbers Quickly and Accurately
with Integers") and printf-%g-like layout rules.  Grisu2 returns a round-trip-safe digit string
that is the SHORTEST one for almost every double but not for all of them (e.g. 4957.0239520958085,
where the shortest is 4957.023952095808), so Python's repr() cannot stand in for it.  This module
restates the algorithm with exact integer arithmetic:

* boundaries m-, m+ of the double (the lower one closer at power-of-two significands);
* a cached power of ten c_k (64-bit significand, round to nearest, k = -300 + 8 i) chosen so the
  scaled upper boundary's binary exponent lies in [alpha, gamma] = [-60, -32] — the table is
  computed here from exact rationals;
* 64 x 64 -> 64-bit multiplication rounded on the discarded half (the "DiyFp" product);
* digit generation from the integral part, then the fractional part, stopping once the remaining
  distance fits in delta, followed by the Grisu2 "round weed" correction;
* layout: fixed notation when the decimal point lands in (-4, 15] (".0" appended to integers),
  otherwise d[.ddd]e+XX with at least two exponent digits.
"""
from __future__ import annotations

import math
import struct
from fractions import Fraction

_ALPHA, _GAMMA = -60, -32
_MIN_DEC_EXP, _DEC_STEP = -300, 8
_M64 = (1 << 64) - 1


def _cached_powers():
    out = []
    for k in range(_MIN_DEC_EXP, 325, _DEC_STEP):
        v = Fraction(10) ** k
        e = v.numerator.bit_length() - v.denominator.bit_length() - 64
        while v / Fraction(2) ** e >= 2 ** 64:
            e += 1
        while v / Fraction(2) ** e < 2 ** 63:
            e -= 1
        q = v / Fraction(2) ** e
        f = int(q) + (1 if q - int(q) >= Fraction(1, 2) else 0)
        if f == 1 << 64:
            f, e = f >> 1, e + 1
        out.append((f, e, k))
    return out


_POWERS = _cached_powers()


def _mul(xf, xe, yf, ye):
    """Upper 64 bits of the 128-bit product, rounded at bit 63 of the discarded half."""
    p = xf * yf
    return ((p + (1 << 63)) >> 64) & _M64, xe + ye + 64


def _normalize(f, e):
    s = 64 - f.bit_length()
    return (f << s) & _M64, e - s


def _boundaries(v: float):
    bits = struct.unpack("<Q", struct.pack("<d", v))[0]
    E, F = bits >> 52, bits & ((1 << 52) - 1)
    if E == 0:
        f, e = F, 1 - 1075
    else:
        f, e = F + (1 << 52), E - 1075
    closer = F == 0 and E > 1
    mp = (2 * f + 1, e - 1)
    mm = (4 * f - 1, e - 2) if closer else (2 * f - 1, e - 1)
    wp = _normalize(*mp)
    wm = (mm[0] << (mm[1] - wp[1]), wp[1])
    return _normalize(f, e), wm, wp


def _cached_power(e: int):
    f = _ALPHA - e - 1
    num = f * 78913
    k = int(num / (1 << 18)) if num >= 0 else -((-num) // (1 << 18))  # C integer division (toward zero)
    k += 1 if f > 0 else 0
    idx = (-_MIN_DEC_EXP + k + (_DEC_STEP - 1)) // _DEC_STEP
    return _POWERS[idx]


def _round_weed(digits, dist, delta, rest, ten_k):
    while rest < dist and delta - rest >= ten_k and (rest + ten_k < dist or dist - rest > rest + ten_k - dist):
        digits[-1] -= 1
        rest += ten_k


def _grisu2(v: float):
    w, m_minus, m_plus = _boundaries(v)
    cf, ce, ck = _cached_power(m_plus[1])
    w_f, w_e = _mul(w[0], w[1], cf, ce)
    lo_f, lo_e = _mul(m_minus[0], m_minus[1], cf, ce)
    hi_f, hi_e = _mul(m_plus[0], m_plus[1], cf, ce)
    M_minus = lo_f + 1
    M_plus = hi_f - 1
    dec_exp = -ck
    delta = M_plus - M_minus
    dist = M_plus - w_f
    shift = -hi_e
    one = 1 << shift
    p1 = M_plus >> shift
    p2 = M_plus & (one - 1)
    digits = []
    n = len(str(p1))  # number of decimal digits of p1 (p1 > 0 here)
    pow10 = 10 ** (n - 1)
    while n > 0:
        d, p1 = divmod(p1, pow10)
        digits.append(d)
        n -= 1
        rest = (p1 << shift) + p2
        if rest <= delta:
            dec_exp += n
            _round_weed(digits, dist, delta, rest, pow10 << shift)
            return digits, dec_exp
        pow10 //= 10
    m = 0
    while True:
        p2 *= 10
        d, p2 = p2 >> shift, p2 & (one - 1)
        digits.append(d)
        m += 1
        delta *= 10
        dist *= 10
        if p2 <= delta:
            break
    dec_exp -= m
    _round_weed(digits, dist, delta, p2, one)
    return digits, dec_exp


def _exponent(e: int) -> str:
    s = "-" if e < 0 else "+"
    e = abs(e)
    return s + (f"0{e}" if e < 10 else str(e))


def dump_float(v: float) -> str:
    """The JSON text of a number_float (non-finite values dump as null)."""
    v = float(v)
    if math.isnan(v) or math.isinf(v):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    sign = "-" if v < 0 else ""
    digits, dec_exp = _grisu2(abs(v))
    s = "".join(map(str, digits))
    k = len(s)
    n = k + dec_exp  # position of the decimal point relative to the digit string
    if k <= n <= 15:
        return sign + s + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + s[:n] + "." + s[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + s
    mant = s if k == 1 else s[0] + "." + s[1:]
    return sign + mant + "e" + _exponent(n - 1)
