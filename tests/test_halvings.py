"""CPU check of the arithmetic claim behind halvings() (csrc/hps_eval.cuh): once a and b share a
binade, the end state of the reference's remaining halvings (ls/provisioner.py:430-436, with
quota_ok(mid) == (mid >= tstar)) is known in closed form. A Python mirror of the device function
(Python floats are IEEE doubles with the same rounding) is compared with the literal loop."""
import math
import random
import struct

import numpy as np


def _bits(x):
    return struct.unpack("<q", struct.pack("<d", x))[0]


def _from_bits(i):
    return struct.unpack("<d", struct.pack("<q", i))[0]


def literal(a, b, tstar, steps):
    for _ in range(steps):
        mid = (a + b) / 2.0
        if mid >= tstar:
            b = mid
        else:
            a = mid
    return b


def fast(a, b, tstar, steps):   # mirror of halvings() in hps_eval.cuh
    for it in range(steps):
        ia, ib = _bits(a), _bits(b)
        ea = ia >> 52
        if ea == (ib >> 52) and 52 < ea < 2047 and ia > 0:
            if ia == ib:
                return b
            u = _from_bits((ea - 52) << 52)
            d = (b - a) / u
            idd = _bits(d)
            need = (idd >> 52) - 1023 + (1 if idd & 0xFFFFFFFFFFFFF else 0) + 1
            if steps - it >= need:
                if not (tstar <= b):
                    return b
                if tstar <= a:
                    return a + u if ia & 1 else a
                return tstar
        mid = (a + b) / 2.0
        last = mid == a or mid == b
        if mid >= tstar:
            b = mid
        else:
            a = mid
        if last:
            break
    return b


def _cases(n, seed):
    rng = random.Random(seed)
    for _ in range(n):
        kind = rng.random()
        if kind < 0.4:      # the provisioner's shape: a = serial floor, b = tau_hi, tstar between
            a = 10 ** rng.uniform(-6, 1)
            b = a * (1 + 10 ** rng.uniform(-12, 2))
            t = a + (b - a) * rng.random()
        elif kind < 0.6:    # tstar a double close to a or b, or on a power of two
            a = 10 ** rng.uniform(-3, 1)
            b = a * (1 + rng.random() * 3)
            t = rng.choice([a, b, math.nextafter(a, math.inf), math.nextafter(b, -math.inf),
                            2.0 ** math.floor(math.log2(b)), 2.0 ** math.ceil(math.log2(a))])
        elif kind < 0.8:    # quota never binds / always binds / NaN
            a = 10 ** rng.uniform(-3, 1)
            b = a * (1 + rng.random())
            t = rng.choice([-math.inf, a / 2, b * 2, math.inf, math.nan])
        else:               # narrow, ulp-level intervals
            a = 10 ** rng.uniform(-3, 1)
            k = rng.randint(0, 70)
            b = a
            for _ in range(k):
                b = math.nextafter(b, math.inf)
            t = a + (b - a) * rng.random()
        yield a, b, t, rng.choice([60, 60, 60, rng.randint(0, 60)])


def test_fast_forward_matches_literal_halvings():
    for a, b, t, steps in _cases(100000, 1234):
        want, got = literal(a, b, t, steps), fast(a, b, t, steps)
        assert _bits(want) == _bits(got), (a, b, t, steps, want, got)


def test_fast_forward_exhaustive_small_binade_gaps():
    # every gap 1..300 ulp, every tstar position (below, on each grid point, above), A odd and even
    for a0 in (1.0, math.nextafter(1.0, 2.0), 1.7, np.float64(1.2345678).item()):
        u = math.nextafter(a0, 2.0) - a0
        for gap in range(1, 301, 7):
            b0 = a0 + gap * u
            for j in range(-2, gap + 3):
                t = a0 + j * u
                for steps in (60, 3, 9):
                    assert _bits(literal(a0, b0, t, steps)) == _bits(fast(a0, b0, t, steps))
