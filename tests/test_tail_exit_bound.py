"""CPU checks of the arithmetic behind the walk's no-op tail exit
(`walk_tail_noop`, csrc/ucp_kernels.cu; DESIGN.md §2 (v)).

The kernel stops a stage-0 Gaussian walk (kernels.py:406-445 of the
reference) once every remaining addend is provably below |acc| * 2^-55.  These
tests check, in IEEE double arithmetic on the host (Python floats are
round-to-nearest binary64), (1) the absorption lemma it relies on and (2) a
scalar restatement of the walk with the same exit rule against the full walk,
bit for bit.  The device path itself is A/B-tested in test_gpu_tail_exit.py.
"""
import math
import random
import struct

import pytest

E = 2.0 ** -55
TINY = 2.0 ** -960


def bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def test_absorption_lemma():
    rng = random.Random(7)
    for _ in range(20000):
        acc = math.ldexp(1.0 + rng.random(), rng.randint(-900, 900)) * rng.choice((1.0, -1.0))
        if rng.random() < 0.2:  # exact powers of two: the ulp below is half the ulp above
            acc = math.copysign(math.ldexp(1.0, rng.randint(-900, 900)), acc)
        lim = abs(acc) * E
        t = lim * rng.random() * rng.choice((1.0, -1.0))
        if rng.random() < 0.1:
            t = math.copysign(math.nextafter(lim, 0.0), t)  # largest addend the rule admits
        assert abs(t) < abs(acc) * E
        assert bits(acc + t) == bits(acc)


def walk(s, a, h, v, exit_rule, chunk=256):
    """Stage-0 walk over nodes a + j*h within s +- 12 (interior weight h, half
    weight at the grid ends), in the reference's order; with exit_rule the
    walk stops between ``chunk``-node chunks (the kernel's 4 x UCP_WALK_CHUNK4)
    once the bounds of walk_tail_noop pass."""
    d = len(v)
    q = math.exp(-h * h)
    jlo = max(0, math.ceil(((s - 12.0) - a) / h))
    jhi = min(d - 1, math.floor(((s + 12.0) - a) / h))
    acc0 = acc1 = acc2 = 0.0
    if jlo > jhi:
        return acc0, acc1, acc2, 0
    tt = (a + jlo * h) - s
    pdf = math.exp((-0.5 * tt) * tt) * (1.0 / math.sqrt(2.0 * math.pi))
    ratio = math.exp(-h * (tt + 0.5 * h))
    visited = 0
    for j in range(jlo, jhi + 1):
        if exit_rule and (j - jlo) % chunk == 0 and j > jlo and ratio <= 1.0:
            vm = max(abs(x) for x in v[j:jhi + 1])
            wpc = h * pdf
            b1 = wpc * vm
            b2 = b1 * vm
            if (acc0 > TINY and abs(acc1) > TINY and acc2 > TINY and wpc < acc0 * E and
                    b1 < abs(acc1) * E and b2 < acc2 * E):
                break
        w = 0.5 * h if j in (0, d - 1) else h
        wp = w * pdf
        acc0 += wp
        wv = wp * v[j]
        acc1 += wv
        acc2 += wv * v[j]
        pdf *= ratio
        ratio *= q
        visited += 1
    return acc0, acc1, acc2, visited


@pytest.mark.parametrize("chunk", [64, 256])
@pytest.mark.parametrize("kind", ["smooth", "spikes", "odd", "huge"])
def test_tail_exit_walk_bitwise(kind, chunk):
    rng = random.Random(["smooth", "spikes", "odd", "huge"].index(kind) + 11)
    a, h, d = -25.0, 50.0 / 2047, 2048
    xs = [a + j * h for j in range(d)]
    if kind == "smooth":
        v = [x + 0.3 * math.sin(x) for x in xs]
    elif kind == "spikes":  # large finite values far in the tail
        v = [x + (rng.choice((1e4, -1e6)) if rng.random() < 0.02 else 0.0) for x in xs]
    elif kind == "odd":  # u1 = y: the first moment cancels around s = 0
        v = list(xs)
    else:  # one value whose square overflows: the bound is +inf, no early stop past it
        v = [x for x in xs]
        v[1500] = 1e200
    saved = 0
    for s in [a + rng.random() * 50.0 for _ in range(60)] + [0.0, -25.0, 25.0, 13.0]:
        full = walk(s, a, h, v, False)
        fast = walk(s, a, h, v, True, chunk)
        assert [bits(x) for x in fast[:3]] == [bits(x) for x in full[:3]], (kind, s)
        saved += full[3] - fast[3]
    if kind != "odd":
        assert saved > 0  # the rule does fire on these windows
