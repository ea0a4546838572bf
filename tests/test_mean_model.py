"""CPU model of the exact parallel row mean (kernels.cu K1, mean_* kernels):
F96 fixed-point prefix sums plus the FP64 chain's rounding steps.  Checks the
algorithm itself -- on random and adversarial sequences, in plain Python
integers -- against the literal sequential chain of engine.cpp:446-461
(np.cumsum over float64 adds strictly in order).  The GPU kernels are checked
against the oracle in tests/test_gpu_mean.py."""
import numpy as np
import pytest

ROUNDS = 6  # kMeanRounds (bmg_internal.h)


def to_f96(x):
    """x * 2^96 as an int, or None when not exact / |x| >= 2^8."""
    u = int(np.float32(x).view(np.uint32))
    e, frac, neg = (u >> 23) & 0xFF, u & 0x7FFFFF, u >> 31
    if e == 0:
        return 0 if frac == 0 else None
    if e >= 127 + 8:
        return None
    m = frac | 0x800000
    if e >= 54:
        mag = m << (e - 54)
    else:
        sh = 54 - e
        if sh >= 24 or m & ((1 << sh) - 1):
            return None
        mag = m >> sh
    return -mag if neg else mag


def fits_double(v):
    a = abs(v)
    if a == 0:
        return True
    top, bot = a.bit_length() - 1, (a & -a).bit_length() - 1
    return top - bot <= 52


def round53(v):
    a = abs(v)
    if a == 0:
        return 0
    sh = a.bit_length() - 53
    if sh > 0:
        q, rem, half = a >> sh, a & ((1 << sh) - 1), 1 << (sh - 1)
        if rem > half or (rem == half and q & 1):
            q += 1
        a = q << sh
    return -a if v < 0 else a


def model_channel(xs):
    """Final chain accumulator of one channel (as F96 int), or None = chain fallback."""
    f = [to_f96(x) for x in xs]
    if any(v is None for v in f):
        return None
    prefix = np.cumsum(np.array(f, dtype=object)) if f else []
    delta, k_start = 0, 0
    for _ in range(ROUNDS):
        event = next((k for k in range(k_start, len(f)) if not fits_double(prefix[k] + delta)), None)
        if event is None:
            return (prefix[-1] if len(f) else 0) + delta
        delta = round53(prefix[event] + delta) - prefix[event]
        k_start = event + 1
    return None


def chain(xs):
    return float(np.cumsum(np.asarray(xs, np.float32).astype(np.float64))[-1]) if len(xs) else 0.0


def check(xs, expect_fallback=False, allow_fallback=False):
    got = model_channel(xs)
    if expect_fallback:
        assert got is None
        return
    if got is None and allow_fallback:
        return
    assert got is not None
    # the accumulator fits a double exactly: compare as such
    assert fits_double(got)
    assert float(got) / 2 ** 96 == chain(xs)


def test_random_unit_descriptor_channels():
    rng = np.random.default_rng(5)
    d = rng.standard_normal((3000, 8)).astype(np.float32)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    for c in range(8):
        check(d[:, c])


def test_rounding_steps_are_replayed():
    # 1.0 then k additions of 2^-54 (each rounds back to 1.0), ties to even
    for k in range(0, ROUNDS):
        check([1.0] + [2.0 ** -54] * k)
    check([1.0, 2.0 ** -52, 2.0 ** -53, 3.0, 2.0 ** -53, -4.0, 2.0 ** -60])
    check([1.5, 2.0 ** -53, 2.0 ** -53])          # tie, even stays
    check([1.0 + 2.0 ** -23, 2.0 ** -53])           # float32 input values only
    check([200.0, 2.0 ** -50, -200.0, 2.0 ** -50])


def test_too_many_rounding_steps_fall_back():
    check([1.0] + [2.0 ** -54] * (ROUNDS + 3), expect_fallback=True)


def test_out_of_range_values_fall_back():
    check([1.0, 300.0], expect_fallback=True)       # |x| >= 2^8
    check([1.0, 1e-40], expect_fallback=True)       # subnormal
    check([1.0, 1e-30], expect_fallback=True)       # lowest bit below 2^-96
    check([1.0, 2.0 ** -80, -1.0])                 # in range


@pytest.mark.parametrize("seed", range(8))
def test_random_magnitudes(seed):
    # wide exponent spreads round often: exact or (correctly) handed to the chain
    rng = np.random.default_rng(seed)
    n = [30, 300, 4000, 4000][seed % 4]
    xs = (rng.standard_normal(n) * np.exp2(rng.integers(-30, 6, n))).astype(np.float32)
    check(xs, allow_fallback=True)
