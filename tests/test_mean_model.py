"""CPU model of the exact parallel row mean (kernels.cu K1, mean_* kernels):
F96 fixed-point prefix sums plus the FP64 chain's rounding steps.  Checks the
algorithm itself -- on random and adversarial sequences, in plain Python
integers -- against the literal sequential chain of engine.cpp:446-461
(np.cumsum over float64 adds strictly in order).  The GPU kernels are checked
against the oracle in tests/test_gpu_mean.py."""
import numpy as np
import pytest

TILE = 128      # kCodesTile: descriptors per tile of the F96 tile sums
MAX_WALKS = 1024  # kMeanMaxWalks (kernels.cu)


def to_f96(x):
    """x * 2^96 as an int, or None when not exact / |x| >= 2^7."""
    u = int(np.float32(x).view(np.uint32))
    e, frac, neg = (u >> 23) & 0xFF, u & 0x7FFFFF, u >> 31
    if e == 0:
        return 0 if frac == 0 else None
    if e >= 127 + 7:
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


def low_bit(v):
    return (abs(v) & -abs(v)).bit_length() - 1


def certified(v, rng, lowx):
    """kernels.cu tile_certified: every partial sum of the tile is a multiple
    of 2^low inside [v + lo, v + hi]."""
    if lowx is None:
        return True
    low = lowx if v == 0 else min(lowx, low_bit(v))
    m = max(abs(v + rng[0]), abs(v + rng[1]))
    return m == 0 or m.bit_length() - 1 - low <= 52


def partial_range(t):
    lo = hi = run = 0
    for v in t:
        run += v
        lo, hi = min(lo, run), max(hi, run)
    return lo, hi


def model_channel(xs, tile=TILE, stats=None):
    """Final chain accumulator of one channel (as F96 int), or None = chain
    fallback: tile sums -> exclusive prefix -> certify tiles against the
    current delta -> walk the first uncertified tile, replaying its rounding
    steps -> resume after it (mean_sums / mean_resolve)."""
    f = [to_f96(x) for x in xs]
    if any(v is None for v in f):
        return None
    tiles = [f[i:i + tile] for i in range(0, len(f), tile)]
    sums = [sum(t) for t in tiles]
    rngs = [partial_range(t) for t in tiles]
    lows = [min((low_bit(v) for v in t if v), default=None) for t in tiles]
    prefix, run = [], 0
    for s_ in sums:
        prefix.append(run)
        run += s_
    delta, cur, walked = 0, 0, 0
    while True:
        fail = next((t for t in range(cur, len(tiles))
                     if not certified(prefix[t] + delta, rngs[t], lows[t])), None)
        if fail is None:
            break
        if walked >= MAX_WALKS:
            return None
        S = prefix[fail]
        for v in tiles[fail]:
            S += v
            if not fits_double(S + delta):
                delta = round53(S + delta) - S
        cur, walked = fail + 1, walked + 1
    if stats is not None:
        stats["walked"] = walked
    return run + delta


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
    for k in range(0, 300, 7):
        check([1.0] + [2.0 ** -54] * k)
    check([1.0, 2.0 ** -52, 2.0 ** -53, 3.0, 2.0 ** -53, -4.0, 2.0 ** -60])
    check([1.5, 2.0 ** -53, 2.0 ** -53])          # tie, even stays
    check([1.0 + 2.0 ** -23, 2.0 ** -53])           # float32 input values only
    check([100.0, 2.0 ** -50, -100.0, 2.0 ** -50])


def test_rounding_steps_spread_over_tiles():
    # events in many tiles: each uncertified tile is walked once
    xs = []
    for t in range(40):
        xs += [1.0 if t == 0 else 0.25] + [2.0 ** -54] * 3 + [0.0] * 124
    stats = {}
    check(xs)
    model_channel(xs, stats=stats)
    assert stats["walked"] >= 39


def test_certificate_skips_clean_tiles():
    rng = np.random.default_rng(9)
    xs = (np.round(rng.standard_normal(5000) * 512) / 512).astype(np.float32)
    stats = {}
    check(xs)
    model_channel(xs, stats=stats)
    assert stats["walked"] == 0


def test_small_tiles_match_the_chain():
    rng = np.random.default_rng(11)
    xs = (rng.standard_normal(600) * np.exp2(rng.integers(-40, 3, 600))).astype(np.float32)
    for tile in (1, 3, 32, 128):
        got = model_channel(xs, tile=tile)
        assert got is not None and float(got) / 2 ** 96 == chain(xs)


def test_too_many_uncertified_tiles_fall_back():
    xs = []
    for t in range(MAX_WALKS + 5):
        xs += [1.0, 2.0 ** -54]
    assert model_channel(xs, tile=2) is None


def test_out_of_range_values_fall_back():
    check([1.0, 300.0], expect_fallback=True)       # |x| >= 2^7
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
