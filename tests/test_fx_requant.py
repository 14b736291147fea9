"""The exact fixed-point requantization ("FX", k_quant.cu fx_channel / k_conv_tc.cu
epi_chunk16_fx) restated in numpy and checked against the reference's fp64 requantize
(/root/reference/pkg/src/ptqtune/intexec.py:72-85: clip(floor(fl(fl(acc*m) + 0.5)) + zp)).

The construction: S = 31 - e (m_max = f * 2^e, so M_max lies in [2^30, 2^31)), per-channel
thresholds t_k = min{acc : floor(fl(fl(acc*m) + 0.5)) + zy >= k} found with the reference's own fp64 arithmetic, then
M = round(m * 2^S) (+-2) and B = max_k (k*2^S - t_k*M) whenever max - min < M.  Claim: for every
int32 accumulator, clip(floor((acc*M + B) / 2^S), lo, 127) equals the reference.  Checked here
densely around every threshold and on random accumulators over the whole int32 range, for
random multipliers, power-of-two multipliers (exact fp64 ties) and decimal ones.
"""
import math

import numpy as np

QMAX = 127


def ref_codes(acc, m, zy, lo):
    r = np.floor(acc.astype(np.float64) * m + 0.5)           # fl(fl(acc*m) + 0.5) (no FMA)
    return np.clip(r + zy, lo, QMAX).astype(np.int64)


def fx_params(m, zy, lo, S):
    def pred(a, j):
        return math.floor(float(a) * m + 0.5) >= j          # fl(fl(a*m) + 0.5) >= j
    ks, ts = [], []
    for k in range(lo + 1, QMAX + 1):
        j = k - zy
        x0 = (j - 0.5) / m
        if not abs(x0) < 2 ** 30:
            return None
        a = math.ceil(x0)
        while pred(a - 1, j):
            a -= 1
        while not pred(a, j):
            a += 1
        ks.append(k)
        ts.append(a)
    M0 = int(round(math.ldexp(m, S)))
    for d in (0, 1, -1, 2, -2):
        M = M0 + d
        if M <= 0 or M >= 2 ** 31:
            continue
        if not ks:
            return M, 0
        L = [k * (1 << S) - t * M for k, t in zip(ks, ts)]
        if max(L) - min(L) < M:
            return M, max(L)
    return None


def fx_codes(acc, M, B, S, lo):
    X = acc.astype(object) * M + B                            # exact (python ints)
    q = np.array([int(x) >> S for x in X], dtype=np.int64)
    return np.clip(q, lo, QMAX)


def layer_S(m_max):
    _, e = math.frexp(m_max)
    return 31 - e


def check(m, zy, lo, rng, must=True):
    S = layer_S(m)
    assert 32 <= S <= 52
    p = fx_params(m, zy, lo, S)
    if p is None:          # no exact 32-bit (M, B): the layer keeps the fp64 epilogue
        assert not must, (m, zy, lo)
        return False
    M, B = p
    # dense windows around every threshold, the int32 extremes and random accumulators
    centers = [int(math.ceil((k - zy - 0.5) / m)) for k in range(lo + 1, QMAX + 1)]
    acc = [c + d for c in centers for d in range(-3, 4)]
    acc += list(rng.integers(-2 ** 31, 2 ** 31, 2000)) + [-2 ** 31, 2 ** 31 - 1, 0, 1, -1]
    acc = np.asarray(acc, dtype=np.int64)
    acc = acc[(acc >= -2 ** 31) & (acc < 2 ** 31)]
    assert np.array_equal(fx_codes(acc, M, B, S, lo), ref_codes(acc, m, zy, lo)), (m, zy, lo)
    return True


def test_fx_random_multipliers():
    """Exact whenever constants are found; always found for m >= 1e-5 (the multipliers of the
    bench networks are ~1e-4 .. 1e-1); below that the LP may fail and fp64 takes over."""
    rng = np.random.default_rng(0)
    found = 0
    for i in range(150):
        m = float(10.0 ** rng.uniform(-6.5, math.log10(0.49)))
        zy = int(rng.integers(-128, 128))
        lo = -128 if rng.random() < 0.5 else max(-128, zy)
        found += check(m, zy, lo, rng, must=m >= 1e-5)
    assert found > 100


def test_fx_exact_ties_and_decimal_multipliers():
    rng = np.random.default_rng(1)
    for m in [2.0 ** -s for s in range(2, 22)] + [0.1, 0.01, 0.2, 1 / 3, 0.001, 0.05, 0.4999, 3e-5]:
        for zy in (-128, -5, 0, 17, 127):
            check(m, zy, -128, rng)
            check(m, zy, max(-128, zy), rng)


def test_fx_uniform_S_for_smaller_channel_multipliers():
    """Per-channel weights: S comes from the layer's largest multiplier, so smaller channels
    get smaller M.  Constants are always found for the per-channel spreads of weight scales
    (m_max / m <= 3) at m >= 1e-4, and are exact whenever found (wider spreads may fail: the
    layer then keeps the fp64 epilogue)."""
    rng = np.random.default_rng(2)
    for i in range(80):
        m_max = float(10.0 ** rng.uniform(-3.5, math.log10(0.49)))
        S = layer_S(m_max)
        ratio = float(rng.uniform(1.0, 3.0 if i % 2 else 30.0))
        m = m_max / ratio
        zy = int(rng.integers(-128, 128))
        p = fx_params(m, zy, -128, S)
        if p is None:
            assert ratio > 3.0 or m < 1e-4, (m_max, m)
            continue
        M, B = p
        acc = np.concatenate([rng.integers(-2 ** 31, 2 ** 31, 3000),
                              np.arange(-300, 300) + int((0 - zy) / m)]).astype(np.int64)
        assert np.array_equal(fx_codes(acc, M, B, S, -128), ref_codes(acc, m, zy, -128))
