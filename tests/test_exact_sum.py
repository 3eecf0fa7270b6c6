"""The exactness test behind the tree-split modes (csrc/ts_stream.cu
split_sum_exact / amax_bound), restated in numpy and checked on the CPU: when
it holds for a row's terms, the f64 sum of those terms is the same in every
order -- so the splits' own sums add up to the reference's tree-order sum (ref
evaluators.py:529-535) -- and when the terms do round it must not hold.

The restatement follows the device code line by line: terms are fp32 leaf
values (unit weights); each split reports its sequential sum, the high word of
its largest |running sum| and its smallest nonzero |leaf| bit pattern minus 1.
"""
import numpy as np
import pytest


def _hi(x: float) -> int:
    return int(np.float64(x).view(np.uint64) >> np.uint64(32)) & 0x7FFFFFFF


def _amax_bound(amax: int) -> float:
    if amax >= 0x7FE00000:
        return float("inf")
    return float(np.uint64((amax + 1) << 32).view(np.float64))


def _split_partials(terms32, cuts):
    """(sum, amax, kmin1) of every split, as k_stream's ORD = 2 walk keeps them."""
    out = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        acc, amax, kmin1 = np.float64(0.0), 0, 0xFFFFFFFF
        for v in terms32[a:b]:
            acc = acc + np.float64(v)
            amax = max(amax, _hi(acc))
            key = int(np.float32(v).view(np.uint32)) & 0x7FFFFFFF
            kmin1 = min(kmin1, (key - 1) & 0xFFFFFFFF)
        out.append((acc, amax, kmin1))
    return out


def _split_sum_exact(M: float, kmin1: int, acc0: float) -> bool:
    if kmin1 == 0xFFFFFFFF:
        return not (acc0 == 0.0 and np.signbit(acc0)) and M < float("inf")
    q = max(((kmin1 + 1) & 0xFFFFFFFF) >> 23, 1) - 150
    if acc0 != 0.0:
        b = int(np.float64(acc0).view(np.uint64))
        ea = (b >> 52) & 0x7FF
        if ea == 0 or ea == 0x7FF:
            return False
        mant = (b & 0xFFFFFFFFFFFFF) | (1 << 52)
        q = min(q, ea - 1075 + ((mant & -mant).bit_length() - 1))
    elif np.signbit(acc0):
        return False
    Mt = M + abs(acc0)
    if not Mt < float("inf"):
        return False
    em = (int(np.float64(Mt).view(np.uint64)) >> 52) & 0x7FF
    return (em - 1022 + 1) - q <= 53


def _verdict(terms32, cuts, acc0):
    parts = _split_partials(terms32, cuts)
    M = sum(_amax_bound(a) for _s, a, _k in parts)
    kmin1 = min(k for _s, _a, k in parts)
    fast = np.float64(acc0)
    total = np.float64(0.0)
    for s, _a, _k in parts:
        total = total + s
    return _split_sum_exact(M, kmin1, acc0), fast + total


def _sequential(terms32, acc0):
    acc = np.float64(acc0)
    for v in terms32:
        acc = acc + np.float64(v)
    return acc


def _cuts(rng, n):
    k = int(rng.integers(1, 9))
    inner = np.sort(rng.choice(np.arange(1, n), size=min(k - 1, n - 1), replace=False)) if n > 1 else []
    return [0, *[int(c) for c in inner], n]


@pytest.mark.parametrize("seed", range(60))
def test_exact_verdict_means_order_free(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 400))
    kind = seed % 4
    if kind == 0:
        t = rng.standard_normal(n) * 0.1
    elif kind == 1:
        t = rng.standard_normal(n) * 10.0 ** rng.uniform(-12, 3, n)
    elif kind == 2:
        t = rng.choice(np.array([0.0, -0.0, 1e-45, -3e-42, 0.25, -1.5, 3.0]), n)
    else:
        t = rng.integers(-1000, 1000, n) * 2.0 ** -int(rng.integers(0, 30))
    t32 = t.astype(np.float32)
    acc0 = float(rng.choice([0.0, 0.375, float(np.float32(rng.standard_normal())), 1e-7]))
    ok, fast = _verdict(t32, _cuts(rng, n), acc0)
    seq = _sequential(t32, acc0)
    if ok:
        assert fast.view(np.uint64) == seq.view(np.uint64)
        # and any other order gives the same bits
        for _ in range(3):
            perm = rng.permutation(n)
            assert _sequential(t32[perm], acc0).view(np.uint64) == seq.view(np.uint64)


def test_rounding_sums_are_refused():
    """A term whose bits fall below the running sum's ulp makes the sum
    order-dependent: the verdict must be 'not exact'."""
    t32 = np.array([1.0, 2.0 ** -60, -1.0, 2.0 ** -60] * 8, np.float32)
    a = _sequential(t32, 0.0)
    b = _sequential(np.sort(t32), 0.0)
    assert a != b  # the order does matter here
    for cuts in ([0, len(t32)], [0, 5, 17, len(t32)]):
        ok, _ = _verdict(t32, cuts, 0.0)
        assert not ok
    # and signed zeros: -0.0 running sum with all-zero terms is the one zero case refused
    z = np.array([-0.0, 0.0, -0.0], np.float32)
    assert _verdict(z, [0, 3], 0.0)[0]
    assert not _verdict(z, [0, 3], -0.0)[0]


def test_narrow_leaves_pass():
    """Leaves like a trained ensemble's (N(0, 0.1), 1000 trees) pass the test,
    so the fast path is what normally runs."""
    rng = np.random.default_rng(7)
    passed = 0
    for _ in range(50):
        t32 = (rng.standard_normal(1000) * 0.1).astype(np.float32)
        t32[np.abs(t32) < 1e-6] = 0.01
        ok, fast = _verdict(t32, _cuts(rng, 1000), 0.0)
        passed += ok
        if ok:
            assert fast.view(np.uint64) == _sequential(t32, 0.0).view(np.uint64)
    assert passed == 50
