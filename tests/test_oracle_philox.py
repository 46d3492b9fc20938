"""Pins for oracle O1 (Philox4x32-10 + unif mapping).  CPU only."""
import os

import numpy as np

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def test_philox_known_answers():
    rows = [l.split() for l in open(GOLDEN) if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        out = oracle.philox(v[:4], v[4:6])
        assert [int(x) for x in out] == v[6:], r


def test_philox_counter_sensitivity():
    # every counter word and key word changes the output (no dropped input)
    base = oracle.philox([1, 2, 3, 4], [5, 6])
    for i in range(4):
        c = [1, 2, 3, 4]
        c[i] ^= 1
        assert not np.array_equal(oracle.philox(c, [5, 6]), base)
    for i in range(2):
        k = [5, 6]
        k[i] ^= 1
        assert not np.array_equal(oracle.philox([1, 2, 3, 4], k), base)


def test_mulhi64_closed_forms():
    rng = np.random.default_rng(0)
    for _ in range(200):
        r = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        # n = 2^k: floor(r * 2^k / 2^64) = top k bits of r
        for k in (0, 1, 7, 31, 48, 63):
            assert oracle.mulhi64(r, 1 << k) == r >> (64 - k)
        n = int(rng.integers(1, 2**49))
        # exact integer definition floor(r*n / 2^64)
        assert oracle.mulhi64(r, n) == (r * n) >> 64
        assert 0 <= oracle.mulhi64(r, n) < n
    assert oracle.mulhi64(2**64 - 1, 12345) == 12344
    assert oracle.mulhi64(0, 12345) == 0
