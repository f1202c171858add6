"""Pins for the oracle's PRNG layer (reading R-O17; the paper only says
"pseudo-random number generator", and "predetermined pseudo-random
sequence")."""
import numpy as np
import pytest

import oracle as O
from oracle import literal as L

# Random123 known-answer vectors for philox4x32_10 (kat_vectors, Salmon et al. SC'11)
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_kat(ctr, key, want):
    assert tuple(int(x) for x in O.philox4x32_10(ctr, key)) == want


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_literal_philox_kat(ctr, key, want):
    assert tuple(L.philox(ctr, key)) == want


def test_splitmix64_reference_stream():
    # Vigna's splitmix64 seeded with 0: first outputs (state += golden, then mix)
    assert O.splitmix64(0) == 0xE220A8397B1DCDAF
    assert O.splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4
    assert L.splitmix64(0) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("n", list(range(1, 131)) + [255, 256, 257, 1000, 1023, 1024, 1025, 4095, 4096])
def test_perm_is_bijection(n):
    for seed in (1, 2, 0x2511137240000001):
        K = O.key(seed, 2, 1, 0)
        img = sorted(O.perm(K, n, x) for x in range(n))
        assert img == list(range(n))


def test_perm_matches_literal_and_is_keyed():
    for n in (2, 3, 17, 64, 1000, 5000, 1 << 20, 1_281_167, 14_197_122):
        K = O.key(7, 3, 2, 5, 1)
        xs = [0, 1, n // 2, n - 1] + [int(v) % n for v in (12345, 999_999, 7_777_777)]
        for x in xs:
            assert O.perm(K, n, x) == L.perm(K, n, x)
    # distinct keys give distinct permutations; not the identity
    n = 1000
    p1 = [O.perm(O.key(1, 2, 0, 0), n, x) for x in range(n)]
    p2 = [O.perm(O.key(1, 2, 0, 1), n, x) for x in range(n)]
    assert p1 != p2 and p1 != list(range(n))
    # fixed points of a random permutation: ~Poisson(1)
    assert sum(1 for x in range(n) if p1[x] == x) < 10


def test_perm_uniformity_first_position():
    # the first request of an epoch is uniform over [0,n): chi-square over keys
    n, trials = 16, 8000
    counts = np.zeros(n)
    for t in range(trials):
        counts[O.perm(O.key(t, 2, 0, 0), n, 0)] += 1
    chi2 = ((counts - trials / n) ** 2 / (trials / n)).sum()
    assert chi2 < 45  # df = 15, p ~ 1e-4


def test_key_domain_separation():
    seen = set()
    for purpose in (1, 2, 3, 4):
        for a in range(4):
            for b in range(4):
                for c in range(4):
                    seen.add(O.key(11, purpose, a, b, c))
    assert len(seen) == 4 * 4 * 4 * 4
    assert O.key(11, 2, 1, 3, 0) == L.key(11, 2, 1, 3, 0)
