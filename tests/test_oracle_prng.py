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


def _bijection_keys(keys):
    """Worker: every n <= 4096 under each key in `keys`; returns the failures."""
    bad = []
    for k in keys:
        K = O.key(0x5EED + k, 2, k % 32, k)
        for n in range(1, 4097):
            img = O.perm_block(K, n)
            if not np.array_equal(np.bincount(img, minlength=n), np.ones(n, np.int64)):
                bad.append((k, n))
    return bad


def test_perm_is_bijection_exhaustive_4096_x_100_keys():
    """perm(K, n, .) is a bijection of [0, n) for EVERY n <= 4096
    under 100 keys (839 M evaluations of the oracle's perm, one process per core)."""
    import multiprocessing as mp
    import os
    cores = max(1, min(16, len(os.sched_getaffinity(0))))
    chunks = [list(range(k, 100, cores)) for k in range(cores)]
    with mp.get_context("fork").Pool(cores) as pool:
        bad = sum(pool.map(_bijection_keys, chunks), [])
    assert bad == []


def _chi2_bound(df, p=1e-6):
    from scipy.stats import chi2
    return chi2.ppf(1.0 - p, df)


def _binned(values, n, bins):
    """Counts of values in `bins` near-equal bins of [0, n) and each bin's size."""
    edges = (np.arange(bins + 1) * n) // bins
    idx = np.searchsorted(edges, values, side="right") - 1
    return np.bincount(idx, minlength=bins), np.diff(edges)


# non-square domains with cycle walking (a*b > n) and a pool size near the
# kernel's largest (ImageNet-22K's 4.38 M E pool)
WALKED = [5, 17, 1000, 65537, 4_376_846]


@pytest.mark.parametrize("n", WALKED)
def test_perm_positions_uniform_over_keys(n):
    """For each of the first 8 positions x, pi_K(x) over 12,000 keys (keys as the
    replay derives them: purpose SUB, job, round, tier) is uniform on [0, n):
    chi-square over min(n, 64) near-equal bins, p > 1e-6 for every position."""
    a = int(np.ceil(np.sqrt(n)))
    b = -(-n // a)
    assert n in (5, 17) or a * b > n          # the sizes really walk
    T = 12_000
    X = min(8, n)
    vals = np.stack([O.perm_block(O.key(7, 3, t % 8, t // 8, 1 + t % 3), n, 0, X) for t in range(T)])
    assert vals.max() < n
    bins = min(n, 64)
    for x in range(X):
        cnt, size = _binned(vals[:, x], n, bins)
        exp = T * size / n
        chi2 = float(((cnt - exp) ** 2 / exp).sum())
        assert chi2 < _chi2_bound(bins - 1), (n, x, chi2)


@pytest.mark.parametrize("n", [5, 17, 63, 64, 1000])
def test_perm_pairs_uniform_over_keys(n):
    """(pi_K(0), pi_K(1)) over 20,000 keys is uniform over the ordered pairs of
    distinct values (exact expected counts per bin pair, the diagonal depleted
    because pi is injective): chi-square, p > 1e-6."""
    T = 20_000
    vals = np.stack([O.perm_block(O.key(11, 3, 1, t, 2), n, 0, 2) for t in range(T)]).astype(np.int64)
    assert np.all(vals[:, 0] != vals[:, 1])
    bins = min(n, 16)
    edges = (np.arange(bins + 1) * n) // bins
    size = np.diff(edges).astype(np.float64)
    i = np.searchsorted(edges, vals[:, 0], side="right") - 1
    j = np.searchsorted(edges, vals[:, 1], side="right") - 1
    cnt = np.bincount(i * bins + j, minlength=bins * bins).reshape(bins, bins)
    exp = np.outer(size, size)
    exp[np.diag_indices(bins)] = size * (size - 1)
    exp *= T / (n * (n - 1))
    keep = exp > 0
    chi2 = float(((cnt[keep] - exp[keep]) ** 2 / exp[keep]).sum())
    assert chi2 < _chi2_bound(int(keep.sum()) - 1), (n, chi2)


@pytest.mark.parametrize("P,k", [(1000, 37), (65537, 300), (4_376_846, 354)])
def test_substitute_ranks_uniform(P, k):
    """Substitution (R-O2) takes pool[sigma(u)], u < k, sigma = perm(key(seed, SUB,
    j, r, t), P, .): over many rounds every pool rank is chosen with probability
    k / P -- chi-square of the chosen ranks over 64 bins, and the k ranks of one
    round are distinct (sampling without replacement)."""
    rounds = max(400, 400_000 // k)
    chosen = []
    for r in range(rounds):
        s = O.perm_block(O.key(0x2511, 3, r % 8, r, 1), P, 0, k)
        assert len(np.unique(s)) == k
        chosen.append(s)
    chosen = np.concatenate(chosen)
    cnt, size = _binned(chosen, P, 64)
    exp = rounds * k * size / P
    chi2 = float(((cnt - exp) ** 2 / exp).sum())
    assert chi2 < _chi2_bound(63), chi2


def test_perm_single_key_looks_random_at_pool_scale():
    """One key, n = 4,376,846 (the 22K E pool): 200,000 consecutive positions are
    uniform over 256 bins, about half are ascents (pi(x+1) > pi(x)), and lag-1
    values are uncorrelated (|rho| < 0.01) -- no structure from the Z_a x Z_b
    Feistel leaks into a job's request stream."""
    n = 4_376_846
    v = O.perm_block(O.key(3, 2, 5, 1), n, 0, 200_000).astype(np.float64)
    cnt, size = _binned(v.astype(np.int64), n, 256)
    exp = len(v) * size / n
    assert float(((cnt - exp) ** 2 / exp).sum()) < _chi2_bound(255)
    asc = float(np.mean(v[1:] > v[:-1]))
    assert abs(asc - 0.5) < 0.006
    rho = float(np.corrcoef(v[1:], v[:-1])[0, 1])
    assert abs(rho) < 0.01


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
