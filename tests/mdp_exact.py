"""Exact-rational brute force for the MDP argmax (test helper, not product).

Independent of oracle.c's argmax loop: the split counts are computed with
Python integers from Eqs. 5-8 read as floor(x S_mem / (M S_data))
(R-M6), Eq. 9 is evaluated in Fractions (no rounding at all) over
the tier throughputs, and the maximum is exact.  Used to pin the FP64 oracle:
its argmax value must be within 1e-12 of the exact maximum, and its index must
equal the exact argmax wherever that maximum is unique by a margin.
"""
from fractions import Fraction


def counts(n, s, cache, m_num, m_den, pe, pd, pa):
    cap_a = (pa * cache * m_den) // (100 * m_num * s)
    cap_d = (pd * cache * m_den) // (100 * m_num * s)
    cap_e = (pe * cache) // (100 * s)
    na = min(n, cap_a)
    nd = min(n - na, cap_d)
    ne = min(n - na - nd, cap_e)
    return na, nd, ne, n - na - nd - ne


def splits(g):
    for pe in range(100, -1, -g):
        for pd in range(100 - pe, -1, -g):
            yield pe, pd, 100 - pe - pd


def exact_values(prof, dsi, g):
    """prof: dict with n_total, s_data, cache_bytes, m_num, m_den; dsi: 4 floats (A,D,E,S)."""
    fa, fd, fe, fs = (Fraction(x) for x in dsi)
    n = prof["n_total"]
    out = []
    for pe, pd, pa in splits(g):
        na, nd, ne, ns = counts(n, prof["s_data"], prof["cache_bytes"], prof["m_num"], prof["m_den"], pe, pd, pa)
        out.append(Fraction(na * fa + nd * fd + ne * fe + ns * fs, n))
    return out
