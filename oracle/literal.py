"""oracle.literal -- TEST INFRASTRUCTURE ONLY.

A second, deliberately literal transcription of the ODS protocol (§5.2,
P:L669-711, readings R-O1..R-O20 of DESIGN.md §3) in pure Python: Python ints
for the PRNG, Python sets for seen / consumer sets, pools materialised as sorted
lists and indexed by rank exactly as "pool_t[sigma(u)]" reads.  It shares no
code with oracle.c; agreement of the two on thousands of random tiny configs is
the pin for the C oracle's exact decisions.  Only for tiny N.
"""
from __future__ import annotations

import math

M32 = 0xFFFFFFFF
M64 = 0xFFFFFFFFFFFFFFFF
S, E, D, A, SUBST = 0, 1, 2, 3, 4


def philox(ctr, key):
    c = list(ctr)
    k0, k1 = key
    for rnd in range(10):
        if rnd:
            k0 = (k0 + 0x9E3779B9) & M32
            k1 = (k1 + 0xBB67AE85) & M32
        p0 = 0xD2511F53 * c[0]
        p1 = 0xCD9E8D57 * c[2]
        c = [((p1 >> 32) ^ c[1] ^ k0) & M32, p1 & M32, ((p0 >> 32) ^ c[3] ^ k1) & M32, p0 & M32]
    return c


def splitmix64(x):
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def key(seed, purpose, a=0, b=0, c=0):
    return splitmix64(seed ^ splitmix64(((purpose << 56) ^ (a << 48) ^ (c << 44) ^ b) & M64))


def perm(K, n, x):
    if n <= 1:
        return 0
    a = math.isqrt(n - 1) + 1          # ceil(sqrt(n))
    b = -(-n // a)
    kk = (K & M32, K >> 32)
    while True:
        left, right = divmod(x, b)
        for rd in range(12 if n < 64 else 4):       # R-O17: more rounds on small domains
            if rd % 2 == 0:
                left = (left + ((philox((right, rd, 0, 0), kk)[0] * a) >> 32)) % a
            else:
                right = (right + ((philox((left, rd, 0, 0), kk)[0] * b) >> 32)) % b
        x = left * b + right
        if x < n:
            return x


class LiteralODS:
    """evict_all: SURVEY 8c.3 "evict_tiers = ALL" as read in DESIGN.md R-O21:
    consumer sets for every cached source, every cached tier evictable, refills
    tier by tier A -> D -> E from one keyed rank stream over the round-start
    storage pool."""

    def __init__(self, n_total, batch, target, cap_e, cap_d, cap_a, seed, evict_all=False, baseline=False,
                 arrival=None, cold=False):
        self.N, self.batch, self.target = n_total, list(batch), list(target)
        self.J = len(batch)
        self.cap_a, self.seed = cap_a, seed
        self.cap = {A: cap_a, D: cap_d, E: cap_e}
        self.evict_all = evict_all
        self.cached = (A, D, E) if evict_all else (A,)        # tiers with consumer sets / eviction
        self.baseline = baseline                              # R-O22: no substitution, no eviction
        if baseline:
            self.cached = ()
        self.tier = [S] * n_total
        iota = [perm(key(seed, 1), n_total, p) for p in range(cap_a + cap_d + cap_e)]
        for p, i in enumerate(iota):
            self.tier[i] = A if p < cap_a else (D if p < cap_a + cap_d else E)
        self.cold, self.warm = cold, not cold                 # R-O24: empty tiers, admission until full
        if cold:
            self.tier = [S] * n_total
        self.seen = [set() for _ in range(self.J)]
        self.cons = [set() for _ in range(self.J)]
        self.c = [0] * self.J
        self.e = [0] * self.J
        self.n = [0] * self.J
        self.arrival = list(arrival) if arrival is not None else [0] * self.J   # R-O23
        self.pending = [a > 0 for a in self.arrival]
        self.active = [not p for p in self.pending]
        self.r = 0
        self.deliveries = [[[] for _ in range(max(target))] for _ in range(self.J)]  # (id, src)
        self.evicted = 0
        self.refilled = 0

    def pool(self, t, j):
        if t == S:
            return [i for i in range(self.N) if self.tier[i] == S]
        return [i for i in range(self.N)
                if self.tier[i] == t and i not in self.seen[j] and (t != A or i not in self.cons[j])]

    def arrive(self):
        for j in range(self.J):
            if self.pending[j] and self.arrival[j] <= self.r:
                self.pending[j], self.active[j] = False, True

    def round(self, jobs):
        self.arrive()
        departing = set()
        a_served = []
        fetched = {}
        for j in jobs:
            need = min(self.batch[j], self.N - self.n[j])
            K = key(self.seed, 2, j, self.e[j])
            req, pos, last = [], self.c[j], self.c[j]
            while len(req) < need:
                i = perm(K, self.N, pos)
                if i not in self.seen[j]:
                    req.append(i)
                    last = pos
                pos = (pos + 1) % self.N
            self.c[j] = (last + 1) % self.N
            out, src, misses = [None] * need, [None] * need, []
            for s, i in enumerate(req):
                t = self.tier[i]
                if t in (E, D) or (t == A and (self.baseline or i not in self.cons[j])):
                    out[s], src[s] = i, t
                    self.seen[j].add(i)
                else:
                    misses.append(s)
            q = 0
            for t in (() if self.baseline else (A, D, E)):
                if q == len(misses):
                    break
                pool = self.pool(t, j)
                k = min(len(misses) - q, len(pool))
                if k == 0:
                    continue
                Ks = key(self.seed, 3, j, self.r, t)
                for u in range(k):
                    out[misses[q + u]] = pool[perm(Ks, len(pool), u)]
                    src[misses[q + u]] = t | SUBST
                q += k
            for s in misses[q:]:
                out[s], src[s] = req[s], S
            for s in range(need):
                self.seen[j].add(out[s])
                if src[s] & 3 in self.cached:
                    self.cons[j].add(out[s])
                    a_served.append(out[s])
                if src[s] == S and not self.warm:
                    fetched.setdefault(j, []).append(out[s])
                self.deliveries[j][self.e[j]].append((out[s], src[s]))
            self.n[j] += need
            if self.n[j] == self.N:
                self.seen[j] = set()
                self.e[j] += 1
                self.c[j] = 0
                self.n[j] = 0
                if self.e[j] == self.target[j]:
                    departing.add(j)
        changed = bool(departing)
        for j in departing:
            self.active[j] = False
        if any(self.active):
            cand = (sorted(i for i in range(self.N) if self.tier[i] in self.cached) if changed
                    else sorted(set(a_served)))
            evict = [i for i in cand if self.tier[i] in self.cached and
                     all(i in self.cons[a] for a in range(self.J) if self.active[a])]
            admit = not self.warm
            deficit = {}
            for t in (A, D, E):
                size = sum(1 for x in self.tier if x == t) - sum(1 for i in evict if self.tier[i] == t)
                deficit[t] = self.cap[t] - size if (t in self.cached or admit) else 0
            want = deficit[A] + deficit[D] + deficit[E]
            if admit:                                        # R-O24: this round's storage fetches
                fill = []
                for j in sorted(fetched):
                    for i in fetched[j]:
                        if self.tier[i] == S and i not in fill and len(fill) < want:
                            fill.append(i)
                k = len(fill)
            else:
                pool_s = self.pool(S, 0)
                k = min(want, len(pool_s))
                Kr = key(self.seed, 4, 0, self.r)
                fill = [pool_s[perm(Kr, len(pool_s), u)] for u in range(k)]
            dest = []
            for t in (A, D, E):                              # tier by tier from one rank stream
                dest += [t] * min(deficit[t], k - len(dest))
            for i in evict:
                self.tier[i] = S
                for a in range(self.J):
                    self.cons[a].discard(i)
            for i, t in zip(fill, dest):
                self.tier[i] = t
            if admit and all(sum(1 for x in self.tier if x == t) == self.cap[t] for t in (A, D, E)):
                self.warm = True
            self.evicted += len(evict)
            self.refilled += k
        self.r += 1

    def replay_all(self):
        while any(self.active) or any(self.pending):
            self.arrive()
            if not any(self.active):
                self.r += 1                                    # idle round (R-O23)
                continue
            self.round([j for j in range(self.J) if self.active[j]])
