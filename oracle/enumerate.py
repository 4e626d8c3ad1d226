"""Exact enumeration for tiny corpora — TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Independent of the oracle's formulas: the joint p(W, Z, T) is obtained by
brute force from the *generative process*, not from the closed form the
sampler uses.

* Table multiplicities: every seating of a restaurant's customer sequence is
  enumerated with the Chinese-restaurant rule of the Poisson–Dirichlet
  process (§2.4.3): customer n joins an existing table
  with probability (c_s - a)/(b + n), or opens a new table with probability
  (b + a J)/(b + n) and draws its dish from the base H.  Summing seatings by
  per-dish table counts gives p(words, t) = coef(t) * prod_w H(w)^{t_w}.
* The shared base phi0_k ~ Dir(beta) is integrated exactly:
  E[prod_w phi0_kw^{Q_kw}] = prod_w (beta)_{Q_kw} / (V beta)_{T_k}.
* theta_d ~ Dir(alpha) is integrated exactly:
  p(z_d) = prod_k (alpha)_{n_dk} / (K alpha)_{L_d}.

All arithmetic is in Fraction, so p(W, Z, T) is exact.  The tables R (which
customer opened a table) satisfy p(W, Z, R) = p(W, Z, T) / prod C(m, t)
(Eq. SPDP-table-to-head).
"""
from __future__ import annotations

import itertools
from collections import defaultdict
from fractions import Fraction
from math import comb


def rising(x, n, y=1):
    """(x|y)_n = prod_{j<n} (x + j y)."""
    out = Fraction(1)
    for j in range(n):
        out *= x + j * y
    return out


def crp_coefficients(words, a, b):
    """{t: coef} with p(sequence, table multiplicities t) = coef * prod_w H(w)^{t_w},
    by enumerating every seating of the customer sequence.
    t is a tuple of (word, tables) pairs sorted by word."""
    a = Fraction(a); b = Fraction(b)
    out = defaultdict(Fraction)

    def rec(j, tables, prob):
        if j == len(words):
            cnt = defaultdict(int)
            for dish, _ in tables:
                cnt[dish] += 1
            out[tuple(sorted(cnt.items()))] += prob
            return
        w = words[j]
        for s, (dish, c) in enumerate(tables):
            if dish == w:
                nt = list(tables); nt[s] = (dish, c + 1)
                rec(j + 1, nt, prob * (c - a) / (b + j))
        rec(j + 1, tables + [(w, 1)], prob * (b + a * len(tables)) / (b + j))

    rec(0, [], Fraction(1))
    return dict(out)


class TinyCorpus:
    def __init__(self, group, doc, word, num_groups, vocab, num_topics, alpha, beta, a, b):
        self.group, self.doc, self.word = list(group), list(doc), list(word)
        self.I, self.V, self.K = num_groups, vocab, num_topics
        self.alpha, self.beta = Fraction(alpha), Fraction(beta)
        self.a, self.b = Fraction(a), Fraction(b)
        self.N = len(self.word)
        self.D = max(self.doc) + 1
        self._coef_cache = {}

    def cells(self, z):
        """m[(i,w,k)] for assignment z."""
        m = defaultdict(int)
        for p in range(self.N):
            m[(self.group[p], self.word[p], z[p])] += 1
        return dict(m)

    def states(self):
        """Every valid (z, t): z in K^N, and 1 <= t_c <= m_c on every occupied cell."""
        for z in itertools.product(range(self.K), repeat=self.N):
            m = self.cells(z)
            keys = sorted(m)
            for ts in itertools.product(*[range(1, m[c] + 1) for c in keys]):
                yield tuple(z), dict(zip(keys, ts))

    def _restaurant_coef(self, words, t_of_word):
        key = tuple(words)
        if key not in self._coef_cache:
            self._coef_cache[key] = crp_coefficients(words, self.a, self.b)
        return self._coef_cache[key].get(tuple(sorted(t_of_word.items())), Fraction(0))

    def joint_WZT(self, z, t):
        """Exact p(W, Z, T) (sequence probability) by the generative process."""
        K, V = self.K, self.V
        p = Fraction(1)
        # theta integrated: prod_d prod_k (alpha)_{n_dk} / (K alpha)_{L_d}
        for d in range(self.D):
            toks = [q for q in range(self.N) if self.doc[q] == d]
            if not toks:
                continue
            for k in range(K):
                p *= rising(self.alpha, sum(1 for q in toks if z[q] == k))
            p /= rising(K * self.alpha, len(toks))
        # restaurants (i,k): sum over seatings with the given table counts
        Q = defaultdict(int)
        for i in range(self.I):
            for k in range(K):
                words = [self.word[q] for q in range(self.N) if self.group[q] == i and z[q] == k]
                if not words:
                    continue
                tw = {w: t[(i, w, k)] for w in set(words)}
                p *= self._restaurant_coef(words, tw)
                for w, tv in tw.items():
                    Q[(k, w)] += tv
        # phi0 integrated: prod_k prod_w (beta)_{Q_kw} / (V beta)_{T_k}
        for k in range(K):
            Tk = 0
            for w in range(V):
                p *= rising(self.beta, Q[(k, w)])
                Tk += Q[(k, w)]
            p /= rising(V * self.beta, Tk)
        return p

    def joint_WZR_per_T(self, z, t):
        """p(W, Z, R) for any R consistent with T: p(W,Z,T) / prod C(m,t)."""
        m = self.cells(z)
        den = 1
        for c, mv in m.items():
            den *= comb(mv, t[c])
        return self.joint_WZT(z, t) / den

    def posterior(self):
        """{(z, frozen t): exact posterior probability}."""
        w = {}
        for z, t in self.states():
            w[(z, tuple(sorted(t.items())))] = self.joint_WZT(z, t)
        tot = sum(w.values())
        return {s: v / tot for s, v in w.items()}

    def exact_conditional(self, z, t, p, r_rem):
        """Exact normalised blocked conditional of (z_p, r_p) (2K slots, j=2k <-> r=1)
        after removing token p with indicator r_rem, as ratios of p(W, Z, R)."""
        i, w, k0 = self.group[p], self.word[p], z[p]
        tm = dict(t)
        tm[(i, w, k0)] -= r_rem
        out = []
        for k in range(self.K):
            for r in (1, 0):
                z2 = list(z); z2[p] = k
                t2 = dict(tm)
                c = (i, w, k)
                t2[c] = t2.get(c, 0) + r
                m2 = self.cells(z2)
                t2 = {cc: v for cc, v in t2.items() if cc in m2}
                ok = all(1 <= t2.get(cc, 0) <= m2[cc] for cc in m2)
                out.append(self.joint_WZR_per_T(tuple(z2), t2) if ok else Fraction(0))
        tot = sum(out)
        return [v / tot for v in out]


def multinomial(n, parts):
    out = Fraction(1)
    rest = n
    for x in parts:
        out *= comb(rest, x)
        rest -= x
    return out


class TinyCorpusP(TinyCorpus):
    """NEXT-4: the same brute force with a transformation matrix P^i per group
    (PAPER.md:985-1014): a table of restaurant (i,k) serving word w takes its
    dish through a source word v with probability p_{i,w,v} phi0_{k,v}
    (P^i phi0 is the base of the group's PDP).  Expanding
    H(w)^{t_w} = (sum_v p_wv phi0_v)^{t_w} over the tables' sources gives, for
    source counts q (sum_v q_v = t_w), multinomial(t_w; q) prod_v (p_wv phi0_v)^{q_v};
    phi0 is integrated exactly as before with Q_kv = sum_{i,w} q_{ikwv}.
    P: {(i, w): [(v, p), ...]} (entries in the sampler's order)."""

    def __init__(self, *args, P=None, **kw):
        super().__init__(*args, **kw)
        self.P = {key: [(v, Fraction(p)) for v, p in ent] for key, ent in P.items()}

    def states_q(self):
        """Every valid (z, t, q): q[(i,w,k)] a tuple of per-entry source counts summing to t."""
        for z, t in self.states():
            keys = sorted(t)
            splits = []
            for c in keys:
                i, w, k = c
                S = len(self.P[(i, w)])
                splits.append([q for q in itertools.product(range(t[c] + 1), repeat=S) if sum(q) == t[c]])
            for qs in itertools.product(*splits):
                yield z, t, dict(zip(keys, qs))

    def joint_WZTQ(self, z, t, q):
        K, V = self.K, self.V
        p = Fraction(1)
        for d in range(self.D):
            toks = [x for x in range(self.N) if self.doc[x] == d]
            if not toks:
                continue
            for k in range(K):
                p *= rising(self.alpha, sum(1 for x in toks if z[x] == k))
            p /= rising(K * self.alpha, len(toks))
        Q = defaultdict(int)
        for i in range(self.I):
            for k in range(K):
                words = [self.word[x] for x in range(self.N) if self.group[x] == i and z[x] == k]
                if not words:
                    continue
                tw = {w: t[(i, w, k)] for w in set(words)}
                p *= self._restaurant_coef(words, tw)
                for w in set(words):
                    qc = q[(i, w, k)]
                    p *= multinomial(t[(i, w, k)], qc)
                    for (v, pv), qv in zip(self.P[(i, w)], qc):
                        p *= pv ** qv
                        Q[(k, v)] += qv
        for k in range(K):
            Tk = 0
            for v in range(V):
                p *= rising(self.beta, Q[(k, v)])
                Tk += Q[(k, v)]
            p /= rising(V * self.beta, Tk)
        return p

    def joint_WZRV(self, z, t, q):
        """p(W, Z, R, V) for any table-creator and per-table source assignment consistent
        with (T, Q): p(W, Z, T, Q) / prod_cells C(m, t) multinomial(t; q)."""
        m = self.cells(z)
        den = Fraction(1)
        for c, mv in m.items():
            den *= comb(mv, t[c]) * multinomial(t[c], q[c])
        return self.joint_WZTQ(z, t, q) / den

    def posterior_q(self):
        w = {}
        for z, t, q in self.states_q():
            w[(z, tuple(sorted(q.items())))] = self.joint_WZTQ(z, t, q)
        tot = sum(w.values())
        return {s: v / tot for s, v in w.items()}

    def exact_conditional_q(self, z, t, q, p, r_rem, e_rem):
        """Exact normalised conditional of (z_p, r_p, source) after removing token p
        (its table with source entry e_rem when r_rem): slots k (S+1) + e (r = 1, entry e),
        k (S+1) + S (r = 0), as ratios of p(W, Z, R, V)."""
        i, w, k0 = self.group[p], self.word[p], z[p]
        S = len(self.P[(i, w)])
        tm, qm = dict(t), dict(q)
        if r_rem:
            tm[(i, w, k0)] -= 1
            qq = list(qm[(i, w, k0)]); qq[e_rem] -= 1; qm[(i, w, k0)] = tuple(qq)
        out = []
        for k in range(self.K):
            for slot in range(S + 1):
                r = slot < S
                z2 = list(z); z2[p] = k
                t2, q2 = dict(tm), dict(qm)
                c = (i, w, k)
                if c not in q2:
                    q2[c] = (0,) * S
                    t2[c] = 0
                if r:
                    t2[c] += 1
                    qq = list(q2[c]); qq[slot] += 1; q2[c] = tuple(qq)
                m2 = self.cells(z2)
                t2 = {cc: v for cc, v in t2.items() if cc in m2}
                q2 = {cc: v for cc, v in q2.items() if cc in m2}
                ok = all(1 <= t2.get(cc, 0) <= m2[cc] for cc in m2) and all(min(v) >= 0 for v in q2.values())
                out.append(self.joint_WZRV(tuple(z2), t2, q2) if ok else Fraction(0))
        tot = sum(out)
        return [v / tot for v in out]
