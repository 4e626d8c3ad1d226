"""Pins of the CPU oracle against what the paper and mathematics fix (CPU only).

Each test names the passage it pins.  None of them re-types the oracle's own
formula: they use published vectors (Philox KAT), closed forms and
identities of the generalised Stirling numbers, brute-force enumeration of
the generative process (oracle/enumerate.py), and exact Markov-chain
stationarity.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle.enumerate import TinyCorpus, crp_coefficients, rising

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                yield line.split()


# --------------------------------------------------------------------------
# RNG (reading c11): Random123 published known-answer vectors
# --------------------------------------------------------------------------
def test_philox_kat():
    n = 0
    for row in _rows("philox4x32_10_kat.txt"):
        v = [int(x, 16) for x in row]
        assert list(oracle.philox(v[0:4], v[4:6])) == v[6:10]
        n += 1
    assert n == 3


# --------------------------------------------------------------------------
# Generalised Stirling numbers
# --------------------------------------------------------------------------
def test_stirling_golden_vectors():
    for a, N, M, val in _rows("stirling_vectors.txt"):
        got = oracle.log_stirling(float(a), int(N), int(M))
        if val == "0":
            assert got == -math.inf
        else:
            assert got == pytest.approx(math.log(float(Fraction(val))), abs=1e-12)


@pytest.mark.parametrize("a", [0.0, 0.3, 0.7, 0.95])
def test_stirling_closed_forms(a):
    for N in [1, 2, 5, 17, 60, 200]:
        # S^N_N = 1
        assert oracle.log_stirling(a, N, N) == pytest.approx(0.0, abs=1e-9)
        # S^N_1 = prod_{j=1}^{N-1} (j - a) = Gamma(N - a) / Gamma(1 - a)
        want = math.lgamma(N - a) - math.lgamma(1 - a)
        assert oracle.log_stirling(a, N, 1) == pytest.approx(want, rel=1e-11, abs=1e-11)
        # S^N_{N-1} = (1 - a) N (N - 1) / 2
        if N >= 2:
            assert oracle.log_stirling(a, N, N - 1) == pytest.approx(math.log((1 - a) * N * (N - 1) / 2), rel=1e-11)
        # S^N_0 = 0 for N >= 1, S^N_M = 0 for M > N
        assert oracle.log_stirling(a, N, 0) == -math.inf
        assert oracle.log_stirling(a, N, N + 1) == -math.inf


def _stirling_explicit(N, M, a):
    """S^N_{M,a} from the explicit alternating sum of generalised Stirling numbers
    (a > 0): S^N_M = 1/(a^M M!) * sum_{j=1}^{M} (-1)^j C(M, j) (-j a)_N with the rising
    factorial (x)_N — a route independent of the recursion P:1454-1455."""
    tot = sum((-1) ** j * math.comb(M, j) * rising(-j * a, N) for j in range(1, M + 1))
    return tot / (a ** M * math.factorial(M))


def test_ratio_table_exact_rationals():
    """A0/A1 (Eqs. r0/r1 P:1683) against exact rationals
    from the explicit Stirling sum, every cell m <= 40 at a = 7/10 and 3/10."""
    for a in (Fraction(7, 10), Fraction(3, 10)):
        mmax = 40
        S = {(N, M): _stirling_explicit(N, M, a) for N in range(0, mmax + 2) for M in range(1, N + 1)}
        A0, A1 = oracle.ratio_table(float(a), mmax)
        assert (A0[0], A1[0]) == (0.0, 1.0)                  # A0(0,0) = 0, A1(0,0) = 1
        for m in range(1, mmax + 1):
            base = m * (m + 1) // 2
            assert (A0[base], A1[base]) == (0.0, 0.0)        # t = 0 < m: not a state
            for t in range(1, m + 1):
                w0 = Fraction(m - t + 1, m + 1) * S[(m + 1, t)] / S[(m, t)]
                w1 = Fraction(t + 1, m + 1) * S[(m + 1, t + 1)] / S[(m, t)]
                assert A0[base + t] == pytest.approx(float(w0), rel=1e-12), (m, t)
                assert A1[base + t] == pytest.approx(float(w1), rel=1e-12), (m, t)


@pytest.mark.parametrize("a", [0.0, 0.7])
def test_ratio_table_closed_forms_to_large_m(a):
    """Closed forms on every row up to m = 5000 (> C5's M_max 4898):
    A1(m,m) = 1, A0(m,m) = (1-a) m / 2, A0(m,1) = m (m - a) / (m + 1); all entries finite, > 0."""
    mmax = 5000
    A0, A1 = oracle.ratio_table(a, mmax)
    m = np.arange(1, mmax + 1)
    base = m * (m + 1) // 2
    np.testing.assert_allclose(A1[base + m], 1.0, rtol=1e-9)
    np.testing.assert_allclose(A0[base + m], (1 - a) * m / 2, rtol=1e-9)
    np.testing.assert_allclose(A0[base + 1], m * (m - a) / (m + 1), rtol=1e-9)
    valid = np.ones_like(A0, bool)
    valid[base] = False
    valid[0] = False                                          # (0, 0): A0 = 0, A1 = 1
    assert (A0[0], A1[0]) == (0.0, 1.0)
    assert np.isfinite(A0).all() and np.isfinite(A1).all()
    assert (A0[valid] > 0).all() and (A1[valid] > 0).all()


@pytest.mark.parametrize("a,b", [(0.7, 100.0), (0.7, 0.5), (0.3, 3.0), (0.0, 2.0)])
def test_stirling_pdp_normalisation(a, b):
    """Sum over table counts of the PDP joint is one (Cor.17):
    sum_M S^N_{M,a} (b|a)_M = (b)_N for every N."""
    for N in [1, 3, 10, 40, 120]:
        terms = [oracle.log_stirling(a, N, M) + math.log(float(rising(Fraction(b), M, Fraction(a)))) for M in range(1, N + 1)]
        mx = max(terms)
        lhs = mx + math.log(sum(math.exp(t - mx) for t in terms))
        rhs = math.lgamma(b + N) - math.lgamma(b)
        assert lhs == pytest.approx(rhs, rel=1e-10)


def test_crp_enumeration_matches_corollary17():
    """Brute-force seating enumeration reproduces the PDP
    joint p(w, t) = (b|a)_T/(b)_N prod_w S^{n_w}_{t_w,a} H(w)^{t_w} (P:1441,
    reading c1), which fixes the oracle's Stirling table."""
    a, b = Fraction(7, 10), Fraction(3, 2)
    for words in ([0, 0, 0], [0, 1, 0, 0], [1, 0, 1, 1, 0], [0, 0, 0, 0, 0, 0]):
        coef = crp_coefficients(words, a, b)
        assert sum(coef.values()) > 0
        for key, val in coef.items():
            tw = dict(key)
            T = sum(tw.values())
            lhs = math.log(float(val))
            rhs = math.log(float(rising(b, T, a))) - math.log(float(rising(b, len(words))))
            for w, t in tw.items():
                rhs += oracle.log_stirling(0.7, words.count(w), t)
            assert lhs == pytest.approx(rhs, abs=1e-12)


# --------------------------------------------------------------------------
# tiny corpora for exact enumeration
# --------------------------------------------------------------------------
TINY = [
    # (groups, docs as word lists, doc_group, V) — SURVEY Appendix A.2 corpus first
    (2, [[0, 0], [0, 1]], [0, 1], 2),
    (1, [[0, 1, 0]], [0], 2),
    (2, [[1], [0, 1], [1]], [0, 1, 1], 2),
]
HYPER = dict(alpha=0.1, beta=0.1, discount=0.7, concentration=100.0)
HYPER2 = dict(alpha=0.5, beta=0.3, discount=0.4, concentration=1.5)


def _tiny(spec, K=2, hyper=HYPER):
    I, docs, dg, V = spec
    group, doc, word = [], [], []
    for d, ws in enumerate(docs):
        for w in ws:
            group.append(dg[d]); doc.append(d); word.append(w)
    tc = TinyCorpus(group, doc, word, I, V, K,
                    Fraction(hyper["alpha"]).limit_denominator(1000), Fraction(hyper["beta"]).limit_denominator(1000),
                    Fraction(hyper["discount"]).limit_denominator(1000),
                    Fraction(hyper["concentration"]).limit_denominator(1000))
    return tc, np.array(group, np.int32), np.array(doc, np.int32), np.array(word, np.int32)


def _oracle_at(tc, arrays, z, t, hyper=HYPER, seed=7):
    group, doc, word = arrays
    o = oracle.Oracle(tc.I, tc.V, tc.K, hyper["alpha"], hyper["beta"], hyper["discount"], hyper["concentration"], seed)
    T = np.zeros((tc.I, tc.V, tc.K), np.int32)
    for (i, w, k), v in t.items():
        T[i, w, k] = v
    o.load(group, doc, word, tc.D, z_init=np.array(z, np.int32), t_init=T)
    return o


@pytest.mark.parametrize("hyper", [HYPER, HYPER2])
@pytest.mark.parametrize("spec", TINY)
def test_log_joint_matches_generative_enumeration(spec, hyper):
    """or_log_joint (P:1654-1665 summed over R) equals the exact p(W,Z,T) of the
    generative process, on every state of the tiny corpus."""
    tc, g, d, w = _tiny(spec, hyper=hyper)
    for z, t in tc.states():
        o = _oracle_at(tc, (g, d, w), z, t, hyper)
        assert o.log_joint() == pytest.approx(math.log(float(tc.joint_WZT(z, t))), abs=1e-10)


@pytest.mark.parametrize("hyper", [HYPER, HYPER2])
@pytest.mark.parametrize("spec", TINY)
def test_conditional_is_exact_joint_ratio(spec, hyper):
    """Eqs. SPDP-sampling-w-z-r0/-r1, as the oracle evaluates them,
    are the exact blocked conditional of p(W,Z,R) (reading c1)."""
    tc, g, d, w = _tiny(spec, hyper=hyper)
    checked = 0
    for z, t in tc.states():
        o = _oracle_at(tc, (g, d, w), z, t, hyper)
        m = tc.cells(z)
        for p in range(tc.N):
            c = (tc.group[p], tc.word[p], z[p])
            for r in (0, 1):
                got = o.conditional(p, r)
                impossible = (r == 0 and t[c] == m[c]) or (r == 1 and t[c] == 1 and m[c] > 1)
                if impossible:
                    assert got is None
                    continue
                want = [float(x) for x in tc.exact_conditional(z, t, p, r)]
                np.testing.assert_allclose(got, want, rtol=1e-11, atol=1e-15)
                checked += 1
    assert checked > 0


def _transition_matrix(tc, arrays, hyper):
    """One mode-S sweep (Alg.1 + keep rule) as an exact matrix over (z, t) states,
    built from the oracle's removal rule and conditional."""
    states = [(z, tuple(sorted(t.items()))) for z, t in tc.states()]
    index = {s: j for j, s in enumerate(states)}
    P = np.eye(len(states))
    for p in range(tc.N):
        Pp = np.zeros_like(P)
        for j, (z, tt) in enumerate(states):
            t = dict(tt)
            o = _oracle_at(tc, arrays, z, t, hyper)
            c = (tc.group[p], tc.word[p], z[p])
            m = tc.cells(z)[c]
            for r, pr in ((1, t[c] / m), (0, 1 - t[c] / m)):
                if pr == 0:
                    continue
                if r == 1 and t[c] == 1 and m > 1:        # keep rule (reading c5)
                    Pp[j, j] += pr
                    continue
                probs = o.conditional(p, r)
                for slot, q in enumerate(probs):
                    if q == 0:
                        continue
                    k, rn = slot // 2, 1 if slot % 2 == 0 else 0
                    z2 = list(z); z2[p] = k
                    t2 = dict(t); t2[c] -= r
                    cn = (tc.group[p], tc.word[p], k)
                    t2[cn] = t2.get(cn, 0) + rn
                    t2 = {cc: v for cc, v in t2.items() if v > 0}
                    Pp[j, index[(tuple(z2), tuple(sorted(t2.items())))]] += pr * q
        P = P @ Pp
    return states, P


@pytest.mark.parametrize("spec", TINY[:2])
def test_sequential_sweep_leaves_posterior_invariant(spec):
    """Alg.1 with Bernoulli(t/m) removal and the keep rule is an
    exact Gibbs sweep: pi P = pi for pi = p(Z,T|W)."""
    tc, g, d, w = _tiny(spec)
    states, P = _transition_matrix(tc, (g, d, w), HYPER)
    post = tc.posterior()
    pi = np.array([float(post[s]) for s in states])
    np.testing.assert_allclose(P.sum(axis=1), 1.0, atol=1e-13)
    assert np.abs(pi @ P - pi).max() < 1e-13


def test_sequential_chain_matches_exact_posterior_3sigma():
    """north_star (4): exact posterior enumeration on a 4-token K=2 corpus vs the
    empirical (z,t)- and z-frequencies of or_sweep_seq, within 3 sigma
    (sigma from 100 batch means)."""
    tc, g, d, w = _tiny(TINY[0])
    post = tc.posterior()
    o = oracle.Oracle(tc.I, tc.V, tc.K, **HYPER, seed=12345)
    o.load(g, d, w, tc.D)
    nsw, nb = 1_000_000, 100
    codes = o.chain_codes(nsw, waves=-1, tbase=5)
    K, N = tc.K, tc.N
    cells = [(i, ww, k) for i in range(tc.I) for ww in range(tc.V) for k in range(tc.K)]

    def code_of(z, t):
        c = sum(z[p] * K ** p for p in range(N))
        tc_ = sum(t.get(cell, 0) * 5 ** j for j, cell in enumerate(cells))
        return c + K ** N * tc_

    zmarg = {}
    for (z, tt), pv in post.items():
        zmarg[z] = zmarg.get(z, 0.0) + float(pv)
    batches = codes.reshape(nb, -1)
    bad = []
    for (z, tt), pv in post.items():
        hits = (batches == code_of(z, dict(tt))).mean(axis=1)
        mean, sig = hits.mean(), hits.std(ddof=1) / math.sqrt(nb)
        if abs(mean - float(pv)) > 3 * sig + 1e-12:
            bad.append(((z, tt), mean, float(pv), sig))
    zcodes = batches % (K ** N)
    for z, pv in zmarg.items():
        hits = (zcodes == sum(z[p] * K ** p for p in range(N))).mean(axis=1)
        mean, sig = hits.mean(), hits.std(ddof=1) / math.sqrt(nb)
        if abs(mean - pv) > 3 * sig + 1e-12:
            bad.append((z, mean, pv, sig))
    assert not bad, bad


# --------------------------------------------------------------------------
# parallel semantics and counts (reading c13-c15)
# --------------------------------------------------------------------------
def test_single_token_waves_equal_algorithm1():
    """Mode P with one token per wave (W=0) is Alg.1 exactly (bit-identical)."""
    import synth
    c = synth.generate(2, 6, 12.0, 40, 4, seed=5)
    a = oracle.from_corpus(c, 4)
    b = oracle.from_corpus(c, 4)
    for _ in range(4):
        a.sweep_seq()
        b.sweep_par(waves=0, shards=1)
        sa, sb = a.state(), b.state()
        for key in sa:
            np.testing.assert_array_equal(sa[key], sb[key])
        assert b.stats()["clamped"] == 0


@pytest.mark.parametrize("waves,shards", [(1, 1), (4, 1), (1, 2), (3, 4), (200, 3)])
def test_count_invariants_hold_after_parallel_sweeps(waves, shards):
    """north_star (4) invariants after mode-P sweeps: n, m recount from z,
    sum m = N, 0 <= t <= m, t > 0 iff m > 0, Q = sum_i t, sums consistent."""
    import synth
    c = synth.corpus_for(synth.CONFIGS["C1"])
    o = oracle.from_corpus(c, 10)
    assert o.check_invariants() == 0
    for _ in range(3):
        o.sweep_par(waves=waves, shards=shards)
        assert o.check_invariants() == 0
        st = o.state()
        assert st["m"].sum() == c.num_tokens


def test_sequential_never_clamps_and_keeps_invariants():
    import synth
    c = synth.corpus_for(synth.CONFIGS["C1"])
    o = oracle.from_corpus(c, 10)
    for _ in range(3):
        o.sweep_seq()
        assert o.check_invariants() == 0
        assert o.stats()["clamped"] == 0


def test_partition_is_balanced_and_covers_every_doc():
    import synth
    c = synth.corpus_for(synth.CONFIGS["C1"])
    o = oracle.from_corpus(c, 10)
    L = np.bincount(c.doc, minlength=c.num_docs)
    for G in (1, 2, 3, 8):
        s = o.partition(G)
        assert s.min() >= 0 and s.max() < G
        load = np.bincount(s, weights=L, minlength=G)
        assert load.max() - load.min() <= 2 * L.max()


def test_k1_only_tables_move():
    """K = 1 special case: z stays 0, only r/t move; sum m = N."""
    import synth
    c = synth.generate(2, 5, 20.0, 30, 3, seed=11)
    o = oracle.from_corpus(c, 1)
    for _ in range(3):
        o.sweep_par(waves=1)
        st = o.state()
        assert (st["z"] == 0).all() and st["m"].sum() == c.num_tokens
        assert o.check_invariants() == 0


# --------------------------------------------------------------------------
# b -> infinity limit: SPDP becomes textbook collapsed-Gibbs LDA
# --------------------------------------------------------------------------
def _textbook_lda(group, doc, word, V, K, alpha, beta, z, seed, sweeps, jacobi, waves=1):
    """Collapsed Gibbs LDA (Griffiths & Steyvers; PAPER.md:1217-1304 background)
    on group-pooled word-topic counts, p(k) ∝ (alpha+n_dk)(beta+n_kw)/(V beta+n_k),
    drawing with the same Philox uniform u and the first-exceeding-CDF rule.
    jacobi: every token of a wave decides against the wave-start counts; the
    waves are the in-document positions l mod `waves` (the paper's round-robin
    reorder P:2289-2299), run in order 0 .. waves-1."""
    z = np.array(z, np.int64)
    N = len(word)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    seen = {}
    pos = np.zeros(N, np.int64)                      # in-document position: order of appearance
    for p in range(N):
        pos[p] = seen.get(int(doc[p]), 0)
        seen[int(doc[p])] = pos[p] + 1
    if jacobi and waves > 1:
        for s in range(sweeps):
            for wv in range(waves):
                ndk = np.zeros((doc.max() + 1, K), np.int64)
                nkw = np.zeros((K, V), np.int64)
                for p in range(N):
                    ndk[doc[p], z[p]] += 1; nkw[z[p], word[p]] += 1
                nk = nkw.sum(axis=1)
                newz = z.copy()
                for p in np.nonzero(pos % waves == wv)[0]:
                    x = oracle.philox([int(p), s, 0, 0], key)
                    u = (float(x[1]) * 2097152.0 + float(int(x[2]) >> 11)) / 9007199254740992.0
                    A, B, C_ = ndk.copy(), nkw.copy(), nk.copy()
                    A[doc[p], z[p]] -= 1; B[z[p], word[p]] -= 1; C_[z[p]] -= 1
                    pk = (alpha + A[doc[p]]) * (beta + B[:, word[p]]) / (V * beta + C_)
                    newz[p] = int(np.argmax(np.cumsum(pk / pk.sum()) > u))
                z = newz
        return z
    for s in range(sweeps):
        ndk = np.zeros((doc.max() + 1, K), np.int64)
        nkw = np.zeros((K, V), np.int64)
        for p in range(N):
            ndk[doc[p], z[p]] += 1; nkw[z[p], word[p]] += 1
        nk = nkw.sum(axis=1)
        snap = (ndk.copy(), nkw.copy(), nk.copy())
        newz = z.copy()
        for p in range(N):
            x = oracle.philox([p, s, 0, 0], key)
            u = (float(x[1]) * 2097152.0 + float(int(x[2]) >> 11)) / 9007199254740992.0
            A, B, C_ = snap if jacobi else (ndk, nkw, nk)
            A = A.copy(); B = B.copy(); C_ = C_.copy()
            A[doc[p], z[p]] -= 1; B[z[p], word[p]] -= 1; C_[z[p]] -= 1
            pk = (alpha + A[doc[p]]) * (beta + B[:, word[p]]) / (V * beta + C_)
            cdf = np.cumsum(pk / pk.sum())
            k = int(np.argmax(cdf > u))
            if jacobi:
                newz[p] = k
            else:
                ndk[doc[p], z[p]] -= 1; nkw[z[p], word[p]] -= 1; nk[z[p]] -= 1
                z[p] = k
                ndk[doc[p], k] += 1; nkw[k, word[p]] += 1; nk[k] += 1
        if jacobi:
            z = newz
    return z


@pytest.mark.parametrize("jacobi,waves", [(False, 1), (True, 1), (True, 2), (True, 3), (True, 4)])
def test_infinite_concentration_is_collapsed_lda(jacobi, waves):
    """b -> infinity (SURVEY §8(c) pin): the SPDP sweep is textbook collapsed-Gibbs
    LDA; for waves > 1 this also pins the wave membership pos % W (an index slip,
    e.g. the canonical token index instead of the in-document position, fails)."""
    import synth
    c = synth.generate(2, 4, 15.0, 25, 3, seed=3)
    K, seed = 3, 99
    z0 = np.random.default_rng(0).integers(0, K, c.num_tokens).astype(np.int32)
    o = oracle.Oracle(2, c.vocab, K, 0.1, 0.1, 0.7, 1e30, seed)
    o.load(c.group, c.doc, c.word, c.num_docs, z_init=z0, r_init=np.ones(c.num_tokens, np.uint8))
    sweeps = 6
    for _ in range(sweeps):
        if jacobi:
            o.sweep_par(waves=waves)
        else:
            o.sweep_seq()
    want = _textbook_lda(c.group, c.doc, c.word, c.vocab, K, 0.1, 0.1, z0, seed, sweeps, jacobi, waves)
    np.testing.assert_array_equal(o.state()["z"], want)
    assert (o.state()["r"] == 1).all()


# --------------------------------------------------------------------------
# perplexity estimator (P:1978-2007 with P:1738)
# --------------------------------------------------------------------------
def test_predictive_distribution_is_normalised():
    """With reading c16 (b + a t_ik.) the estimator of P:1754 is a distribution:
    sum_w p(w | d) = 1 for every document (the printed a t_ik. would not be)."""
    import synth
    c = synth.generate(2, 4, 10.0, 15, 3, seed=8)
    o = oracle.from_corpus(c, 3)
    for _ in range(2):
        o.sweep_par(waves=1)
    for d in range(c.num_docs):
        assert sum(o.word_prob(d, w) for w in range(c.vocab)) == pytest.approx(1.0, abs=1e-12)
    ppl = o.perplexity()
    ll = sum(math.log(o.word_prob(int(c.doc[p]), int(c.word[p]))) for p in range(c.num_tokens))
    assert ppl == pytest.approx(math.exp(-ll / c.num_tokens), rel=1e-12)


def test_perplexity_degenerate_cases():
    import synth
    # V = 1: every predicted probability is 1 -> perplexity exactly 1
    c = synth.generate(2, 3, 8.0, 1, 2, seed=4)
    o = oracle.from_corpus(c, 3)
    o.sweep_par(waves=1)
    assert o.perplexity() == pytest.approx(1.0, abs=1e-12)
    # uniform limit (uniform model -> perplexity V)
    c = synth.generate(2, 3, 8.0, 17, 2, seed=4)
    o = oracle.Oracle(2, 17, 3, 1e12, 1e12, 0.7, 1e15, 1)
    o.load(c.group, c.doc, c.word, c.num_docs)
    assert o.perplexity() == pytest.approx(17.0, rel=1e-9)


# --------------------------------------------------------------------------
# NEXT-3: exchanges every E waves (bounded staleness) and training-data duplication
# --------------------------------------------------------------------------
def test_per_wave_exchange_with_one_token_waves_is_algorithm1():
    """G shards exchanging after every one-token wave see every earlier decision:
    exactly the sequential sampler (Alg.1, pinned against exact enumeration)."""
    import synth
    c = synth.generate(2, 6, 12.0, 40, 4, seed=5)
    a = oracle.from_corpus(c, 4)
    b = oracle.from_corpus(c, 4)
    for _ in range(4):
        a.sweep_seq()
        b.sweep_par(waves=0, shards=3, merge_every=1)
        sa, sb = a.state(), b.state()
        for k in ("z", "r", "n", "m", "t", "Q"):
            assert np.array_equal(sa[k], sb[k]), k
    assert b.stats()["clamped"] == 0


@pytest.mark.parametrize("E", [1, 2, 3])
def test_exchange_cadence_single_shard_and_invariants(E):
    import synth
    c = synth.generate(2, 10, 15.0, 30, 4, seed=9)
    a = oracle.from_corpus(c, 4)
    b = oracle.from_corpus(c, 4)
    for _ in range(3):                       # one shard: the exchange cadence changes nothing
        a.sweep_par(waves=4)
        b.sweep_par(waves=4, merge_every=E)
    assert all(np.array_equal(a.state()[k], b.state()[k]) for k in ("z", "r", "n", "m", "t", "Q"))
    d = oracle.from_corpus(c, 4)
    for _ in range(3):                       # several shards: a valid state after every sweep
        d.sweep_par(waves=4, shards=3, merge_every=E)
        assert d.check_invariants() == 0
    e = oracle.from_corpus(c, 4)
    f = oracle.from_corpus(c, 4)
    e.sweep_par(waves=4, shards=3, merge_every=99)
    f.sweep_par(waves=4, shards=3)
    assert all(np.array_equal(e.state()[k], f.state()[k]) for k in ("z", "r", "n", "m", "t", "Q"))
