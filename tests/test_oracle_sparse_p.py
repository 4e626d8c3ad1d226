"""Pins of the oracle's NEXT-4 sampler (sparse non-identity transformation
matrices P^i), CPU only:
  * with P^i = identity it is the identity-P sampler bit for bit (itself pinned
    against exact enumeration in test_oracle_pins.py);
  * its conditional equals the exact ratio of p(W, Z, R, V) obtained by brute
    force from the generative process with P (oracle/enumerate.py
    TinyCorpusP), on every state, token and removal outcome;
  * its sequential chain visits every (z, q) state with the exact posterior
    frequency (3 sigma, batch means);
  * the wave mode keeps a valid state (q >= 0, t = sum q in [min(1,m), m],
    Q = sum_{i,w} q).
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from oracle.enumerate import TinyCorpusP

HYPER = dict(alpha=0.1, beta=0.1, discount=0.7, concentration=100.0)
HYPER2 = dict(alpha=0.5, beta=0.3, discount=0.4, concentration=1.5)


def identity_P(I, V):
    return np.arange(I * V + 1), np.tile(np.arange(V), I), np.ones(I * V)


def mixing_P(I, V, rng, density=2):
    """Doubly stochastic sparse rows: each P^i = (1 - e) Id + e Perm (columns and rows sum to 1)."""
    pptr, pv, pp = [0], [], []
    for i in range(I):
        perm = rng.permutation(V)
        eps = 0.2 + 0.1 * i
        for w in range(V):
            ent = {w: 1.0 - eps}
            ent[int(perm[w])] = ent.get(int(perm[w]), 0.0) + eps
            for v in sorted(ent):
                pv.append(v); pp.append(ent[v])
            pptr.append(len(pv))
    return np.array(pptr), np.array(pv), np.array(pp)


@pytest.mark.parametrize("waves", [-1, 1, 3])
def test_identity_P_is_the_identity_sampler(waves):
    c = synth.generate(2, 6, 12.0, 40, 4, seed=5)
    a = oracle.from_corpus(c, 4)
    b = oracle.from_corpus(c, 4)
    sp = oracle.SparseOracle(b, *identity_P(2, 40))
    for _ in range(4):
        if waves < 0:
            a.sweep_seq(); sp.sweep_seq()
        else:
            a.sweep_par(waves=waves); sp.sweep_par(waves=waves)
        sa, sb = a.state(), sp.state()
        for k in ("z", "r", "n", "m", "t"):
            assert np.array_equal(sa[k], sb[k]), k
        assert np.array_equal(sa["Q"], sb["Qs"])
    assert a.stats() == b.stats()


def test_invalid_P_is_rejected():
    c = synth.generate(1, 2, 5.0, 3, 2, seed=1)
    o = oracle.from_corpus(c, 2)
    with pytest.raises(ValueError):
        oracle.SparseOracle(o, np.array([0, 1, 2, 3]), np.array([0, 1, 2]), np.array([0.5, 1.0, 1.0]))  # column 0 sums to 0.5
    with pytest.raises(ValueError):
        oracle.SparseOracle(o, np.array([0, 1, 1, 2]), np.array([0, 2]), np.array([1.0, 1.0]))            # row 1 empty


# tiny corpora with 2-entry rows: V = 2, P^i = [[1-e, e], [e, 1-e]] (doubly stochastic)
TINY = [(2, [[0, 0], [0, 1]], [0, 1], 2), (1, [[0, 1, 0]], [0], 2)]


def _tiny(spec, K=2, hyper=HYPER):
    I, docs, dg, V = spec
    group, doc, word = [], [], []
    for d, ws in enumerate(docs):
        for w in ws:
            group.append(dg[d]); doc.append(d); word.append(w)
    eps = [Fraction(3, 10), Fraction(1, 5)]
    P = {}
    pptr, pv, pp = [0], [], []
    for i in range(I):
        for w in range(V):
            ent = [(0, 1 - eps[i] if w == 0 else eps[i]), (1, eps[i] if w == 0 else 1 - eps[i])]
            P[(i, w)] = ent
            for v, p in ent:
                pv.append(v); pp.append(float(p))
            pptr.append(len(pv))
    f = lambda x: Fraction(x).limit_denominator(1000)
    tc = TinyCorpusP(group, doc, word, I, V, K, f(hyper["alpha"]), f(hyper["beta"]), f(hyper["discount"]),
                     f(hyper["concentration"]), P=P)
    arr = lambda x: np.array(x, np.int32)
    return tc, arr(group), arr(doc), arr(word), (np.array(pptr), np.array(pv), np.array(pp))


def _q_array(tc, q, pptr, K):
    out = np.zeros((int(pptr[-1]), K), np.int32)
    for (i, w, k), qs in q.items():
        for j, x in enumerate(qs):
            out[pptr[i * tc.V + w] + j, k] = x
    return out


@pytest.mark.parametrize("spec,hyper", [(TINY[0], HYPER), (TINY[1], HYPER2)])
def test_conditional_is_exact_joint_ratio_with_P(spec, hyper):
    tc, g, d, w, (pptr, pv, pp) = _tiny(spec, hyper=hyper)
    worst, checked = 0.0, 0
    for z, t, q in tc.states_q():
        o = oracle.Oracle(tc.I, tc.V, tc.K, **hyper, seed=1)
        tarr = np.zeros((tc.I, tc.V, tc.K), np.int32)
        for (i, ww, k), tv in t.items():
            tarr[i, ww, k] = tv
        o.load(g, d, w, tc.D, z_init=np.array(z, np.int32), t_init=tarr)
        sp = oracle.SparseOracle(o, pptr, pv, pp)
        sp.set_q(_q_array(tc, q, pptr, tc.K))
        for p in range(tc.N):
            c = (int(g[p]), int(w[p]), z[p])
            S = len(tc.P[(c[0], c[1])])
            outcomes = [(0, 0)] + [(1, e) for e in range(S)]
            for r_rem, e_rem in outcomes:
                if r_rem and q[c][e_rem] < 1:
                    continue
                got = sp.conditional(p, r_rem, int(pptr[c[0] * tc.V + c[1]]) + e_rem)
                removable = (t[c] < tc.cells(z)[c]) if not r_rem else not (t[c] == 1 and tc.cells(z)[c] > 1)
                if not removable:
                    assert got is None
                    continue
                want = np.array([float(x) for x in tc.exact_conditional_q(z, t, q, p, r_rem, e_rem)])
                worst = max(worst, float(np.max(np.abs(got - want) / np.maximum(want, 1e-300) * (want > 0))))
                assert np.all((got > 0) == (want > 0))
                checked += 1
    assert checked > 100 and worst < 1e-11, (checked, worst)


def test_sequential_chain_matches_exact_posterior_with_P_3sigma():
    tc, g, d, w, (pptr, pv, pp) = _tiny(TINY[0])
    post = tc.posterior_q()
    o = oracle.Oracle(tc.I, tc.V, tc.K, **HYPER, seed=4321)
    o.load(g, d, w, tc.D)
    sp = oracle.SparseOracle(o, pptr, pv, pp)
    nsw, nb, qbase = 400_000, 100, 5
    codes = sp.chain_codes(nsw, waves=-1, qbase=qbase)
    K, N = tc.K, tc.N

    def code_of(z, q):
        c = sum(z[p] * K ** p for p in range(N))
        qa = _q_array(tc, dict(q), pptr, K).reshape(-1)
        return c + K ** N * sum(int(x) * qbase ** j for j, x in enumerate(qa))

    batches = codes.reshape(nb, -1)
    bad = []
    for (z, q), pv_ in post.items():
        hits = (batches == code_of(z, q)).mean(axis=1)
        mean, sig = hits.mean(), hits.std(ddof=1) / math.sqrt(nb)
        sig = max(sig, 2 * math.sqrt(float(pv_) / nsw))     # rare states: Poisson floor (x2 for autocorrelation)
        if abs(mean - float(pv_)) > 3 * sig + 1e-12:
            bad.append(((z, q), mean, float(pv_), sig))
    assert len(post) > 20
    assert not bad, bad[:5]


@pytest.mark.parametrize("waves", [1, 4])
def test_wave_mode_keeps_a_valid_state_with_P(waves):
    c = synth.generate(2, 12, 15.0, 30, 4, seed=9)
    rng = np.random.default_rng(3)
    pptr, pv, pp = mixing_P(2, 30, rng)
    o = oracle.from_corpus(c, 4)
    sp = oracle.SparseOracle(o, pptr, pv, pp)
    for _ in range(4):
        sp.sweep_par(waves=waves)
        st = sp.state()
        q, m, t = st["q"], st["m"], st["t"]
        assert (q >= 0).all()
        tq = np.zeros_like(t)
        Qs = np.zeros((4, 30), np.int64)
        for i in range(2):
            for ww in range(30):
                for e in range(pptr[i * 30 + ww], pptr[i * 30 + ww + 1]):
                    tq[i, ww] += q[e]
                    Qs[:, pv[e]] += q[e]
        assert np.array_equal(tq, t)
        assert (t <= m).all() and ((t > 0) == (m > 0)).all()
        assert np.array_equal(Qs, st["Qs"])
        assert m.sum() == c.num_tokens


def test_sparse_estimators_normalised_and_identity_reduction():
    """With P^i = I the estimators are those of P:1753-1754 (pinned in
    test_oracle_heldout.py); with a sparse doubly-stochastic P^i the rows of
    phi~^i still sum to 1 (because the columns of P^i do), and the training
    perplexity equals the held-out perplexity of the training documents."""
    c = synth.generate(2, 8, 12.0, 30, 3, seed=3)
    a = oracle.from_corpus(c, 4)
    b = oracle.from_corpus(c, 4)
    sp = oracle.SparseOracle(b, *identity_P(2, 30))
    for _ in range(2):
        a.sweep_par(waves=1); sp.sweep_par(waves=1)
    p0a, pa = a.topics(); p0b, pb = sp.topics()
    assert np.array_equal(p0a, p0b) and np.array_equal(pa, pb)
    assert sp.perplexity() == a.perplexity()
    o = oracle.from_corpus(c, 4)
    P = mixing_P(2, 30, np.random.default_rng(5))
    s2 = oracle.SparseOracle(o, *P)
    for _ in range(3):
        s2.sweep_par(waves=2)
    p0, ph = s2.topics()
    assert np.allclose(p0.sum(axis=1), 1.0, atol=1e-12) and np.allclose(ph.sum(axis=2), 1.0, atol=1e-12)
    z = s2.state()["z"]
    assert s2.heldout_perplexity(c.group, c.doc, c.word, c.num_docs, z) == pytest.approx(s2.perplexity(), rel=1e-12)
    te = synth.generate(2, 3, 9.0, 30, 3, seed=6)
    zf = s2.foldin(te.group, te.doc, te.word, te.num_docs, seed=2, iterations=3)
    assert np.isfinite(s2.heldout_perplexity(te.group, te.doc, te.word, te.num_docs, zf))


@pytest.mark.parametrize("G,waves", [(1, 1), (2, 1), (3, 2)])
def test_sharded_sweep_identity_reduction_and_validity(G, waves):
    """Several shards with one exchange per sweep: with P^i = I exactly the pinned
    G-shard identity sampler (or_sweep_par); with a sparse P a valid state."""
    c = synth.generate(2, 10, 12.0, 30, 4, seed=5)
    a = oracle.from_corpus(c, 4)
    b = oracle.from_corpus(c, 4)
    sp = oracle.SparseOracle(b, *identity_P(2, 30))
    for _ in range(3):
        a.sweep_par(waves=waves, shards=G)
        sp.sweep_shards(waves=waves, shards=G)
        sa, sb = a.state(), sp.state()
        for k in ("z", "r", "n", "m", "t"):
            assert np.array_equal(sa[k], sb[k]), k
        assert np.array_equal(sa["Q"], sb["Qs"])
    o = oracle.from_corpus(c, 4)
    s2 = oracle.SparseOracle(o, *mixing_P(2, 30, np.random.default_rng(7)))
    if G == 1:
        o2 = oracle.from_corpus(c, 4)
        s3 = oracle.SparseOracle(o2, *mixing_P(2, 30, np.random.default_rng(7)))
    for _ in range(3):
        s2.sweep_shards(waves=waves, shards=G)
        st = s2.state()
        assert (st["q"] >= 0).all() and (st["t"] <= st["m"]).all() and ((st["t"] > 0) == (st["m"] > 0)).all()
        if G == 1:
            s3.sweep_par(waves=waves)
            assert all(np.array_equal(st[k], s3.state()[k]) for k in ("z", "r", "m", "t", "q"))


@pytest.mark.parametrize("spec,hyper", [(TINY[0], HYPER), (TINY[1], HYPER2)])
def test_sparse_log_joint_is_exact(spec, hyper):
    """log p(W, Z, T, Q) of the oracle equals the brute-force joint of the
    generative process with P (TinyCorpusP) on every state."""
    tc, g, d, w, (pptr, pv, pp) = _tiny(spec, hyper=hyper)
    n = 0
    for z, t, q in tc.states_q():
        o = oracle.Oracle(tc.I, tc.V, tc.K, **hyper, seed=1)
        tarr = np.zeros((tc.I, tc.V, tc.K), np.int32)
        for (i, ww, k), tv in t.items():
            tarr[i, ww, k] = tv
        o.load(g, d, w, tc.D, z_init=np.array(z, np.int32), t_init=tarr)
        sp = oracle.SparseOracle(o, pptr, pv, pp)
        sp.set_q(_q_array(tc, q, pptr, tc.K))
        want = math.log(float(tc.joint_WZTQ(z, t, q)))
        assert sp.log_joint() == pytest.approx(want, abs=1e-9), (z, t, q)
        n += 1
    assert n > 20
