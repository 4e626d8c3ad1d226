"""Pins of the oracle's NEXT-1 functions (held-out evaluation),
CPU only.  Each pin comes from outside the oracle: closed forms of the
Hellinger distance, normalisation and limits of the estimators P:1753-1754,
exact posterior enumeration of the fold-in chain, the already-pinned training
perplexity, and label-permutation symmetry.
"""
import itertools
import math

import numpy as np
import pytest

import oracle
import synth

HYPER = dict(alpha=0.1, beta=0.1, discount=0.7, concentration=100.0)


def _trained(seed=3, K=4, sweeps=3, V=30):
    c = synth.generate(2, 8, 12.0, V, 3, seed=seed)
    o = oracle.from_corpus(c, K, **HYPER)
    for _ in range(sweeps):
        o.sweep_par(waves=1)
    return c, o


# --------------------------------------------------------------------------
# Hellinger distance (§4.2.6; reading c22 = the standard formula)
# --------------------------------------------------------------------------
def test_hellinger_closed_forms():
    p = np.array([0.2, 0.3, 0.5])
    assert oracle.hellinger(p, p) == pytest.approx(0.0, abs=1e-7)
    assert oracle.hellinger([1.0, 0.0, 0.0, 0.0], [0.0, 0.5, 0.5, 0.0]) == 1.0          # disjoint supports
    assert oracle.hellinger([1.0, 0.0], [0.5, 0.5]) == pytest.approx(math.sqrt(1 - math.sqrt(0.5)), abs=1e-15)
    # two Bernoullis: H^2 = 1 - sqrt(pq) - sqrt((1-p)(1-q))
    for a, b in [(0.1, 0.7), (0.5, 0.25), (0.9, 0.05)]:
        h = oracle.hellinger([a, 1 - a], [b, 1 - b])
        assert h * h == pytest.approx(1 - math.sqrt(a * b) - math.sqrt((1 - a) * (1 - b)), abs=1e-14)
        assert h == oracle.hellinger([b, 1 - b], [a, 1 - a])


def test_greedy_match_hand_example():
    # global greedy: 0.05 (1,2) first, then 0.1 (0,1)... (0,1) conflicts with nothing -> taken, then (2,0)
    d = np.array([[0.9, 0.1, 0.3],
                  [0.2, 0.4, 0.05],
                  [0.15, 0.6, 0.7]])
    assert list(oracle.greedy_match(d)) == [1, 2, 0]
    assert list(oracle.greedy_match(np.ones((4, 4)) - np.eye(4))) == [0, 1, 2, 3]
    rng = np.random.default_rng(0)
    for _ in range(20):
        K = int(rng.integers(1, 9))
        perm = oracle.greedy_match(rng.random((K, K)))
        assert sorted(perm) == list(range(K))                                              # a bijection


def test_topic_align_self_and_label_swap():
    c, o = _trained()
    st = o.state()
    dist, perm = o.topic_align(o)
    assert np.allclose(np.diag(dist), 0.0, atol=1e-7) and list(perm) == [0, 1, 2, 3]
    # relabel topics 0 <-> 2 (z and the table counts): the model is the same up to labels
    swap = np.array([2, 1, 0, 3])
    o2 = oracle.Oracle(c.num_groups, c.vocab, 4, **HYPER, seed=7)
    o2.load(c.group, c.doc, c.word, c.num_docs, z_init=swap[st["z"]], t_init=st["t"][:, :, np.argsort(swap)])
    d2, p2 = o.topic_align(o2)
    assert list(p2) == [2, 1, 0, 3]
    assert d2[0, 2] == pytest.approx(0.0, abs=1e-7) and d2[2, 0] == pytest.approx(0.0, abs=1e-7)


# --------------------------------------------------------------------------
# estimators P:1753-1754 (reading c16)
# --------------------------------------------------------------------------
def test_topic_estimates_are_distributions_and_limits():
    c, o = _trained()
    phi0, phi = o.topics()
    assert np.allclose(phi0.sum(axis=1), 1.0, atol=1e-12)
    assert np.allclose(phi.sum(axis=2), 1.0, atol=1e-12)                                   # reading c16
    assert (phi0 > 0).all() and (phi > 0).all()
    # b -> inf: the group distribution collapses onto the shared base phi0
    st = o.state()
    ob = oracle.Oracle(c.num_groups, c.vocab, 4, 0.1, 0.1, 0.7, 1e15, 7)
    ob.load(c.group, c.doc, c.word, c.num_docs, z_init=st["z"], t_init=st["t"])
    p0b, pb = ob.topics()
    assert np.allclose(pb, p0b[None], rtol=1e-9, atol=1e-15)


# --------------------------------------------------------------------------
# held-out perplexity (reading c17) and fold-in (reading c21)
# --------------------------------------------------------------------------
def test_heldout_perplexity_of_training_docs_is_training_perplexity():
    """Evaluating the training documents as the 'held-out' set with their own
    z reproduces the (pinned) training perplexity: same equation, other code."""
    c, o = _trained()
    z = o.state()["z"]
    ppl = o.heldout_perplexity(c.group, c.doc, c.word, c.num_docs, z)
    assert ppl == pytest.approx(o.perplexity(), rel=1e-12)


def test_heldout_perplexity_degenerate_cases():
    # V = 1: every word probability is 1
    c = synth.generate(2, 3, 8.0, 1, 2, seed=4)
    o = oracle.from_corpus(c, 3)
    o.sweep_par(waves=1)
    te = synth.generate(2, 2, 6.0, 1, 2, seed=9)
    z = o.foldin(te.group, te.doc, te.word, te.num_docs, seed=1, iterations=3)
    assert o.heldout_perplexity(te.group, te.doc, te.word, te.num_docs, z) == pytest.approx(1.0, abs=1e-12)
    # uniform limit: perplexity V
    c = synth.generate(2, 3, 8.0, 17, 2, seed=4)
    o = oracle.Oracle(2, 17, 3, 1e12, 1e12, 0.7, 1e15, 1)
    o.load(c.group, c.doc, c.word, c.num_docs)
    te = synth.generate(2, 2, 6.0, 17, 2, seed=9)
    z = o.foldin(te.group, te.doc, te.word, te.num_docs, seed=1, iterations=2)
    assert o.heldout_perplexity(te.group, te.doc, te.word, te.num_docs, z) == pytest.approx(17.0, rel=1e-9)


def test_foldin_k1_and_determinism():
    c = synth.generate(2, 4, 10.0, 15, 3, seed=8)
    o = oracle.from_corpus(c, 1)
    o.sweep_par(waves=1)
    te = synth.generate(2, 3, 7.0, 15, 3, seed=2)
    z, th = o.foldin(te.group, te.doc, te.word, te.num_docs, seed=5, iterations=4), None
    assert (z == 0).all()
    _, th = o.heldout_perplexity(te.group, te.doc, te.word, te.num_docs, z, want_theta=True)
    assert np.allclose(th, 1.0)
    # RNG keyed by (token, iteration): one call of 5 iterations == 5 calls of 1
    c, o = _trained()
    te = synth.generate(2, 3, 9.0, 30, 3, seed=6)
    z5 = o.foldin(te.group, te.doc, te.word, te.num_docs, seed=11, iterations=5)
    z = o.foldin(te.group, te.doc, te.word, te.num_docs, seed=11, iterations=0)
    for it in range(5):
        z = o.foldin(te.group, te.doc, te.word, te.num_docs, seed=11, iterations=1, first_iteration=it, z=z)
    assert np.array_equal(z, z5)
    assert not np.array_equal(z5, o.foldin(te.group, te.doc, te.word, te.num_docs, seed=12, iterations=5))


def test_foldin_follows_the_dominant_topic():
    """a document whose words only topic k explains folds into k."""
    # training: word 0 always topic 1, word 1 always topic 0; every customer at its own table
    docs = [[0, 0, 0, 1, 1], [0, 0, 1], [1, 1, 0, 0]]
    c = synth.tiny_corpus(1, docs, [0, 0, 0], 6)
    z = np.where(c.word == 0, 1, 0).astype(np.int32)
    o = oracle.Oracle(1, 6, 3, 0.1, 1e-6, 0.0, 1e-3, 1)
    o.load(c.group, c.doc, c.word, c.num_docs, z_init=z, r_init=np.ones(c.num_tokens, np.uint8))
    te = synth.tiny_corpus(1, [[0, 0, 0, 0, 0, 0]], [0], 6)
    zt = o.foldin(te.group, te.doc, te.word, te.num_docs, seed=3, iterations=5)
    _, th = o.heldout_perplexity(te.group, te.doc, te.word, te.num_docs, zt, want_theta=True)
    assert int(np.argmax(th[0])) == 1 and (zt == 1).all()


def test_foldin_chain_matches_exact_posterior_3sigma():
    """The fold-in chain's z-frequencies on a 3-token held-out document (K = 2)
    match the exact posterior p(z | w, phi~) ∝ prod_k Gamma(alpha + n_k) *
    prod_p phi~_{z_p w_p} (Dirichlet-multinomial times the frozen likelihoods)
    within 3 sigma (100 batch means)."""
    c = synth.generate(1, 5, 8.0, 3, 2, seed=21)
    o = oracle.from_corpus(c, 2, **HYPER)
    for _ in range(2):
        o.sweep_par(waves=1)
    _, phi = o.topics()
    te = synth.tiny_corpus(1, [[0, 2, 0]], [0], 3)
    K, N = 2, 3
    post = {}
    for z in itertools.product(range(K), repeat=N):
        n = np.bincount(z, minlength=K)
        lp = sum(math.lgamma(0.1 + n[k]) for k in range(K)) + sum(math.log(phi[0, z[p], te.word[p]]) for p in range(N))
        post[z] = lp
    mx = max(post.values())
    tot = sum(math.exp(v - mx) for v in post.values())
    post = {z: math.exp(v - mx) / tot for z, v in post.items()}
    iters, nb = 40_000, 100
    codes = np.zeros(iters, np.int64)
    z = o.foldin(te.group, te.doc, te.word, 1, seed=77, iterations=0)
    for it in range(iters):
        z = o.foldin(te.group, te.doc, te.word, 1, seed=77, iterations=1, first_iteration=it, z=z)
        codes[it] = z[0] + 2 * z[1] + 4 * z[2]
    batches = codes.reshape(nb, -1)
    for zc, pv in post.items():
        hits = (batches == zc[0] + 2 * zc[1] + 4 * zc[2]).mean(axis=1)
        mean, sig = hits.mean(), hits.std(ddof=1) / math.sqrt(nb)
        assert abs(mean - pv) <= 3 * sig + 1e-12, (zc, mean, pv, sig)
