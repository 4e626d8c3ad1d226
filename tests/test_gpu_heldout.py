"""GPU parity of NEXT-1 (held-out evaluation) through the C ABI:
spdp_topics, spdp_heldout (fold-in + held-out perplexity) and
spdp_topic_hellinger against the oracle, on the same trained state.

Fold-in draws are compared in lock-step (the oracle replays each iteration
with the GPU's draws forced and reports its own draws and their margins), as
for the sweep: mismatches only where the uniform lies within 1e-6 of a CDF
boundary, and at most 1e-4 of the tokens.
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import HYPER, corpus, require_gpu
import paper_1510_06549_b200 as spdp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    require_gpu()


def _trained(name, K, sweeps=3, seed=7):
    """(train, test, GPU sampler after `sweeps`, oracle loaded with the GPU's state)."""
    train, test = synth.holdout_split(corpus(name), 0.1, seed=1)
    g = spdp.sampler_for(train, K, seed=seed, **HYPER)
    g.sweep(sweeps)
    gc = g.counts()
    o = oracle.Oracle(train.num_groups, train.vocab, K, **HYPER, seed=seed)
    o.load(train.group, train.doc, train.word, train.num_docs, z_init=gc["z"], t_init=gc["t"])
    return train, test, g, o


@pytest.mark.parametrize("name,K", [("C1", 10), ("C2", 50)])
def test_topics_match_oracle(name, K):
    _, _, g, o = _trained(name, K)
    gp0, gp = g.topics()
    op0, op = o.topics()
    np.testing.assert_allclose(gp0, op0, rtol=1e-12, atol=0)
    np.testing.assert_allclose(gp, op, rtol=1e-11, atol=1e-300)
    assert np.allclose(gp.sum(axis=2), 1.0, atol=1e-12)


@pytest.mark.parametrize("name,K,iters", [("C1", 10, 5), ("C2", 50, 3), ("C1", 1, 2), ("C1", 37, 3)])
def test_foldin_lockstep_and_perplexity(name, K, iters):
    _, test, g, o = _trained(name, K)
    seed = 99
    z_o = o.foldin(test.group, test.doc, test.word, test.num_docs, seed=seed, iterations=0)    # Philox init
    r0 = g.heldout(test, seed, 0)
    np.testing.assert_array_equal(r0["z"], z_o)
    z = r0["z"]
    bad = 0
    for it in range(iters):
        r = g.heldout(test, seed, 1, first_iteration=it, z_init=z)
        zf, margin, own = o.foldin(test.group, test.doc, test.word, test.num_docs, seed=seed, iterations=1,
                                   first_iteration=it, z=z, force_z=r["z"], want_margin=True)
        np.testing.assert_array_equal(zf, r["z"])
        mism = np.nonzero(own != r["z"])[0]
        assert (margin[mism] <= 1e-6).all(), (it, mism[:5], margin[mism[:5]])
        bad += len(mism)
        z = r["z"]
    assert bad <= max(1, 1e-4 * test.num_tokens * iters)
    res = g.heldout(test, seed, 0, z_init=z, want_theta=True)
    ppl_o, th_o = o.heldout_perplexity(test.group, test.doc, test.word, test.num_docs, z, want_theta=True)
    assert res["perplexity"] == pytest.approx(ppl_o, rel=1e-10)
    np.testing.assert_allclose(res["theta"], th_o, rtol=1e-12)
    if K == 1:
        assert (z == 0).all()


def test_foldin_one_call_equals_single_iterations():
    _, test, g, _ = _trained("C1", 10)
    full = g.heldout(test, 5, 4)
    z = g.heldout(test, 5, 0)["z"]
    for it in range(4):
        z = g.heldout(test, 5, 1, first_iteration=it, z_init=z)["z"]
    np.testing.assert_array_equal(full["z"], z)
    assert full["perplexity"] == g.heldout(test, 5, 0, z_init=z)["perplexity"]


def test_heldout_input_errors():
    _, test, g, _ = _trained("C1", 10, sweeps=1)
    bad = synth.Corpus(test.group, test.doc, test.word.copy(), test.z_gen, test.num_groups, test.num_docs, test.vocab)
    bad.word[3] = test.vocab
    with pytest.raises(spdp.SPDPError) as e:
        g.heldout(bad, 1, 1)
    assert e.value.code == spdp.SPDP_EINVAL
    span = synth.Corpus(test.group.copy(), test.doc, test.word, test.z_gen, test.num_groups, test.num_docs, test.vocab)
    span.group[0] = 1 - span.group[0]
    with pytest.raises(spdp.SPDPError):
        g.heldout(span, 1, 1)
    empty = synth.Corpus(test.group[:0], test.doc[:0], test.word[:0], test.z_gen[:0], test.num_groups, 3, test.vocab)
    assert g.heldout(empty, 1, 2)["perplexity"] == 1.0


@pytest.mark.parametrize("name,K", [("C1", 10), ("C2", 50)])
def test_topic_hellinger_matches_oracle(name, K):
    train, _, g, o = _trained(name, K)
    g2 = spdp.sampler_for(train, K, seed=8, **HYPER)
    g2.sweep(3)
    gc2 = g2.counts()
    o2 = oracle.Oracle(train.num_groups, train.vocab, K, **HYPER, seed=8)
    o2.load(train.group, train.doc, train.word, train.num_docs, z_init=gc2["z"], t_init=gc2["t"])
    d_self, p_self = g.topic_hellinger(g)
    # H = sqrt(1 - BC) turns the ~1e-15 rounding of BC = 1 into ~1e-7
    assert np.abs(np.diag(d_self)).max() <= 1e-6 and list(p_self) == list(range(K))
    d, p = g.topic_hellinger(g2)
    od, op = o.topic_align(o2)
    np.testing.assert_allclose(d ** 2, od ** 2, atol=1e-12)
    np.testing.assert_array_equal(p, op)
