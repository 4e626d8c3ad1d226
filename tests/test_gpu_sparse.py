"""GPU parity of NEXT-4 (sparse transformation matrices P^i)
through the C ABI: spdp_set_transform + spdp_sweep against the oracle's
sparse sampler (tests/test_oracle_sparse_p.py pins it), in lock-step: the
oracle replays each sweep with every draw forced to the GPU's (topic, table
indicator and source entry) and reports its own; mismatches only within 1e-6
of a CDF boundary; counts (m, t, q, Q) bit-exact when the draws agree."""
import numpy as np
import pytest

import oracle
import paper_1510_06549_b200 as spdp
from gpu_util import HYPER, corpus, require_gpu
from test_oracle_sparse_p import identity_P, mixing_P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    require_gpu()


def _pair(c, K, P, waves):
    g = spdp.sampler_for(c, K, num_waves=waves, transform=P, **HYPER)
    o = oracle.from_corpus(c, K, **HYPER)
    return g, o, oracle.SparseOracle(o, *P)


def _lockstep(g, sp, P, waves):
    pptr = np.asarray(P[0])
    g.sweep(1)
    gc = g.counts()
    gs = g.sparse_state()
    rows = pptr[np.asarray(sp.base._tok[0]) * sp.base.V + np.asarray(sp.base._tok[2])]
    S = pptr[np.asarray(sp.base._tok[0]) * sp.base.V + np.asarray(sp.base._tok[2]) + 1] - rows
    force = gc["z"] * (S + 1) + np.where(gc["r"] == 1, gs["src"], S)
    force = np.where(gs["src"] == -1, np.where(gc["r"] == 1, -1, force), force)   # kept tokens: no draw
    mg, own = sp.sweep_par(waves=waves, force=force.astype(np.int32), want_margin=True, want_own=True)
    drawn = force >= 0
    mism = np.nonzero(drawn & (own != force))[0]
    return gc, gs, mism, mg


@pytest.mark.parametrize("K,waves,kind", [(10, 1, "mix"), (10, 3, "mix"), (10, 1, "id"), (100, 1, "mix"),
                                          (37, 2, "mix")])
def test_sparse_sweep_lockstep(K, waves, kind):
    c = corpus("C1")
    P = identity_P(c.num_groups, c.vocab) if kind == "id" else mixing_P(c.num_groups, c.vocab, np.random.default_rng(1))
    g, o, sp = _pair(c, K, P, waves)
    for s in range(3):
        gc, gs, mism, mg = _lockstep(g, sp, P, waves)
        assert len(mism) <= max(1, 1e-4 * c.num_tokens), len(mism)
        assert (mg[mism] <= 1e-6).all(), mg[mism]
        st = sp.state()
        if len(mism) == 0:
            for k in ("z", "r", "n", "m", "t"):
                np.testing.assert_array_equal(gc[k], st[k], err_msg=k)
            np.testing.assert_array_equal(gs["q"], st["q"])
            np.testing.assert_array_equal(gs["Qs"], st["Qs"])
    assert (gs["q"] >= 0).all()


def test_sparse_transform_validation():
    c = corpus("C1")
    g = spdp.Sampler(c.num_groups, c.vocab, 10, **HYPER)
    pptr, pv, pp = mixing_P(c.num_groups, c.vocab, np.random.default_rng(2))
    bad = pp.copy(); bad[0] *= 0.5
    with pytest.raises(spdp.SPDPError) as e:
        g.set_transform(pptr, pv, bad)
    assert e.value.code == spdp.SPDP_EINVAL
    g.set_transform(pptr, pv, pp)
    g.load_corpus(c.group, c.doc, c.word, c.num_docs)
    with pytest.raises(spdp.SPDPError) as e:
        g.set_transform(pptr, pv, pp)
    assert e.value.code == spdp.SPDP_ESTATE
    assert np.isfinite(g.log_joint())


@pytest.mark.parametrize("K", [10, 37])
def test_sparse_estimators_match_oracle(K):
    """phi~ with sum_v p phi0~, training perplexity and held-out fold-in
    with a sparse P, GPU vs the oracle on the same state."""
    import synth
    train, test = synth.holdout_split(corpus("C1"), 0.1, seed=1)
    P = mixing_P(train.num_groups, train.vocab, np.random.default_rng(4))
    g, o, sp = _pair(train, K, P, 1)
    for s in range(2):
        gc, gs, mism, mg = _lockstep(g, sp, P, 1)
        assert len(mism) <= 1 and (mg[mism] <= 1e-6).all()     # lock-step: the oracle follows the GPU's draws
    p0g, pg = g.topics()
    p0o, po = sp.topics()
    np.testing.assert_allclose(p0g, p0o, rtol=1e-12)
    np.testing.assert_allclose(pg, po, rtol=1e-11)
    assert np.allclose(pg.sum(axis=2), 1.0, atol=1e-12)
    assert g.perplexity() == pytest.approx(sp.perplexity(), rel=1e-10)
    assert g.log_joint() == pytest.approx(sp.log_joint(), rel=1e-10)
    r = g.heldout(test, 3, 0)
    z = r["z"]
    zf, margin, own = sp.foldin(test.group, test.doc, test.word, test.num_docs, seed=3, iterations=1, z=z,
                                force_z=g.heldout(test, 3, 1, z_init=z)["z"], want_margin=True)
    res = g.heldout(test, 3, 0, z_init=zf)
    assert res["perplexity"] == pytest.approx(sp.heldout_perplexity(test.group, test.doc, test.word, test.num_docs, zf),
                                              rel=1e-10)


@pytest.mark.parametrize("G,waves", [(2, 1), (3, 2)])
def test_sparse_multi_rank_matches_oracle_shards(G, waves):
    """NEXT-4 on several ranks (G contexts on one GPU, external exchange of the
    m and q net changes): the oracle's G-shard sweep with sources, bit for bit
    when the draws agree."""
    c = corpus("C1")
    P = mixing_P(c.num_groups, c.vocab, np.random.default_rng(3))
    ranks = [spdp.sampler_for(c, 10, num_waves=waves, rank=r, world_size=G, exchange=spdp.SPDP_EXCHANGE_EXTERNAL,
                              transform=P, **HYPER) for r in range(G)]
    o = oracle.from_corpus(c, 10, **HYPER)
    sp = oracle.SparseOracle(o, *P)
    part = np.asarray(spdp.spdp_partition(7, G, c.doc, c.num_docs))[c.doc]
    for s in range(2):
        for r in ranks:
            r.sweep_local()
        bufs = [r.exchange_get() for r in ranks]
        tot = sum(b.astype(np.int64) for b in bufs).astype(np.int32)
        for r in ranks:
            r.exchange_put(tot)
            r.sweep_merge()
        sp.sweep_shards(waves=waves, shards=G)
        st = sp.state()
        z = np.full(c.num_tokens, -1, np.int32)
        for j, r in enumerate(ranks):
            z[part == j] = r.counts()["z"][part == j]
        mism = np.count_nonzero(z != st["z"])
        assert mism <= max(1, 1e-4 * c.num_tokens), mism
        if mism == 0:
            g0 = ranks[0].counts()
            for k in ("m", "t"):
                np.testing.assert_array_equal(g0[k], st[k], err_msg=k)
            gs = ranks[0].sparse_state()
            np.testing.assert_array_equal(gs["q"], st["q"])
            np.testing.assert_array_equal(gs["Qs"], st["Qs"])
            for r in ranks[1:]:
                np.testing.assert_array_equal(r.sparse_state()["q"], gs["q"])
