"""GPU parity: the CUDA path (through the C ABI) against the oracle.

north_star (5): conditional probabilities within 1e-5 relative error; draw
mismatches <= 1e-4 of tokens and only where the uniform lies within 1e-6 of
a CDF boundary; count tables bit-exact whenever the draws agree.
"""
import numpy as np
import pytest

import oracle
import paper_1510_06549_b200 as spdp
import synth
from gpu_util import (HYPER, assert_counts_equal, assert_draw_parity, corpus, lockstep_sweep, pack, pair,
                      require_gpu)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    require_gpu()


def _probs_parity(g, o, toks, sweep):
    gp, info = g.debug_probs(toks)
    for j, p in enumerate(toks):
        d = o.debug_token(int(p), sweep)
        assert (info[j, 0], info[j, 1]) == (d["r_rem"], d["keep"]), (p, info[j], d)
        op = d["prob"]
        big = op >= 1e-30
        rel = np.abs(gp[j][big] - op[big]) / op[big]
        assert rel.max() <= 1e-5, (p, rel.max())
        assert np.abs(gp[j][~big] - op[~big]).max(initial=0.0) <= 1e-12
        if d["margin"] > 1e-6:
            assert (info[j, 2], info[j, 3]) == (d["z"], d["r"]), (p, info[j], d)


@pytest.mark.parametrize("name,K", [("C1", 10), ("C2", 50)])
def test_conditionals_match_oracle(name, K):
    c = corpus(name)
    g, o = pair(c, K)
    rng = np.random.default_rng(0)
    toks = rng.choice(c.num_tokens, size=min(c.num_tokens, 3000), replace=False)
    _probs_parity(g, o, toks, 0)
    # after a few lock-step sweeps (non-trivial t, clamps)
    for _ in range(3):
        rep, gc = lockstep_sweep(g, o)
        assert_draw_parity(rep)
    _probs_parity(g, o, toks, o.sweep_index)


@pytest.mark.parametrize("name,K,waves", [("C1", 10, 1), ("C1", 10, 4), ("C1", 10, 200), ("C2", 50, 1),
                                          ("C2", 50, 3), ("C1", 100, 3), ("C1", 128, 2)])
def test_one_sweep_from_identical_state(name, K, waves):
    c = corpus(name)
    g, o = pair(c, K, waves=waves)
    rep, gc = lockstep_sweep(g, o, waves=waves)
    assert_draw_parity(rep)
    assert_counts_equal(gc, o.state())


def test_twenty_lockstep_sweeps_c1():
    c = corpus("C1")
    g, o = pair(c, 10, waves=1)
    for s in range(20):
        rep, gc = lockstep_sweep(g, o)
        assert_draw_parity(rep)
        assert_counts_equal(gc, o.state())
    st = g.stats()
    assert st["sweeps"] == 20


@pytest.mark.parametrize("K", [1, 3, 16, 17, 33, 100, 130, 300, 700, 1024])
def test_topic_counts_edge_cases(K):
    """Every kernel configuration (lanes-per-token x topics-per-lane), ragged K."""
    c = synth.generate(2, 30, 40.0, 300, 8, seed=K)
    g, o = pair(c, K, waves=2)
    for _ in range(2):
        rep, gc = lockstep_sweep(g, o, waves=2)
        assert_draw_parity(rep)
        assert_counts_equal(gc, o.state())


@pytest.mark.parametrize("forced,waves", [("0", 2), ("2", 1)])
def test_kernel_choice_override_lockstep(monkeypatch, forced, waves):
    """Both sample paths at 64 < K <= 128 whatever the automatic choice (it
    depends on the tokens per segment and wave): the chunk kernel with several
    waves (SPDP_TOKEN_KERNEL=0) and the token kernel with one (=2) stay in
    lock-step with the oracle."""
    monkeypatch.setenv("SPDP_TOKEN_KERNEL", forced)
    c = synth.generate(2, 40, 60.0, 200, 8, seed=5)
    g, o = pair(c, 100, waves=waves)
    assert g.stats()["token_kernel"] == (1 if forced == "2" else 0)
    for _ in range(2):
        rep, gc = lockstep_sweep(g, o, waves=waves)
        assert_draw_parity(rep)
        assert_counts_equal(gc, o.state())


def test_tiny_and_degenerate_corpora():
    # single-token docs, a doc with one repeated word, unused words and groups
    c = synth.tiny_corpus(3, [[0], [1, 1, 1, 1], [2, 0, 2], [5]], [0, 0, 1, 1], vocab=7)
    g, o = pair(c, 2, waves=1)
    for _ in range(5):
        rep, gc = lockstep_sweep(g, o)
        assert_draw_parity(rep)
        assert_counts_equal(gc, o.state())


def test_loglik_matches_oracle():
    c = corpus("C1")
    g, o = pair(c, 10)
    for _ in range(3):
        rep, gc = lockstep_sweep(g, o)
    lj, ppl = g.loglik()
    assert ppl == pytest.approx(o.perplexity(), rel=1e-9)
    assert lj == pytest.approx(o.log_joint(), rel=1e-9)


def test_determinism_and_invariants():
    c = corpus("C1")
    a = spdp.sampler_for(c, 10, seed=3, debug_checks=True, **HYPER)
    b = spdp.sampler_for(c, 10, seed=3, **HYPER)
    a.sweep(4); b.sweep(4)
    ca, cb = a.counts(), b.counts()
    for k in ca:
        np.testing.assert_array_equal(ca[k], cb[k])
    assert ca["m"].sum() == c.num_tokens
    assert (ca["t"] <= ca["m"]).all() and ((ca["t"] > 0) == (ca["m"] > 0)).all()
    np.testing.assert_array_equal(ca["Q"], ca["t"].sum(axis=0).T)


def test_set_state_roundtrip_with_tables():
    c = corpus("C1")
    g, o = pair(c, 10)
    for _ in range(2):
        lockstep_sweep(g, o)
    st = o.state()
    h = spdp.sampler_for(c, 10, **HYPER)
    h.set_state(st["z"], st["r"], st["t"])
    hc = h.counts()
    assert_counts_equal(hc, st, keys=("z", "n", "m", "t", "Q"))


@pytest.mark.parametrize("G,waves,pack", [(2, 1, 32), (3, 2, 32), (8, 1, 32), (2, 1, 64), (3, 2, 64)])
def test_multi_rank_exchange_matches_oracle_shards(G, waves, pack, monkeypatch):
    """G ranks as G contexts on one GPU with the external exchange (host sum of
    the packed dm*2^B + dt buffers, B = 16 and 32): bit-exact against the
    oracle's G-shard simulation (reading c13-c15)."""
    if pack == 64:
        monkeypatch.setenv("SPDP_EXCHANGE_PACK64", "1")
    c = corpus("C1")
    ranks = [spdp.sampler_for(c, 10, num_waves=waves, rank=r, world_size=G,
                              exchange=spdp.SPDP_EXCHANGE_EXTERNAL, **HYPER) for r in range(G)]
    o = oracle.from_corpus(c, 10, **HYPER)
    for s in range(3):
        for r in ranks:
            r.sweep_local()
        bufs = [r.exchange_get() for r in ranks]
        assert bufs[0].dtype == (np.int32 if pack == 32 else np.int64)
        with np.errstate(over="ignore"):
            tot = sum(b.astype(np.int64) for b in bufs).astype(bufs[0].dtype)   # wrapping integer sum
        for r in ranks:
            r.exchange_put(tot)
            r.sweep_merge()
        # gather the per-rank token state (each rank writes only its own tokens)
        z = np.full(c.num_tokens, -1, np.int32); rr = np.zeros(c.num_tokens, np.uint8)
        n = np.zeros((c.num_docs, 10), np.int32)
        for r in ranks:
            cr = r.counts()
            own = np.asarray(spdp.spdp_partition(7, G, c.doc, c.num_docs))[c.doc] == ranks.index(r)
            z[own] = cr["z"][own]; rr[own] = cr["r"][own]
            owndoc = np.asarray(spdp.spdp_partition(7, G, c.doc, c.num_docs)) == ranks.index(r)
            n[owndoc] = cr["n"][owndoc]
        gc = ranks[0].counts()
        gc.update(z=z, r=rr, n=n)
        for r in ranks[1:]:
            cr = r.counts()
            for k in ("m", "t", "Q"):
                np.testing.assert_array_equal(cr[k], gc[k])
        rep, _ = lockstep_sweep(None, o, waves=waves, shards=G, gpu_counts=gc)
        assert_draw_parity(rep)
        assert_counts_equal(gc, o.state())


def test_perplexity_trajectory_lockstep_c1_100_sweeps():
    """north_star (5), lock-step form: 100 sweeps of C1, counts bit-exact and the
    perplexity trajectories identical (to fp64 summation order)."""
    c = corpus("C1")
    g, o = pair(c, 10, waves=1)
    worst = 0
    for s in range(100):
        rep, gc = lockstep_sweep(g, o)
        assert_draw_parity(rep)
        worst = max(worst, rep["mismatch"])
        if s % 10 == 9:
            assert_counts_equal(gc, o.state(), keys=("m", "t", "Q", "n"))
            assert g.perplexity() == pytest.approx(o.perplexity(), rel=1e-9)


@pytest.mark.slow
def test_perplexity_trajectory_free_running_c2_100_sweeps():
    """north_star (5): the free-running 1-GPU chain stays within 1% of the oracle's
    (same seed, same corpus, W = 1) after 100 sweeps on C2 (1M tokens)."""
    c = corpus("C2")
    g, o = pair(c, 50, waves=1)
    traj = []
    for s in range(100):
        g.sweep(1)
        o.sweep_par(waves=1)
        if s % 10 == 9:
            traj.append((s + 1, g.perplexity(), o.perplexity()))
    last = traj[-1]
    assert abs(last[1] / last[2] - 1) <= 0.01, traj


@pytest.mark.parametrize("name,K", [("C1", 10), ("C1", 100), ("C2", 50)])
def test_word_range_parts_equal_single_wave(name, K, monkeypatch):
    """The sweep in P word-range parts (the exchange pipeline's schedule)
    is the same W = 1 sweep: identical state after 3 sweeps, for the token kernel
    (K <= 64) and the chunk kernel."""
    c = corpus(name)
    ref = spdp.sampler_for(c, K, **HYPER)
    ref.sweep(3)
    want = ref.counts()
    monkeypatch.setenv("SPDP_EXCHANGE_PARTS", "4")
    g = spdp.sampler_for(c, K, **HYPER)
    g.sweep(3)
    got = g.counts()
    for k in ("z", "r", "n", "m", "t", "Q"):
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    assert g.perplexity() == pytest.approx(ref.perplexity(), rel=1e-12)   # per-chunk partials in another order


@pytest.mark.parametrize("G", [2, 3])
def test_multi_rank_parts_match_oracle_shards(G, monkeypatch):
    """G ranks (external exchange) sampling in word-range parts: still the oracle's
    G-shard sweep, bit for bit."""
    monkeypatch.setenv("SPDP_EXCHANGE_PARTS", "3")
    c = corpus("C1")
    ranks = [spdp.sampler_for(c, 10, rank=r, world_size=G, exchange=spdp.SPDP_EXCHANGE_EXTERNAL, **HYPER)
             for r in range(G)]
    o = oracle.from_corpus(c, 10, **HYPER)
    for s in range(2):
        for r in ranks:
            r.sweep_local()
        bufs = [r.exchange_get() for r in ranks]
        with np.errstate(over="ignore"):
            tot = sum(b.astype(np.int64) for b in bufs).astype(bufs[0].dtype)
        for r in ranks:
            r.exchange_put(tot)
            r.sweep_merge()
        z = np.full(c.num_tokens, -1, np.int32)
        for r in ranks:
            cr = r.counts()
            own = np.asarray(spdp.spdp_partition(7, G, c.doc, c.num_docs))[c.doc] == ranks.index(r)
            z[own] = cr["z"][own]
        forced = np.full(c.num_tokens, -1, np.int32)
        o.sweep_par(waves=1, shards=G)
        oc = o.state()
        mism = np.count_nonzero(z != oc["z"])
        assert mism <= max(1, 1e-4 * c.num_tokens), mism
        if mism == 0:
            for k in ("m", "t", "Q"):
                np.testing.assert_array_equal(ranks[0].counts()[k], oc[k], err_msg=k)


@pytest.mark.parametrize("G,waves,E", [(2, 4, 1), (3, 4, 2), (2, 3, 1)])
def test_bounded_staleness_exchange_matches_oracle(G, waves, E):
    """NEXT-3: ranks exchanging after every E waves (external exchange, G contexts on
    one GPU) follow the oracle's G-shard sweep with the same cadence."""
    c = corpus("C1")
    ranks = [spdp.sampler_for(c, 10, num_waves=waves, rank=r, world_size=G, merge_every=E,
                              exchange=spdp.SPDP_EXCHANGE_EXTERNAL, **HYPER) for r in range(G)]
    nb = ranks[0].exchange_blocks()
    assert nb == -(-waves // E)
    o = oracle.from_corpus(c, 10, **HYPER)
    part = np.asarray(spdp.spdp_partition(7, G, c.doc, c.num_docs))[c.doc]
    for s in range(2):
        for b in range(nb):
            for r in ranks:
                r.sweep_local()
            bufs = [r.exchange_get() for r in ranks]
            with np.errstate(over="ignore"):
                tot = sum(x.astype(np.int64) for x in bufs).astype(bufs[0].dtype)
            for r in ranks:
                r.exchange_put(tot)
                r.sweep_merge()
        o.sweep_par(waves=waves, shards=G, merge_every=E)
        oc = o.state()
        z = np.full(c.num_tokens, -1, np.int32)
        for j, r in enumerate(ranks):
            z[part == j] = r.counts()["z"][part == j]
        mism = np.count_nonzero(z != oc["z"])
        assert mism <= max(1, 1e-4 * c.num_tokens), mism
        if mism == 0:
            got = ranks[0].counts()
            for k in ("m", "t", "Q"):
                np.testing.assert_array_equal(got[k], oc[k], err_msg=k)


def test_duplicated_corpus_parity():
    """NEXT-3 duplication: the duplicated corpus is an ordinary input; one lock-step
    sweep against the oracle on it."""
    c = synth.duplicate(corpus("C1"), 1)
    assert c.num_tokens == 2 * corpus("C1").num_tokens
    g, o = pair(c, 10)
    rep, gc = lockstep_sweep(g, o)
    assert_draw_parity(rep)
    assert_counts_equal(gc, o.state())


def test_packed_assignments_match_counts():
    c = corpus("C1")
    g = spdp.sampler_for(c, 10, **HYPER)
    g.sweep(2)
    cnt = g.counts(doc_topic=False, customers=False, tables=False, shadow=False)
    zr = g.zr()
    np.testing.assert_array_equal(zr & 0x7FFF, cnt["z"])
    np.testing.assert_array_equal(zr >> 15, cnt["r"])


def test_async_assignment_copies_overlap_sweeps():
    """spdp_zr_async (include/spdp.h): copies queued between sweeps land by
    spdp_wait, each holding the state of its own step; a synchronous spdp_zr and
    spdp_counts after a pending copy see the current state."""
    import torch
    c = corpus("C2")
    g = spdp.sampler_for(c, 50, **HYPER)
    ref = spdp.sampler_for(c, 50, **HYPER)
    bufs = [torch.empty(c.num_tokens, dtype=torch.int16, pin_memory=True).numpy().view(np.uint16)
            for _ in range(3)]
    for s in range(3):
        g.sweep(1)
        g.zr_async(bufs[s])
    cnt = g.counts(doc_topic=False, customers=False, tables=False, shadow=False)   # ordered after the copies
    g.wait()
    for s in range(3):
        ref.sweep(1)
        np.testing.assert_array_equal(bufs[s], ref.zr())
    np.testing.assert_array_equal(bufs[2] & 0x7FFF, cnt["z"])
    g.sweep(1)
    g.zr_async(bufs[0])
    now = g.zr()                                             # after the queued copy, same state
    g.wait()
    np.testing.assert_array_equal(bufs[0], now)
    g.close(); ref.close()


def test_call_order_and_input_errors():
    """The boundary's error behaviour (include/spdp.h): state errors for calls out of
    order, SPDP_EINVAL for invalid inputs, and the context stays usable after a
    rejected call."""
    c = corpus("C1")
    g = spdp.Sampler(c.num_groups, c.vocab, 10, **HYPER)
    for call in (lambda: g.sweep(1), lambda: g.counts(), lambda: g.loglik(), lambda: g.zr()):
        with pytest.raises(spdp.SPDPError) as e:
            call()
        assert e.value.code == spdp.SPDP_ESTATE
    bad = c.word.copy(); bad[5] = c.vocab
    with pytest.raises(spdp.SPDPError) as e:
        g.load_corpus(c.group, c.doc, bad, c.num_docs)
    assert e.value.code == spdp.SPDP_EINVAL
    g.close()
    g = spdp.Sampler(c.num_groups, c.vocab, 10, **HYPER)
    span = c.group.copy(); span[0] = 1 - span[0]           # document 0 now spans two groups
    with pytest.raises(spdp.SPDPError) as e:
        g.load_corpus(span, c.doc, c.word, c.num_docs)
    assert e.value.code == spdp.SPDP_EINVAL
    g.close()
    g = spdp.sampler_for(c, 10, **HYPER)
    with pytest.raises(spdp.SPDPError) as e:
        g.load_corpus(c.group, c.doc, c.word, c.num_docs)   # once per context
    assert e.value.code == spdp.SPDP_ESTATE
    z = np.full(c.num_tokens, 10, np.int32)                # z out of [0, K)
    with pytest.raises(spdp.SPDPError) as e:
        g.set_state(z)
    assert e.value.code == spdp.SPDP_EINVAL
    with pytest.raises(spdp.SPDPError) as e:
        g.sweep(-1)
    assert e.value.code == spdp.SPDP_EINVAL
    g.sweep(2)                                             # still usable
    assert g.counts()["m"].sum() == c.num_tokens
