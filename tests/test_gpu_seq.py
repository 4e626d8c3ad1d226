"""W = 0 test mode: the exact sequential sampler — Algorithm 1
 with the keep rule (reading c5) — on the device, through
the C ABI.

  * lock-step against the oracle's one-token-wave sweep (mode P with W = 0,
    which the CPU pins show equals Alg.1 bit for bit): draw mismatches only
    within 1e-6 of a CDF boundary, counts bit-exact;
  * north_star (4) on the GPU itself: exact posterior enumeration on a
    4-token, K = 2 corpus vs the empirical (z, t)- and z-frequencies of
    10^6 device sweeps, within 3 sigma (100 batch means) — the same pin the
    oracle's mode S carries, now on the CUDA path.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import paper_1510_06549_b200 as spdp
import synth
from gpu_util import HYPER, assert_counts_equal, assert_draw_parity, corpus, lockstep_sweep, pair, require_gpu
from oracle.enumerate import TinyCorpus

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    require_gpu()


@pytest.mark.parametrize("name,K", [("C1", 10), ("C1", 100)])
def test_sequential_mode_lockstep(name, K):
    c = corpus(name)
    g, o = pair(c, K, waves=0)
    for _ in range(3):
        rep, gc = lockstep_sweep(g, o, waves=0)
        assert_draw_parity(rep)
        assert_counts_equal(gc, o.state())
    assert g.stats()["clamped"] == 0


def test_sequential_mode_ragged_and_uint16(monkeypatch):
    monkeypatch.setenv("SPDP_ROW16", "1")
    c = synth.tiny_corpus(3, [[0], [1, 1, 1, 1], [2, 0, 2], [5], [4] * 40], [0, 0, 1, 1, 2], vocab=7)
    g, o = pair(c, 3, waves=0)
    assert g.stats()["row_bytes"] == 2
    for _ in range(5):
        rep, gc = lockstep_sweep(g, o, waves=0)
        assert_draw_parity(rep)
        assert_counts_equal(gc, o.state())


def test_sequential_mode_rejects_several_ranks():
    with pytest.raises(spdp.SPDPError) as e:
        spdp.Sampler(2, 10, 4, num_waves=0, rank=0, world_size=2, exchange=spdp.SPDP_EXCHANGE_EXTERNAL)
    assert e.value.code == spdp.SPDP_EINVAL


@pytest.mark.slow
def test_device_chain_matches_exact_posterior_3sigma():
    """10^6 sequential device sweeps of the SURVEY A.2 corpus (K = 2): every (z, t)
    state's and every z's frequency within 3 sigma (batch means) of the exact
    posterior p(Z, T | W) by enumeration (oracle/enumerate.py)."""
    I, docs, dg, V, K = 2, [[0, 0], [0, 1]], [0, 1], 2, 2
    group, doc, word = [], [], []
    for d, ws in enumerate(docs):
        for w in ws:
            group.append(dg[d]); doc.append(d); word.append(w)
    fr = lambda x: Fraction(x).limit_denominator(1000)
    tc = TinyCorpus(group, doc, word, I, V, K, fr(HYPER["alpha"]), fr(HYPER["beta"]), fr(HYPER["discount"]),
                    fr(HYPER["concentration"]))
    post = tc.posterior()
    c = synth.tiny_corpus(I, docs, dg, V)
    g = spdp.sampler_for(c, K, seed=4242, num_waves=0, **HYPER)
    nsw, nb = 1_000_000, 100
    codes = g.debug_chain(nsw, tbase=5)
    N = tc.N
    cells = [(i, w, k) for i in range(I) for w in range(V) for k in range(K)]

    def code_of(z, t):
        return sum(z[p] * K ** p for p in range(N)) + K ** N * sum(t.get(cc, 0) * 5 ** j for j, cc in enumerate(cells))

    batches = codes.reshape(nb, -1)
    bad = []
    zmarg = {}
    for (z, tt), pv in post.items():
        zmarg[z] = zmarg.get(z, 0.0) + float(pv)
        hits = (batches == code_of(z, dict(tt))).mean(axis=1)
        mean, sig = hits.mean(), hits.std(ddof=1) / math.sqrt(nb)
        if abs(mean - float(pv)) > 3 * sig + 1e-12:
            bad.append(((z, tt), mean, float(pv), sig))
    zc = batches % (K ** N)
    for z, pv in zmarg.items():
        hits = (zc == sum(z[p] * K ** p for p in range(N))).mean(axis=1)
        mean, sig = hits.mean(), hits.std(ddof=1) / math.sqrt(nb)
        if abs(mean - pv) > 3 * sig + 1e-12:
            bad.append((z, mean, pv, sig))
    assert not bad, bad
    # every state the chain visits is a valid one
    valid = {code_of(z, dict(tt)) for (z, tt) in post}
    assert set(np.unique(codes).tolist()) <= valid
