"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (W = 1, default kernels): sampled outputs the oracle computes one by one
(the sweep's own conditionals via spdp_debug_probs, on tokens drawn across the
corpus, from the GPU's state after a few sweeps), and properties that hold at
any size (count invariants after the sweeps, the Stirling-table edge K)."""
import numpy as np
import pytest

import oracle
import paper_1510_06549_b200 as spdp
import synth
from gpu_util import HYPER, require_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    require_gpu()


def _state_oracle(c, K, g):
    gc = g.counts()
    o = oracle.Oracle(c.num_groups, c.vocab, K, **HYPER, seed=7)
    o.load(c.group, c.doc, c.word, c.num_docs, z_init=gc["z"], t_init=gc["t"])
    o.sweep_index = g.stats()["sweeps"]
    return gc, o


def _check_conditionals(g, o, toks):
    gp, info = g.debug_probs(toks)
    worst = 0.0
    for j, p in enumerate(toks):
        d = o.debug_token(int(p), o.sweep_index)
        assert (info[j, 0], info[j, 1]) == (d["r_rem"], d["keep"]), (p, info[j], d)
        op = d["prob"]
        big = op >= 1e-30
        worst = max(worst, float((np.abs(gp[j][big] - op[big]) / op[big]).max()))
        assert np.abs(gp[j][~big] - op[~big]).max(initial=0.0) <= 1e-12
        if d["margin"] > 1e-6:
            assert (info[j, 2], info[j, 3]) == (d["z"], d["r"]), (p, info[j], d)
    assert worst <= 1e-5, worst


@pytest.mark.parametrize("name,K,sweeps,ntok", [("C3", 100, 3, 3000), ("C4", 1000, 1, 400)])
def test_full_size_sampled_conditionals(name, K, sweeps, ntok):
    """C3 (the bench workload, 10 M tokens) and C4 at K = 1000 (the largest K
    configuration): after a few sweeps, the conditionals of tokens sampled across
    the corpus match the oracle's to 1e-5, with the same draws away from CDF
    boundaries; the count invariants hold on the full state."""
    c = synth.corpus_for(synth.CONFIGS[name])
    g = spdp.sampler_for(c, K, **HYPER)
    g.sweep(sweeps)
    gc, o = _state_oracle(c, K, g)
    assert gc["m"].sum() == c.num_tokens and gc["n"].sum() == c.num_tokens
    assert (gc["t"] <= gc["m"]).all() and ((gc["t"] > 0) == (gc["m"] > 0)).all()
    np.testing.assert_array_equal(gc["Q"], gc["t"].sum(axis=0).T)
    assert o.check_invariants() == 0
    rng = np.random.default_rng(11)
    toks = np.sort(rng.choice(c.num_tokens, size=ntok, replace=False))
    _check_conditionals(g, o, toks)


def test_maximum_K_and_ragged_tiny_corpus_lockstep():
    """K = 1024 (the maximum) on a tiny ragged corpus (documents of 1..7 tokens,
    one segment longer than a chunk): one sweep from identical state is the
    oracle's, bit for bit when the draws agree."""
    docs = [[0], [1, 1], [2, 0, 1], [3] * 7, [0, 4, 4, 4, 1], [5]]
    docs += [[6] * 3 for _ in range(200)]            # word 6 in group 0: a 600-token segment (> 512-token chunks)
    c = synth.tiny_corpus(2, docs, [0, 1, 0, 1, 1, 0] + [0] * 200, 8)
    from gpu_util import assert_counts_equal, assert_draw_parity, lockstep_sweep, pair
    for K in (1024, 1):
        g, o = pair(c, K)
        for _ in range(2):
            rep, gc = lockstep_sweep(g, o)
            assert_draw_parity(rep)
            if rep["mismatch"] == 0:
                assert_counts_equal(gc, o.state())
