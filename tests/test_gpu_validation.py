"""spdp_load_corpus input validation on the device (validate_tokens_kernel, warp-aggregated per
document): out-of-range triples and documents spanning groups fail with SPDP_EINVAL; document
lengths of a valid corpus (the CSR the W = 1 recount uses) match a host recount."""
import numpy as np
import pytest

import paper_1510_06549_b200 as spdp
import synth
from gpu_util import require_gpu

pytestmark = pytest.mark.gpu


def _load(group, doc, word, num_docs, I=2, V=50, K=8):
    h = spdp.Sampler(I, V, K, alpha=0.1, beta=0.1, discount=0.7, concentration=10.0, seed=3)
    try:
        h.load_corpus(np.asarray(group, np.int32), np.asarray(doc, np.int32), np.asarray(word, np.int32), num_docs)
    finally:
        h.close()


def test_out_of_range_token_is_rejected():
    require_gpu()
    n = 4000
    rng = np.random.default_rng(1)
    doc = np.sort(rng.integers(0, 40, n)).astype(np.int32)
    group = (doc % 2).astype(np.int32)
    word = rng.integers(0, 50, n).astype(np.int32)
    word[1234] = 50                                   # V = 50
    with pytest.raises(spdp.SPDPError) as e:
        _load(group, doc, word, 40)
    assert e.value.code == spdp.SPDP_EINVAL and "out of range" in str(e.value)


@pytest.mark.parametrize("where", ["same_warp", "other_warp"])
def test_document_spanning_groups_is_rejected(where):
    require_gpu()
    n = 4000
    rng = np.random.default_rng(2)
    doc = np.sort(rng.integers(0, 40, n)).astype(np.int32)   # consecutive tokens share documents
    group = (doc % 2).astype(np.int32)
    word = rng.integers(0, 50, n).astype(np.int32)
    d = int(doc[2000])
    idx = np.nonzero(doc == d)[0]
    j = idx[1] if where == "same_warp" else idx[-1]
    group[j] = 1 - group[j]
    with pytest.raises(spdp.SPDPError) as e:
        _load(group, doc, word, 40)
    assert e.value.code == spdp.SPDP_EINVAL and "spans several groups" in str(e.value)


def test_valid_corpus_loads_and_counts_match():
    require_gpu()
    c = synth.generate(2, 60, 40.0, 300, 5, seed=4)
    g = spdp.sampler_for(c, 12, seed=5, alpha=0.1, beta=0.1, discount=0.7, concentration=10.0)
    try:
        cnt = g.counts()
        n = cnt["n"]
        assert np.array_equal(n.sum(axis=1), np.bincount(c.doc, minlength=c.num_docs))
        g.sweep(2)
        n2 = g.counts()["n"]
        assert np.array_equal(n2.sum(axis=1), np.bincount(c.doc, minlength=c.num_docs))
    finally:
        g.close()
