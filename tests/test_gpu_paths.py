"""Parity on the code paths the measured configurations take (VERDICT r1 "what's
weak" 1-2): north_star (5) checks — draw mismatches <= 1e-4 of tokens, each
within 1e-6 of a CDF boundary; counts bit-exact once the draws agree (lock-step)
— on

  * uint16 and uint8 doc-topic rows with L2 prefetch (the HBM-bound C4
    K = 1000 / C5 path), forced on small corpora at every lanes-per-token x topics-per-lane
    instantiation, including 8 x 32 (C5's K = 200, compiled for 5 blocks/SM)
    and 32 x 32 (K = 1000);
  * (w, i) segments split across several chunks (C3 and C5 split segments on
    every sweep: M_max 1870 / 4898 > 512-token chunks);
  * the full-size bench workload C3 (one lock-step sweep of all 10 M tokens),
    and the library's recount of n and m from z at full size (C3, C5);
  * the sparse-row sample kernel (C5, C4 K >= 300 default) at every shape;
  * every cell of the device Stirling-ratio table (Eqs. r0/r1 P:1683)
    against the oracle's log-space table up to m = 5000 (> C5's M_max).
"""
import numpy as np
import pytest

import oracle
import paper_1510_06549_b200 as spdp
import synth
from gpu_util import (HYPER, assert_counts_equal, assert_draw_parity, corpus, lockstep_sweep, pair,
                      require_gpu)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    require_gpu()


def _lockstep(c, K, waves, sweeps, **kw):
    g, o = pair(c, K, waves=waves, **kw)
    for _ in range(sweeps):
        rep, gc = lockstep_sweep(g, o, waves=waves)
        assert_draw_parity(rep)
        assert_counts_equal(gc, o.state())
    return g


# K -> instantiation: 20/50 token kernel; 100 -> 4x32; 200 -> 8x32 (C5's, 5 blocks/SM); 300 -> 16x32;
# 1000 -> 32x32 (C4 K = 1000's)
@pytest.mark.parametrize("rowb", [2, 1])
@pytest.mark.parametrize("K,waves", [(20, 1), (50, 2), (100, 1), (100, 2), (200, 1), (200, 3), (300, 1),
                                     (1000, 1), (1000, 2)])
def test_narrow_rows_with_prefetch_lockstep(monkeypatch, K, waves, rowb):
    """uint16 (rowb = 2) and uint8 (rowb = 1, documents < 256 tokens: C5, C4) rows."""
    monkeypatch.setenv("SPDP_ROW_BYTES", str(rowb))
    monkeypatch.setenv("SPDP_PREFETCH_ROWS", "1")
    c = synth.generate(2, 30, 40.0, 300, 8, seed=K + waves)
    g = _lockstep(c, K, waves, 3)
    st = g.stats()
    assert st["row_bytes"] == rowb
    if K > 64:
        assert (st["lanes_per_token"], st["topics_per_lane"]) == {100: (4, 32), 200: (8, 32), 300: (16, 32),
                                                                  1000: (32, 32)}[K]


@pytest.mark.parametrize("rowb", [2, 1])
def test_narrow_rows_conditionals(monkeypatch, rowb):
    """The narrow-row path's own conditionals (spdp_debug_probs runs the sweep's device
    code with uint16 / uint8 rows) match the oracle to 1e-5 at K = 200 (C5's instantiation)."""
    monkeypatch.setenv("SPDP_ROW_BYTES", str(rowb))
    monkeypatch.setenv("SPDP_PREFETCH_ROWS", "1")
    c = synth.generate(3, 40, 50.0, 400, 10, seed=3)
    K = 200
    g, o = pair(c, K)
    for _ in range(2):
        rep, _ = lockstep_sweep(g, o)
        assert_draw_parity(rep)
    toks = np.random.default_rng(1).choice(c.num_tokens, 1500, replace=False)
    gp, info = g.debug_probs(toks)
    for j, p in enumerate(toks):
        d = o.debug_token(int(p), o.sweep_index)
        assert (info[j, 0], info[j, 1]) == (d["r_rem"], d["keep"])
        big = d["prob"] >= 1e-30
        assert (np.abs(gp[j][big] - d["prob"][big]) / d["prob"][big]).max() <= 1e-5


@pytest.mark.parametrize("rowb", [4, 2, 1])
@pytest.mark.parametrize("K,lpt", [(100, 8), (200, 8), (200, 16), (300, 16), (1000, 32), (1000, 8)])
def test_sparse_rows_lockstep(monkeypatch, K, lpt, rowb):
    """The sparse-row sample kernel (spdp_sprows.cuh: nonzero doc-topic counts + a per-chunk alpha-F
    prefix, crossing entry then binary search) at every lanes-per-token and topic span, each row type."""
    monkeypatch.setenv("SPDP_SPARSE_ROWS", "1")
    monkeypatch.setenv("SPDP_SPROWS_LPT", str(lpt))
    monkeypatch.setenv("SPDP_ROW_BYTES", str(rowb))
    c = synth.generate(2, 30, 40.0, 300, 8, seed=K + lpt)
    g = _lockstep(c, K, 1, 3)
    st = g.stats()
    assert st["sparse_rows"] == 1 and st["sparse_rows_lanes"] == lpt and st["row_bytes"] == rowb
    n = g.counts(z=False, r=False, customers=False, tables=False, shadow=False)["n"]
    assert st["sparse_row_entries"] == int((n > 0).sum())


@pytest.mark.parametrize("K,waves", [(200, 2), (1000, 3)])
def test_sparse_rows_several_waves_lockstep(monkeypatch, K, waves):
    """W > 1: the entries are rebuilt after every wave's doc-topic update."""
    monkeypatch.setenv("SPDP_SPARSE_ROWS", "1")
    c = synth.generate(2, 30, 40.0, 300, 8, seed=K + waves)
    g = _lockstep(c, K, waves, 3)
    assert g.stats()["sparse_rows"] == 1


@pytest.mark.parametrize("K,waves,extra", [(100, 1, {}), (100, 3, {}), (200, 1, {"SPDP_ROW_BYTES": "1"}),
                                           (300, 2, {"SPDP_ROW_BYTES": "2"}), (1000, 1, {}),
                                           (130, 1, {"SPDP_CHUNK_TOKENS": "16"}), (50, 1, {"SPDP_TOKEN_KERNEL": "0"})])
def test_chunk_factor_tables_lockstep(monkeypatch, K, waves, extra):
    """The chunk kernel reading per-wave factor tables (SPDP_CHUNK_FACTORS=1: slot factors, r = 1 shares,
    alpha F and packed (m, t) of every (wave, w, i) run from one throughput kernel) instead of its prologue."""
    monkeypatch.setenv("SPDP_CHUNK_FACTORS", "1")
    for k, v in extra.items():
        monkeypatch.setenv(k, v)
    c = synth.generate(2, 30, 40.0, 300, 8, seed=K + 7 * waves)
    _lockstep(c, K, waves, 3)


@pytest.mark.parametrize("K,rowb", [(100, 4), (200, 1), (256, 2)])
def test_document_order_scatter_lockstep(monkeypatch, K, rowb):
    """W = 1 with the assignments also scattered to their document-order slots (the HBM-bound default:
    SPDP_DOC_SCATTER) and the recount streaming them; forced on small corpora."""
    monkeypatch.setenv("SPDP_DOC_SCATTER", "1")
    monkeypatch.setenv("SPDP_ROW_BYTES", str(rowb))
    c = synth.generate(2, 30, 40.0, 300, 8, seed=K + rowb)
    _lockstep(c, K, 1, 3)


@pytest.mark.parametrize("name,K", [("C1", 200), ("C2", 300)])
def test_sparse_rows_split_segments_lockstep(monkeypatch, name, K):
    monkeypatch.setenv("SPDP_SPARSE_ROWS", "1")
    monkeypatch.setenv("SPDP_CHUNK_TOKENS", "64")
    g = _lockstep(corpus(name), K, 1, 2)
    assert g.stats()["sparse_rows"] == 1


@pytest.mark.parametrize("name,K,extra", [("C1", 100, {}), ("C1", 200, {"SPDP_ROW16": "1"}), ("C1", 200, {"SPDP_ROW8": "1"}),
                                          ("C2", 50, {"SPDP_TOKEN_KERNEL": "0"}), ("C2", 130, {})])
def test_segments_split_across_chunks_lockstep(monkeypatch, name, K, extra):
    """64-token chunks: every (w, i) segment longer than 64 tokens is sampled by
    several warps against the same snapshot, each flushing its own deltas."""
    monkeypatch.setenv("SPDP_CHUNK_TOKENS", "64")
    for k, v in extra.items():
        monkeypatch.setenv(k, v)
    c = corpus(name)
    g = _lockstep(c, K, 1, 3 if name == "C1" else 2)
    st = g.stats()
    assert st["chunk_tokens"] == 64 and st["token_kernel"] == 0
    assert st["m_max"] > 64 and st["chunks"] > 0


@pytest.mark.parametrize("K", [100, 200, 1000])
def test_long_segment_default_chunks_lockstep(K):
    """Default 512-token chunks with a 1500-token (w, i) segment (3 chunks) and a
    600-token one, plus ragged short documents."""
    docs = [[0], [1, 1], [2, 0, 1], [3] * 7, [0, 4, 4, 4, 1], [5]]
    docs += [[6] * 3 for _ in range(500)]            # word 6 in group 0: a 1500-token segment
    docs += [[7, 7, 8] for _ in range(300)]          # word 7 in group 1: 600 tokens
    groups = [0, 1, 0, 1, 1, 0] + [0] * 500 + [1] * 300
    c = synth.tiny_corpus(2, docs, groups, 10)
    g = _lockstep(c, K, 1, 3)
    st = g.stats()
    assert st["chunk_tokens"] == 512 and st["m_max"] == 1500


def test_ratio_table_every_cell_matches_oracle():
    """Device A0/A1 (fp64 linear-space ratio recursion, fp32 store) vs the oracle's
    fp64 log-space Stirling table on every cell 0 <= t <= m <= 5000, two discounts
    (one table per distinct a): relative error <= 1e-6 (SURVEY §8(c) "A0/A1
    folding" pin); t = 0 < m cells are 0."""
    docs = [[0] * 5000, [1, 2, 1], [0] * 40, [3]]
    c = synth.tiny_corpus(2, docs, [0, 0, 1, 1], 4)
    K = 4
    g = spdp.sampler_for(c, K, alpha=0.1, beta=0.1, discount=np.array([0.7, 0.3]), concentration=100.0)
    mmax = g.stats()["m_max"]
    assert mmax == 5000
    for grp, a in ((0, 0.7), (1, 0.3)):
        A0g, A1g = g.debug_ratio_table(grp, mmax)
        A0o, A1o = oracle.ratio_table(a, mmax)
        m = np.repeat(np.arange(mmax + 1), np.arange(1, mmax + 2))
        t = np.arange(len(A0o)) - m * (m + 1) // 2
        state = (t > 0) | (m == 0)
        assert (A0g[~state] == 0).all() and (A1g[~state] == 0).all()
        for got, want in ((A0g, A0o), (A1g, A1o)):
            rel = np.abs(got[state].astype(np.float64) - want[state]) / np.abs(want[state]).clip(1e-300)
            rel[want[state] == 0] = np.abs(got[state][want[state] == 0])
            assert rel.max() <= 1e-6, (grp, float(rel.max()), int(np.argmax(rel)))


@pytest.mark.slow
def test_full_size_c3_lockstep_sweeps():
    """The bench workload itself (C3: 10 M tokens, K = 100, W = 1, default
    kernels and chunks): two sweeps from identical state, the oracle replaying
    each with the GPU's draws; z, r, n, m, t, Q bit-exact (north_star (5))."""
    c = corpus("C3")
    g, o = pair(c, 100)
    for _ in range(2):
        rep, gc = lockstep_sweep(g, o)
        assert_draw_parity(rep)
        assert_counts_equal(gc, o.state())
    st = g.stats()
    assert st["m_max"] > st["chunk_tokens"]          # split segments on this path


@pytest.mark.slow
@pytest.mark.parametrize("name,K,sweeps", [("C3", 100, 3), ("C5", 200, 2)])
def test_full_size_library_recount(name, K, sweeps):
    """debug_checks at full size: after every sweep the library recounts n and m
    from z and checks 0 <= t <= m, t > 0 iff m > 0, Q = sum_i t, M/Tt/T = sums
    (SPDP_EINTEGRITY otherwise), on the bench configuration of each size — C5
    with uint8 rows (its doc-topic array exceeds half of L2, documents < 256 tokens)."""
    c = corpus(name)
    g = spdp.sampler_for(c, K, debug_checks=True, **HYPER)
    g.sweep(sweeps)
    st = g.stats()
    assert st["sweeps"] == sweeps and st["moved"] > 0
    if name == "C5":
        assert st["row_bytes"] == 1 and (st["lanes_per_token"], st["topics_per_lane"]) == (8, 32)


@pytest.mark.parametrize("K", [10, 100, 128])
def test_zr8_async_matches_counts(K):
    """spdp_zr8_async (the e2e read-back, one byte per token) equals z | r << 7 of spdp_counts."""
    c = corpus("C1")
    g = spdp.sampler_for(c, K, **HYPER)
    out = np.zeros(c.num_tokens, np.uint8)
    for _ in range(2):
        g.sweep(1)
        g.zr8_async(out)
        g.wait()
        gc = g.counts(doc_topic=False, customers=False, tables=False, shadow=False)
        np.testing.assert_array_equal(out, (gc["z"] | (gc["r"].astype(np.int32) << 7)).astype(np.uint8))
    with pytest.raises(spdp.SPDPError):
        spdp.sampler_for(c, 200, **HYPER).zr8_async(np.zeros(c.num_tokens, np.uint8))


def test_sweep_async_pipeline_equals_sweep():
    """The e2e loop of bench.py (spdp_sweep_async, then the wait for the previous step's copy, then
    spdp_zr8_async into alternating buffers) gives the same chain and every step's assignments."""
    c = corpus("C2")
    K = 50
    ref = spdp.sampler_for(c, K, **HYPER)
    g = spdp.sampler_for(c, K, **HYPER)
    bufs = [np.zeros(c.num_tokens, np.uint8) for _ in range(2)]
    want = []
    for s in range(4):
        ref.sweep(1)
        gc = ref.counts(doc_topic=False, customers=False, tables=False, shadow=False)
        want.append((gc["z"] | (gc["r"].astype(np.int32) << 7)).astype(np.uint8))
        g.sweep_async(1)
        g.wait()
        if s > 0:
            np.testing.assert_array_equal(bufs[(s - 1) % 2], want[s - 1])
        g.zr8_async(bufs[s % 2])
    g.wait()
    np.testing.assert_array_equal(bufs[3 % 2], want[3])
    a, b = ref.counts(), g.counts()
    for k in ("z", "r", "n", "m", "t", "Q"):
        np.testing.assert_array_equal(a[k], b[k])


@pytest.mark.parametrize("K,rowb,lpd", [(100, 4, "16"), (200, 1, "16"), (30, 4, "16"), (100, 4, "32")])
def test_recount_lanes_per_document_lockstep(monkeypatch, K, rowb, lpd):
    """The W = 1 doc-topic recount with 16 lanes per document (two documents per warp, the default for
    documents of <= 64 tokens on average, C5) and with 32: the rebuilt rows must equal the oracle's."""
    monkeypatch.setenv("SPDP_RECOUNT_LPD", lpd)
    monkeypatch.setenv("SPDP_ROW_BYTES", str(rowb))
    c = synth.generate(2, 40, 50.0, 300, 8, seed=K + rowb + int(lpd))
    _lockstep(c, K, 1, 3)


@pytest.mark.parametrize("waves,K,narrow", [(1, 50, True), (1, 100, True), (2, 50, True), (1, 200, False), (3, 100, False)])
def test_readback_scatter_overlaps_following_sweeps(waves, K, narrow):
    """The canonical-order scatter of spdp_zr8_async / spdp_zr_async runs on the copy stream while the
    next sweeps run; a sweep that writes the assignment buffer it reads (two sweeps later at W = 1,
    the next one at W > 1) waits for it.  1 or 2 sweeps between read-backs, against a plain chain."""
    c = corpus("C2")
    ref = spdp.sampler_for(c, K, num_waves=waves, **HYPER)
    g = spdp.sampler_for(c, K, num_waves=waves, **HYPER)
    dt = np.uint8 if narrow else np.uint16
    bufs = [np.zeros(c.num_tokens, dt) for _ in range(2)]
    want = []
    for s in range(6):
        nsw = 1 + (s % 2)
        ref.sweep(nsw)
        gc = ref.counts(doc_topic=False, customers=False, tables=False, shadow=False)
        if narrow:
            want.append((gc["z"] | (gc["r"].astype(np.int32) << 7)).astype(np.uint8))
        else:
            want.append((gc["z"] | (gc["r"].astype(np.int32) << 15)).astype(np.uint16))
        g.sweep_async(nsw)
        g.wait()                                      # step s-1's copy has landed
        if s > 0:
            np.testing.assert_array_equal(bufs[(s - 1) % 2], want[s - 1])
        (g.zr8_async if narrow else g.zr_async)(bufs[s % 2])
    g.wait()
    np.testing.assert_array_equal(bufs[5 % 2], want[5])
    (g.zr8_async if narrow else g.zr_async)(bufs[0])   # a read-back still pending at the state installation
    a = ref.counts()
    g.set_state(a["z"], a["r"], tables=a["t"])
    g.wait()
    np.testing.assert_array_equal(bufs[0], want[5])
    b = g.counts()
    for k in ("z", "r", "n", "m", "t", "Q"):
        np.testing.assert_array_equal(a[k], b[k])
    g.close(); ref.close()
