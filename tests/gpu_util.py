"""Helpers for the -m gpu parity tests: the CUDA path vs the oracle."""
import numpy as np
import pytest

import oracle
import paper_1510_06549_b200 as spdp
import synth

HYPER = dict(alpha=0.1, beta=0.1, discount=0.7, concentration=100.0)


def require_gpu():
    try:
        spdp.build()
        spdp.Sampler(1, 1, 1).close()
    except spdp.SPDPError as e:
        if e.code == spdp.SPDP_ECUDA:
            pytest.skip(f"no CUDA device: {e}")
        raise


def pack(z, r):
    return (np.asarray(z, np.int32) | (np.asarray(r, np.int32) << 15)).astype(np.int32)


def pair(corpus, K, seed=7, waves=1, hyper=HYPER, z_init=None, r_init=None, **kw):
    """A GPU sampler and an oracle at the same initial state."""
    g = spdp.sampler_for(corpus, K, seed=seed, num_waves=waves, z_init=z_init, r_init=r_init, **hyper, **kw)
    o = oracle.from_corpus(corpus, K, seed=seed, z_init=z_init, r_init=r_init, **hyper)
    return g, o


def lockstep_sweep(g, o, waves=1, shards=1, gpu_counts=None):
    """One GPU sweep; the oracle replays the same sweep with every draw forced to
    the GPU's, reporting its own draws and margins.  Returns (report, gpu counts).

    north_star (5): draw mismatches <= 1e-4 of tokens, each with the uniform
    within 1e-6 of a CDF boundary; counts bit-exact once the draws agree."""
    if gpu_counts is None:
        g.sweep(1)
        gpu_counts = g.counts(customers=False, tables=False, shadow=False, doc_topic=False)
        gpu_counts.update(g.counts(z=False, r=False))
    forced = pack(gpu_counts["z"], gpu_counts["r"])
    margin, own = o.sweep_par(waves=waves, shards=shards, force_zr=forced, want_margin=True, want_own=True)
    mism = np.nonzero(own != forced)[0]
    rep = {"mismatch": len(mism), "N": len(forced), "max_margin": float(margin[mism].max()) if len(mism) else 0.0}
    return rep, gpu_counts


def assert_counts_equal(gc, oc, keys=("z", "r", "n", "m", "t", "Q")):
    for k in keys:
        np.testing.assert_array_equal(gc[k], oc[k], err_msg=f"count table {k} differs")


def assert_draw_parity(rep):
    assert rep["mismatch"] <= max(1, 1e-4 * rep["N"]), rep
    assert rep["max_margin"] <= 1e-6, rep


def corpus(name):
    return synth.corpus_for(synth.CONFIGS[name])
