"""A short sweep job for ncu captures (not a measurement):
    python tools/prof_sweeps.py --config C5 [--topics K] [--waves W] [--sweeps 4] [--update async]
Loads the config's synthetic corpus and runs --sweeps sweeps one call at a time (SPDP_GRAPHS=0 unless
set, so every kernel is a plain launch)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SPDP_GRAPHS", "0")

import paper_1510_06549_b200 as spdp  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--topics", type=int, default=0)
ap.add_argument("--waves", type=int, default=1)
ap.add_argument("--sweeps", type=int, default=4)
ap.add_argument("--update", default="wave", choices=["wave", "async"])
ap.add_argument("--transform", default="none", choices=["none", "mix"])
ap.add_argument("--nnz", action="store_true", help="print the distribution of nonzero doc-topic counts per document")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
K = a.topics or cfg.k
c = synth.corpus_for(cfg)
tr = None
if a.transform == "mix":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import mixing_transform
    tr = mixing_transform(cfg.groups, cfg.vocab, cfg.seed)
g = spdp.sampler_for(c, K, alpha=cfg.alpha, beta=cfg.beta, discount=cfg.discount, concentration=cfg.concentration,
                     seed=cfg.seed, num_waves=a.waves, transform=tr,
                     update_mode=spdp.SPDP_UPDATE_ASYNC if a.update == "async" else spdp.SPDP_UPDATE_WAVE)
for _ in range(a.sweeps):
    g.sweep(1)
print(a.config, K, a.waves, g.stats(), flush=True)
if a.nnz:
    import numpy as np
    n = g.counts(z=False, r=False, customers=False, tables=False, shadow=False)["n"]
    nz = (n > 0).sum(axis=1)
    L = n.sum(axis=1)
    print("nnz per doc: mean %.2f p50 %d p90 %d max %d; doc length mean %.2f max %d; nnz/K %.3f" % (
        nz.mean(), np.percentile(nz, 50), np.percentile(nz, 90), nz.max(), L.mean(), L.max(), nz.mean() / K), flush=True)
g.close()
