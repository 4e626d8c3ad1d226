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
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
K = a.topics or cfg.k
c = synth.corpus_for(cfg)
g = spdp.sampler_for(c, K, alpha=cfg.alpha, beta=cfg.beta, discount=cfg.discount, concentration=cfg.concentration,
                     seed=cfg.seed, num_waves=a.waves,
                     update_mode=spdp.SPDP_UPDATE_ASYNC if a.update == "async" else spdp.SPDP_UPDATE_WAVE)
for _ in range(a.sweeps):
    g.sweep(1)
print(a.config, K, a.waves, g.stats(), flush=True)
g.close()
