"""NEXT-3 measurement: effect of the cross-rank exchange cadence
(bounded staleness) and of training-data duplication on model quality, with G
ranks simulated as G contexts on one GPU (external exchange, host sum).

Quality = held-out perplexity (10% of each group's documents, fold-in of 20
iterations) and training perplexity after S sweeps.
Prints one JSON line per configuration.  Usage:
    python tools/next3_experiment.py [--config C2] [--sweeps 30] [--ranks 4]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1510_06549_b200 as spdp  # noqa: E402
import synth  # noqa: E402


def run(train, test, K, G, waves, E, sweeps, seed=7):
    kw = dict(alpha=0.1, beta=0.1, discount=0.7, concentration=100.0, seed=seed, num_waves=waves)
    if G == 1:
        g = spdp.sampler_for(train, K, **kw)
        t0 = time.perf_counter()
        g.sweep(sweeps)
        dt = time.perf_counter() - t0
        ranks = [g]
    else:
        ranks = [spdp.sampler_for(train, K, rank=r, world_size=G, merge_every=E,
                                  exchange=spdp.SPDP_EXCHANGE_EXTERNAL, **kw) for r in range(G)]
        nb = ranks[0].exchange_blocks()
        t0 = time.perf_counter()
        for _ in range(sweeps):
            for _ in range(nb):
                for r in ranks:
                    r.sweep_local()
                bufs = [r.exchange_get() for r in ranks]
                with np.errstate(over="ignore"):
                    tot = sum(b.astype(np.int64) for b in bufs).astype(bufs[0].dtype)
                for r in ranks:
                    r.exchange_put(tot)
                    r.sweep_merge()
        dt = time.perf_counter() - t0
    # the word-topic state is replicated: rank 0 scores the held-out documents
    held = ranks[0].heldout(test, seed=1, iterations=20, want_z=False)["perplexity"]
    # training perplexity over all ranks' documents: per-rank log-likelihood sums
    ll, n = 0.0, 0
    for r in ranks:
        p = r.perplexity()
        st = r.stats()
        ll += -np.log(p) * st["local_tokens"]
        n += st["local_tokens"]
    for r in ranks:
        r.close()
    return {"heldout_ppl": round(held, 3), "train_ppl": round(float(np.exp(-ll / n)), 3), "wall_s": round(dt, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--sweeps", type=int, default=30)
    ap.add_argument("--ranks", type=int, default=4)
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    train, test = synth.holdout_split(synth.corpus_for(cfg), 0.1, seed=1)
    G = args.ranks
    cases = [("1 rank, W=1", train, 1, 1, 0), ("1 rank, W=4", train, 1, 4, 0),
             (f"{G} ranks, W=1 (exchange per sweep)", train, G, 1, 0),
             (f"{G} ranks, W=4, exchange per sweep", train, G, 4, 0),
             (f"{G} ranks, W=4, exchange per 2 waves", train, G, 4, 2),
             (f"{G} ranks, W=4, exchange per wave", train, G, 4, 1),
             (f"{G} ranks, W=1, training data duplicated once", synth.duplicate(train, 1), G, 1, 0)]
    for name, tr, g, w, e in cases:
        r = run(tr, test, cfg.k, g, w, e, args.sweeps)
        print(json.dumps({"config": args.config, "case": name, "ranks": g, "waves": w, "merge_every": e,
                          "train_tokens": tr.num_tokens, "sweeps": args.sweeps, **r}), flush=True)


if __name__ == "__main__":
    main()
