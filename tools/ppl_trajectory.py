"""Perplexity trajectories of the oracle: mode S (Alg.1) vs wave-snapshot mode P
(W waves, G shards) on a config — the "perplexity gap" of BASELINE.json's metric.
Usage: python tools/ppl_trajectory.py C2 20 "S,P1,P8" [seed] > out.json"""
import json
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1]]
sweeps = int(sys.argv[2])
modes = sys.argv[3].split(",")
seed = int(sys.argv[4]) if len(sys.argv) > 4 else cfg.seed
c = synth.corpus_for(cfg)
out = {"config": cfg.name, "tokens": c.num_tokens, "seed": seed, "sweeps": sweeps, "traj": {}}
for m in modes:
    o = oracle.from_corpus(c, cfg.k, cfg.alpha, cfg.beta, cfg.discount, cfg.concentration, seed)
    tr = [o.perplexity()]
    t0 = time.time()
    for s in range(sweeps):
        if m == "S":
            o.sweep_seq()
        else:
            W = int(m[1:].split("g")[0]); G = int(m.split("g")[1]) if "g" in m else 1
            o.sweep_par(waves=W, shards=G)
        tr.append(o.perplexity())
    out["traj"][m] = tr
    out.setdefault("seconds", {})[m] = time.time() - t0
    print(m, [round(x, 1) for x in tr[::max(1, sweeps // 10)]], file=sys.stderr, flush=True)
print(json.dumps(out))
