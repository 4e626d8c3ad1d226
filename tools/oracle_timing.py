"""Oracle timing (SURVEY §8(d) "Oracle, timed in the same bench run on the host"):
the plain C oracle as it stands, on a config's corpus.

    python tools/oracle_timing.py --config C3 [--topics K] [--waves 1] --mode P|S [--tokens N] [--sweeps 1]

--mode P: one mode-P sweep (wave snapshots, G = 1) — with ORACLE_OPENMP=1 the -fopenmp build of the
same source spreads each wave's decisions over the host cores; --mode S: Algorithm 1 (sequential, one
thread by construction).  --tokens bounds the sampled tokens of each sweep (0 = all).  Prints one JSON
line: tokens/s, threads used, seconds, the sample.  Test/measurement infrastructure (loads oracle/)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def threads_used():
    if os.environ.get("ORACLE_OPENMP") != "1":
        return 1
    n = os.environ.get("OMP_NUM_THREADS")
    return int(n) if n else (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())


def time_oracle(corpus, cfg, K, waves, mode, tokens, sweeps=1):
    import oracle
    o = oracle.from_corpus(corpus, K, cfg.alpha, cfg.beta, cfg.discount, cfg.concentration, cfg.seed)
    n = tokens if tokens > 0 else corpus.num_tokens
    t0 = time.perf_counter()
    for _ in range(sweeps):
        if mode == "S":
            o.sweep_seq(max_tokens=n)
        else:
            o.sweep_par(waves=waves, shards=1, max_tokens=n)
    dt = time.perf_counter() - t0
    o.close()
    return {"value": n * sweeps / dt, "unit": "tokens/s", "cores": threads_used() if mode == "P" else 1,
            "kind": "oracle", "mode": mode, "seconds": round(dt, 3),
            "sample": f"{'all' if n == corpus.num_tokens else 'first ' + str(n)} tokens of {sweeps} mode-{mode}"
                      f"{' (W=' + str(waves) + ')' if mode == 'P' else ''} sweep(s) of {cfg.name} "
                      f"(N={corpus.num_tokens}, K={K}); plain C oracle, fp64 log space"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--topics", type=int, default=0)
    ap.add_argument("--waves", type=int, default=1)
    ap.add_argument("--mode", default="P", choices=["P", "S"])
    ap.add_argument("--tokens", type=int, default=0)
    ap.add_argument("--sweeps", type=int, default=1)
    a = ap.parse_args()
    import synth
    cfg = synth.CONFIGS[a.config]
    K = a.topics or cfg.k
    print(json.dumps(time_oracle(synth.corpus_for(cfg), cfg, K, a.waves, a.mode, a.tokens, a.sweeps)), flush=True)


if __name__ == "__main__":
    main()
