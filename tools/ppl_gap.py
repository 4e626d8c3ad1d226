"""The BASELINE metric's "perplexity gap": training perplexity after S sweeps of
the GPU sampler's schedules (W = 1, 4, 16 waves; the paper's async scheme;
4 ranks) against the oracle's exact sequential sampler (Alg.1), same corpus,
several seeds; the seed spread is the noise floor the gap is read against
(SURVEY §8(c) "approximation quality").  The oracle chains run in parallel
host processes while the GPU chains run.  One JSON line per (method, seed)
plus a summary line.  Usage: python tools/ppl_gap.py [--config C2] [--sweeps 100]
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

HYPER = dict(alpha=0.1, beta=0.1, discount=0.7, concentration=100.0)


def oracle_chain(args):
    cfg_name, K, seed, sweeps, every = args
    import oracle
    import synth
    c = synth.corpus_for(synth.CONFIGS[cfg_name])
    o = oracle.from_corpus(c, K, seed=seed, **HYPER)
    traj = []
    for s in range(1, sweeps + 1):
        o.sweep_seq()
        if s % every == 0:
            traj.append(o.perplexity())
    return seed, traj


def gpu_chain(c, K, seed, sweeps, every, waves=1, update=0, ranks=1):
    import paper_1510_06549_b200 as spdp
    if ranks == 1:
        g = spdp.sampler_for(c, K, seed=seed, num_waves=waves, update_mode=update, **HYPER)
        traj = []
        for s in range(1, sweeps + 1):
            g.sweep(1)
            if s % every == 0:
                traj.append(g.perplexity())
        g.close()
        return traj
    rs = [spdp.sampler_for(c, K, seed=seed, num_waves=waves, rank=r, world_size=ranks,
                           exchange=spdp.SPDP_EXCHANGE_EXTERNAL, **HYPER) for r in range(ranks)]
    traj = []
    for s in range(1, sweeps + 1):
        for r in rs:
            r.sweep_local()
        bufs = [r.exchange_get() for r in rs]
        with np.errstate(over="ignore"):
            tot = sum(b.astype(np.int64) for b in bufs).astype(bufs[0].dtype)
        for r in rs:
            r.exchange_put(tot)
            r.sweep_merge()
        if s % every == 0:
            ll, n = 0.0, 0
            for r in rs:
                st = r.stats()
                ll += -np.log(r.perplexity()) * st["local_tokens"]
                n += st["local_tokens"]
            traj.append(float(np.exp(-ll / n)))
    for r in rs:
        r.close()
    return traj


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--sweeps", type=int, default=100)
    ap.add_argument("--every", type=int, default=10)
    ap.add_argument("--seeds", default="7,8,9")
    ap.add_argument("--methods", default="", help="comma-separated subset of the method names (default: all)")
    ap.add_argument("--oracle-from", default="", help="reuse the oracle chains of an earlier run's JSON lines "
                                                      "(same config, seeds, sweeps; the oracle is deterministic)")
    args = ap.parse_args()
    import synth
    cfg = synth.CONFIGS[args.config]
    K = cfg.k
    seeds = [int(x) for x in args.seeds.split(",")]
    t0 = time.time()
    reuse = {}
    if args.oracle_from:
        for line in open(args.oracle_from):
            d = json.loads(line)
            if d.get("method") == "oracle sequential (Alg.1)" and d.get("config") == args.config and d["seed"] in seeds \
                    and d["every"] == args.every and len(d["perplexity"]) == args.sweeps // args.every:
                reuse[d["seed"]] = d["perplexity"]
    todo = [s for s in seeds if s not in reuse]
    pool = mp.get_context("spawn").Pool(max(len(todo), 1))
    pending = pool.map_async(oracle_chain, [(args.config, K, s, args.sweeps, args.every) for s in todo])
    c = synth.corpus_for(cfg)
    methods = {"gpu W=1": dict(waves=1), "gpu W=2": dict(waves=2), "gpu W=4": dict(waves=4),
               "gpu W=8": dict(waves=8), "gpu W=16": dict(waves=16),
               "gpu async (NEXT-2)": dict(update=1), "gpu 4 ranks W=1": dict(ranks=4),
               "gpu 4 ranks W=2": dict(waves=2, ranks=4), "gpu 4 ranks W=4": dict(waves=4, ranks=4)}
    if args.methods:
        keep = [m.strip() for m in args.methods.split(",")]
        methods = {k: v for k, v in methods.items() if k in keep}
    results = {}
    for name, kw in methods.items():
        for s in seeds:
            traj = gpu_chain(c, K, s, args.sweeps, args.every, **kw)
            results.setdefault(name, []).append(traj)
            print(json.dumps({"config": args.config, "method": name, "seed": s, "every": args.every,
                              "perplexity": [round(x, 3) for x in traj]}), flush=True)
    got = dict(pending.get()) if todo else {}
    for s in seeds:
        traj = reuse.get(s, got.get(s))
        results.setdefault("oracle sequential (Alg.1)", []).append(traj)
        print(json.dumps({"config": args.config, "method": "oracle sequential (Alg.1)", "seed": s,
                          "every": args.every, "perplexity": [round(x, 3) for x in traj],
                          "reused_from": args.oracle_from if s in reuse else None}), flush=True)
    ref = np.array(results["oracle sequential (Alg.1)"])[:, -1]
    summary = {"config": args.config, "sweeps": args.sweeps, "seeds": seeds,
               "oracle_host_minutes": round((time.time() - t0) / 60, 1), "final": {}}
    for name, trajs in results.items():
        fin = np.array(trajs)[:, -1]
        summary["final"][name] = {"mean": round(float(fin.mean()), 2), "sd": round(float(fin.std(ddof=1)), 2),
                                  "gap_vs_sequential_pct": round(100 * (fin.mean() / ref.mean() - 1), 2)}
    print(json.dumps({"summary": summary}), flush=True)


if __name__ == "__main__":
    main()
