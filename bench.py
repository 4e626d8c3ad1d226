#!/usr/bin/env python
"""bench.py — sampled tokens/sec of the SPDP Gibbs sweep on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--waves 1] [--impl reference]

One step = one full sweep (every token of the corpus sampled once) on a
synthetic SPDP corpus shaped like the paper's multi-group collections
(synth/).  N > 1 is launched with torch.distributed.run; the
corpus (fixed total) is sharded by document over the ranks (strong scaling)
and the count deltas are all-reduced over NCCL inside the library.

Prints ONE JSON line (rank 0).  See DESIGN.md §7 for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--topics", type=int, default=0, help="override K (C4's K sweep)")
    ap.add_argument("--waves", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-tokens", type=int, default=0)
    ap.add_argument("--mode", default="sweep", choices=["sweep", "heldout"],
                    help="heldout: NEXT-1 fold-in + held-out perplexity of the 10%% hold-out (separate line)")
    ap.add_argument("--foldin-iters", type=int, default=20)
    ap.add_argument("--transform", default="none", choices=["none", "mix"],
                    help="mix: NEXT-4 sparse P^i = (1-e) I + e Perm_i (2 sources per word, seeded)")
    ap.add_argument("--update", default="wave", choices=["wave", "async"],
                    help="async: NEXT-2, the paper's immediate-update in-GPU scheme (nondeterministic)")
    ap.add_argument("--train-sweeps", type=int, default=20)
    ap.add_argument("--largest", default="C5", help="also time the largest config on the same GPUs ('' = skip)")
    ap.add_argument("--largest-steps", type=int, default=10)
    ap.add_argument("--largest-warmup", type=int, default=3)
    return ap.parse_args()


# ------------------------------------------------------------------ helpers
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy b.copy_(a))"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 9:
                for n, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def alg_bytes(plan, K, row_bytes=4):
    """Algorithmic HBM bytes of one sample-kernel pass:
    per token 12 B of token record (doc, id, zr in; zr out) + row_bytes*K B doc-topic row
    (4: the canonical int32 model of SURVEY §8(d); 2: the uint16 rows the library stores when
    the doc-topic array exceeds half of L2, i.e. the bytes the kernel actually has to move);
    per (w, i) segment 28K B (m, t, Q rows, A0/A1 table row in; dm, dt rows out)."""
    return plan["tokens"] * (12 + row_bytes * K) + plan["segments"] * 28 * K


def plan_stats(corpus, shard_docs, waves):
    """Distinct (wave, w, i) segments and tokens of this rank (from the wave plan)."""
    mask = np.isin(corpus.doc, shard_docs) if shard_docs is not None else np.ones(corpus.num_tokens, bool)
    doc = corpus.doc[mask]
    # in-document position l
    order = np.argsort(corpus.doc, kind="stable")
    pos = np.empty(corpus.num_tokens, np.int64)
    d_sorted = corpus.doc[order]
    starts = np.r_[0, np.nonzero(np.diff(d_sorted))[0] + 1]
    run = np.arange(corpus.num_tokens) - np.repeat(starts, np.diff(np.r_[starts, corpus.num_tokens]))
    pos[order] = run
    key = ((pos[mask] % waves) * corpus.vocab + corpus.word[mask]).astype(np.int64) * corpus.num_groups + corpus.group[mask]
    return {"tokens": int(doc.shape[0]), "segments": int(np.unique(key).shape[0])}


def ncu_summary(cfg_name, K, kernel="sample"):
    """The latest round's committed ncu --set full summary of the kernel (profiles/), or {}."""
    import glob
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_ncu_{cfg_name}_K{K}_{kernel}.json")))
    if paths:
        with open(paths[-1]) as f:
            d = json.load(f)
        if isinstance(d, list):
            d = d[0]
        d["file"] = os.path.relpath(paths[-1], ROOT)
        return d
    return {}


def load_traffic(cfg_name, K, kernel="sample"):
    """DRAM bytes per launch from the latest round's committed ncu --set full summary."""
    return ncu_summary(cfg_name, K, kernel).get("dram_bytes_per_launch")


class LoadPhases:
    """Captures spdp_load_corpus's SPDP_VERBOSE phase times (written by the library to fd 2)
    for the JSON line: where the e2e setup time goes."""

    def __enter__(self):
        import tempfile
        self.ms = {}
        self.prev = os.environ.get("SPDP_VERBOSE")
        os.environ["SPDP_VERBOSE"] = "1"
        sys.stderr.flush()
        self.tmp = tempfile.TemporaryFile(mode="w+b")
        self.saved = os.dup(2)
        os.dup2(self.tmp.fileno(), 2)
        return self

    def __exit__(self, *a):
        os.dup2(self.saved, 2)
        os.close(self.saved)
        if self.prev is None:
            os.environ.pop("SPDP_VERBOSE", None)
        else:
            os.environ["SPDP_VERBOSE"] = self.prev
        self.tmp.seek(0)
        for line in self.tmp.read().decode(errors="replace").splitlines():
            if line.startswith("[spdp] load "):
                name, _, val = line[len("[spdp] load "):].rpartition("  ")
                try:
                    self.ms[name.strip()] = float(val.strip().split()[0])
                except ValueError:
                    pass
        self.tmp.close()


def cpu_baseline(corpus, cfg, K, waves, sample_tokens, topics_arg):
    """The oracle as it stands, timed on this host: the -fopenmp build of the same
    source on all host cores for one whole mode-P sweep of the workload (the headline baseline),
    plus single-thread samples of mode P and mode S (Algorithm 1) on the first `sample_tokens`
    tokens.  The OpenMP leg runs in a subprocess (its library is process-global)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from oracle_timing import time_oracle
    one = time_oracle(corpus, cfg, K, waves, "P", sample_tokens)
    seq = time_oracle(corpus, cfg, K, waves, "S", sample_tokens)
    out = None
    try:
        env = dict(os.environ, ORACLE_OPENMP="1")
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "oracle_timing.py"), "--config", cfg.name,
                            "--topics", str(topics_arg), "--waves", str(waves), "--mode", "P"],
                           env=env, capture_output=True, text=True, timeout=600)
        out = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:   # the single-thread numbers still stand
        out = {"error": f"{type(e).__name__}: {e}"}
    if "value" in out:
        line = dict(out)
        line["single_thread_mode_P"] = one
        line["single_thread_mode_S"] = seq
        return line
    one["all_cores"] = out
    one["single_thread_mode_S"] = seq
    return one


def mixing_transform(I, V, seed):
    """NEXT-4 workload: P^i = (1 - e_i) Id + e_i Perm_i (doubly stochastic, 2 sources per word)."""
    rng = np.random.default_rng(seed)
    pptr, pv, pp = [0], [], []
    for i in range(I):
        perm = rng.permutation(V)
        eps = 0.1 + 0.05 * (i % 4)
        for w in range(V):
            ent = {w: 1.0 - eps}
            ent[int(perm[w])] = ent.get(int(perm[w]), 0.0) + eps
            for v in sorted(ent):
                pv.append(v); pp.append(ent[v])
            pptr.append(len(pv))
    return np.array(pptr, np.int32), np.array(pv, np.int32), np.array(pp)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def static_config(cfg, corpus, K, waves, world, workload):
    """The workload description both arms print (identical dicts)."""
    return {"workload": workload, "tokens": corpus.num_tokens, "groups": cfg.groups, "docs": corpus.num_docs,
            "vocab": cfg.vocab, "topics": K, "waves": waves, "parallelism": f"doc-shard x{world}",
            "l2": "flushed between timed sweeps"}


def recorded_ppl_gap(waves, update):
    """The BASELINE metric's third part, from the latest committed measurement (tools/ppl_gap.py:
    training perplexity after 100 sweeps of C2, 3 seeds per schedule, against the exact sequential
    sampler, i.e. the oracle's Algorithm 1); not re-measured here (the oracle chains take ~10 CPU-minutes)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ppl_gap_C2*.jsonl")))
    summary, src = {}, []
    for f in files:                     # later files refine earlier ones (same corpus, seeds, oracle chains)
        for ln in open(f):
            d = json.loads(ln)
            if "summary" in d:
                summary.update(d["summary"]["final"])
                src.append(os.path.relpath(f, ROOT))
    if not summary:
        return None
    this = "gpu async (NEXT-2)" if update == "async" else f"gpu W={waves}"
    return {"config": "C2 (1 M tokens, K = 50), 100 sweeps, seeds 7/8/9", "reference": "oracle sequential (Alg.1)",
            "this_schedule": this, "this_schedule_gap_pct": summary.get(this, {}).get("gap_vs_sequential_pct"),
            "by_schedule": summary, "files": src}


def measure_largest(args, spdp, torch, dist, world, rank, local_rank, stream, barrier, peak):
    """The largest BASELINE config (C5, ~200 M tokens, K = 200) on the same GPUs: device-resident sweep
    throughput and the sample kernel's roofline (no e2e / CPU legs), so that every driver run records it."""
    import synth
    cfg = synth.CONFIGS[args.largest]
    corpus = synth.corpus_for(cfg)
    N = corpus.num_tokens
    uid = None
    if world > 1:
        t = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            t = torch.tensor(list(spdp.spdp_nccl_unique_id()), dtype=torch.uint8)
        dist.broadcast(t, 0)
        uid = bytes(t.tolist())
    g = spdp.Sampler(cfg.groups, cfg.vocab, cfg.k, alpha=cfg.alpha, beta=cfg.beta, discount=cfg.discount,
                     concentration=cfg.concentration, seed=cfg.seed, num_waves=1, device=local_rank, rank=rank,
                     world_size=world, nccl_unique_id=uid, stream=stream.cuda_stream)
    t0 = time.perf_counter()
    g.load_corpus(corpus.group, corpus.doc, corpus.word, corpus.num_docs)
    load_s = time.perf_counter() - t0
    for _ in range(args.largest_warmup):
        g.sweep(1)

    def timed(steps):
        evs = []
        torch.cuda.synchronize(); barrier()
        for _ in range(steps):
            s_ = torch.cuda.Event(enable_timing=True); e_ = torch.cuda.Event(enable_timing=True)
            s_.record(stream); g.sweep(1); e_.record(stream)
            evs.append((s_, e_))
        torch.cuda.synchronize(); barrier()
        return [a.elapsed_time(b) for a, b in evs]

    step_ms = timed(args.largest_steps)
    g.profile(True)
    timed(max(3, min(args.largest_steps, 10)))
    tm = g.timings()
    g.profile(False)
    stats = g.stats()
    g.close()
    ms = float(np.mean(step_ms))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    sample_ms = tm["sample_ms"] / max(tm["sweeps"], 1)
    shard_docs = None
    if world > 1:
        part = spdp.spdp_partition(cfg.seed, world, corpus.doc, corpus.num_docs)
        shard_docs = np.nonzero(part == rank)[0]
    plan = plan_stats(corpus, shard_docs, 1)
    if stats.get("sparse_rows"):       # entries (4 B each) + the document's {first entry, count} record
        bytes_sweep = plan["tokens"] * (12 + 8) + stats["sparse_row_entries_read"] * 4 + plan["segments"] * 28 * cfg.k
        model = "sparse rows: per token 12 B record + 8 B doc record + (its document's entries x 4 B); per segment 28K B"
    else:
        bytes_sweep = alg_bytes(plan, cfg.k, stats.get("row_bytes", 4))
        model = f"dense rows: per token 12 B + {stats.get('row_bytes', 4)}K B; per segment 28K B"
    bytes_i32 = alg_bytes(plan, cfg.k, 4)
    ach = bytes_sweep / (sample_ms / 1e3) / 1e9
    nc = ncu_summary(cfg.name, cfg.k, "sample")
    return {"workload": f"{cfg.name}: I={cfg.groups} groups x {cfg.docs_per_group} docs, mean len {cfg.mean_len}, "
                        f"V={cfg.vocab}, K={cfg.k}, W=1", "tokens": N, "value": round(N / (ms / 1e3), 1), "unit": "tokens/s",
            "ms_per_step": round(ms, 4), "steps": args.largest_steps, "warmup": args.largest_warmup,
            "sweep_ms": [round(x, 3) for x in step_ms], "load_s": round(load_s, 3),
            "sample_ms_per_sweep": round(sample_ms, 4),
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(ach / peak, 4), "byte_model": model,
                         "int32_model": {"achieved": round(bytes_i32 / (sample_ms / 1e3) / 1e9, 1),
                                         "frac": round(bytes_i32 / (sample_ms / 1e3) / 1e9 / peak, 4)},
                         "traffic": nc.get("dram_bytes_per_launch"), "ncu": {k: nc.get(k) for k in (
                             "file", "kernel", "duration_ms", "dram_bytes_per_launch", "l2_hit_pct", "issue_active_pct",
                             "warp_instructions")} if nc else None},
            "stats": {k: stats.get(k) for k in ("row_bytes", "sparse_rows", "sparse_rows_lanes", "sparse_row_entries",
                                                "lanes_per_token", "topics_per_lane", "m_max", "parts", "local_tokens")},
            "timings_ms": {k: round(v, 3) for k, v in tm.items()}}


# ------------------------------------------------------------------ main
def main():
    args = parse()
    world0 = int(os.environ.get("WORLD_SIZE", "1"))
    if world0 > 1 and "OMP_NUM_THREADS" not in os.environ:   # corpus generation threads: share the host cores
        os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or 1) // world0))
    import synth
    cfg = synth.CONFIGS[args.config]
    K = args.topics or cfg.k
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    workload = f"{cfg.name}: I={cfg.groups} groups x {cfg.docs_per_group} docs, mean len {cfg.mean_len}, " \
               f"V={cfg.vocab}, K={K}, W={args.waves}" + (", async updates (NEXT-2)" if args.update == "async" else "") \
               + (", sparse P^i with 2 sources per word (NEXT-4)" if args.transform == "mix" else "")

    if args.impl == "reference":
        return run_reference(args, cfg, K, world, rank, workload)
    if args.mode == "heldout":
        return run_heldout(args, cfg, K, workload)

    import torch
    import torch.distributed as dist
    import paper_1510_06549_b200 as spdp

    spdp.build()
    # SPDP_BENCH_SHARE_GPU=1 (functional test only, with SPDP_NCCL_LIB=tests/libnccl_shim.so): every rank on
    # GPU 0, torch.distributed over gloo; the numbers of such a run are not measurements
    share = os.environ.get("SPDP_BENCH_SHARE_GPU") == "1"
    if share:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device("cuda", local_rank))
    corpus = synth.corpus_for(cfg)
    N = corpus.num_tokens
    def new_uid():   # one fresh NCCL unique id per communicator (an id bootstraps exactly one ncclCommInitRank)
        if world == 1:
            return None
        t = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            t = torch.tensor(list(spdp.spdp_nccl_unique_id()), dtype=torch.uint8)
        dist.broadcast(t, 0)
        return bytes(t.tolist())

    uid = new_uid()
    stream = torch.cuda.current_stream()
    kw = dict(alpha=cfg.alpha, beta=cfg.beta, discount=cfg.discount, concentration=cfg.concentration,
              seed=cfg.seed, num_waves=args.waves, device=local_rank, rank=rank, world_size=world,
              nccl_unique_id=uid, stream=stream.cuda_stream,
              update_mode=spdp.SPDP_UPDATE_ASYNC if args.update == "async" else spdp.SPDP_UPDATE_WAVE)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---------------- device-resident throughput (value) ----------------
    transform = mixing_transform(cfg.groups, cfg.vocab, cfg.seed) if args.transform == "mix" else None
    g = spdp.Sampler(cfg.groups, cfg.vocab, K, **kw)
    if transform is not None:
        g.set_transform(*transform)
    g.load_corpus(corpus.group, corpus.doc, corpus.word, corpus.num_docs)
    flush = None if args.no_flush else torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        g.sweep(1)

    def timed(steps):
        evs = []
        torch.cuda.synchronize(); barrier()
        for _ in range(steps):
            if flush is not None:
                flush.fill_(1)                      # evict L2 between timed sweeps (outside the events)
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(stream)
            g.sweep(1)
            e.record(stream)
            evs.append((s, e))
        torch.cuda.synchronize(); barrier()
        return [s.elapsed_time(e) for s, e in evs]

    # (1) the timed region of `value`: each sweep replays a captured CUDA graph (single rank)
    with ClockSampler(local_rank) as clk:
        step_ms = timed(args.steps)
    # (2) the same sweeps again with the library's per-phase CUDA events (which run the sweep
    #     uncaptured): the dominant kernel's duration for the roofline and the launch count
    psteps = max(3, min(args.steps, 30))
    g.profile(True)
    prof_ms = timed(psteps)
    tm = g.timings()
    g.profile(False)
    ms = float(np.mean(step_ms))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = N / (ms / 1e3)
    stats = g.stats()
    ppl = g.loglik(log_joint=False)[1] if transform is None else None
    g.close()

    # roofline of the dominant kernel (sample_kernel), from this run's CUDA events
    shard_docs = None
    if world > 1:
        part = spdp.spdp_partition(cfg.seed, world, corpus.doc, corpus.num_docs)
        shard_docs = np.nonzero(part == rank)[0]
    plan = plan_stats(corpus, shard_docs, args.waves)
    peak, peak_src = measured_peaks()
    sample_ms = tm["sample_ms"] / max(tm["sweeps"], 1)       # per sweep (all waves), from the profiled pass
    row_bytes = stats.get("row_bytes", 4)
    bytes_sweep = alg_bytes(plan, K, row_bytes)                 # the bytes this kernel has to move
    bytes_i32 = alg_bytes(plan, K, 4)                           # SURVEY §8(d)'s canonical int32 model
    achieved = bytes_sweep / (sample_ms / 1e3) / 1e9
    kname = "sp_token_kernel" if transform is not None else ("token_kernel" if stats.get("token_kernel") else "sample_kernel")
    pkey = kname.split("_")[0] + ("_async" if args.update == "async" else "")   # which committed ncu capture
    traffic = load_traffic(cfg.name, K, pkey)
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": kname,
            "alg_bytes_per_launch": int(bytes_sweep / max(args.waves, 1)), "peak_source": peak_src,
            "doc_topic_row_bytes_per_topic": row_bytes,
            "int32_model": {"alg_bytes_per_launch": int(bytes_i32 / max(args.waves, 1)),
                            "achieved": round(bytes_i32 / (sample_ms / 1e3) / 1e9, 1),
                            "frac": round(bytes_i32 / (sample_ms / 1e3) / 1e9 / peak, 4)},
            "sample_ms_per_sweep": round(sample_ms, 4), "share_of_step": round(sample_ms / ms, 3)}
    if traffic:   # measured DRAM bytes (committed ncu capture) over this run's kernel time
        roof["traffic_source"] = "committed ncu --set full capture (dram__bytes_read.sum + dram__bytes_write.sum per launch)"
        roof["dram_achieved"] = round(traffic / (sample_ms / max(args.waves, 1) / 1e3) / 1e9, 1)
        roof["dram_frac"] = round(roof["dram_achieved"] / peak, 4)
    nc = ncu_summary(cfg.name, K, pkey)
    if nc:   # what actually limits the kernel (from the committed ncu capture, not this run)
        roof["ncu"] = {k: nc.get(k) for k in ("file", "l2_hit_pct", "l1_pct_of_peak", "issue_active_pct",
                                               "achieved_occupancy_pct", "warp_instructions", "duration_ms")}

    # ---------------- end to end through the C ABI with host buffers ----------------
    torch.cuda.synchronize(); barrier()
    e2e_steps = args.steps
    # the caller's host buffers, pinned and filled before the job starts: the token arrays (inputs)
    # and two output buffers for the assignments
    t_pin = time.perf_counter()
    hin = [torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).pin_memory().numpy()
           for a in (corpus.group, corpus.doc, corpus.word)]
    narrow = K <= 128                                            # the step's result in one byte per token
    zr = [torch.empty(N, dtype=torch.uint8, pin_memory=True).numpy() if narrow else
          torch.empty(N, dtype=torch.int16, pin_memory=True).numpy().view(np.uint16) for _ in range(2)]
    t_pin = time.perf_counter() - t_pin
    kw["nccl_unique_id"] = new_uid()                            # (a collective: outside the clock)
    t0 = time.perf_counter()
    h = spdp.Sampler(cfg.groups, cfg.vocab, K, **kw)
    t_create = time.perf_counter() - t0
    if transform is not None:
        h.set_transform(*transform)
    with LoadPhases() as phases:                                 # the library's own phase timer (stderr)
        h.load_corpus(hin[0], hin[1], hin[2], corpus.num_docs)     # H2D of the job's inputs (pinned)
    t_setup = time.perf_counter() - t0
    for s in range(e2e_steps):
        h.sweep_async(1)                                # queued behind step s-1's staging; the host goes on
        h.wait()                                        # step s-1's assignments have landed in zr[(s-1) % 2]
        if narrow:
            h.zr8_async(zr[s % 2])                      # D2H of step s's z | r << 7, overlapping sweep s+1
        else:
            h.zr_async(zr[s % 2])                       # D2H of step s's z | r << 15, overlapping sweep s+1
    h.wait()
    torch.cuda.synchronize(); barrier()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h.close()
    e2e = {"value": N * e2e_steps / e2e_s, "unit": "tokens/s", "setup_ms": round(t_setup * 1e3, 2), "create_ms": round(t_create * 1e3, 2),
           "load_phases_ms": phases.ms,
           "host_buffer_pin_ms_untimed": round(t_pin * 1e3, 2),
           "ms_per_step_after_setup": round((e2e_s - t_setup) * 1e3 / e2e_steps, 4),
           "h2d_bytes_per_step": int(N * 12 / e2e_steps), "d2h_bytes_per_step": int(N * (1 if narrow else 2)),
           "includes": "spdp_create + spdp_load_corpus (host token arrays) + per step spdp_sweep_async(1) + "
                       + ("spdp_zr8_async (z | r << 7, one byte per token)" if narrow else
                          "spdp_zr_async (z | r << 15, two bytes per token)")
                       + " of every token into pinned host memory, the copy of step s overlapping "
                       "sweep s+1, spdp_wait each step; wall clock, max over ranks"}

    line = {
        "metric": "sampled tokens/sec per sweep", "value": round(value, 1), "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic SPDP-generated corpus (synth/, seeded)",
        "config": static_config(cfg, corpus, K, args.waves, world, workload),
        "timing": {"arithmetic": "f32 slot masses, f64 CDF prefix and uniform, int32 counts, exact integer removal draw",
                   "l2": "flushed between timed sweeps (256 MiB write outside the events)" if flush is not None else "not flushed",
                   "sweep_ms": [round(x, 4) for x in step_ms],
                   "sweep": "one CUDA-graph replay per step (single rank); the roofline's kernel time comes from "
                            "a second pass of the same sweeps with per-phase events (profiled_sweep_ms)",
                   "profiled_sweep_ms": round(float(np.mean(prof_ms)), 4)},
        "roofline": roof,
        "e2e": e2e,
        "gpu_launches": int(round(tm["launches"] / max(tm["sweeps"], 1) * args.steps)),
        "clocks": clk.summary(),
        "perplexity_after": round(ppl, 4) if ppl is not None else None,
        "stats": stats,
        "timings_ms": {k: round(v, 4) for k, v in tm.items()},
    }
    if world > 1:   # the exchange of this run: one packed int32 per (w, i, k) cell, all-reduced per sweep
        kp = (K + 3) // 4 * 4
        line["multi_gpu"] = {"ranks": world, "backend": "NCCL all-reduce over NVLink (library-owned communicator)",
                             "exchange_bytes_per_sweep": cfg.vocab * cfg.groups * kp * 4,
                             "parts": stats.get("parts"), "exchange_ms_per_sweep": round(tm["exchange_ms"] / max(tm["sweeps"], 1), 4),
                             "merge_ms_per_sweep": round(tm["merge_ms"] / max(tm["sweeps"], 1), 4),
                             "sample_ms_per_sweep": round(tm["sample_ms"] / max(tm["sweeps"], 1), 4)}
    line["perplexity_gap"] = recorded_ppl_gap(args.waves, args.update)
    if rank == 0 and world == 1 and not args.no_cpu_baseline and transform is None:
        st = args.cpu_sample_tokens or min(N, 400_000 if K <= 100 else 100_000)
        line["cpu_baseline"] = cpu_baseline(corpus, cfg, K, args.waves, st, K)
        line["cpu_baseline"]["cpu"] = cpu_model()
    if args.largest and args.largest != args.config and transform is None and args.update == "wave":
        del corpus
        try:
            line["largest_config"] = measure_largest(args, spdp, torch, dist, world, rank, local_rank, stream, barrier, peak)
        except Exception as e:   # the headline line stands without it
            line["largest_config"] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_heldout(args, cfg, K, workload):
    """NEXT-1 measurement (one GPU): train on 90% of the corpus, then time
    spdp_heldout (fold-in of the held-out 10% per group + held-out perplexity,
    DESIGN.md §10) per step; the fold-in kernel's own CUDA-event time gives the
    roofline (fp64 phi~ row of 8K bytes + 16 B of token record per
    token-iteration, plus one 8K-byte row per token for the likelihood pass)."""
    import torch
    import paper_1510_06549_b200 as spdp
    import synth
    spdp.build()
    torch.cuda.set_device(0)
    train, test = synth.holdout_split(synth.corpus_for(cfg), 0.1, seed=1)
    stream = torch.cuda.current_stream()
    g = spdp.Sampler(cfg.groups, cfg.vocab, K, alpha=cfg.alpha, beta=cfg.beta, discount=cfg.discount,
                     concentration=cfg.concentration, seed=cfg.seed, num_waves=args.waves, stream=stream.cuda_stream)
    g.load_corpus(train.group, train.doc, train.word, train.num_docs)
    g.sweep(args.train_sweeps)
    F = args.foldin_iters
    for s_ in range(args.warmup):
        g.heldout(test, 1000 + s_, F, want_z=False)
    g.profile(True)
    torch.cuda.synchronize()
    ms, ppl = [], []
    with ClockSampler(0) as clk:
        for s_ in range(args.steps):
            t0 = time.perf_counter()
            r = g.heldout(test, s_, F, want_z=False)          # host prep + H2D + phi table + fold-in + D2H
            ms.append((time.perf_counter() - t0) * 1e3)
            ppl.append(r["perplexity"])
    tm = g.timings()
    _, train_ppl = g.loglik(log_joint=False)
    g.close()
    Nh = test.num_tokens
    units = Nh * F
    kern_ms = tm["foldin_ms"] / max(args.steps, 1)
    alg = Nh * F * (8 * K + 16) + Nh * (8 * K + 8)
    peak, src = measured_peaks()
    line = {
        "metric": "held-out fold-in token-iterations/sec", "value": round(units / (float(np.mean(ms)) / 1e3), 1),
        "unit": "token-iterations/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(float(np.mean(ms)), 4), "higher_is_better": True, "scaling": "none",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic SPDP-generated corpus (synth/, seeded), 10% per group held out",
        "config": {"workload": f"{workload} | train {train.num_tokens} tokens x {args.train_sweeps} sweeps, "
                               f"held-out {Nh} tokens / {test.num_docs} docs x {F} fold-in iterations",
                   "timing": "wall clock per spdp_heldout call (host prep, H2D, phi table, fold-in, reduce, D2H)"},
        "kernel_ms_per_step": round(kern_ms, 4),
        "kernel_value": round(units / (kern_ms / 1e3), 1) if kern_ms > 0 else None,
        "roofline": {"bound": "hbm", "achieved": round(alg / (kern_ms / 1e3) / 1e9, 1) if kern_ms > 0 else None,
                     "peak": peak, "unit": "GB/s",
                     "frac": round(alg / (kern_ms / 1e3) / 1e9 / peak, 4) if kern_ms > 0 else None,
                     "traffic": load_traffic(cfg.name, K, "foldin"), "kernel": "foldin_kernel",
                     "alg_bytes_per_launch": int(alg), "peak_source": src},
        "heldout_perplexity": round(float(np.mean(ppl)), 4), "train_perplexity": round(train_ppl, 4),
        "clocks": clk.summary(), "gpu_launches": int(tm["launches"]),
    }
    print(json.dumps(line), flush=True)


def run_reference(args, cfg, K, world, rank, workload):
    """--impl reference: the oracle as it stands on the host cores (the paper ships
    no code; the CPU oracle is this tier's reference arm).  Rank 0 only."""
    if rank != 0:
        return
    os.environ.setdefault("ORACLE_OPENMP", "1")      # the -fopenmp build of the same source, all host cores
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from oracle_timing import threads_used
    import synth
    corpus = synth.corpus_for(cfg)
    # whole sweeps (C3 on 16 cores: ~4 s each) unless the workload is larger; per-call fixed passes over the
    # count tables make short prefixes understate the oracle's throughput
    sample = args.cpu_sample_tokens or min(corpus.num_tokens, 12_000_000 if K <= 100 else 2_000_000)
    import oracle
    o = oracle.from_corpus(corpus, K, cfg.alpha, cfg.beta, cfg.discount, cfg.concentration, cfg.seed)
    for _ in range(args.warmup):
        o.sweep_par(waves=args.waves, max_tokens=sample)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o.sweep_par(waves=args.waves, max_tokens=sample)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(times))
    value = sample / (ms / 1e3)
    cb = {"value": value, "unit": "tokens/s", "cores": threads_used(), "kind": "oracle",
          "sample": f"{'all' if sample >= corpus.num_tokens else 'first ' + str(sample)} tokens of a mode-P (W={args.waves}) sweep of {cfg.name} per step "
                    f"(plain C oracle, fp64 log space; -fopenmp build over the wave's decisions)"}
    line = {"impl": "reference", "metric": "sampled tokens/sec per sweep", "value": round(value, 1),
            "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic SPDP-generated corpus (synth/, seeded)",
            "config": static_config(cfg, corpus, K, args.waves, world, workload),
            "cpu_baseline": cb,
            "e2e": {"value": round(value, 1), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
