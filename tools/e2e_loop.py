"""Per-step cost of bench.py's e2e loop pieces at one config (wall clock, after warm-up):
sweep_async alone, zr8_async + wait alone, and the pipelined loop bench.py times.
Usage: python tools/e2e_loop.py [C3] [steps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1510_06549_b200 as spdp  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
c = synth.corpus_for(cfg)
kw = dict(alpha=0.1, beta=0.1, discount=0.7, concentration=100.0, seed=7)
zb = [torch.empty(c.num_tokens, dtype=torch.uint8, pin_memory=True).numpy() for _ in range(2)]
h = spdp.Sampler(cfg.groups, cfg.vocab, cfg.k, **kw)
h.load_corpus(c.group, c.doc, c.word, c.num_docs)


def timed(fn):
    fn(5)
    torch.cuda.synchronize()
    a = time.perf_counter()
    fn(steps)
    h.wait()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / steps * 1e3


def sweeps(n):
    for _ in range(n):
        h.sweep_async(1)


def copies(n):
    for s in range(n):
        h.zr8_async(zb[s % 2])
        h.wait()


def pipelined(n):
    for s in range(n):
        h.sweep_async(1)
        h.wait()
        h.zr8_async(zb[s % 2])


def serial(n):
    for s in range(n):
        h.sweep(1)
        h.zr8_async(zb[s % 2])
        h.wait()


print(f"{cfg.name}: sweep_async alone {timed(sweeps):.3f} ms/step; zr8_async+wait alone {timed(copies):.3f}; "
      f"pipelined (bench loop) {timed(pipelined):.3f}; serial {timed(serial):.3f}")
h.close()
