"""Wall time of each of the first e2e steps of a fresh context (bench.py's e2e loop: sweep_async,
wait, zr8_async), to see what the first steps cost beyond the steady state.  Usage: python tools/first_steps.py [C3]"""
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
c = synth.corpus_for(cfg)
hin = [torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).pin_memory().numpy() for a in (c.group, c.doc, c.word)]
zb = [torch.empty(c.num_tokens, dtype=torch.uint8, pin_memory=True).numpy() for _ in range(2)]
kw = dict(alpha=0.1, beta=0.1, discount=0.7, concentration=100.0, seed=7)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = spdp.Sampler(cfg.groups, cfg.vocab, cfg.k, **kw)
    h.load_corpus(hin[0], hin[1], hin[2], c.num_docs)
    t1 = time.perf_counter()
    ts = []
    for s in range(8):
        a = time.perf_counter()
        h.sweep_async(1)
        b = time.perf_counter()
        h.wait()
        d = time.perf_counter()
        h.zr8_async(zb[s % 2])
        e = time.perf_counter()
        ts.append((round(1e3 * (b - a), 2), round(1e3 * (d - b), 2), round(1e3 * (e - d), 2)))
    h.wait()
    torch.cuda.synchronize()
    print(f"rep {rep}: setup {1e3*(t1-t0):.1f} ms; per step (sweep_async, wait, zr8_async) ms: {ts}", flush=True)
    h.close()
