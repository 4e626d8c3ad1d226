"""Wall-clock breakdown of bench.py's e2e leg (create, load_corpus, sweep, zr)
at one config.  Usage: python tools/e2e_breakdown.py [C3] [steps]"""
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
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = synth.corpus_for(cfg)
kw = dict(alpha=0.1, beta=0.1, discount=0.7, concentration=100.0, seed=7)
if len(sys.argv) > 3 and sys.argv[3] == "async":
    kw["update_mode"] = spdp.SPDP_UPDATE_ASYNC
zr = torch.empty(c.num_tokens, dtype=torch.int16, pin_memory=True).numpy().view(np.uint16)
for rep in range(2):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    h = spdp.Sampler(cfg.groups, cfg.vocab, cfg.k, **kw)
    t.append(time.perf_counter())
    h.load_corpus(c.group, c.doc, c.word, c.num_docs)
    t.append(time.perf_counter())
    sw, zt = 0.0, 0.0
    for _ in range(steps):
        a = time.perf_counter()
        h.sweep(1)
        b = time.perf_counter()
        h.zr(zr)
        sw += b - a
        zt += time.perf_counter() - b
    t_first = time.perf_counter()
    h.sweep(1)
    first = time.perf_counter() - t_first
    zb = [zr, zr.copy()]
    zb[1] = torch.empty(c.num_tokens, dtype=torch.int16, pin_memory=True).numpy().view(np.uint16)
    a = time.perf_counter()
    for s in range(steps):
        h.sweep(1)
        h.wait()
        h.zr_async(zb[s % 2])
    h.wait()
    pipe = (time.perf_counter() - a) / steps
    a = time.perf_counter()
    for s in range(steps):
        h.sweep(1)
    sw_only = (time.perf_counter() - a) / steps
    a = time.perf_counter()
    for s in range(steps):
        h.zr_async(zb[s % 2])
        h.wait()
    zr_only = (time.perf_counter() - a) / steps
    print(f"   sweep alone {1e3*sw_only:.3f} ms; zr_async+wait alone {1e3*zr_only:.3f} ms")
    h.close()
    t.append(time.perf_counter())
    print(f"   one more sweep {1e3*first:.3f} ms; pipelined sweep+zr_async {1e3*pipe:.3f} ms/step")
    print(f"rep {rep}: create {1e3*(t[1]-t[0]):.1f} ms, load {1e3*(t[2]-t[1]):.1f} ms, "
          f"sweep {1e3*sw/steps:.3f} ms/step, zr {1e3*zt/steps:.3f} ms/step, total {1e3*(t[3]-t[0]):.1f} ms")
