"""spdp_load_corpus phase times (SPDP_VERBOSE=2: the library drains the device at each mark) with pinned
host token arrays, as bench.py's e2e leg loads them; three contexts in a row.
Usage: SPDP_VERBOSE=2 python tools/load_phases.py [C3]"""
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
kw = dict(alpha=0.1, beta=0.1, discount=0.7, concentration=100.0, seed=7)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = spdp.Sampler(cfg.groups, cfg.vocab, cfg.k, **kw)
    t1 = time.perf_counter()
    h.load_corpus(hin[0], hin[1], hin[2], c.num_docs)
    t2 = time.perf_counter()
    h.sweep(1)
    t3 = time.perf_counter()
    h.close()
    print(f"rep {rep}: create {1e3*(t1-t0):.1f} ms, load {1e3*(t2-t1):.1f} ms, first sweep {1e3*(t3-t2):.1f} ms", flush=True)
