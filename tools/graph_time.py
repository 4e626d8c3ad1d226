import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np, synth, paper_1510_06549_b200 as spdp
for name in ["C1", "C2", "C3"]:
    cfg = synth.CONFIGS[name]; c = synth.corpus_for(cfg)
    for gflag in ["1", "0"]:
        os.environ["SPDP_GRAPHS"] = gflag
        g = spdp.sampler_for(c, cfg.k, seed=7)
        g.sweep(5)
        torch.cuda.synchronize()
        ms = []
        for _ in range(50):
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(); g.sweep(1); e.record(); torch.cuda.synchronize(); ms.append(s.elapsed_time(e))
        print(name, "graphs" if gflag == "1" else "direct", round(float(np.mean(ms)), 4), flush=True)
        g.close()
