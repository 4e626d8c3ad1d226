import os, sys
sys.path.insert(0, os.getcwd())
os.environ["SPDP_SPARSE_ROWS"] = "1"
os.environ["SPDP_GRAPHS"] = "0"
import synth, paper_1510_06549_b200 as spdp
c = synth.generate(2, 30, 40.0, 300, 8, seed=101)
g = spdp.sampler_for(c, 100)
print(g.stats(), flush=True)
g.sweep(1)
print("ok", g.stats(), flush=True)
