import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_1510_06549_b200 as spdp
c = synth.corpus_for(synth.CONFIGS["C1"])
g = spdp.sampler_for(c, 10, seed=7)
st = g.stats(); print(st)
g.sweep(1)
print("ok")
