"""One rank of a multi-process NCCL-path run on a single GPU (tests/nccl_shim.c).
Usage: python nccl_shim_worker.py RANK WORLD UIDFILE OUT.npz K WAVES MERGE_EVERY SWEEPS"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1510_06549_b200 as spdp  # noqa: E402
import synth  # noqa: E402

rank, world, uidfile, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
K, waves, E, sweeps = (int(x) for x in sys.argv[5:9])
sparse = len(sys.argv) > 9 and sys.argv[9] == "sparse"
if rank == 0:
    uid = spdp.spdp_nccl_unique_id()
    with open(uidfile + ".tmp", "wb") as f:
        f.write(uid)
    os.rename(uidfile + ".tmp", uidfile)
else:
    while not os.path.exists(uidfile):
        time.sleep(0.05)
    uid = open(uidfile, "rb").read()
c = synth.corpus_for(synth.CONFIGS["C1"])
transform = None
if sparse:
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_oracle_sparse_p import mixing_P
    transform = mixing_P(c.num_groups, c.vocab, np.random.default_rng(3))
g = spdp.sampler_for(c, K, num_waves=waves, merge_every=E, rank=rank, world_size=world, nccl_unique_id=uid,
                     alpha=0.1, beta=0.1, discount=0.7, concentration=100.0, transform=transform)
g.sweep(sweeps)
st = g.counts()
if sparse:
    lj, ppl = 0.0, 2.0
    st["q"] = g.sparse_state()["q"]
else:
    lj, ppl = g.loglik()
if rank == 0:
    np.savez(out, lj=lj, ppl=ppl, parts=g.stats()["parts"], **st)
g.close()
