"""Multi-process (world_size 2, gloo, CPU) coverage of the multi-GPU protocol.

The library's multi-GPU sweep is: every rank samples its document shard
against the sweep-start counts, hands out its net count changes D_g, the
ranks all-reduce them, and every rank merges S1 = clamp(S0 + sum_g D_g)
(Alg.3; readings c13-c15).  Here two CPU
processes run that protocol with the oracle's per-shard sweep and a gloo
all-reduce, and must reproduce the single-process G-shard simulation bit for
bit; each rank's shard is also the library's own partition (host code)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, waves, sweeps, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import paper_1510_06549_b200 as spdp
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = synth.corpus_for(synth.CONFIGS["C1"])
    o = oracle.from_corpus(c, 10)
    part_lib = spdp.spdp_partition(7, world, c.doc, c.num_docs)
    assert np.array_equal(part_lib, o.partition(world))
    for _ in range(sweeps):
        Dm, Dt = o.sweep_shard(waves, world, rank)
        t = torch.from_numpy(np.concatenate([Dm, Dt]))
        dist.all_reduce(t)                       # the exchange step (NCCL in the library)
        tot = t.numpy()
        o.merge(tot[:Dm.size], tot[Dm.size:])
    st = o.state()
    mine = part_lib[c.doc] == rank
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), z=st["z"][mine], r=st["r"][mine], m=st["m"], t=st["t"],
             Q=st["Q"], mine=mine)
    dist.destroy_process_group()


@pytest.mark.parametrize("waves", [1, 3])
def test_two_ranks_over_gloo_match_the_sharded_oracle(tmp_path, waves):
    world, sweeps = 2, 3
    mp.spawn(_worker, args=(world, _free_port(), waves, sweeps, str(tmp_path)), nprocs=world, join=True)
    import oracle
    import synth
    c = synth.corpus_for(synth.CONFIGS["C1"])
    ref = oracle.from_corpus(c, 10)
    for _ in range(sweeps):
        ref.sweep_par(waves=waves, shards=world)
    st = ref.state()
    for r in range(world):
        d = np.load(os.path.join(tmp_path, f"rank{r}.npz"))
        for k in ("m", "t", "Q"):
            np.testing.assert_array_equal(d[k], st[k])
        np.testing.assert_array_equal(d["z"], st["z"][d["mine"]])
        np.testing.assert_array_equal(d["r"], st["r"][d["mine"]])
