"""The library's NCCL code path (SPDP_EXCHANGE_NCCL: communicator, packed
all-reduce, exchange-pipelining slices on the second stream, exchange blocks,
the gathers of spdp_counts / spdp_loglik) with 2 processes on ONE GPU, through
tests/nccl_shim.c (real NCCL refuses two ranks on one device).  Each run must
equal the in-process external-exchange run of the same ranks bit for bit; that
one is pinned to the oracle's G-shard sweep (test_gpu_parity.py)."""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import paper_1510_06549_b200 as spdp
import synth
from gpu_util import HYPER, corpus, require_gpu

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def shim():
    require_gpu()
    so = os.path.join(HERE, "libnccl_shim.so")
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-I/usr/local/cuda/include", os.path.join(HERE, "nccl_shim.c"),
                           "-o", so, "-L/usr/local/cuda/lib64", "-Wl,-rpath,/usr/local/cuda/lib64", "-lcudart"])
    return so


def external(K, waves, E, sweeps, G=2):
    c = corpus("C1")
    ranks = [spdp.sampler_for(c, K, num_waves=waves, merge_every=E, rank=r, world_size=G,
                              exchange=spdp.SPDP_EXCHANGE_EXTERNAL, **HYPER) for r in range(G)]
    nb = ranks[0].exchange_blocks()
    for _ in range(sweeps):
        for _ in range(nb):
            for r in ranks:
                r.sweep_local()
            bufs = [r.exchange_get() for r in ranks]
            with np.errstate(over="ignore"):
                tot = sum(b.astype(np.int64) for b in bufs).astype(bufs[0].dtype)
            for r in ranks:
                r.exchange_put(tot)
                r.sweep_merge()
    part = np.asarray(spdp.spdp_partition(7, G, c.doc, c.num_docs))
    z = np.full(c.num_tokens, -1, np.int32); r_ = np.zeros(c.num_tokens, np.uint8)
    n = np.zeros((c.num_docs, K), np.int32)
    for j, r in enumerate(ranks):
        cr = r.counts()
        own = part[c.doc] == j
        z[own] = cr["z"][own]; r_[own] = cr["r"][own]
        n[part == j] = cr["n"][part == j]
    out = dict(z=z, r=r_, n=n, m=ranks[0].counts()["m"], t=ranks[0].counts()["t"], Q=ranks[0].counts()["Q"])
    return out


@pytest.mark.parametrize("K,waves,E,parts", [(10, 1, 0, 1), (100, 1, 0, 1), (100, 1, 0, 3), (10, 1, 0, 3),
                                             (100, 4, 1, 1), (10, 3, 2, 1)])
def test_nccl_path_equals_external_exchange(shim, K, waves, E, parts):
    sweeps = 3
    with tempfile.TemporaryDirectory() as d:
        env = dict(os.environ, SPDP_NCCL_LIB=shim, SPDP_EXCHANGE_PARTS=str(parts))
        uid = os.path.join(d, "uid")
        out = os.path.join(d, "out.npz")
        procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "nccl_shim_worker.py"), str(r), "2", uid, out,
                                   str(K), str(waves), str(E), str(sweeps)], env=env) for r in range(2)]
        for p in procs:
            assert p.wait(timeout=300) == 0
        got = dict(np.load(out))
    if parts > 1:
        assert int(got["parts"]) == parts          # the pipelined exchange ran
    want = external(K, waves, E, sweeps)
    for k in ("z", "r", "n", "m", "t", "Q"):
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    assert np.isfinite(got["lj"]) and got["ppl"] > 1


def test_nccl_path_sparse_transform(shim):
    """NEXT-4 with NCCL: 2 processes, sparse P, vs the in-process external exchange."""
    from test_oracle_sparse_p import mixing_P
    K, sweeps = 10, 2
    with tempfile.TemporaryDirectory() as d:
        env = dict(os.environ, SPDP_NCCL_LIB=shim)
        uid = os.path.join(d, "uid"); out = os.path.join(d, "out.npz")
        procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "nccl_shim_worker.py"), str(r), "2", uid, out,
                                   str(K), "1", "0", str(sweeps), "sparse"], env=env) for r in range(2)]
        for p in procs:
            assert p.wait(timeout=300) == 0
        got = dict(np.load(out))
    c = corpus("C1")
    P = mixing_P(c.num_groups, c.vocab, np.random.default_rng(3))
    ranks = [spdp.sampler_for(c, K, rank=r, world_size=2, exchange=spdp.SPDP_EXCHANGE_EXTERNAL, transform=P, **HYPER)
             for r in range(2)]
    for _ in range(sweeps):
        for r in ranks:
            r.sweep_local()
        tot = sum(r.exchange_get().astype(np.int64) for r in ranks).astype(np.int32)
        for r in ranks:
            r.exchange_put(tot)
            r.sweep_merge()
    want = ranks[0].counts()
    for k in ("m", "t", "Q"):
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    np.testing.assert_array_equal(got["q"], ranks[0].sparse_state()["q"])
