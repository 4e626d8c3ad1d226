"""Seeded synthetic corpora shaped like the paper's multi-group collections.

INPUT GENERATION ONLY: this module holds none of the sampler's arithmetic.
It is the one module both the oracle tests and the CUDA path may share
(SURVEY.md §8(d) "Synthetic inputs").  The corpus is drawn from the SPDP
generative process with identity P (§2.3.4) realised
with the Pitman–Yor seating rule; see synth/gen.c.

Configs C1..C5 are BASELINE.json's `configs`, with the per-config recipe of
SURVEY.md §8(d) (groups x docs per group, Poisson mean length, V, K_gen, K,
generator seed).  Sampler hyper-parameters are the paper's
alpha = beta = 0.1, a = 0.7, b = 100 (§4.1).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libsynth.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-shared", "-fPIC", _SRC, "-o", _LIB, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.synth_num_tokens.restype = ctypes.c_int64
        lib.synth_num_tokens.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_uint64, ctypes.c_int]
        lib.synth_spdp_corpus.restype = ctypes.c_int
        lib.synth_spdp_corpus.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_uint64, ctypes.c_int] + [ctypes.c_void_p] * 4
        _lib = lib
    return _lib


@dataclass(frozen=True)
class CorpusConfig:
    name: str
    groups: int            # I
    docs_per_group: int    # D_i
    mean_len: float        # Poisson lambda of document length
    vocab: int             # V
    k_gen: int             # topics of the generating process
    k: int                 # topics of the sampler
    gen_seed: int
    # sampler settings
    alpha: float = 0.1
    beta: float = 0.1
    discount: float = 0.7
    concentration: float = 100.0
    seed: int = 7
    sweeps: int = 20
    # generator hyper-parameters
    alpha_gen: float = 0.1
    beta_gen: float = 0.1
    # one generator per document / topic / restaurant, drawn in parallel (synth/gen.c per_unit)
    per_unit_streams: bool = False

    def with_k(self, k: int) -> "CorpusConfig":
        return replace(self, k=k, name=f"{self.name}_K{k}")


CONFIGS = {
    "C1": CorpusConfig("C1", 2, 100, 100.0, 1_000, 10, 10, 101, sweeps=20),
    "C2": CorpusConfig("C2", 3, 3_000, 111.0, 10_000, 50, 50, 102, sweeps=20),
    "C3": CorpusConfig("C3", 4, 20_000, 125.0, 30_000, 100, 100, 103, sweeps=20),
    "C4": CorpusConfig("C4", 4, 10_000, 125.0, 30_000, 100, 100, 104, sweeps=10),
    # C5 (~200 M tokens) is drawn with per-unit generator streams, in parallel (round 2; round 1's C5
    # used the single-stream draw, ~110 s on 8 cores: same process and shape, a different draw)
    "C5": CorpusConfig("C5", 16, 200_000, 62.5, 100_000, 200, 200, 105, sweeps=10, per_unit_streams=True),
}


@dataclass
class Corpus:
    group: np.ndarray   # int32 [N]
    doc: np.ndarray     # int32 [N], global doc ids in [0, num_docs)
    word: np.ndarray    # int32 [N]
    z_gen: np.ndarray   # int32 [N], generating topic (not used by the sampler)
    num_groups: int
    num_docs: int
    vocab: int

    @property
    def num_tokens(self) -> int:
        return int(self.word.shape[0])


def generate(groups: int, docs_per_group: int, mean_len: float, vocab: int, k_gen: int,
             seed: int, alpha_gen: float = 0.1, beta_gen: float = 0.1,
             discount: float = 0.7, concentration: float = 100.0, per_unit_streams: bool = False) -> Corpus:
    lib = _load()
    n = lib.synth_num_tokens(groups, docs_per_group, mean_len, seed, int(per_unit_streams))
    if n < 0:
        raise MemoryError("synth_num_tokens failed")
    g = np.empty(n, np.int32); d = np.empty(n, np.int32); w = np.empty(n, np.int32); z = np.empty(n, np.int32)
    rc = lib.synth_spdp_corpus(groups, docs_per_group, mean_len, vocab, k_gen, alpha_gen, beta_gen,
                               discount, concentration, seed, int(per_unit_streams),
                               g.ctypes.data, d.ctypes.data, w.ctypes.data, z.ctypes.data)
    if rc != 0:
        raise MemoryError("synth_spdp_corpus failed")
    return Corpus(g, d, w, z, groups, groups * docs_per_group, vocab)


def corpus_for(cfg: CorpusConfig) -> Corpus:
    return generate(cfg.groups, cfg.docs_per_group, cfg.mean_len, cfg.vocab, cfg.k_gen, cfg.gen_seed,
                    cfg.alpha_gen, cfg.beta_gen, cfg.discount, cfg.concentration, cfg.per_unit_streams)


def tiny_corpus(groups: int, docs: list[list[int]], doc_group: list[int], vocab: int) -> Corpus:
    """Hand-written corpus: docs[d] = list of word ids, doc_group[d] = its group."""
    g, d, w = [], [], []
    for di, words in enumerate(docs):
        for x in words:
            g.append(doc_group[di]); d.append(di); w.append(x)
    a = lambda v: np.asarray(v, np.int32)
    return Corpus(a(g), a(d), a(w), np.zeros(len(w), np.int32), groups, len(docs), vocab)


def holdout_split(corpus: Corpus, fraction: float = 0.1, seed: int = 0) -> tuple[Corpus, Corpus]:
    """(train, test): hold out ``fraction`` of the documents of every group
    (§4.1: "For each group, 10% of the data is held out
    from training for computing the perplexity").  Seeded choice of
    round(fraction * D_i) documents per group; doc ids renumbered densely in
    each part, token order kept (canonical: group, doc, position)."""
    rng = np.random.default_rng(seed)
    doc_group = np.full(corpus.num_docs, -1, np.int64)
    doc_group[corpus.doc] = corpus.group
    test_doc = np.zeros(corpus.num_docs, bool)
    for i in range(corpus.num_groups):
        ids = np.nonzero(doc_group == i)[0]
        k = int(round(fraction * len(ids)))
        if k:
            test_doc[rng.choice(ids, size=k, replace=False)] = True

    def part(mask_doc):
        keep = mask_doc[corpus.doc]
        old = np.nonzero(mask_doc)[0]
        new_id = np.full(corpus.num_docs, -1, np.int64)
        new_id[old] = np.arange(len(old))
        return Corpus(corpus.group[keep].copy(), new_id[corpus.doc[keep]].astype(np.int32), corpus.word[keep].copy(),
                      corpus.z_gen[keep].copy(), corpus.num_groups, int(len(old)), corpus.vocab)

    return part(~test_doc), part(test_doc)


def duplicate(corpus: Corpus, copies: int) -> Corpus:
    """Training-data duplication (§3.3):
    the corpus followed by `copies` more copies of every document, as new
    documents (copy j of doc d is doc j*D + d; its tokens follow all tokens of
    copy j-1, so canonical token j*N + p is copy j of token p).  With several
    ranks the copies of a document usually land on different ranks (the
    partition keys on the doc id), which is what averages out their errors."""
    if copies < 0:
        raise ValueError("copies must be >= 0")
    n = copies + 1
    rep = lambda a: np.tile(a, n)
    doc = np.concatenate([corpus.doc + j * corpus.num_docs for j in range(n)]).astype(np.int32)
    return Corpus(rep(corpus.group).astype(np.int32), doc, rep(corpus.word).astype(np.int32),
                  rep(corpus.z_gen).astype(np.int32), corpus.num_groups, corpus.num_docs * n, corpus.vocab)
