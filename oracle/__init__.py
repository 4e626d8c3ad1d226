"""CPU oracle for the SPDP Gibbs sweep — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1510_06549_b200``) never imports, links or executes
anything under ``oracle/``; the two share no code.

The arithmetic lives in ``spdp_oracle.c`` (plain C, fp64, log space), which
cites the paper passage each function follows.  This module only builds it
with gcc and marshals arguments through ctypes.

Parity status of every oracle function is listed in DESIGN.md §4; each one
is pinned by a ``-m "not gpu"`` test in ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spdp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

P = C.c_void_p


_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")


def build(force: bool = False, openmp: bool = False) -> str:
    """gcc -O2 build of spdp_oracle.c.  openmp=True: the same source with -fopenmp (mode P's
    per-wave decisions over the host cores; the timing protocol of SURVEY §8(d) item (2))."""
    out = _LIB_OMP if openmp else _LIB
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", *(["-fopenmp"] if openmp else []), "-shared", "-fPIC", _SRC,
                               "-o", out, "-lm"])
    return out


def lib():
    """The oracle library; ORACLE_OPENMP=1 loads the -fopenmp build (timing only)."""
    global _lib
    if _lib is None:
        omp = os.environ.get("ORACLE_OPENMP") == "1"
        path = build(openmp=omp)
        L = C.CDLL(path)
        L.or_philox.argtypes = [P, P, P]
        L.or_log_stirling.restype = C.c_double
        L.or_log_stirling.argtypes = [C.c_double, C.c_int, C.c_int]
        L.or_ratio_table.restype = C.c_int
        L.or_ratio_table.argtypes = [C.c_double, C.c_int, P, P]
        L.or_create.restype = P
        L.or_create.argtypes = [C.c_int, C.c_int, C.c_int, P, C.c_double, P, P, C.c_uint64]
        L.or_destroy.argtypes = [P]
        L.or_load.restype = C.c_int
        L.or_load.argtypes = [P, C.c_int64, C.c_int32, P, P, P, P, P, P]
        L.or_sweep_seq.restype = C.c_int
        L.or_sweep_seq.argtypes = [P, C.c_int64]
        L.or_sweep_par.restype = C.c_int
        L.or_sweep_par.argtypes = [P, C.c_int, C.c_int, P, P, C.c_int64, P]
        L.or_sweep_par_e.restype = C.c_int
        L.or_sweep_par_e.argtypes = [P, C.c_int, C.c_int, C.c_int, P, P, C.c_int64, P]
        L.or_get.argtypes = [P] + [P] * 6
        L.or_sweep_index.restype = C.c_uint32
        L.or_sweep_index.argtypes = [P]
        L.or_set_sweep_index.argtypes = [P, C.c_uint32]
        L.or_stats.argtypes = [P, P]
        L.or_conditional.restype = C.c_int
        L.or_conditional.argtypes = [P, C.c_int64, C.c_int, P]
        L.or_debug_token.restype = C.c_int
        L.or_debug_token.argtypes = [P, C.c_int64, C.c_uint32, P, P, P, P]
        L.or_perplexity.restype = C.c_double
        L.or_perplexity.argtypes = [P]
        L.or_log_joint.restype = C.c_double
        L.or_log_joint.argtypes = [P]
        L.or_check_invariants.restype = C.c_int
        L.or_check_invariants.argtypes = [P]
        L.or_partition.argtypes = [P, C.c_int, P]
        L.or_sweep_shard.restype = C.c_int
        L.or_sweep_shard.argtypes = [P, C.c_int, C.c_int, C.c_int, P, P]
        L.or_merge.restype = C.c_int
        L.or_merge.argtypes = [P, P, P]
        L.or_word_prob.restype = C.c_double
        L.or_word_prob.argtypes = [P, C.c_int32, C.c_int32]
        L.or_chain_codes.restype = C.c_int
        L.or_chain_codes.argtypes = [P, C.c_int64, C.c_int, C.c_int, P]
        L.or_phi0.argtypes = [P, C.c_int, C.c_int]
        L.or_phi0.restype = C.c_double
        L.or_phi.argtypes = [P, C.c_int, C.c_int, C.c_int]
        L.or_phi.restype = C.c_double
        L.or_topics.argtypes = [P, P, P]
        L.or_topics.restype = None
        L.or_foldin.argtypes = [P, C.c_int64, C.c_int32, P, P, P, C.c_uint64, C.c_int32, C.c_int32, C.c_int, P, P, P, P]
        L.or_heldout_perplexity.argtypes = [P, C.c_int64, C.c_int32, P, P, P, P, P]
        L.or_heldout_perplexity.restype = C.c_double
        L.or_hellinger.argtypes = [C.c_int64, P, P]
        L.or_hellinger.restype = C.c_double
        L.or_greedy_match.argtypes = [C.c_int, P, P]
        L.or_greedy_match.restype = None
        L.or_topic_align.argtypes = [P, P, P, P]
        # NEXT-4 (sparse P^i)
        L.or_sp_create.restype = P
        L.or_sp_create.argtypes = [P, P, P, P]
        L.or_sp_destroy.argtypes = [P]
        L.or_sp_destroy.restype = None
        L.or_sp_sweep_seq.argtypes = [P]
        L.or_sp_sweep_par.argtypes = [P, C.c_int, P, P, P]
        L.or_sp_get.argtypes = [P, P, P]
        L.or_sp_get.restype = None
        L.or_sp_set_q.argtypes = [P, P]
        L.or_sp_conditional.argtypes = [P, C.c_int64, C.c_int, C.c_int32, P]
        L.or_sp_chain_codes.argtypes = [P, C.c_int64, C.c_int, C.c_int, P]
        L.or_sp_topics.argtypes = [P, P, P]
        L.or_sp_topics.restype = None
        L.or_sp_foldin.argtypes = [P, C.c_int64, C.c_int32, P, P, P, C.c_uint64, C.c_int32, C.c_int32, C.c_int, P, P, P, P]
        L.or_sp_heldout_perplexity.argtypes = [P, C.c_int64, C.c_int32, P, P, P, P, P]
        L.or_sp_heldout_perplexity.restype = C.c_double
        L.or_sp_perplexity.argtypes = [P]
        L.or_sp_sweep_shards.argtypes = [P, C.c_int, C.c_int]
        L.or_sp_log_joint.argtypes = [P]
        L.or_sp_log_joint.restype = C.c_double
        L.or_sp_perplexity.restype = C.c_double
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def philox(ctr, key):
    """Philox4x32-10 of a 4-word counter and 2-word key (both uint32)."""
    c = np.asarray(ctr, np.uint32); k = np.asarray(key, np.uint32); out = np.zeros(4, np.uint32)
    lib().or_philox(_ptr(c), _ptr(k), _ptr(out))
    return out


def ratio_table(a: float, mmax: int):
    """(A0, A1) fp64 at m(m+1)/2 + t, 0 <= t <= m <= mmax (spdp_oracle.c or_ratio_table)."""
    n = (mmax + 1) * (mmax + 2) // 2
    A0, A1 = np.zeros(n), np.zeros(n)
    if lib().or_ratio_table(float(a), int(mmax), _ptr(A0), _ptr(A1)) != 0:
        raise MemoryError("or_ratio_table")
    return A0, A1


def log_stirling(a: float, n: int, m: int) -> float:
    """log S^n_{m,a} by the recursion of PAPER.md:1454-1455 (fp64, log space)."""
    return lib().or_log_stirling(float(a), int(n), int(m))


class Oracle:
    """Sequential (mode S) and wave-snapshot (mode P) SPDP Gibbs sampler."""

    def __init__(self, num_groups, vocab, num_topics, alpha, beta, discount, concentration, seed):
        L = lib()
        I, V, K = int(num_groups), int(vocab), int(num_topics)
        al = np.asarray(alpha, np.float64)
        al = np.full((I, K), float(al)) if al.ndim == 0 else al.reshape(I, K).astype(np.float64)
        a = np.asarray(discount, np.float64); a = np.full(I, float(a)) if a.ndim == 0 else a.astype(np.float64)
        b = np.asarray(concentration, np.float64); b = np.full(I, float(b)) if b.ndim == 0 else b.astype(np.float64)
        self._keep = (np.ascontiguousarray(al), np.ascontiguousarray(a), np.ascontiguousarray(b))
        self.I, self.V, self.K = I, V, K
        self.h = L.or_create(I, V, K, _ptr(self._keep[0]), float(beta), _ptr(self._keep[1]), _ptr(self._keep[2]),
                             C.c_uint64(int(seed) & (2**64 - 1)))
        if not self.h:
            raise ValueError("or_create: invalid parameters")
        self.N = 0
        self.D = 0

    def close(self):
        if self.h:
            lib().or_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, group, doc, word, num_docs, z_init=None, r_init=None, t_init=None):
        g = np.ascontiguousarray(group, np.int32); d = np.ascontiguousarray(doc, np.int32)
        w = np.ascontiguousarray(word, np.int32)
        z = None if z_init is None else np.ascontiguousarray(z_init, np.int32)
        r = None if r_init is None else np.ascontiguousarray(r_init, np.uint8)
        t = None if t_init is None else np.ascontiguousarray(np.asarray(t_init).reshape(-1), np.int32)
        rc = lib().or_load(self.h, len(w), int(num_docs), _ptr(g), _ptr(d), _ptr(w), _ptr(z), _ptr(r), _ptr(t))
        if rc != 0:
            raise ValueError(f"or_load failed ({rc})")
        self.N, self.D = len(w), int(num_docs)
        self._tok = (g, d, w)

    def sweep_seq(self, max_tokens: int = -1):
        if lib().or_sweep_seq(self.h, int(max_tokens)) != 0:
            raise RuntimeError("or_sweep_seq failed")

    def sweep_par(self, waves: int = 1, shards: int = 1, force_zr=None, want_margin=False, max_tokens: int = -1,
                  want_own=False, merge_every: int = 0):
        """Mode-P sweep.  Returns margin [N] (or None), and with want_own also the
        oracle's own draws z | r<<15 [N] (before force_zr replaced them).
        merge_every E >= 1: the shards exchange after every E waves (NEXT-3)."""
        f = None if force_zr is None else np.ascontiguousarray(force_zr, np.int32)
        mg = np.full(self.N, np.inf) if want_margin else None
        own = np.full(self.N, -1, np.int32) if want_own else None
        rc = lib().or_sweep_par_e(self.h, int(waves), int(shards), int(merge_every), _ptr(f), _ptr(mg),
                                  int(max_tokens), _ptr(own))
        if rc != 0:
            raise RuntimeError("or_sweep_par failed")
        return (mg, own) if want_own else mg

    def sweep_shard(self, waves: int, shards: int, shard: int):
        """One shard's part of a distributed mode-P sweep: returns its net changes
        (Dm, Dt) as int32 [I*V*K]; the global counts are left untouched."""
        cells = self.I * self.V * self.K
        Dm = np.zeros(cells, np.int32); Dt = np.zeros(cells, np.int32)
        if lib().or_sweep_shard(self.h, int(waves), int(shards), int(shard), _ptr(Dm), _ptr(Dt)) != 0:
            raise RuntimeError("or_sweep_shard failed")
        return Dm, Dt

    def merge(self, Dm_sum, Dt_sum):
        Dm = np.ascontiguousarray(Dm_sum, np.int32); Dt = np.ascontiguousarray(Dt_sum, np.int32)
        lib().or_merge(self.h, _ptr(Dm), _ptr(Dt))

    @property
    def sweep_index(self) -> int:
        return int(lib().or_sweep_index(self.h))

    @sweep_index.setter
    def sweep_index(self, v: int):
        lib().or_set_sweep_index(self.h, int(v))

    def stats(self):
        s = np.zeros(8, np.int64)
        lib().or_stats(self.h, _ptr(s))
        return {"keeps": int(s[0]), "moved": int(s[1]), "clamped": int(s[2]), "forced_differ": int(s[3])}

    def state(self):
        """dict of z [N], r [N], n [D,K], m [I,V,K], t [I,V,K], Q [K,V]."""
        I, V, K = self.I, self.V, self.K
        z = np.zeros(self.N, np.int32); r = np.zeros(self.N, np.uint8)
        n = np.zeros((self.D, K), np.int32); m = np.zeros((I, V, K), np.int32); t = np.zeros((I, V, K), np.int32)
        Q = np.zeros((K, V), np.int32)
        lib().or_get(self.h, _ptr(z), _ptr(r), _ptr(n), _ptr(m), _ptr(t), _ptr(Q))
        return {"z": z, "r": r, "n": n, "m": m, "t": t, "Q": Q}

    def conditional(self, tok: int, r_rem: int):
        p = np.zeros(2 * self.K)
        rc = lib().or_conditional(self.h, int(tok), int(r_rem), _ptr(p))
        return None if rc != 0 else p

    def debug_token(self, tok: int, sweep: int):
        p = np.zeros(2 * self.K); info = np.zeros(4, np.int32); u = C.c_double(); mg = C.c_double()
        rc = lib().or_debug_token(self.h, int(tok), int(sweep), _ptr(p), _ptr(info), C.byref(u), C.byref(mg))
        if rc != 0:
            raise RuntimeError("or_debug_token failed")
        return {"prob": p, "r_rem": int(info[0]), "keep": int(info[1]), "z": int(info[2]), "r": int(info[3]),
                "u": u.value, "margin": mg.value}

    def perplexity(self) -> float:
        return float(lib().or_perplexity(self.h))

    def log_joint(self) -> float:
        return float(lib().or_log_joint(self.h))

    def word_prob(self, doc: int, word: int) -> float:
        return float(lib().or_word_prob(self.h, int(doc), int(word)))

    def chain_codes(self, nsweeps: int, waves: int = -1, tbase: int = 5):
        out = np.zeros(int(nsweeps), np.int64)
        if lib().or_chain_codes(self.h, int(nsweeps), int(waves), int(tbase), _ptr(out)) != 0:
            raise RuntimeError("or_chain_codes failed")
        return out

    def check_invariants(self) -> int:
        return int(lib().or_check_invariants(self.h))

    # ---------------- NEXT-1: held-out evaluation ----------------
    def topics(self):
        """(phi0 [K,V], phi [I,K,V]): Eqs. P:1753-1754 of the current state."""
        p0 = np.zeros((self.K, self.V)); p = np.zeros((self.I, self.K, self.V))
        lib().or_topics(self.h, _ptr(p0), _ptr(p))
        return p0, p

    def foldin(self, group, doc, word, num_docs, seed, iterations, first_iteration=0, z=None,
               force_z=None, want_margin=False):
        """Fold-in (reading c21).  z None: Philox initial topics.  Returns z, or with
        want_margin (z, margins, own draws before forcing)."""
        g = np.ascontiguousarray(group, np.int32); d = np.ascontiguousarray(doc, np.int32)
        w = np.ascontiguousarray(word, np.int32)
        init = z is None
        zz = np.full(len(g), -1, np.int32) if init else np.array(z, np.int32, copy=True)
        fz = None if force_z is None else np.ascontiguousarray(force_z, np.int32)
        mg = np.zeros(len(g)) if want_margin else None
        own = np.zeros(len(g), np.int32) if want_margin else None
        rc = lib().or_foldin(self.h, len(g), int(num_docs), _ptr(g), _ptr(d), _ptr(w), int(seed) & (2**64 - 1),
                             int(first_iteration), int(iterations), int(init), _ptr(zz), _ptr(fz), _ptr(mg),
                             _ptr(own))
        if rc != 0:
            raise RuntimeError(f"or_foldin failed ({rc})")
        return (zz, mg, own) if want_margin else zz

    def heldout_perplexity(self, group, doc, word, num_docs, z, want_theta=False):
        g = np.ascontiguousarray(group, np.int32); d = np.ascontiguousarray(doc, np.int32)
        w = np.ascontiguousarray(word, np.int32); zz = np.ascontiguousarray(z, np.int32)
        th = np.zeros((int(num_docs), self.K)) if want_theta else None
        ppl = float(lib().or_heldout_perplexity(self.h, len(g), int(num_docs), _ptr(g), _ptr(d), _ptr(w), _ptr(zz),
                                                _ptr(th)))
        return (ppl, th) if want_theta else ppl

    def topic_align(self, other):
        """(dist [K,K] Hellinger on phi0~, perm [K]) against another oracle state."""
        dist = np.zeros((self.K, self.K)); perm = np.zeros(self.K, np.int32)
        if lib().or_topic_align(self.h, other.h, _ptr(dist), _ptr(perm)) != 0:
            raise RuntimeError("or_topic_align: K or V mismatch")
        return dist, perm

    def partition(self, shards: int):
        out = np.zeros(self.D, np.int32)
        lib().or_partition(self.h, int(shards), _ptr(out))
        return out


class SparseOracle:
    """NEXT-4: the sampler with sparse transformation matrices P^i (spdp_oracle.c
    "NEXT-4").  P as CSR rows over (i, w): pptr [I*V+1], pv [E] source words,
    pp [E] weights (columns of each P^i sum to 1).  Wraps a loaded Oracle."""

    def __init__(self, base: "Oracle", pptr, pv, pp):
        self.base = base
        self._keep = (np.ascontiguousarray(pptr, np.int32), np.ascontiguousarray(pv, np.int32),
                      np.ascontiguousarray(pp, np.float64))
        self.E = int(self._keep[0][-1])
        self.h = lib().or_sp_create(base.h, *(_ptr(a) for a in self._keep))
        if not self.h:
            raise ValueError("invalid P (rows need a source, columns must sum to 1)")

    def close(self):
        if getattr(self, "h", None):
            lib().or_sp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sweep_seq(self):
        if lib().or_sp_sweep_seq(self.h) != 0:
            raise RuntimeError("or_sp_sweep_seq failed")

    def sweep_par(self, waves=1, force=None, want_margin=False, want_own=False):
        f = None if force is None else np.ascontiguousarray(force, np.int32)
        mg = np.full(self.base.N, np.inf) if want_margin else None
        own = np.full(self.base.N, -1, np.int32) if want_own else None
        if lib().or_sp_sweep_par(self.h, int(waves), _ptr(f), _ptr(mg), _ptr(own)) != 0:
            raise RuntimeError("or_sp_sweep_par failed")
        return mg, own

    def sweep_shards(self, waves=1, shards=1):
        """Mode P over several shards with one exchange per sweep (NEXT-4 on several GPUs)."""
        if lib().or_sp_sweep_shards(self.h, int(waves), int(shards)) != 0:
            raise RuntimeError("or_sp_sweep_shards failed")

    def state(self):
        st = self.base.state()
        q = np.zeros((self.E, self.base.K), np.int32); Qs = np.zeros((self.base.K, self.base.V), np.int64)
        lib().or_sp_get(self.h, _ptr(q), _ptr(Qs))
        st["q"], st["Qs"] = q, Qs
        return st

    def set_q(self, q):
        q = np.ascontiguousarray(q, np.int32)
        lib().or_sp_set_q(self.h, _ptr(q))

    def conditional(self, tok, r_rem, e_rem):
        i, w = int(self.base._tok[0][tok]), int(self.base._tok[2][tok])
        r = i * self.base.V + w
        S = int(self._keep[0][r + 1] - self._keep[0][r])
        out = np.zeros(self.base.K * (S + 1))
        rc = lib().or_sp_conditional(self.h, int(tok), int(r_rem), int(e_rem), _ptr(out))
        return None if rc != 0 else out

    def topics(self):
        p0 = np.zeros((self.base.K, self.base.V)); p = np.zeros((self.base.I, self.base.K, self.base.V))
        lib().or_sp_topics(self.h, _ptr(p0), _ptr(p))
        return p0, p

    def perplexity(self):
        return float(lib().or_sp_perplexity(self.h))

    def log_joint(self):
        return float(lib().or_sp_log_joint(self.h))

    def foldin(self, group, doc, word, num_docs, seed, iterations, first_iteration=0, z=None, force_z=None,
               want_margin=False):
        g = np.ascontiguousarray(group, np.int32); d = np.ascontiguousarray(doc, np.int32)
        w = np.ascontiguousarray(word, np.int32)
        init = z is None
        zz = np.full(len(g), -1, np.int32) if init else np.array(z, np.int32, copy=True)
        fz = None if force_z is None else np.ascontiguousarray(force_z, np.int32)
        mg = np.zeros(len(g)) if want_margin else None
        own = np.zeros(len(g), np.int32) if want_margin else None
        rc = lib().or_sp_foldin(self.h, len(g), int(num_docs), _ptr(g), _ptr(d), _ptr(w), int(seed) & (2**64 - 1),
                                int(first_iteration), int(iterations), int(init), _ptr(zz), _ptr(fz), _ptr(mg), _ptr(own))
        if rc != 0:
            raise RuntimeError(f"or_sp_foldin failed ({rc})")
        return (zz, mg, own) if want_margin else zz

    def heldout_perplexity(self, group, doc, word, num_docs, z, want_theta=False):
        g = np.ascontiguousarray(group, np.int32); d = np.ascontiguousarray(doc, np.int32)
        w = np.ascontiguousarray(word, np.int32); zz = np.ascontiguousarray(z, np.int32)
        th = np.zeros((int(num_docs), self.base.K)) if want_theta else None
        ppl = float(lib().or_sp_heldout_perplexity(self.h, len(g), int(num_docs), _ptr(g), _ptr(d), _ptr(w),
                                                   _ptr(zz), _ptr(th)))
        return (ppl, th) if want_theta else ppl

    def chain_codes(self, nsweeps, waves=-1, qbase=5):
        out = np.zeros(int(nsweeps), np.int64)
        if lib().or_sp_chain_codes(self.h, int(nsweeps), int(waves), int(qbase), _ptr(out)) != 0:
            raise RuntimeError("or_sp_chain_codes failed")
        return out


def hellinger(p, q) -> float:
    p = np.ascontiguousarray(p, np.float64); q = np.ascontiguousarray(q, np.float64)
    assert p.shape == q.shape
    return float(lib().or_hellinger(p.size, _ptr(p), _ptr(q)))


def greedy_match(dist):
    d = np.ascontiguousarray(dist, np.float64); K = d.shape[0]
    perm = np.zeros(K, np.int32)
    lib().or_greedy_match(K, _ptr(d), _ptr(perm))
    return perm


def from_corpus(corpus, num_topics, alpha=0.1, beta=0.1, discount=0.7, concentration=100.0, seed=7,
                z_init=None, r_init=None, t_init=None) -> Oracle:
    o = Oracle(corpus.num_groups, corpus.vocab, num_topics, alpha, beta, discount, concentration, seed)
    o.load(corpus.group, corpus.doc, corpus.word, corpus.num_docs, z_init, r_init, t_init)
    return o
