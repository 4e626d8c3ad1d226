"""paper_1510_06549_b200 — B200-native SPDP Gibbs sweep (MGPU-DP-SPDP hot path).

Thin Python binding over ``libspdp.so`` (C ABI in ``include/spdp.h``): the
functions below carry the C names and only marshal arguments (numpy arrays ->
host pointers).  Every step of the sweep runs in the library's sm_100a
kernels; there is no CPU fallback, and importing fails loudly when the
library is missing or cannot be loaded.

``Sampler`` is a small convenience object over the same calls.
"""
from __future__ import annotations

import ctypes as C
import glob
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
LIB_PATH = os.environ.get("SPDP_LIB") or os.path.join(_HERE, "libspdp.so")   # SPDP_LIB: tuning variants
# every source the library is compiled from (spdp.cu includes the headers): a change to any of them rebuilds it
_SOURCES = sorted(glob.glob(os.path.join(_HERE, "csrc", "*.cu")) + glob.glob(os.path.join(_HERE, "csrc", "*.cuh"))) + [
    os.path.join(_ROOT, "include", "spdp.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]

SPDP_OK, SPDP_EINVAL, SPDP_ENOMEM, SPDP_ECUDA, SPDP_ENCCL, SPDP_ESTATE, SPDP_ETABLE, SPDP_EINTEGRITY = 0, -1, -2, -3, -4, -5, -6, -7
SPDP_EXCHANGE_NCCL, SPDP_EXCHANGE_EXTERNAL = 0, 1
SPDP_UPDATE_WAVE, SPDP_UPDATE_ASYNC = 0, 1
_NAMES = {0: "SPDP_OK", -1: "SPDP_EINVAL", -2: "SPDP_ENOMEM", -3: "SPDP_ECUDA", -4: "SPDP_ENCCL",
          -5: "SPDP_ESTATE", -6: "SPDP_ETABLE", -7: "SPDP_EINTEGRITY"}

# every symbol include/spdp.h declares
EXPORTS = ["spdp_create", "spdp_load_corpus", "spdp_set_state", "spdp_sweep", "spdp_sweep_local",
           "spdp_exchange_buffer", "spdp_exchange_copy", "spdp_sweep_merge", "spdp_counts", "spdp_loglik", "spdp_debug_probs",
           "spdp_stats", "spdp_profile", "spdp_timings", "spdp_partition", "spdp_nccl_unique_id", "spdp_destroy", "spdp_last_error",
           "spdp_version", "spdp_topics", "spdp_heldout", "spdp_topic_hellinger", "spdp_exchange_blocks", "spdp_zr",
           "spdp_set_transform", "spdp_sparse_state", "spdp_zr_async", "spdp_wait", "spdp_debug_ratio_table",
           "spdp_debug_chain", "spdp_zr8_async", "spdp_sweep_async"]


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libspdp.so for sm_100a in-tree (nvcc cross-compiles without a GPU)."""
    # a variant library named by SPDP_LIB (tuning A/B) is used as built, never recompiled from the tree
    variant = bool(os.environ.get("SPDP_LIB")) and os.path.exists(LIB_PATH)
    stale = force or not os.path.exists(LIB_PATH) or (not variant and any(
        os.path.getmtime(s) > os.path.getmtime(LIB_PATH) for s in _SOURCES))
    if stale:
        cmd = ["nvcc", *NVCC_FLAGS, os.path.join(_HERE, "csrc", "spdp.cu"), "-o", LIB_PATH, "-ldl", "-lpthread"]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
    return LIB_PATH


class SPDPError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


class spdp_config(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("num_groups", C.c_int32), ("vocab_size", C.c_int32),
                ("num_topics", C.c_int32), ("alpha", C.c_double), ("alpha_ik", C.c_void_p), ("beta", C.c_double),
                ("discount", C.c_void_p), ("concentration", C.c_void_p), ("seed", C.c_uint64),
                ("num_waves", C.c_int32), ("device", C.c_int32), ("rank", C.c_int32), ("world_size", C.c_int32),
                ("exchange", C.c_int32), ("nccl_unique_id", C.c_void_p), ("stream", C.c_void_p),
                ("debug_checks", C.c_int32), ("update_mode", C.c_int32), ("merge_every", C.c_int32)]


_lib = None


def lib():
    """Load libspdp.so (fails loudly: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc sm_100a) first")
        L = C.CDLL(LIB_PATH)
        P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "spdp_create": [P, P], "spdp_load_corpus": [P, I64, I32, P, P, P, P, P],
            "spdp_set_state": [P, P, P, P], "spdp_sweep": [P, I32], "spdp_sweep_local": [P],
            "spdp_exchange_buffer": [P, P, P, P], "spdp_exchange_copy": [P, P, I32], "spdp_sweep_merge": [P], "spdp_counts": [P, P, P, P, P, P, P],
            "spdp_loglik": [P, P, P], "spdp_debug_probs": [P, I64, P, P, P], "spdp_stats": [P, P],
            "spdp_profile": [P, I32], "spdp_timings": [P, P],
            "spdp_partition": [C.c_uint64, I32, I64, I32, P, P], "spdp_nccl_unique_id": [P],
            "spdp_topics": [P, P, P],
            "spdp_heldout": [P, I64, I32, P, P, P, C.c_uint64, I32, I32, P, P, P, P],
            "spdp_topic_hellinger": [P, P, P, P], "spdp_exchange_blocks": [P, P], "spdp_zr": [P, P], "spdp_zr_async": [P, P], "spdp_wait": [P], "spdp_set_transform": [P, P, P, P], "spdp_sparse_state": [P, P, P, P],
            "spdp_debug_ratio_table": [P, I32, I32, P], "spdp_debug_chain": [P, I32, I32, P], "spdp_zr8_async": [P, P], "spdp_sweep_async": [P, I32],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.spdp_destroy.argtypes = [P]
        L.spdp_destroy.restype = None
        L.spdp_last_error.argtypes = [P]
        L.spdp_last_error.restype = C.c_char_p
        L.spdp_version.argtypes = []
        L.spdp_version.restype = C.c_char_p
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _check(code, ctx=None):
    if code != SPDP_OK:
        msg = lib().spdp_last_error(ctx).decode() if ctx else ""
        raise SPDPError(code, msg)


# ---------------------------------------------------------------- C-named calls
def spdp_version() -> str:
    return lib().spdp_version().decode()


def spdp_partition(seed: int, world_size: int, doc, num_docs: int):
    d = np.ascontiguousarray(doc, np.int32)
    out = np.zeros(int(num_docs), np.int32)
    _check(lib().spdp_partition(C.c_uint64(int(seed) & (2**64 - 1)), int(world_size), len(d), int(num_docs), _p(d), _p(out)))
    return out


def spdp_nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().spdp_nccl_unique_id(buf))
    return bytes(buf)


def spdp_create(num_groups, vocab_size, num_topics, alpha=0.1, beta=0.1, discount=0.7, concentration=100.0,
                seed=7, num_waves=1, device=0, rank=0, world_size=1, exchange=SPDP_EXCHANGE_NCCL,
                nccl_unique_id=None, stream=None, debug_checks=False, alpha_ik=None, update_mode=SPDP_UPDATE_WAVE,
                merge_every=0):
    """Returns (ctx handle, keep-alive tuple)."""
    I, K = int(num_groups), int(num_topics)
    disc = np.ascontiguousarray(np.broadcast_to(np.asarray(discount, np.float64), (I,)))
    conc = np.ascontiguousarray(np.broadcast_to(np.asarray(concentration, np.float64), (I,)))
    aik = None if alpha_ik is None else np.ascontiguousarray(np.asarray(alpha_ik, np.float64).reshape(I, K))
    uid = None if nccl_unique_id is None else C.create_string_buffer(bytes(nccl_unique_id), 128)
    cfg = spdp_config(C.sizeof(spdp_config), I, int(vocab_size), K, float(alpha), _p(aik), float(beta),
                      _p(disc), _p(conc), int(seed) & (2**64 - 1), int(num_waves), int(device), int(rank),
                      int(world_size), int(exchange), C.cast(uid, C.c_void_p) if uid is not None else None,
                      stream, int(bool(debug_checks)), int(update_mode), int(merge_every))
    h = C.c_void_p()
    code = lib().spdp_create(C.byref(cfg), C.byref(h))
    if code != SPDP_OK:
        msg = lib().spdp_last_error(h).decode() if h else ""
        if h:
            lib().spdp_destroy(h)
        raise SPDPError(code, msg)
    return h


def spdp_load_corpus(ctx, group, doc, word, num_docs, z_init=None, r_init=None):
    g = np.ascontiguousarray(group, np.int32); d = np.ascontiguousarray(doc, np.int32)
    w = np.ascontiguousarray(word, np.int32)
    z = None if z_init is None else np.ascontiguousarray(z_init, np.int32)
    r = None if r_init is None else np.ascontiguousarray(r_init, np.uint8)
    _check(lib().spdp_load_corpus(ctx, len(w), int(num_docs), _p(g), _p(d), _p(w), _p(z), _p(r)), ctx)


def spdp_set_state(ctx, z, r=None, tables=None):
    z = np.ascontiguousarray(z, np.int32)
    r = None if r is None else np.ascontiguousarray(r, np.uint8)
    t = None if tables is None else np.ascontiguousarray(np.asarray(tables).reshape(-1), np.int32)
    _check(lib().spdp_set_state(ctx, _p(z), _p(r), _p(t)), ctx)


def spdp_sweep(ctx, num_sweeps=1):
    _check(lib().spdp_sweep(ctx, int(num_sweeps)), ctx)


def spdp_sweep_local(ctx):
    _check(lib().spdp_sweep_local(ctx), ctx)


def spdp_exchange_buffer(ctx):
    """(device pointer, element count, element bytes): packed dm*2^B + dt per cell (B = 16 or 32)."""
    ptr, cnt, eb = C.c_void_p(), C.c_int64(), C.c_int32()
    _check(lib().spdp_exchange_buffer(ctx, C.byref(ptr), C.byref(cnt), C.byref(eb)), ctx)
    return ptr.value, cnt.value, eb.value


def spdp_exchange_copy(ctx, host, to_device):
    """host: contiguous int32 (4-byte elements) or int64 numpy array of spdp_exchange_buffer()[1] elements."""
    assert host.dtype in (np.int32, np.int64) and host.flags["C_CONTIGUOUS"]
    _check(lib().spdp_exchange_copy(ctx, _p(host), int(bool(to_device))), ctx)
    return host


def spdp_sweep_merge(ctx):
    _check(lib().spdp_sweep_merge(ctx), ctx)


def spdp_counts(ctx, N, D, I, V, K, z=True, r=True, doc_topic=True, customers=True, tables=True, shadow=True,
                out=None):
    """State read-out.  out: optional dict of caller-owned arrays to fill (reused across calls)."""
    out = {} if out is None else out
    shapes = {"z": ((N,), np.int32, z), "r": ((N,), np.uint8, r), "n": ((D, K), np.int32, doc_topic),
              "m": ((I, V, K), np.int32, customers), "t": ((I, V, K), np.int32, tables), "Q": ((K, V), np.int32, shadow)}
    for k, (shape, dt, want) in shapes.items():
        if not want:
            out.pop(k, None)
        elif k not in out:
            out[k] = np.zeros(shape, dt)
        else:
            assert out[k].shape == shape and out[k].dtype == dt and out[k].flags["C_CONTIGUOUS"], k
    _check(lib().spdp_counts(ctx, _p(out.get("z")), _p(out.get("r")), _p(out.get("n")), _p(out.get("m")),
                             _p(out.get("t")), _p(out.get("Q"))), ctx)
    return out


def spdp_zr(ctx, N, out=None):
    """Packed assignments z | r << 15 [N] uint16 (out: caller-owned, e.g. pinned, reused)."""
    out = np.empty(N, np.uint16) if out is None else out
    assert out.dtype == np.uint16 and out.shape == (N,) and out.flags["C_CONTIGUOUS"]
    _check(lib().spdp_zr(ctx, _p(out)), ctx)
    return out


def spdp_zr_async(ctx, N, out):
    """Queue the packed assignments' copy into out (caller-owned, pinned, kept alive
    until spdp_wait); returns at once (include/spdp.h)."""
    assert out.dtype == np.uint16 and out.shape == (N,) and out.flags["C_CONTIGUOUS"]
    _check(lib().spdp_zr_async(ctx, _p(out)), ctx)
    return out


def spdp_sweep_async(ctx, num_sweeps):
    _check(lib().spdp_sweep_async(ctx, int(num_sweeps)), ctx)


def spdp_zr8_async(ctx, N, out):
    """spdp_zr_async with one byte per token (z | r << 7, K <= 128)."""
    assert out.dtype == np.uint8 and out.shape == (N,) and out.flags["C_CONTIGUOUS"]
    _check(lib().spdp_zr8_async(ctx, _p(out)), ctx)
    return out


def spdp_wait(ctx):
    _check(lib().spdp_wait(ctx), ctx)


def spdp_loglik(ctx, log_joint=True, perplexity=True):
    lj, pp = C.c_double(np.nan), C.c_double(np.nan)
    _check(lib().spdp_loglik(ctx, C.byref(lj) if log_joint else None, C.byref(pp) if perplexity else None), ctx)
    return (lj.value if log_joint else None), (pp.value if perplexity else None)


def spdp_topics(ctx, I, V, K, phi0=True, phi=True):
    """(phi0 [K,V], phi [I,K,V]) fp64 estimates, or None for a skipped one."""
    p0 = np.zeros((K, V)) if phi0 else None
    p = np.zeros((I, K, V)) if phi else None
    _check(lib().spdp_topics(ctx, _p(p0), _p(p)), ctx)
    return p0, p


def spdp_heldout(ctx, K, group, doc, word, num_docs, seed, iterations, first_iteration=0, z_init=None,
                 want_z=True, want_theta=False):
    """Fold-in + held-out perplexity (NEXT-1).  Returns dict(perplexity, z, theta)."""
    g = np.ascontiguousarray(group, np.int32); d = np.ascontiguousarray(doc, np.int32)
    w = np.ascontiguousarray(word, np.int32)
    zi = None if z_init is None else np.ascontiguousarray(z_init, np.int32)
    zo = np.zeros(len(w), np.int32) if want_z else None
    th = np.zeros((int(num_docs), K)) if want_theta else None
    ppl = C.c_double(np.nan)
    _check(lib().spdp_heldout(ctx, len(w), int(num_docs), _p(g), _p(d), _p(w), int(seed) & (2**64 - 1),
                              int(first_iteration), int(iterations), _p(zi), _p(zo), _p(th), C.byref(ppl)), ctx)
    return {"perplexity": ppl.value, "z": zo, "theta": th}


def spdp_topic_hellinger(ctx_a, ctx_b, K):
    """(dist [K,K], perm [K]): Hellinger distances of phi0~ rows and the greedy alignment."""
    dist = np.zeros((K, K)); perm = np.zeros(K, np.int32)
    _check(lib().spdp_topic_hellinger(ctx_a, ctx_b, _p(dist), _p(perm)), ctx_a)
    return dist, perm


def spdp_debug_probs(ctx, tok_ids, K):
    ids = np.ascontiguousarray(tok_ids, np.int64)
    probs = np.zeros((len(ids), 2 * K)); info = np.zeros((len(ids), 4), np.int32)
    _check(lib().spdp_debug_probs(ctx, len(ids), _p(ids), _p(probs), _p(info)), ctx)
    return probs, info


def spdp_debug_ratio_table(ctx, group, mmax):
    """The device A0/A1 table of a group: (A0, A1) fp32 arrays at m(m+1)/2 + t, m <= mmax."""
    out = np.zeros(((mmax + 1) * (mmax + 2) // 2, 2), np.float32)
    _check(lib().spdp_debug_ratio_table(ctx, int(group), int(mmax), _p(out)), ctx)
    return out[:, 0], out[:, 1]


def spdp_debug_chain(ctx, nsweeps, tbase=5):
    """W = 0 test mode: nsweeps exact sequential sweeps; the state code after each (int64 [nsweeps])."""
    out = np.zeros(int(nsweeps), np.int64)
    _check(lib().spdp_debug_chain(ctx, int(nsweeps), int(tbase), _p(out)), ctx)
    return out


def spdp_stats(ctx):
    out = np.zeros(20, np.int64)
    _check(lib().spdp_stats(ctx, _p(out)), ctx)
    keys = ["keeps", "moved", "clamped", "sweeps", "local_tokens", "local_docs", "m_max", "chunks",
            "lanes_per_token", "topics_per_lane", "chunk_tokens", "sample_grid", "token_kernel", "parts", "row_bytes",
            "async", "sparse_rows", "sparse_rows_lanes", "sparse_row_entries", "sparse_row_entries_read"]
    return dict(zip(keys, (int(x) for x in out)))


def spdp_profile(ctx, enable=True):
    _check(lib().spdp_profile(ctx, int(bool(enable))), ctx)


def spdp_timings(ctx):
    out = np.zeros(10)
    _check(lib().spdp_timings(ctx, _p(out)), ctx)
    keys = ["sample_ms", "apply_ms", "merge_ms", "exchange_ms", "sweep_ms", "sample_launches", "launches", "sweeps",
            "foldin_ms", "foldin_token_iters"]
    return dict(zip(keys, (float(x) for x in out)))


def spdp_destroy(ctx):
    if ctx:
        lib().spdp_destroy(ctx)


# ---------------------------------------------------------------- convenience
class Sampler:
    """One SPDP chain on one GPU (or one rank of a multi-GPU chain)."""

    def __init__(self, num_groups, vocab_size, num_topics, **kw):
        self.I, self.V, self.K = int(num_groups), int(vocab_size), int(num_topics)
        self.ctx = spdp_create(num_groups, vocab_size, num_topics, **kw)
        self.N = self.D = 0
        self._zr_pending = []        # host buffers of queued zr_async copies (alive until wait/close)

    def load_corpus(self, group, doc, word, num_docs, z_init=None, r_init=None):
        spdp_load_corpus(self.ctx, group, doc, word, num_docs, z_init, r_init)
        self.N, self.D = len(word), int(num_docs)
        return self

    def set_state(self, z, r=None, tables=None):
        spdp_set_state(self.ctx, z, r, tables)

    def sweep(self, n=1):
        spdp_sweep(self.ctx, n)

    def sweep_async(self, n=1):
        """Queue n sweeps and return (see spdp_sweep_async)."""
        spdp_sweep_async(self.ctx, n)

    def sweep_local(self):
        spdp_sweep_local(self.ctx)

    def exchange_blocks(self):
        n = C.c_int32()
        _check(lib().spdp_exchange_blocks(self.ctx, C.byref(n)), self.ctx)
        return n.value

    def exchange_buffer(self):
        return spdp_exchange_buffer(self.ctx)

    def exchange_get(self):
        _, n, eb = spdp_exchange_buffer(self.ctx)
        return spdp_exchange_copy(self.ctx, np.zeros(n, np.int32 if eb == 4 else np.int64), False)

    def exchange_put(self, host):
        _, n, eb = spdp_exchange_buffer(self.ctx)
        spdp_exchange_copy(self.ctx, np.ascontiguousarray(host, np.int32 if eb == 4 else np.int64), True)

    def sweep_merge(self):
        spdp_sweep_merge(self.ctx)

    def counts(self, out=None, **which):
        return spdp_counts(self.ctx, self.N, self.D, self.I, self.V, self.K, out=out, **which)

    def set_transform(self, pptr, pv, pp):
        """NEXT-4: sparse P^i rows over r = i * V + w (before load_corpus)."""
        self._P = (np.ascontiguousarray(pptr, np.int32), np.ascontiguousarray(pv, np.int32),
                   np.ascontiguousarray(pp, np.float64))
        _check(lib().spdp_set_transform(self.ctx, *(_p(a) for a in self._P)), self.ctx)
        return self

    def sparse_state(self):
        E = int(self._P[0][-1])
        q = np.zeros((E, self.K), np.int32); Q = np.zeros((self.K, self.V), np.int32)
        src = np.zeros(self.N, np.int16)
        _check(lib().spdp_sparse_state(self.ctx, _p(q), _p(Q), _p(src)), self.ctx)
        return {"q": q, "Qs": Q, "src": src}

    def zr(self, out=None):
        return spdp_zr(self.ctx, self.N, out)

    def zr_async(self, out):
        """Copy of the assignments into out, landing by the next wait() (overlaps the next sweep)."""
        self._zr_pending.append(spdp_zr_async(self.ctx, self.N, out))
        return out

    def zr8_async(self, out):
        """One byte per token (z | r << 7, K <= 128), landing by the next wait()."""
        self._zr_pending.append(spdp_zr8_async(self.ctx, self.N, out))
        return out

    def wait(self):
        spdp_wait(self.ctx)
        self._zr_pending.clear()

    def loglik(self, log_joint=True, perplexity=True):
        return spdp_loglik(self.ctx, log_joint, perplexity)

    def perplexity(self):
        return spdp_loglik(self.ctx, False, True)[1]

    def log_joint(self):
        return spdp_loglik(self.ctx, True, False)[0]

    def debug_probs(self, tok_ids):
        return spdp_debug_probs(self.ctx, tok_ids, self.K)

    def debug_chain(self, nsweeps, tbase=5):
        return spdp_debug_chain(self.ctx, nsweeps, tbase)

    def debug_ratio_table(self, group, mmax):
        return spdp_debug_ratio_table(self.ctx, group, mmax)

    def topics(self, phi0=True, phi=True):
        return spdp_topics(self.ctx, self.I, self.V, self.K, phi0, phi)

    def heldout(self, corpus, seed, iterations, first_iteration=0, z_init=None, want_z=True, want_theta=False):
        return spdp_heldout(self.ctx, self.K, corpus.group, corpus.doc, corpus.word, corpus.num_docs, seed,
                            iterations, first_iteration, z_init, want_z, want_theta)

    def topic_hellinger(self, other):
        return spdp_topic_hellinger(self.ctx, other.ctx, self.K)

    def stats(self):
        return spdp_stats(self.ctx)

    def profile(self, enable=True):
        spdp_profile(self.ctx, enable)

    def timings(self):
        return spdp_timings(self.ctx)

    def close(self):
        if self.ctx:
            spdp_destroy(self.ctx)       # waits for queued copies
            self.ctx = None
            self._zr_pending.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def sampler_for(corpus, num_topics, alpha=0.1, beta=0.1, discount=0.7, concentration=100.0, seed=7,
                num_waves=1, z_init=None, r_init=None, transform=None, **kw) -> Sampler:
    s = Sampler(corpus.num_groups, corpus.vocab, num_topics, alpha=alpha, beta=beta, discount=discount,
                concentration=concentration, seed=seed, num_waves=num_waves, **kw)
    if transform is not None:
        s.set_transform(*transform)
    return s.load_corpus(corpus.group, corpus.doc, corpus.word, corpus.num_docs, z_init, r_init)
