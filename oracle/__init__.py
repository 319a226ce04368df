"""CPU oracle of the C^2 hot path (ctypes binding of ``c2o.cpp``).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product (``paper_2010_11497_b200``) never imports it; the two share
no code.  See ``c2o.h`` for the paper passages each function follows and
DESIGN.md "Oracle pins" for what pins it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = [os.path.join(_HERE, "c2o.cpp"), os.path.join(_HERE, "c2o.h")]
_LIB = os.path.join(_HERE, "libc2oracle.so")
_lib = None

CAND = np.dtype([("id", "<i4"), ("inter", "<u2"), ("uni", "<u2")])
ABSENT = 0xFFFF
GF_BITS = 1024
NTHREADS = os.cpu_count() or 1


def build(force: bool = False) -> str:
    newest = max(os.path.getmtime(s) for s in _SRC)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC[0]])
        os.replace(tmp, _LIB)
    return _LIB


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_U64 = ctypes.c_uint64


def _load():
    global _lib
    if _lib is not None:
        return _lib
    L = ctypes.CDLL(build())
    sig = {
        "c2o_splitmix64_next": (_U64, [_P]),
        "c2o_hash_params": (None, [_U64, _I, _P, _P]),
        "c2o_gf_params": (None, [_U64, _P, _P]),
        "c2o_item_hash": (ctypes.c_uint32, [_U64, _U64, _U64, ctypes.c_uint32]),
        "c2o_hash_table": (_I, [_U64, _I, ctypes.c_uint32, _I64, _P]),
        "c2o_gf_table": (_I, [_U64, _I64, _P]),
        "c2o_frh": (_I, [_I64, _P, _P, _I, _I64, _P, _P]),
        "c2o_sketch": (_I, [_I64, _P, _P, _I, _I64, _P, _I, _P]),
        "c2o_cluster": (_I, [_I64, _P, _P, _I, _I64, _P, _I64, _I, _P, _P, _P, _P, _P]),
        "c2o_minhash_cluster": (_I, [_I64, _P, _P, _I, _U64, _I64, _P, _P, _P, _P, _P]),
        "c2o_local_knn": (_I, [_I64, _P, _P, _I, _P, _P, _P, _I, _I, _P, _I64, _I, _P]),
        "c2o_local_knn2": (_I, [_I64, _P, _P, _I, _P, _P, _P, _I, _I, _P, _I64, _I, _I, _U64, _P, _P]),
        "c2o_merge": (_I, [_I64, _I, _I, _P, _I, _P, _P, _P, _P]),
        "c2o_knn_union": (_I, [_I64, _P, _P, _I, _P, _P, _P, _I, _I, _P, _I64, _I, _P, _P, _P]),
        "c2o_knn_union_users": (_I, [_I64, _P, _P, _I, _P, _P, _P, _I, _I, _P, _I64, _I64, _P, _I, _P, _P, _P]),
        "c2o_exact_knn": (_I, [_I64, _P, _P, _I, _I, _P, _I64, _I64, _P, _I, _P, _P, _P]),
        "c2o_pair_counts": (_I, [_I64, _P, _P, _I64, _P, _P, _P, _P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _ptr(a):
    return None if a is None else a.ctypes.data


def _chk(rc, what):
    if rc != 0:
        raise ValueError(f"oracle {what} failed with code {rc}")


def _csr(offs, items):
    offs = np.ascontiguousarray(offs, dtype=np.int32)
    items = np.ascontiguousarray(items, dtype=np.int32)
    return offs, items, len(offs) - 1


# ------------------------------------------------------------------ hashing
def splitmix64(seed: int, count: int) -> list[int]:
    st = ctypes.c_uint64(seed)
    return [_load().c2o_splitmix64_next(ctypes.byref(st)) for _ in range(count)]


def hash_params(seed: int, t: int):
    a = np.zeros(t, np.uint64)
    c = np.zeros(t, np.uint64)
    _load().c2o_hash_params(seed, t, _ptr(a), _ptr(c))
    return a, c


def gf_params(seed: int):
    a = ctypes.c_uint64()
    c = ctypes.c_uint64()
    _load().c2o_gf_params(seed, ctypes.byref(a), ctypes.byref(c))
    return a.value, c.value


def item_hash(a: int, c: int, x: int, b: int) -> int:
    return _load().c2o_item_hash(a, c, x, b)


def hash_table(seed: int, t: int, b: int, m: int) -> np.ndarray:
    h = np.zeros((t, m), np.uint16)
    _chk(_load().c2o_hash_table(seed, t, b, m, _ptr(h)), "hash_table")
    return h


def gf_table(seed: int, m: int) -> np.ndarray:
    g = np.zeros(m, np.uint16)
    _chk(_load().c2o_gf_table(seed, m, _ptr(g)), "gf_table")
    return g


# ------------------------------------------------------------------ step 1
def frh(offs, items, htab) -> np.ndarray:
    offs, items, n = _csr(offs, items)
    htab = np.ascontiguousarray(htab, np.uint16)
    t, m = htab.shape
    H = np.zeros((t, n), np.int32)
    _chk(_load().c2o_frh(n, _ptr(offs), _ptr(items), t, m, _ptr(htab), _ptr(H)), "frh")
    return H


def sketch(offs, items, htab, D: int = 8) -> np.ndarray:
    offs, items, n = _csr(offs, items)
    htab = np.ascontiguousarray(htab, np.uint16)
    t, m = htab.shape
    sk = np.zeros((t, n, D), np.uint16)
    _chk(_load().c2o_sketch(n, _ptr(offs), _ptr(items), t, m, _ptr(htab), D, _ptr(sk)), "sketch")
    return sk


STAT_KEYS = ["clusters", "max_depth", "split_nodes", "folded_singletons", "chunked_residuals", "pairs",
             "max_cluster_size", "residual_clusters"]


def cluster(offs, items, htab, N: int, formulation: int = 0) -> dict:
    offs, items, n = _csr(offs, items)
    htab = np.ascontiguousarray(htab, np.uint16)
    t, m = htab.shape
    out = dict(offsets=np.zeros((t, n + 1), np.int32), members=np.zeros((t, n), np.int32),
               cluster_of=np.zeros((t, n), np.int32), n_clusters=np.zeros(t, np.int32))
    st = np.zeros(8, np.int64)
    _chk(_load().c2o_cluster(n, _ptr(offs), _ptr(items), t, m, _ptr(htab), N, formulation, _ptr(out["offsets"]),
                             _ptr(out["members"]), _ptr(out["cluster_of"]), _ptr(out["n_clusters"]), _ptr(st)),
         "cluster")
    out["stats"] = dict(zip(STAT_KEYS, (int(x) for x in st)))
    return out


def cluster_minhash(offs, items, seed: int, t: int, N: int) -> dict:
    """C^2/MinHash variant clustering: one cluster per min-hash item, no split."""
    offs, items, n = _csr(offs, items)
    out = dict(offsets=np.zeros((t, n + 1), np.int32), members=np.zeros((t, n), np.int32),
               cluster_of=np.zeros((t, n), np.int32), n_clusters=np.zeros(t, np.int32))
    st = np.zeros(8, np.int64)
    _chk(_load().c2o_minhash_cluster(n, _ptr(offs), _ptr(items), t, seed, N, _ptr(out["offsets"]),
                                     _ptr(out["members"]), _ptr(out["cluster_of"]), _ptr(out["n_clusters"]),
                                     _ptr(st)), "minhash_cluster")
    out["stats"] = dict(zip(STAT_KEYS, (int(x) for x in st)))
    return out


# ------------------------------------------------------------------ steps 2-3
def local_knn(offs, items, cl: dict, k: int, sim_mode: int = 0, gtab=None, nthreads: int | None = None,
              solver: int = 0, seed: int = 0, stats: dict | None = None):
    """Alg. 2 per cluster: brute force (solver 0), or the hybrid with Hyrec for |C| >= 5k^2 (solver 1)."""
    offs, items, n = _csr(offs, items)
    t = cl["offsets"].shape[0]
    m = 0 if gtab is None else len(gtab)
    cand = np.zeros((t, n, k), CAND)
    its = ctypes.c_int64(0)
    _chk(_load().c2o_local_knn2(n, _ptr(offs), _ptr(items), t, _ptr(cl["offsets"]), _ptr(cl["members"]),
                                _ptr(cl["n_clusters"]), k, sim_mode, _ptr(gtab), m, nthreads or NTHREADS, solver,
                                seed, _ptr(cand), ctypes.byref(its)), "local_knn")
    if stats is not None:
        stats["hyrec_iters"] = its.value
    return cand


def merge(cand: np.ndarray, nthreads: int | None = None):
    cand = np.ascontiguousarray(cand, CAND)
    t, n, k = cand.shape
    nbr = np.zeros((n, k), np.int32)
    inter = np.zeros((n, k), np.uint16)
    uni = np.zeros((n, k), np.uint16)
    sim = np.zeros((n, k), np.float32)
    _chk(_load().c2o_merge(n, t, k, _ptr(cand), nthreads or NTHREADS, _ptr(nbr), _ptr(inter), _ptr(uni),
                           _ptr(sim)), "merge")
    return nbr, inter, uni, sim


def knn_union(offs, items, cl: dict, k: int, sim_mode: int = 0, gtab=None, nthreads: int | None = None):
    offs, items, n = _csr(offs, items)
    t = cl["offsets"].shape[0]
    m = 0 if gtab is None else len(gtab)
    nbr = np.zeros((n, k), np.int32)
    inter = np.zeros((n, k), np.uint16)
    uni = np.zeros((n, k), np.uint16)
    _chk(_load().c2o_knn_union(n, _ptr(offs), _ptr(items), t, _ptr(cl["offsets"]), _ptr(cl["members"]),
                               _ptr(cl["cluster_of"]), k, sim_mode, _ptr(gtab), m, nthreads or NTHREADS, _ptr(nbr),
                               _ptr(inter), _ptr(uni)), "knn_union")
    return nbr, inter, uni


def knn_union_users(offs, items, cl: dict, k: int, users, sim_mode: int = 0, gtab=None,
                    nthreads: int | None = None):
    offs, items, n = _csr(offs, items)
    t = cl["offsets"].shape[0]
    m = 0 if gtab is None else len(gtab)
    users = np.ascontiguousarray(users, np.int32)
    q = len(users)
    nbr = np.zeros((q, k), np.int32)
    inter = np.zeros((q, k), np.uint16)
    uni = np.zeros((q, k), np.uint16)
    _chk(_load().c2o_knn_union_users(n, _ptr(offs), _ptr(items), t, _ptr(cl["offsets"]), _ptr(cl["members"]),
                                     _ptr(cl["cluster_of"]), k, sim_mode, _ptr(gtab), m, q, _ptr(users),
                                     nthreads or NTHREADS, _ptr(nbr), _ptr(inter), _ptr(uni)), "knn_union_users")
    return nbr, inter, uni


def exact_knn(offs, items, k: int, users=None, sim_mode: int = 0, gtab=None, nthreads: int | None = None):
    offs, items, n = _csr(offs, items)
    users = np.arange(n, dtype=np.int32) if users is None else np.ascontiguousarray(users, np.int32)
    m = 0 if gtab is None else len(gtab)
    q = len(users)
    nbr = np.zeros((q, k), np.int32)
    inter = np.zeros((q, k), np.uint16)
    uni = np.zeros((q, k), np.uint16)
    _chk(_load().c2o_exact_knn(n, _ptr(offs), _ptr(items), k, sim_mode, _ptr(gtab), m, q, _ptr(users),
                               nthreads or NTHREADS, _ptr(nbr), _ptr(inter), _ptr(uni)), "exact_knn")
    return nbr, inter, uni


def pair_counts(offs, items, u, v):
    offs, items, n = _csr(offs, items)
    u = np.ascontiguousarray(u, np.int32)
    v = np.ascontiguousarray(v, np.int32)
    inter = np.zeros(len(u), np.int32)
    uni = np.zeros(len(u), np.int32)
    _chk(_load().c2o_pair_counts(n, _ptr(offs), _ptr(items), len(u), _ptr(u), _ptr(v), _ptr(inter), _ptr(uni)),
         "pair_counts")
    return inter, uni


def build_graph(offs, items, *, k: int, t: int, b: int, N: int, seed: int, sim_mode: int = 0, htab=None,
                nthreads: int | None = None, formulation: int = 0, clustering: str = "frh",
                solver: int = 0) -> dict:
    """Whole C^2 pipeline on the CPU: FRH (or MinHash) clustering -> local brute force -> Alg. 3."""
    offs, items, n = _csr(offs, items)
    m = int(items.max()) + 1 if len(items) else 1
    gtab = gf_table(seed, m) if sim_mode == 1 else None
    if clustering == "minhash":
        cl = cluster_minhash(offs, items, seed, t, N)
    else:
        if htab is None:
            htab = hash_table(seed, t, b, m)
        cl = cluster(offs, items, htab, N, formulation)
    st = {}
    cand = local_knn(offs, items, cl, k, sim_mode, gtab, nthreads, solver=solver, seed=seed, stats=st)
    nbr, inter, uni, sim = merge(cand, nthreads)
    return dict(clusters=cl, cand=cand, nbr=nbr, inter=inter, uni=uni, sim=sim, htab=htab, gtab=gtab,
                hyrec_iters=st.get("hyrec_iters", 0))
