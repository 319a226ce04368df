"""Seeded synthetic inputs shaped like the paper's workloads.

Shared by the oracle tests, the GPU parity tests and ``bench.py``.  This module
holds NO arithmetic of the method (no item hash, FastRandomHash or Jaccard): it
only produces CSR user/item sets and the run parameters (t, b, N, k, seeds) of
the five BASELINE.json configs.  The heavy lifting is ``gen.c`` (counter-based
RNG, so results do not depend on the thread count).

Configs (BASELINE.json ``configs[0..4]``, called c1..c5):
  c1  2,000 users x 1,000 items, lognormal(median 20, sigma 1) in [5,200], Zipf 1.0, k10 t2 b64 N500
  c2  6,040 x 3,706, bounded Pareto [20,2000] mean 165, Zipf 0.9, k30 t8 b1024 N2000
  c3  18,889 x 203,030, bounded Pareto [5,1000] mean 37, Zipf 1.1, k30 t8 b1024 N2000
  c4  69,878 x 10,677, bounded Pareto [20,3000] mean 143, Zipf 0.9, k30 t8 b1024 N2000 (+GF-1024)
  c5  1,000,000 x 100,000, lognormal(median 60, sigma 1) in [10,2000], Zipf 1.0, k30 t8 b4096 N2000
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

HASH_SEED = 42  # hash seed 42 for every config


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-fPIC", "-shared", "-o", tmp,
                               _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.synth_sizes.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p]
        _lib.synth_sizes.restype = ctypes.c_int
        _lib.synth_fill.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        _lib.synth_fill.restype = ctypes.c_int
        _lib.synth_fit_pareto_alpha.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double]
        _lib.synth_fit_pareto_alpha.restype = ctypes.c_double
    return _lib


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    m: int
    dist: str          # "lognormal" | "bpareto"
    p1: float          # lognormal median | bounded-Pareto target mean
    p2: float          # lognormal sigma (unused for bpareto)
    lo: int
    hi: int
    zipf: float
    k: int
    t: int
    b: int
    N: int
    data_seed: int
    hash_seed: int = HASH_SEED


CONFIGS = {
    "c1": Config("c1", 2000, 1000, "lognormal", 20.0, 1.0, 5, 200, 1.0, 10, 2, 64, 500, 1),
    "c2": Config("c2", 6040, 3706, "bpareto", 165.0, 0.0, 20, 2000, 0.9, 30, 8, 1024, 2000, 2),
    "c3": Config("c3", 18889, 203030, "bpareto", 37.0, 0.0, 5, 1000, 1.1, 30, 8, 1024, 2000, 3),
    "c4": Config("c4", 69878, 10677, "bpareto", 143.0, 0.0, 20, 3000, 0.9, 30, 8, 1024, 2000, 4),
    "c5": Config("c5", 1000000, 100000, "lognormal", 60.0, 1.0, 10, 2000, 1.0, 30, 8, 4096, 2000, 5),
}


def config(name: str, **over) -> Config:
    return replace(CONFIGS[name], **over) if over else CONFIGS[name]


def sizes(cfg: Config) -> np.ndarray:
    lib = _load()
    out = np.empty(cfg.n, dtype=np.int32)
    if cfg.dist == "lognormal":
        rc = lib.synth_sizes(cfg.n, 0, cfg.p1, cfg.p2, cfg.lo, cfg.hi, cfg.data_seed, out.ctypes.data)
    else:
        alpha = lib.synth_fit_pareto_alpha(float(cfg.lo), float(cfg.hi), cfg.p1)
        rc = lib.synth_sizes(cfg.n, 1, alpha, 0.0, cfg.lo, cfg.hi, cfg.data_seed, out.ctypes.data)
    if rc:
        raise RuntimeError(f"synth_sizes failed ({rc})")
    return out


def generate(cfg: Config | str, nthreads: int | None = None, cache: bool = True):
    """Return (offsets int32[n+1], items int32[nnz]) for a config (rows ascending)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    cpath = None
    if cache:
        cdir = os.path.join(os.path.dirname(_HERE), "data")
        key = f"{cfg.name}_{cfg.n}_{cfg.m}_{cfg.dist}_{cfg.p1}_{cfg.p2}_{cfg.lo}_{cfg.hi}_{cfg.zipf}_{cfg.data_seed}"
        cpath = os.path.join(cdir, key + ".npz")
        if os.path.exists(cpath):
            z = np.load(cpath)
            return z["offsets"], z["items"]
    sz = sizes(cfg)
    offsets = np.zeros(cfg.n + 1, dtype=np.int64)
    np.cumsum(sz, out=offsets[1:])
    if offsets[-1] >= 2**31:
        raise ValueError("nnz too large for int32 CSR")
    offsets = offsets.astype(np.int32)
    items = np.empty(int(offsets[-1]), dtype=np.int32)
    rc = _load().synth_fill(cfg.n, cfg.m, cfg.zipf, cfg.data_seed, offsets.ctypes.data, items.ctypes.data,
                            nthreads or os.cpu_count() or 1)
    if rc:
        raise RuntimeError(f"synth_fill failed ({rc})")
    if cpath is not None:
        os.makedirs(os.path.dirname(cpath), exist_ok=True)
        tmp = cpath + f".tmp{os.getpid()}.npz"
        np.savez(tmp, offsets=offsets, items=items)
        os.replace(tmp, cpath)
    return offsets, items


def random_instance(rng: np.random.Generator, n: int, m: int, lo: int = 1, hi: int = 12, zipf: float = 1.0):
    """Tiny random CSR for property tests (numpy RNG; rows ascending, distinct, non-empty)."""
    w = 1.0 / np.arange(1, m + 1) ** zipf
    w /= w.sum()
    perm = rng.permutation(m)
    offs = [0]
    items = []
    for _ in range(n):
        s = int(rng.integers(lo, min(hi, m) + 1))
        row = np.sort(perm[rng.choice(m, size=s, replace=False, p=w)])
        items.extend(row.tolist())
        offs.append(len(items))
    return np.asarray(offs, dtype=np.int32), np.asarray(items, dtype=np.int32)
