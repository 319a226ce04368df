"""B200 (sm_100a) Cluster-and-Conquer hot path: thin Python binding of ``include/c2.h``.

Argument marshalling only: every step runs in the CUDA kernels of ``libc2.so``.  There is
no CPU fallback -- importing works without a GPU (for symbol checks), but every compute
call raises if the library or a CUDA device is missing.

Entry points (same names as the C ABI, torch CUDA tensors in/out):
  fastrandomhash(offsets, items, t, b, N, seed)            Step 1
  fastrandomhash_table(offsets, items, t, b, N, htab)      Step 1 with an injected h table
  sketch(offsets, items, t, b, seed, D)                    stage hook (H_f and H\\eta chain)
  local_knn(offsets, items, clusters, k, sim_mode, seed)   Step 2
  merge(cand, k)                                           Step 3  (Alg. 3)
  build(offsets, items, k, t, b, N, seed, sim_mode)        Steps 1-3
  build_host(offsets_np, items_np, ...)                    Steps 1-3 from/to host memory
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# C2_LIB: dev override for A/B runs of a variant build of the same sources (tools/ab.sh)
LIB_PATH = os.environ.get("C2_LIB") or os.path.join(HERE, "lib", "libc2.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "c2.h")

C2_OK, C2_EINVAL, C2_EDATA, C2_ENOMEM, C2_ECUDA = 0, -1, -2, -3, -4
SIM_EXACT, SIM_GF1024 = 0, 1
OPT_SKETCH_DEPTH, OPT_SYNC_CHECK, OPT_TIMING, OPT_KSTATS, OPT_RELABEL, OPT_CLUSTERING, OPT_FUNC_OFFSET, \
    OPT_LOCAL_SOLVER, OPT_SURVIVORS, OPT_GF_TENSOR, OPT_SPLIT_DEVICE = 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11
SOLVER_BRUTE, SOLVER_HYBRID = 0, 1
CLUSTER_FRH, CLUSTER_MINHASH = 0, 1
ABSENT = 0xFFFF
CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: the legacy default stream

_lib = None
_lock = threading.Lock()


class C2Error(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"c2 error {code}: {msg}")
        self.code = code


class _Clusters(ctypes.Structure):
    _fields_ = [("offsets", ctypes.c_void_p), ("members", ctypes.c_void_p), ("cluster_of", ctypes.c_void_p),
                ("n_clusters", ctypes.c_void_p)]


class Stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in ("pairs", "clusters", "max_cluster_size", "split_nodes", "max_depth",
                                              "folded_singletons", "chunked_residuals", "launches", "host_syncs")] + \
               [(k, ctypes.c_double) for k in ("ms_sketch", "ms_cluster", "ms_local", "ms_merge", "ms_total")] + \
               [("work_steps", ctypes.c_int64), ("tile_launches", ctypes.c_int64), ("ms_tile", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_U64 = ctypes.c_uint64
SIGNATURES = {
    "c2_ctx_create": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, _P]),
    "c2_ctx_destroy": (None, [_P]),
    "c2_last_error": (ctypes.c_char_p, [_P]),
    "c2_ctx_set_option": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int64]),
    "c2_fastrandomhash": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, _U64, ctypes.POINTER(_Clusters)]),
    "c2_fastrandomhash_table": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, _P, _I32,
                                               ctypes.POINTER(_Clusters)]),
    "c2_sketch": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _U64, _I32, _P]),
    "c2_local_knn": (ctypes.c_int, [_P, _P, _P, _I32, _I32, ctypes.POINTER(_Clusters), _I32, _I32, _U64, _P]),
    "c2_merge": (ctypes.c_int, [_P, _I32, _I32, _I32, _P, _P, _P, _P, _P]),
    "c2_build": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32, _U64, _P, _P, _P, _P]),
    "c2_build_host": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32, _U64, _P, _P, _P, _P]),
    "c2_get_stats": (ctypes.c_int, [_P, ctypes.POINTER(Stats)]),
}


def lib():
    """Load libc2.so (never a fallback: raises if it is missing)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2010_11497_b200.build` "
                                  "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


class Context:
    """A c2_ctx bound to one device and one CUDA stream."""

    def __init__(self, device: int = 0, stream=None, timing: bool = False):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2010_11497_b200 needs a CUDA device (no CPU fallback)")
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = _P()
        # torch's default stream has handle 0, which c2_ctx_create reads as "make your own
        # stream"; pass cudaStreamLegacy for it so the library's work is ordered with torch's
        handle = self.stream.cuda_stream or CUDA_STREAM_LEGACY
        rc = lib().c2_ctx_create(ctypes.byref(h), device, _P(handle))
        if rc != C2_OK:
            raise C2Error(rc, "c2_ctx_create failed")
        self.h = h
        if timing:
            self.set_option(OPT_TIMING, 1)

    def close(self):
        if getattr(self, "h", None):
            lib().c2_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc):
        if rc != C2_OK:
            msg = lib().c2_last_error(self.h)
            raise C2Error(rc, msg.decode() if msg else "")

    def set_option(self, key, value):
        self.check(lib().c2_ctx_set_option(self.h, key, int(value)))

    def stats(self) -> dict:
        s = Stats()
        self.check(lib().c2_get_stats(self.h, ctypes.byref(s)))
        return s.as_dict()


_default = {}


def default_context(device: int = 0) -> Context:
    import torch
    key = (device, torch.cuda.current_stream(device).cuda_stream)
    if key not in _default:
        _default[key] = Context(device)
    return _default[key]


def _ptr(t):
    return None if t is None else _P(t.data_ptr())


def _check_csr(offsets, items):
    import torch
    for x in (offsets, items):
        if not (x.is_cuda and x.dtype == torch.int32 and x.is_contiguous()):
            raise TypeError("offsets/items must be contiguous int32 CUDA tensors")
    return offsets.numel() - 1


def _alloc_clusters(t, n, device):
    import torch
    return dict(offsets=torch.empty((t, n + 1), dtype=torch.int32, device=device),
                members=torch.empty((t, n), dtype=torch.int32, device=device),
                cluster_of=torch.empty((t, n), dtype=torch.int32, device=device),
                n_clusters=(ctypes.c_int32 * t)())


def _cl_struct(cl):
    return _Clusters(_ptr(cl["offsets"]), _ptr(cl["members"]), _ptr(cl["cluster_of"]),
                     ctypes.cast(cl["n_clusters"], _P))


def fastrandomhash(offsets, items, t, b, N, seed, ctx: Context | None = None) -> dict:
    ctx = ctx or default_context(offsets.device.index or 0)
    n = _check_csr(offsets, items)
    cl = _alloc_clusters(t, n, offsets.device)
    s = _cl_struct(cl)
    ctx.check(lib().c2_fastrandomhash(ctx.h, _ptr(offsets), _ptr(items), n, t, b, N, seed, ctypes.byref(s)))
    cl["n_clusters"] = list(cl["n_clusters"])
    return cl


def fastrandomhash_table(offsets, items, t, b, N, htab, ctx: Context | None = None) -> dict:
    import torch
    ctx = ctx or default_context(offsets.device.index or 0)
    n = _check_csr(offsets, items)
    assert htab.is_cuda and htab.dtype == torch.uint16 and htab.is_contiguous() and htab.shape[0] == t
    cl = _alloc_clusters(t, n, offsets.device)
    s = _cl_struct(cl)
    ctx.check(lib().c2_fastrandomhash_table(ctx.h, _ptr(offsets), _ptr(items), n, t, b, N, _ptr(htab),
                                            htab.shape[1], ctypes.byref(s)))
    cl["n_clusters"] = list(cl["n_clusters"])
    return cl


def sketch(offsets, items, t, b, seed, D=8, ctx: Context | None = None):
    import torch
    ctx = ctx or default_context(offsets.device.index or 0)
    n = _check_csr(offsets, items)
    out = torch.empty((t, n, D), dtype=torch.uint16, device=offsets.device)
    ctx.check(lib().c2_sketch(ctx.h, _ptr(offsets), _ptr(items), n, t, b, seed, D, _ptr(out)))
    return out


def local_knn(offsets, items, clusters: dict, k, sim_mode=SIM_EXACT, seed=0, ctx: Context | None = None):
    """Returns cand as an int32 tensor [t, n, k, 2]: [...,0] = id, [...,1] = inter | uni << 16."""
    import torch
    ctx = ctx or default_context(offsets.device.index or 0)
    n = _check_csr(offsets, items)
    t = clusters["offsets"].shape[0]
    ncl = (ctypes.c_int32 * t)(*clusters["n_clusters"])
    s = _Clusters(_ptr(clusters["offsets"]), _ptr(clusters["members"]), _ptr(clusters["cluster_of"]),
                  ctypes.cast(ncl, _P))
    cand = torch.empty((t, n, k, 2), dtype=torch.int32, device=offsets.device)
    ctx.check(lib().c2_local_knn(ctx.h, _ptr(offsets), _ptr(items), n, t, ctypes.byref(s), k, sim_mode, seed,
                                 _ptr(cand)))
    return cand


def split_cand(cand):
    """int32 [..., 2] cand tensor -> (id, inter, uni) int64 tensors."""
    ident = cand[..., 0].long()
    packed = cand[..., 1].long() & 0xFFFFFFFF
    return ident, packed & 0xFFFF, packed >> 16


def merge(cand, k=None, with_sim=True, ctx: Context | None = None):
    import torch
    if not (cand.is_cuda and cand.dtype == torch.int32 and cand.is_contiguous() and cand.dim() == 4
            and cand.shape[3] == 2):
        raise TypeError("cand must be a contiguous int32 CUDA tensor [t][n][k][2] (c2_cand records)")
    ctx = ctx or default_context(cand.device.index or 0)
    t, n, kk, _ = cand.shape
    if k is not None and k != kk:
        raise ValueError(f"k={k} differs from the list length cand.shape[2]={kk} (c2_merge uses k as both)")
    k = kk
    dev = cand.device
    nbr = torch.empty((n, k), dtype=torch.int32, device=dev)
    inter = torch.empty((n, k), dtype=torch.uint16, device=dev)
    uni = torch.empty((n, k), dtype=torch.uint16, device=dev)
    sim = torch.empty((n, k), dtype=torch.float32, device=dev) if with_sim else None
    ctx.check(lib().c2_merge(ctx.h, t, n, k, _ptr(cand), _ptr(nbr), _ptr(inter), _ptr(uni), _ptr(sim)))
    return nbr, inter, uni, sim


def build(offsets, items, *, k, t, b, N, seed, sim_mode=SIM_EXACT, with_sim=True, out=None,
          ctx: Context | None = None):
    """Steps 1-3 on device-resident CSR.  Returns (nbr int32, inter u16, uni u16, sim f32|None)."""
    import torch
    ctx = ctx or default_context(offsets.device.index or 0)
    n = _check_csr(offsets, items)
    dev = offsets.device
    if out is None:
        out = (torch.empty((n, k), dtype=torch.int32, device=dev),
               torch.empty((n, k), dtype=torch.uint16, device=dev),
               torch.empty((n, k), dtype=torch.uint16, device=dev),
               torch.empty((n, k), dtype=torch.float32, device=dev) if with_sim else None)
    nbr, inter, uni, sim = out
    ctx.check(lib().c2_build(ctx.h, _ptr(offsets), _ptr(items), n, t, b, N, k, sim_mode, seed, _ptr(nbr),
                             _ptr(inter), _ptr(uni), _ptr(sim)))
    return nbr, inter, uni, sim


def build_host(offsets, items, *, k, t, b, N, seed, sim_mode=SIM_EXACT, with_sim=True, out=None,
               ctx: Context | None = None):
    """Steps 1-3 from host numpy CSR to host numpy outputs (copies inside the call)."""
    import numpy as np
    ctx = ctx or default_context(0)
    offsets = np.ascontiguousarray(offsets, np.int32)
    items = np.ascontiguousarray(items, np.int32)
    n = len(offsets) - 1
    if out is None:
        out = (np.empty((n, k), np.int32), np.empty((n, k), np.uint16), np.empty((n, k), np.uint16),
               np.empty((n, k), np.float32) if with_sim else None)
    nbr, inter, uni, sim = out
    ctx.check(lib().c2_build_host(ctx.h, offsets.ctypes.data, items.ctypes.data, n, t, b, N, k, sim_mode, seed,
                                  nbr.ctypes.data, inter.ctypes.data, uni.ctypes.data,
                                  None if sim is None else sim.ctypes.data))
    return nbr, inter, uni, sim
