"""Multi-GPU C^2 sharded by hash function.

The t clustering configurations are independent until the merge: Alg. 1, the split and each
cluster's local KNN "do not need to be synchronized with any other computation", and the
paper notes the method's map-reduce shape.  With G ranks (one process per GPU,
``torch.distributed`` over NCCL):

1. rank g runs functions [g*t/G, (g+1)*t/G) of the seed's stream (C2_OPT_FUNC_OFFSET, reading A2)
   through the fused c2_build: Steps 1-2 plus the Alg. 3 merge of ITS functions -> a partial list
   per user [n][k] (ids, inter, union);
2. ONE all-to-all exchanges the partial lists by user block (rank j owns users
   [j*n/G, (j+1)*n/G)): (G-1)/G * n * k * 8 bytes leave each rank;
3. each rank merges the G partial lists of its users with c2_merge (Alg. 3 with t = G lists).

Alg. 3 keeps the k best of the union with duplicates dropped (A16), an associative and
commutative operation, so the result equals the single-process t-function build bytewise.  The
CSR is replicated (each rank holds the full input; `broadcast_csr` sends it from rank 0).

The arithmetic of every step runs in libc2 (CUDA); this module only moves tensors between ranks.
``local_fn`` / ``merge_fn`` are injectable so the exchange logic can be tested on CPU ranks
(gloo) with the oracle standing in for the GPU steps (tests/test_dist.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import C2_OK  # noqa: F401  (package import: fails loudly if libc2 cannot be loaded)


def function_range(t: int, G: int, g: int) -> tuple[int, int]:
    """Functions [f0, f1) of rank g: a balanced contiguous split of t functions over G ranks."""
    return (g * t) // G, ((g + 1) * t) // G


def user_block(n: int, G: int, j: int) -> tuple[int, int]:
    return (j * n) // G, ((j + 1) * n) // G


def pack_lists(nbr, inter, uni):
    """(nbr int32, inter u16, uni u16) [n][k] -> c2_cand records as int32 [n][k][2]."""
    packed = inter.to(torch.int32) | (uni.to(torch.int32) << 16)
    return torch.stack([nbr.to(torch.int32), packed], dim=-1).contiguous()


def pad_lists(n: int, k: int, device) -> torch.Tensor:
    out = torch.zeros((n, k, 2), dtype=torch.int32, device=device)
    out[..., 0] = -1
    return out


def gpu_local(offsets, items, *, k, t, b, N, seed, f0, t_g, sim_mode, ctx):
    """Steps 1-2 + Alg. 3 over functions [f0, f0 + t_g) on this rank's GPU (fused c2_build)."""
    from . import OPT_FUNC_OFFSET, build
    n = offsets.numel() - 1
    if t_g == 0:
        return pad_lists(n, k, offsets.device)
    ctx.set_option(OPT_FUNC_OFFSET, f0)
    try:
        nbr, inter, uni, _ = build(offsets, items, k=k, t=t_g, b=b, N=N, seed=seed, sim_mode=sim_mode,
                                   with_sim=False, ctx=ctx)
    finally:
        ctx.set_option(OPT_FUNC_OFFSET, 0)
    return pack_lists(nbr, inter, uni)


def gpu_merge(lists, ctx):
    """Alg. 3 over the G partial lists [G][n_blk][k][2] of this rank's users (c2_merge)."""
    from . import merge
    return merge(lists, ctx=ctx)


def build_sharded(offsets, items, *, k, t, b, N, seed, sim_mode=0, group=None, ctx=None, local_fn=None,
                  merge_fn=None, gather=True):
    """C^2 over the ranks of `group` (one GPU each).  Returns (nbr, inter, uni, sim) for ALL users
    on every rank when gather=True, else this rank's block (and its user range).

    Every rank passes the same CSR (device tensors on its own GPU, or host tensors with CPU
    stand-ins for local_fn / merge_fn)."""
    G = dist.get_world_size(group)
    g = dist.get_rank(group)
    n = offsets.numel() - 1
    f0, f1 = function_range(t, G, g)
    if local_fn is None:
        local_fn = lambda o, i, **kw: gpu_local(o, i, ctx=ctx, **kw)  # noqa: E731
    if merge_fn is None:
        merge_fn = lambda lists: gpu_merge(lists, ctx)  # noqa: E731
    part = local_fn(offsets, items, k=k, t=t, b=b, N=N, seed=seed, f0=f0, t_g=f1 - f0, sim_mode=sim_mode)
    # ---- the one exchange: partial lists by user block (all-to-all, uneven blocks)
    blocks = [user_block(n, G, j) for j in range(G)]
    send_sizes = [(hi - lo) * k * 2 for lo, hi in blocks]
    mlo, mhi = blocks[g]
    recv = torch.empty(G * (mhi - mlo) * k * 2, dtype=torch.int32, device=part.device)
    dist.all_to_all_single(recv, part.reshape(-1), [(mhi - mlo) * k * 2] * G, send_sizes, group=group)
    lists = recv.view(G, mhi - mlo, k, 2)
    nbr, inter, uni, sim = merge_fn(lists)
    if not gather:
        return (nbr, inter, uni, sim), (mlo, mhi)
    # ---- gather the blocks (padded to equal length for all_gather_into_tensor)
    bmax = max(hi - lo for lo, hi in blocks)
    rec = pack_lists(nbr, inter, uni)
    pad = pad_lists(bmax, k, rec.device)
    pad[: mhi - mlo] = rec
    allb = torch.empty((G * bmax, k, 2), dtype=torch.int32, device=rec.device)
    dist.all_gather_into_tensor(allb, pad, group=group)
    allb = allb.view(G, bmax, k, 2)
    full = torch.cat([allb[j, : hi - lo] for j, (lo, hi) in enumerate(blocks)], dim=0)
    nbr_all = full[..., 0].contiguous()
    iu = full[..., 1]
    inter_all = (iu & 0xFFFF).to(torch.int32)
    uni_all = ((iu >> 16) & 0xFFFF).to(torch.int32)
    return nbr_all, inter_all, uni_all, None


def broadcast_csr(offsets, items, src=0, group=None):
    """Replicate the CSR from rank `src` (its shapes first, then the arrays)."""
    shape = torch.tensor([offsets.numel(), items.numel()], dtype=torch.int64, device=offsets.device)
    dist.broadcast(shape, src, group=group)
    if dist.get_rank(group) != src:
        offsets = torch.empty(int(shape[0]), dtype=torch.int32, device=offsets.device)
        items = torch.empty(int(shape[1]), dtype=torch.int32, device=items.device)
    dist.broadcast(offsets, src, group=group)
    dist.broadcast(items, src, group=group)
    return offsets, items
