"""Multi-GPU plumbing for the sweep and the forest.

One process per GPU (torchrun), ``torch.distributed`` over NCCL.  The data
path is sharded so that no collective is needed while computing:

* energy sweep -- shard by KERNEL (all configs x archs of a kernel stay on one
  rank, so its tokens are read once): :func:`kernel_shard`;
* forest fit   -- shard by TREE (tree t on rank t % world); per-tree seeds come
  from the global ``RandomState(seed)`` sequence, so the forest does not depend
  on the world size: ``RandomForestRegressor(shard=(rank, world))`` then
  :func:`allgather_forest`;
* the only exchanges are the ones the reference's outputs need: the results
  (:func:`allgather_results`) and the ensemble (:func:`broadcast_flat`).
Collectives run on whatever backend the process group uses (``nccl`` on the
GPU box, ``gloo`` in the CPU tests).
"""

from __future__ import annotations

import numpy as np


def kernel_shard(n_kernels: int, rank: int, world: int) -> np.ndarray:
    """Contiguous kernel ranges, sizes differing by at most one."""
    lo = n_kernels * rank // world
    hi = n_kernels * (rank + 1) // world
    return np.arange(lo, hi, dtype=np.uint32)


def allgather_results(tensors: list, group=None) -> list:
    """All-gather per-rank result vectors of unequal length (e.g. status,
    time_us, power, energy of each rank's points); returns, per input tensor,
    the concatenation over ranks in rank order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = torch.tensor([tensors[0].shape[0]], dtype=torch.int64, device=tensors[0].device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes)
    out = []
    for t in tensors:
        pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad, group=group)
        out.append(torch.cat([b[:s] for b, s in zip(bufs, sizes)]))
    return out


def broadcast_flat(flat, src: int = 0, group=None, device=None):
    """Broadcast a FlatEnsemble (node arrays + scaling) from `src` to all ranks;
    returns the FlatEnsemble on every rank."""
    import torch
    import torch.distributed as dist

    from .ensemble import NODE_DT, FlatEnsemble

    rank = dist.get_rank(group)
    dev = device or torch.device("cpu")
    meta = [None]
    if rank == src:
        meta = [dict(n_nodes=len(flat.nodes), n_trees=flat.n_trees, n_feat=flat.n_feat,
                     base=float(flat.base_score), max_depth=int(flat.max_depth),
                     manifest=list(flat.manifest))]
    dist.broadcast_object_list(meta, src=src, group=group)
    m = meta[0]
    if rank == src:
        nodes = torch.from_numpy(flat.nodes.view(np.uint8).copy()).to(dev)
        off = torch.from_numpy(flat.tree_off.copy()).to(dev)
        dep = torch.from_numpy(np.asarray(flat.tree_depth, np.int32).copy()).to(dev)
        sc = torch.from_numpy(np.stack([flat.scale_lo, flat.scale_hi])).to(dev)
    else:
        nodes = torch.empty(m["n_nodes"] * NODE_DT.itemsize, dtype=torch.uint8, device=dev)
        off = torch.empty(m["n_trees"], dtype=torch.int64, device=dev)
        dep = torch.empty(m["n_trees"], dtype=torch.int32, device=dev)
        sc = torch.empty((2, m["n_feat"]), dtype=torch.float64, device=dev)
    for t in (nodes, off, dep, sc):
        dist.broadcast(t, src=src, group=group)
    if rank == src:
        return flat
    return FlatEnsemble(nodes=nodes.cpu().numpy().view(NODE_DT).copy(),
                        tree_off=off.cpu().numpy(), scale_lo=sc[0].cpu().numpy(),
                        scale_hi=sc[1].cpu().numpy(), base_score=m["base"],
                        max_depth=m["max_depth"], manifest=tuple(m["manifest"]),
                        tree_depth=dep.cpu().numpy())


def allgather_forest(model, group=None):
    """Complete a tree-sharded forest on every rank: each rank contributes the
    trees it built (estimators_[t] for t % world == rank), in global tree order."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    mine = {t: e for t, e in enumerate(model.estimators_) if e is not None}
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    merged = {}
    for p in parts:
        merged.update(p)
    if sorted(merged) != list(range(model.n_estimators)):
        raise RuntimeError("tree shards do not cover the forest")
    model.estimators_ = [merged[t] for t in range(model.n_estimators)]
    model.shard = None
    model._flat = None
    return model
