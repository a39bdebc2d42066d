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
  (:class:`ResultGather`, :func:`allgather_results`) and the ensemble
  (:func:`broadcast_tensors` / :func:`broadcast_device_ensemble`, device
  buffers broadcast in place -- no host round trip).
Collectives run on whatever backend the process group uses (``nccl`` on the
GPU box, ``gloo`` in the CPU tests); tensors live on the device the group
needs (``collective_device``).
"""

from __future__ import annotations

import numpy as np


def kernel_shard(n_kernels: int, rank: int, world: int) -> np.ndarray:
    """Contiguous kernel ranges, sizes differing by at most one."""
    lo = n_kernels * rank // world
    hi = n_kernels * (rank + 1) // world
    return np.arange(lo, hi, dtype=np.uint32)


def chunk_shard(n_chunks: int, rank: int, world: int) -> range:
    """Contiguous ranges of generator chunks (workloads.synth_chunks) per rank:
    a rank builds only its own kernels, and the union over ranks is the global
    corpus in kernel order."""
    return range(n_chunks * rank // world, n_chunks * (rank + 1) // world)


def collective_device(group=None):
    """Where a collective's tensors must live: the current CUDA device for
    NCCL, host memory for gloo."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


class ResultGather:
    """Preallocated all-gather of equal-length per-rank result vectors (the
    sweep's status / time / power / energy of each rank's kernel shard) into
    rank-order concatenations on every rank: one ``all_gather_into_tensor``
    per vector (ncclAllGather over NVLink on the GPU box).  ``run`` is what
    the timed multi-GPU step calls after the sweep."""

    def __init__(self, like: list, group=None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.out = [torch.empty((self.world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype,
                                device=t.device) for t in like]

    @property
    def nbytes(self) -> int:
        return sum(o.numel() * o.element_size() for o in self.out)

    def run(self, tensors: list) -> list:
        import torch.distributed as dist

        nccl = dist.get_backend(self.group) == "nccl"
        for o, t in zip(self.out, tensors):
            if nccl:
                dist.all_gather_into_tensor(o, t.contiguous(), group=self.group)
            else:   # gloo (CPU tests, the 2-rank one-GPU bench test): list form
                dist.all_gather(list(o.chunk(self.world)), t.contiguous(), group=self.group)
        return self.out


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


def broadcast_tensors(bufs: dict | None, src: int = 0, group=None, device=None) -> dict:
    """Broadcast a dict of tensors from rank `src`: shapes / dtypes go as one
    object broadcast, then every tensor in place (NCCL: device to device over
    NVLink, no host staging).  Other ranks pass None and get the dict back on
    `device` (default: the group's collective device)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    dev = device or collective_device(group)
    meta = [None]
    if rank == src:
        meta = [{k: (tuple(v.shape), str(v.dtype).replace("torch.", "")) for k, v in bufs.items()}]
    dist.broadcast_object_list(meta, src=src, group=group)
    if rank != src:
        bufs = {k: torch.empty(shape, dtype=getattr(torch, dt), device=dev)
                for k, (shape, dt) in meta[0].items()}
    for k in sorted(bufs):
        # as raw bytes: collectives lack some dtypes (uint32 roots, uint16)
        raw = bufs[k].view(-1).view(torch.uint8) if bufs[k].numel() else None
        if raw is not None:
            dist.broadcast(raw, src=src, group=group)
    return bufs


def broadcast_device_ensemble(de, src: int = 0, group=None):
    """the ensemble replicated once, ncclBroadcast from rank 0.
    Rank `src` passes its DeviceEnsemble (every walk layout's buffers: the
    16-byte nodes, blocks, exact thresholds, leaves, scaling); the others pass
    None and get a DeviceEnsemble over the received device buffers."""
    import torch.distributed as dist

    from .runtime import DeviceEnsemble

    rank = dist.get_rank(group)
    meta = [None]
    if rank == src:
        meta = [dict(base=float(de.desc.base_score), n_trees=int(de.desc.n_trees),
                     n_feat=int(de.desc.n_feat), max_depth=int(de.desc.max_depth))]
    dist.broadcast_object_list(meta, src=src, group=group)
    import torch

    # the buffers stay device buffers whatever the backend (gloo ships CUDA
    # tensors through the host; NCCL device to device)
    bufs = broadcast_tensors(de.bufs if rank == src else None, src=src, group=group,
                             device=torch.device("cuda", torch.cuda.current_device()))
    if rank == src:
        return de
    return DeviceEnsemble.from_buffers(bufs, **meta[0])


def broadcast_flat(flat, src: int = 0, group=None, device=None):
    """Broadcast a FlatEnsemble (node arrays + scaling) from `src` to all ranks;
    returns the FlatEnsemble on every rank (host arrays; the tensors travel
    on the group's collective device)."""
    import torch
    import torch.distributed as dist

    from .ensemble import NODE_DT, FlatEnsemble
    from .runtime import upload

    rank = dist.get_rank(group)
    dev = device or collective_device(group)
    meta = [None]
    if rank == src:
        meta = [dict(n_nodes=len(flat.nodes), n_trees=flat.n_trees, n_feat=flat.n_feat,
                     base=float(flat.base_score), max_depth=int(flat.max_depth),
                     manifest=list(flat.manifest))]
    dist.broadcast_object_list(meta, src=src, group=group)
    m = meta[0]
    if rank == src:
        nodes = upload(flat.nodes.view(np.uint8).reshape(-1), dev)
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


_TREE_INT = ("children_left", "children_right", "feature", "n_node_samples")
_TREE_F64 = ("threshold", "impurity", "weighted_n_node_samples")


def _pack_trees(items) -> np.ndarray:
    """[(tree id, TreeEstimator)] -> one byte buffer (int64 header + arrays)."""
    parts = []
    for t, est in items:
        tr = est.tree_
        nc = int(tr.node_count)
        parts.append(np.array([t, nc, int(tr.max_depth), int(est.random_state)], np.int64))
        parts += [np.asarray(getattr(tr, k), np.int64).reshape(nc) for k in _TREE_INT]
        parts += [np.asarray(getattr(tr, k), np.float64).reshape(nc) for k in _TREE_F64]
        parts.append(np.asarray(tr.value, np.float64).reshape(nc))
    if not parts:
        return np.zeros(0, np.uint8)
    return np.concatenate([p.view(np.uint8) for p in parts])


def _unpack_trees(buf: np.ndarray) -> dict:
    from .forest import Tree, TreeEstimator

    out, at = {}, 0
    w = buf.view(np.int64) if len(buf) else np.zeros(0, np.int64)
    while at < len(w):
        t, nc, md, rs = (int(v) for v in w[at:at + 4])
        at += 4
        cols = {}
        for k in _TREE_INT:
            cols[k] = w[at:at + nc].copy()
            at += nc
        f = buf.view(np.float64)
        for k in _TREE_F64:
            cols[k] = f[at:at + nc].copy()
            at += nc
        value = f[at:at + nc].copy().reshape(nc, 1, 1)
        at += nc
        out[t] = TreeEstimator(tree_=Tree(node_count=nc, value=value, max_depth=md, **cols),
                               random_state=rs)
    return out


def _pack_trees_dev(items):
    """[(tree id, device-resident TreeEstimator)] -> one int64 device tensor:
    [n, n x (id, node_count, max_depth, random_state), per tree it (4 x nc)
    then fl (4 x nc, f64 bits)] -- built with device copies only."""
    import torch

    from .runtime import device

    dev = device()
    hdr = torch.tensor([len(items)] + [v for t, e in items for v in
                                       (t, e.tree_.node_count, e.tree_.max_depth,
                                        int(e.random_state))], dtype=torch.int64, device=dev)
    parts = [hdr]
    for _, e in items:
        fl, it = e.tree_.device_slices()
        parts += [it.reshape(-1), fl.contiguous().view(torch.int64).reshape(-1)]
    return torch.cat(parts)


def _unpack_trees_dev(buf) -> dict:
    import torch

    from .forest import Tree, TreeBatch, TreeEstimator

    n = int(buf[0].item())
    if n == 0:
        return {}
    hdr = buf[1: 1 + 4 * n].view(n, 4).cpu().numpy()
    at = 1 + 4 * n
    fls, its = [], []
    for t, nc, md, rs in hdr:
        nc = int(nc)
        its.append(buf[at: at + 4 * nc].view(4, nc))
        fls.append(buf[at + 4 * nc: at + 8 * nc].view(4, nc).view(torch.float64))
        at += 8 * nc
    counts = hdr[:, 1].astype(np.int64)
    base = np.concatenate([[0], np.cumsum(counts)[:-1]])
    batch = TreeBatch(torch.cat(fls, dim=1), torch.cat(its, dim=1), base, counts, hdr[:, 2])
    return {int(t): TreeEstimator(tree_=Tree(node_count=int(nc), max_depth=int(md), batch=batch,
                                             start=int(b)), random_state=int(rs))
            for (t, nc, md, rs), b in zip(hdr, base)}


def allgather_forest(model, group=None, device=None):
    """Complete a tree-sharded forest on every rank: each rank's trees
    (estimators_[t] for t % world == rank) are packed into one buffer and
    all-gathered, then unpacked in global tree order.  Device-resident trees
    (the K5 fit's TreeBatch) on an NCCL group go device to device -- packed
    by device copies, ncclAllGather over NVLink, unpacked into one TreeBatch
    per source rank, no host round trip; host trees (or gloo groups) travel
    as one host-packed byte buffer."""
    import torch
    import torch.distributed as dist

    mine = [(t, e) for t, e in enumerate(model.estimators_) if e is not None]
    nccl = dist.get_backend(group) == "nccl"
    on_dev = nccl and all(e.tree_.on_device for _, e in mine)
    flag = torch.tensor([int(on_dev)], dtype=torch.int64, device=collective_device(group))
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    on_dev = bool(flag.item())
    world = dist.get_world_size(group)
    merged = {}
    if on_dev:
        buf = _pack_trees_dev(mine)
        sizes = [torch.zeros(1, dtype=torch.int64, device=buf.device) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([buf.numel()], dtype=torch.int64, device=buf.device),
                        group=group)
        sizes = [int(v.item()) for v in sizes]
        pad = torch.zeros(max(sizes), dtype=torch.int64, device=buf.device)
        pad[: buf.numel()] = buf
        out = torch.empty(world * max(sizes), dtype=torch.int64, device=buf.device)
        dist.all_gather_into_tensor(out, pad, group=group)
        for r, sz in enumerate(sizes):
            merged.update(_unpack_trees_dev(out[r * max(sizes): r * max(sizes) + sz]))
    else:
        dev = device or collective_device(group)
        buf = torch.from_numpy(_pack_trees(mine)).to(dev)
        (gathered,) = allgather_results([buf], group=group)
        # the concatenation is in rank order; each rank's part parses independently
        sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([buf.numel()], dtype=torch.int64, device=dev),
                        group=group)
        host = gathered.cpu().numpy()
        at = 0
        for sz in (int(s.item()) for s in sizes):
            merged.update(_unpack_trees(host[at:at + sz]))
            at += sz
    if sorted(merged) != list(range(model.n_estimators)):
        raise RuntimeError("tree shards do not cover the forest")
    model.estimators_ = [merged[t] for t in range(model.n_estimators)]
    model.shard = None
    model._flat = None
    return model
