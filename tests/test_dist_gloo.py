"""Multi-process (world_size 2, gloo, CPU) tests of the sharding + collective
plumbing used on NVLink/NCCL at N > 1 GPUs (paper_2305_01886_b200/dist.py)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, fn, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _gather_fn(rank, world):
    import torch

    from paper_2305_01886_b200.dist import allgather_results

    n = 5 + 3 * rank  # unequal shards
    st = torch.full((n,), rank, dtype=torch.uint8)
    tu = torch.arange(n, dtype=torch.float64) + 100 * rank
    a, b = allgather_results([st, tu])
    return a.tolist(), b.tolist()


def test_allgather_results_unequal_shards():
    out = _spawn(_gather_fn)
    want_st = [0] * 5 + [1] * 8
    want_tu = [float(i) for i in range(5)] + [100.0 + i for i in range(8)]
    for r in (0, 1):
        assert out[r][0] == want_st and out[r][1] == want_tu


def _bcast_fn(rank, world):
    from paper_2305_01886_b200.dist import broadcast_flat
    from paper_2305_01886_b200.ensemble import random_forest_flat

    flat = None
    if rank == 0:
        flat = random_forest_flat(6, 7, ["a", "b", "c"], np.zeros(3), np.ones(3), seed=9)
    got = broadcast_flat(flat)
    return got.nodes.tobytes(), got.tree_off.tolist(), list(got.tree_depth), got.manifest


def test_broadcast_flat_ensemble():
    from paper_2305_01886_b200.ensemble import random_forest_flat

    out = _spawn(_bcast_fn)
    ref = random_forest_flat(6, 7, ["a", "b", "c"], np.zeros(3), np.ones(3), seed=9)
    for r in (0, 1):
        nodes, off, dep, man = out[r]
        assert nodes == ref.nodes.tobytes() and off == ref.tree_off.tolist()
        assert dep == list(ref.tree_depth) and man == ("a", "b", "c")


def _tiny_tree(t):
    from paper_2305_01886_b200.forest import Tree

    nc = 3 + 2 * (t % 2)
    rng = np.random.default_rng(t)
    return Tree(node_count=nc, children_left=np.r_[1, [-1] * (nc - 1)].astype(np.int64),
                children_right=np.r_[2, [-1] * (nc - 1)].astype(np.int64),
                feature=rng.integers(0, 4, nc), threshold=rng.random(nc),
                value=rng.random((nc, 1, 1)), impurity=rng.random(nc),
                n_node_samples=rng.integers(1, 99, nc),
                weighted_n_node_samples=rng.random(nc) * 10, max_depth=1 + t % 3)


def _forest_fn(rank, world):
    from paper_2305_01886_b200.dist import allgather_forest
    from paper_2305_01886_b200.forest import RandomForestRegressor, TreeEstimator

    # a tree-sharded forest as fit(shard=(rank, world)) leaves it (no GPU needed)
    m = RandomForestRegressor(5, random_state=0, shard=(rank, world))
    m.estimators_ = [TreeEstimator(tree_=_tiny_tree(t), random_state=100 + t)
                     if t % world == rank else None for t in range(5)]
    allgather_forest(m)
    return [(e.random_state, e.tree_.node_count, e.tree_.max_depth,
             e.tree_.threshold.tolist(), e.tree_.value.tolist(), e.tree_.feature.tolist(),
             e.tree_.children_left.tolist(), e.tree_.weighted_n_node_samples.tolist())
            for e in m.estimators_]


def test_tree_sharded_forest_reassembles_in_order():
    out = _spawn(_forest_fn)
    want = []
    for t in range(5):
        tr = _tiny_tree(t)
        want.append((100 + t, tr.node_count, tr.max_depth, tr.threshold.tolist(),
                     tr.value.tolist(), tr.feature.tolist(), tr.children_left.tolist(),
                     tr.weighted_n_node_samples.tolist()))
    for r in (0, 1):
        assert out[r] == want


def test_kernel_shards_partition_the_corpus():
    from paper_2305_01886_b200.dist import kernel_shard

    for n, w in ((10, 3), (7, 8), (10000, 8)):
        parts = [kernel_shard(n, r, w) for r in range(w)]
        allk = np.concatenate(parts)
        assert np.array_equal(allk, np.arange(n))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_tree_seeds_independent_of_world_size():
    from paper_2305_01886_b200.forest import tree_seeds

    s = tree_seeds(0, 12)
    for w in (1, 2, 4, 8):
        got = {t: s[t] for r in range(w) for t in range(12) if t % w == r}
        assert [got[t] for t in range(12)] == list(s)


def _result_gather_fn(rank, world):
    import torch

    from paper_2305_01886_b200.dist import ResultGather

    n = 6   # equal shards (chunk-granular kernel shards)
    st = torch.full((n,), rank + 1, dtype=torch.uint8)
    tu = torch.arange(n, dtype=torch.float64) + 100 * rank
    g = ResultGather([st, tu])
    for _ in range(2):                       # reused buffers, every timed step
        a, b = g.run([st, tu])
    return a.tolist(), b.tolist(), g.nbytes


def test_result_gather_rank_order():
    out = _spawn(_result_gather_fn)
    for r in (0, 1):
        st, tu, nb = out[r]
        assert st == [1] * 6 + [2] * 6
        assert tu == [float(i) for i in range(6)] + [100.0 + i for i in range(6)]
        assert nb == 12 * 1 + 12 * 8


def _bcast_tensors_fn(rank, world):
    import torch

    from paper_2305_01886_b200.dist import broadcast_tensors

    bufs = None
    if rank == 0:
        bufs = {"nodes": torch.arange(40, dtype=torch.uint8), "lo": torch.tensor([1.5, -2.0]),
                "off": torch.tensor([0, 7, 19], dtype=torch.int64),
                "blocks": torch.arange(24, dtype=torch.int32).view(3, 8),
                "root": torch.tensor([1, 2 ** 31 + 5], dtype=torch.uint32)}
    got = broadcast_tensors(bufs)
    return {k: (str(v.dtype), tuple(v.shape), v.flatten().tolist()) for k, v in got.items()}


def test_broadcast_tensors_every_layout_buffer():
    """The device-ensemble broadcast (dist.broadcast_device_ensemble) ships
    every walk-layout buffer with its dtype and shape."""
    out = _spawn(_bcast_tensors_fn)
    assert out[0] == out[1]
    assert out[1]["blocks"] == ("torch.int32", (3, 8), list(range(24)))
    assert out[1]["lo"] == ("torch.float32", (2,), [1.5, -2.0])
    assert out[1]["root"] == ("torch.uint32", (2,), [1, 2 ** 31 + 5])


def test_chunk_shards_cover_the_corpus_in_order():
    from paper_2305_01886_b200.dist import chunk_shard

    for n, w in ((2000, 1), (2000, 8), (5, 2), (13, 4)):
        parts = [list(chunk_shard(n, r, w)) for r in range(w)]
        assert sum(parts, []) == list(range(n))
        assert parts[0][0] == 0


pytestmark = pytest.mark.timeout(300) if hasattr(pytest.mark, "timeout") else []
