"""GPU random forest (K5) behind scikit-learn's estimator shape.

Drop-in for the estimator the reference trainer builds in
``gpukalc_trainer.training._make_model`` (``training.py:73-76``):
``RandomForestRegressor(n_estimators, max_depth, random_state)`` with
``fit(X, y)``, ``predict(X)`` and ``estimators_[k].tree_`` carrying the arrays
``gpukalc_trainer.export.ensemble_document`` reads (``export.py:26-50``):
node_count, children_left/right, feature, threshold, value, impurity,
weighted_n_node_samples (+ n_node_samples, max_depth).

Semantics kept from scikit-learn: per-tree seeds are
successive ``RandomState(seed).randint(2**31 - 1)`` draws
(SK/ensemble/_base.py:77-81); bootstrap weights are
``bincount(RandomState(tree_seed).randint(0, n, n))`` (SK/ensemble/_forest.py:
95-112, 150-156), generated bit-exactly on the device; X is fitted as float32
(SK/tree/_classes.py:244); squared error, all features, min_samples_split 2,
min_samples_leaf 1; thresholds are midpoints between adjacent training values
(SK/tree/_splitter.pyx:459-460); predictions average the trees in order.
Split search is histogram-based (<= 256 bins per feature), so trees differ
from sklearn's exact search; the parity bar is R^2 / MAPE (BASELINE.json).
"""

from __future__ import annotations

import ctypes as C
import functools
import os
from dataclasses import dataclass

import numpy as np

from .ensemble import NODE_DT, FlatEnsemble

N_BINS = 256
SMALL, MEDIUM = 64, 32768  # SMALL = 32 x GK_SMALL_RPL of gk_rftrain.cu (128 / 256 measured slower)
TASK_DT = np.dtype([("tree", "<i4"), ("begin", "<i4"), ("end", "<i4"), ("parity", "<i4")])
SPLIT_DT = np.dtype({"names": ["feat", "bin", "n_left", "pad", "proxy"],
                     "formats": ["<i4", "<i4", "<i4", "<i4", "<f8"],
                     "offsets": [0, 4, 8, 12, 16], "itemsize": 24})
TREE_LEAF, TREE_UNDEFINED = -1, -2
_LEVEL_LOG = None   # set to a list to record per-level kernel times (tools/k5_levels.py)


def _lib():
    from .runtime import load_library

    L = load_library()
    if not getattr(L, "_rf_bound", False):
        vp, i32, i64, u32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32
        L.gk_rf_bootstrap.argtypes = [vp, u32, i64, vp, vp]
        L.gk_rf_compact.argtypes = [vp, u32, i64, vp, i32, vp, vp, vp, vp, vp]
        L.gk_rf_record_bytes.argtypes = [i32]
        L.gk_rf_record_bytes.restype = C.c_size_t
        L.gk_rf_bin.argtypes = [vp, i64, i32, i64, vp, vp, vp, vp, vp, vp]
        L.gk_rf_split_level.argtypes = [vp, vp, vp, vp, i64, i32, vp, vp, i32, vp, i32, vp, i32,
                                        i32, vp, vp, vp, vp, vp, vp, vp, i32, vp]
        L.gk_rf_hist_bytes.argtypes = [i32, i32]
        L.gk_rf_hist_bytes.restype = C.c_size_t
        L.gk_rf_partition.argtypes = [vp, vp, vp, vp, i64, i32, vp, i32, vp, vp, i32, i32, vp,
                                      vp, vp, vp]
        L.gk_rf_leaf_stats.argtypes = [vp, i64, i32, vp, vp, vp, i32, vp, vp, vp, i32, vp]
        L.gk_rf_assemble_nodes.argtypes = [vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp]
        L.gk_rf_assemble_up.argtypes = [vp, vp, vp, vp, i32, vp, vp, vp]
        L.gk_rf_assemble_final.argtypes = [i64, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp]
        L.gk_rf_level_scratch_bytes.argtypes = [i32, i32]
        L.gk_rf_level_scratch_bytes.restype = C.c_size_t
        L.gk_rf_next_level.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, vp, vp, vp, vp, vp,
                                       i32, vp, vp, vp, vp, vp]
        L.gk_rf_partition_lists.argtypes = [vp, vp, i64, i32, vp, i32, vp, vp, i32, vp, i32, i32,
                                            vp, i32, i32, vp, vp, vp, vp]
        L._rf_bound = True
    return L


def _check(rc):
    from .runtime import _check as chk

    chk(rc)


class _Read:
    """An asynchronous device -> pinned host read: the copy and an event are
    queued on the current stream; `.get()` waits for that event only.  A batch
    generator yields the read (so the driver can launch other batches' work
    meanwhile) and calls `.get()` when resumed."""

    def __init__(self, t):
        import torch

        self.h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
        self.h.copy_(t, non_blocking=True)
        self.ev = torch.cuda.Event()
        self.ev.record()

    def ready(self) -> bool:
        return self.ev.query()

    def get(self) -> np.ndarray:
        self.ev.synchronize()
        return self.h.numpy()


_STREAMS: dict = {}


def _stream_pool(dev, n: int) -> list:
    """Streams reused across fits: torch's caching allocator pools memory per
    stream, so fresh streams per fit re-allocated every level buffer with
    cudaMalloc (~150 ms of host time and GPU-idle gaps per 500-tree fit)."""
    import torch

    pool = _STREAMS.setdefault(str(dev), [])
    while len(pool) < n:
        pool.append(torch.cuda.Stream(device=dev))
    return pool[:n]


def _drive(gen):
    """Run one batch generator to completion on the current stream."""
    try:
        while True:
            next(gen).get()
    except StopIteration as stop:
        return stop.value


def _drive_many(gens, streams):
    """Round-robin the batch generators over `streams` from ONE host thread:
    each resume launches a batch's next level (or assembly step) on its own
    stream and returns at its next device -> host read; a batch is resumed
    once that read has landed, ready ones first.  No host threads, so no GIL
    hand-offs between the batches' Python bookkeeping."""
    import collections

    import torch

    todo = collections.deque(enumerate(gens))
    slots = []  # [index, generator, stream, pending read]
    results = {}
    free = list(streams)

    def start():
        while todo and free:
            k, g = todo.popleft()
            slots.append([k, g, free.pop(0), None])

    start()
    while slots:
        pick = next((sl for sl in slots if sl[3] is None or sl[3].ready()), slots[0])
        k, g, st, rd = pick
        if rd is not None:
            rd.ev.synchronize()
        with torch.cuda.stream(st):
            try:
                pick[3] = g.send(None)
            except StopIteration as stop:
                results[k] = stop.value
                slots.remove(pick)
                free.append(st)
                start()
    return [results[k] for k in range(len(results))]


def tree_seeds(random_state, n_estimators: int) -> np.ndarray:
    """Per-tree seeds as scikit-learn draws them (SK/ensemble/_base.py:77-81)."""
    rs = random_state if isinstance(random_state, np.random.RandomState) else \
        np.random.RandomState(random_state)
    return np.array([rs.randint(np.iinfo(np.int32).max) for _ in range(n_estimators)],
                    dtype=np.int64)


@functools.lru_cache(maxsize=8)
def _sample_rows(n: int, sample: int) -> np.ndarray:
    """The deterministic edge sample: sorted row ids of default_rng(0).choice
    (n, sample, replace=False), cached per table height (folds and repeated
    fits of one table reuse it; the draw costs ~10-30 ms at 1M rows)."""
    idx = np.sort(np.random.default_rng(0).choice(n, sample, replace=False))
    idx.setflags(write=False)
    return idx


def bin_edges(Xf: np.ndarray, n_bins: int = N_BINS, sample: int = 65_536, device=None):
    """Per-feature bin edges on float32 data: one bin per distinct value when a
    feature has <= n_bins of them, else quantile edges of a deterministic
    row sample (>= 256 sample rows per bin).  One column-wise sort -- on
    `device` when given (sorting is exact: the same sorted columns; it was
    ~1/3 of a 50-stage boosting fit on the host)."""
    n, F = Xf.shape
    # the sorted sample is kept transposed ([feature][row], each column
    # contiguous) for the per-feature scan below
    if is_device_tensor(Xf):   # the same rows, sorted on the tensor's device
        import torch

        S = Xf
        if n > sample:
            S = Xf.index_select(0, torch.from_numpy(_sample_rows(n, sample).copy()).to(Xf.device))
        S = torch.sort(S.to(torch.float32), dim=0).values.t().contiguous().cpu().numpy()
    elif n > sample:
        S = Xf[_sample_rows(n, sample)]
    else:
        S = Xf
    if is_device_tensor(Xf):
        pass
    elif device is not None:
        import torch

        S = torch.sort(torch.from_numpy(np.ascontiguousarray(S, dtype=np.float32)).to(device),
                       dim=0).values.t().contiguous().cpu().numpy()
    else:
        S = np.ascontiguousarray(np.sort(S.astype(np.float32), axis=0).T)
    m = S.shape[1]
    # k5_bin reads a fixed (N_BINS - 1)-wide edge row per feature; fewer bins
    # use a prefix of it (n_edges[f] <= n_bins - 1)
    edges = np.zeros((F, N_BINS - 1), np.float32)
    n_edges = np.zeros(F, np.int32)
    qpos = (np.linspace(0.0, 1.0, n_bins + 1)[1:-1] * (m - 1)).astype(np.int64)  # "lower"
    for f in range(F):
        col = S[f]
        new = np.empty(m, bool)
        new[0] = True
        np.not_equal(col[1:], col[:-1], out=new[1:])
        u = col[new]
        if len(u) <= n_bins:
            e = u[:-1]
        else:
            q = col[qpos]
            e = q[np.r_[True, q[1:] != q[:-1]]]
        edges[f, : len(e)] = e
        n_edges[f] = len(e)
    return edges, n_edges


def is_device_tensor(a) -> bool:
    """A torch tensor (the trainer passes its folds as device tensors: no host
    copies of the scaled folds, no re-upload)."""
    return type(a).__module__.split(".")[0] == "torch"


def check_n_bins(n_bins) -> int:
    """K5 bins are u8 ids with a fixed 256-entry table per feature: any
    2 <= n_bins <= 256 is exact (fewer bins use a prefix of the edge row)."""
    if isinstance(n_bins, bool) or not isinstance(n_bins, (int, np.integer)) \
            or not 2 <= int(n_bins) <= N_BINS:
        raise ValueError(f"n_bins must be an integer in [2, {N_BINS}], got {n_bins!r}")
    return int(n_bins)


def check_finite(X: np.ndarray, y: np.ndarray) -> None:
    """NaN / inf in X or y raise ValueError before anything reaches the device.
    scikit-learn raises the same for inf, and for NaN in boosting; its forest
    (>= 1.4) would route NaN as a missing value, which K5 does not implement --
    the reference never passes NaN (its Dataset rejects missing values before
    any fit, dataset.py:57-58)."""
    if not np.isfinite(X).all():
        raise ValueError("Input X contains NaN or infinity.")
    if not np.isfinite(y).all():
        raise ValueError("Input y contains NaN or infinity.")


_TREE_ARRAYS = ("children_left", "children_right", "feature", "threshold", "value", "impurity",
                "n_node_samples", "weighted_n_node_samples")


class TreeBatch:
    """The K5 output of one batch of trees, resident in HBM: fl [4, N] f64
    (threshold, value, impurity, weighted_n_node_samples) and it [4, N] int64
    (children_left, children_right, feature, n_node_samples), trees contiguous
    from node_base[k].  A fitted forest keeps its trees here -- predict() walks
    them on the device -- and copies them to host numpy arrays only when
    something reads a ``tree_`` array (export, sklearn-style inspection):
    one DMA per batch through a pinned staging buffer."""

    _STAGE = 32 << 20   # bytes per staging buffer (two, alternating)

    def __init__(self, fl_d, it_d, node_base, next_id, tree_depth):
        import threading

        self.fl_d, self.it_d = fl_d, it_d
        self.node_base = np.asarray(node_base, np.int64)
        self.next_id = np.asarray(next_id, np.int64)
        self.tree_depth = np.asarray(tree_depth, np.int64)
        self._host = None
        self._nodes = None
        self._lock = threading.Lock()

    @property
    def n_nodes(self) -> int:
        return int(self.fl_d.shape[1])

    def host(self):
        """(fl, it) as host numpy arrays (copied once)."""
        with self._lock:
            if self._host is None:
                self._host = (_to_host(self.fl_d), _to_host(self.it_d))
        return self._host

    def device_nodes(self, leaf_scale: float = 1.0):
        """[N] gk_node records (16 B: {v, feature, left}) of the batch built on
        the device: splits {threshold, feature, left}, leaves {value *
        leaf_scale, -1, self - 1} (include/gk.h gk_node)."""
        import torch

        key = float(leaf_scale)
        if self._nodes is not None and self._nodes[0] == key:
            return self._nodes[1]
        fl, it = self.fl_d, self.it_d
        N = self.n_nodes
        dev = fl.device
        split = it[0] >= 0
        tree = torch.repeat_interleave(torch.arange(len(self.next_id), device=dev),
                                       _h2d(self.next_id, dev), output_size=N)
        local = torch.arange(N, device=dev) - _h2d(self.node_base, dev)[tree]
        rec = torch.empty((N, 4), dtype=torch.int32, device=dev)
        v = torch.where(split, fl[0], fl[1] * key).contiguous()
        rec[:, 0:2] = v.view(torch.int32).view(N, 2)
        rec[:, 2] = torch.where(split, it[2], torch.full_like(it[2], -1)).to(torch.int32)
        rec[:, 3] = torch.where(split, it[0], local - 1).to(torch.int32)
        self._nodes = (key, rec)
        return rec


def _h2d(a: np.ndarray, dev):
    """Small host array -> device, asynchronously through pinned memory.  A
    pageable copy blocks the driving thread until the stream's queued work
    drains: ~4 ms per batch start with 4 batches in flight (cProfile of
    train(), 0.36 s of 8 s).  torch's caching host allocator keeps the
    pinned block until the copy is done."""
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(dev, non_blocking=True)


def _to_host(t) -> np.ndarray:
    """Device tensor -> host numpy through two alternating pinned staging
    buffers (DMA of chunk k + 1 overlaps the host copy of chunk k; a pageable
    .cpu() ran at ~2 GB/s)."""
    import torch

    out = np.empty(tuple(t.shape), dtype=np.dtype(str(t.dtype).replace("torch.", "")))
    src = t.contiguous().view(-1).view(torch.uint8)
    dst = out.reshape(-1).view(np.uint8)
    n = src.numel()
    if n == 0:
        return out
    st = torch.cuda.current_stream()
    cap = TreeBatch._STAGE
    bufs = [torch.empty(min(cap, n), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    evs = [torch.cuda.Event(), torch.cuda.Event()]
    chunks = [(a, min(n, a + cap)) for a in range(0, n, cap)]

    def issue(k):
        a, b = chunks[k]
        bufs[k % 2][: b - a].copy_(src[a:b], non_blocking=True)
        evs[k % 2].record(st)

    issue(0)
    for k, (a, b) in enumerate(chunks):
        if k + 1 < len(chunks):   # its buffer was drained by chunk k - 1's host copy
            issue(k + 1)
        evs[k % 2].synchronize()
        np.copyto(dst[a:b], bufs[k % 2][: b - a].numpy())
    return out


class Tree:
    """The subset of sklearn's ``Tree`` the reference exporter reads
    (``export.py:26-50``): node_count, max_depth and the per-node arrays
    children_left / children_right / feature / threshold / value [n, 1, 1] /
    impurity / n_node_samples / weighted_n_node_samples.  Built either from
    host arrays or as a view of a device-resident :class:`TreeBatch`, whose
    arrays are copied to the host on first access."""

    def __init__(self, node_count: int, children_left=None, children_right=None, feature=None,
                 threshold=None, value=None, impurity=None, n_node_samples=None,
                 weighted_n_node_samples=None, max_depth: int = 0, *, batch=None, start: int = 0):
        self.node_count = int(node_count)
        self.max_depth = int(max_depth)
        self._batch, self._start = batch, int(start)
        self._arrays = None
        if batch is None:
            self._arrays = dict(children_left=children_left, children_right=children_right,
                                feature=feature, threshold=threshold, value=value,
                                impurity=impurity, n_node_samples=n_node_samples,
                                weighted_n_node_samples=weighted_n_node_samples)

    @property
    def on_device(self) -> bool:
        return self._batch is not None

    def _load(self) -> dict:
        if self._arrays is None:
            fl, it = self._batch.host()
            g = slice(self._start, self._start + self.node_count)
            self._arrays = dict(children_left=it[0, g], children_right=it[1, g], feature=it[2, g],
                                threshold=fl[0, g], value=fl[1, g].reshape(-1, 1, 1),
                                impurity=fl[2, g], n_node_samples=it[3, g],
                                weighted_n_node_samples=fl[3, g])
        return self._arrays

    def device_slices(self):
        """(fl [4, n], it [4, n]) device views of a device-resident tree."""
        g = slice(self._start, self._start + self.node_count)
        return self._batch.fl_d[:, g], self._batch.it_d[:, g]


def _tree_array(name):
    return property(lambda self: self._load()[name], doc=f"sklearn Tree.{name}")


for _n in _TREE_ARRAYS:
    setattr(Tree, _n, _tree_array(_n))
del _n


@dataclass
class TreeEstimator:
    tree_: Tree
    random_state: int


class _LevelGrower:
    """Shared K5 machinery: device binning + midpoint threshold tables
    (`_prepare_bins`, `_thr_tables`) and level-wise growth of a batch of trees
    over row lists (`_grow`).  Used by the random forest and by gradient
    boosting (boosting.py)."""

    def _prepare_bins(self, X):
        """Bin X on the device (float32 cast like sklearn) and build the
        midpoint threshold table; returns the [n][F] u8 bin matrix."""
        import torch

        from .runtime import _dev, _ptr, device

        n, F = X.shape
        L = _lib()
        dev = device()
        edges, n_edges = bin_edges(X, self.n_bins, device=dev)   # float32 sample inside
        # k5_bin casts to float32 (sklearn)
        Xd = X.contiguous() if is_device_tensor(X) else _dev(X, dev)
        Xb = torch.empty(n * F, dtype=torch.uint8, device=dev)
        bmin = torch.empty(F * N_BINS, dtype=torch.int32, device=dev)
        bmax = torch.empty(F * N_BINS, dtype=torch.int32, device=dev)
        ed = torch.from_numpy(edges).to(dev)
        ne = torch.from_numpy(n_edges).to(dev)
        _check(L.gk_rf_bin(_ptr(Xd), n, F, F, _ptr(ed), _ptr(ne), _ptr(Xb), _ptr(bmin), _ptr(bmax),
                           torch.cuda.current_stream().cuda_stream))
        del Xd
        self._thr_tables(bmin.cpu().numpy().view(np.uint32).reshape(F, N_BINS),
                         bmax.cpu().numpy().view(np.uint32).reshape(F, N_BINS))
        # device copy for the tree assembly, complete before any batch stream reads it
        self._dev_thr = torch.from_numpy(self._thr).to(dev)
        torch.cuda.current_stream().synchronize()
        return Xb

    def _thr_tables(self, bmin_ord, bmax_ord):
        def ord2f(u):
            u = u.astype(np.uint32)
            bits = np.where(u & 0x80000000, u & 0x7FFFFFFF, ~u)
            return bits.astype(np.uint32).view(np.float32).astype(np.float64)

        empty = bmin_ord == 0xFFFFFFFF
        vmin = np.where(empty, np.inf, ord2f(bmin_ord))
        vmax = np.where(empty, -np.inf, ord2f(bmax_ord))
        F = vmin.shape[0]
        # last non-empty bin <= b (its max) and first non-empty bin > b (its min)
        lo = np.full((F, N_BINS), -np.inf)
        hi = np.full((F, N_BINS), np.inf)
        cur = np.full(F, -np.inf)
        for b in range(N_BINS):
            cur = np.where(empty[:, b], cur, vmax[:, b])
            lo[:, b] = cur
        cur = np.full(F, np.inf)
        for b in range(N_BINS - 1, -1, -1):
            hi[:, b] = cur
            cur = np.where(empty[:, b], cur, vmin[:, b])
        thr = lo / 2.0 + hi / 2.0              # SK/tree/_splitter.pyx:459-460
        bad = (thr == hi) | ~np.isfinite(thr)
        self._thr = np.where(bad, lo, thr)

    def _grow(self, counts, base, m, rows0, rows1, TB):
        """Grow TB trees level-wise over the row lists rows0[base[t] .. +m[t]]
        (weights counts[t][row]); returns (sklearn-shaped trees, leaf records)
        where the leaf records are (TASK_DT tasks, per-leaf node value).

        The level loop's bookkeeping runs on the device (gk_rf_next_level: one
        small stats read per level); GK_RF_HOST_LEVELS=1 selects the numpy
        form it replaced (same trees, node for node -- kept for A/B tests)."""
        if os.environ.get("GK_RF_HOST_LEVELS", "0") == "1":
            return self._grow_host(counts, base, m, rows0, rows1, TB)
        return _drive(self._grow_dev(counts, base, m, rows0, rows1, TB))

    def _grow_dev(self, counts, base, m, rows0, rows1, TB):
        """Generator: yields a _Read before every host read of device results
        (one per level, a few in the assembly); returns (trees, leaf records)."""
        import torch

        from .runtime import _ptr, device

        L = _lib()
        dev = device()
        D = self._dev
        n, F = D["n"], D["F"]
        st = torch.cuda.current_stream().cuda_stream
        max_depth = self.max_depth if self.max_depth is not None else 1 << 30
        max_depth = min(int(max_depth), (1 << 31) - 1)
        i32 = torch.int32

        # level 0 on the host: one root per tree
        tasks = np.zeros(TB, TASK_DT)
        tasks["tree"] = np.arange(TB)
        tasks["begin"], tasks["end"] = base, base + m
        size = np.asarray(m, np.int64)
        cls = np.where((size >= 2) & (max_depth > 0),
                       (size > SMALL).astype(np.int64) + (size > MEDIUM), -1)
        cap = 2 * TB
        lists = np.zeros(3 * cap, np.int32)
        stats = np.zeros(8, np.int64)
        stats[0] = TB
        for c in range(3):
            ids = np.nonzero(cls == c)[0]
            lists[c * cap: c * cap + len(ids)] = ids
            stats[1 + c] = len(ids)
        stats[4] = size[cls == 1].max() if (cls == 1).any() else 0
        stats[5] = size[cls == 2].max() if (cls == 2).any() else 0
        tasks_d = _h2d(tasks.view(np.int32), dev)
        node_d = torch.zeros(TB, dtype=i32, device=dev)
        lists_d = _h2d(lists, dev)
        next_id_d = torch.ones(TB, dtype=i32, device=dev)
        stats_d = torch.empty(8, dtype=i32, device=dev)
        # two histogram workspaces for the batch (a big task has > MEDIUM rows),
        # alternating by level: the previous level's big histograms stay for
        # the sibling subtraction (GK_RF_SUBTRACT=0: every big task builds)
        n_big_cap = int(np.sum(m)) // (MEDIUM + 1) + 1
        hists = [torch.empty(max(int(L.gk_rf_hist_bytes(n_big_cap, F)), 8), dtype=torch.uint8,
                             device=dev) for _ in range(2)]
        subtract = os.environ.get("GK_RF_SUBTRACT", "1") != "0"
        par_slot = None
        cursor = torch.empty(0, dtype=i32, device=dev)
        records = []  # per level: (tasks, node, split, lid, n_tasks, n_split), device tensors
        depth = 0
        while True:
            nt = int(stats[0])
            n_s, n_m, n_b = (int(v) for v in stats[1:4])
            split_d = torch.full((6 * nt,), -1, dtype=i32, device=dev)  # feat -1: leaf
            lp = _ptr(lists_d)
            if n_s + n_m + n_b == 0:
                records.append((tasks_d, node_d, split_d, None, nt, 0))
                break
            if n_b > n_big_cap:
                raise RuntimeError("forest: big-task workspace undersized")
            big_chunks = -(-int(stats[5]) // MEDIUM) if n_b else 0
            hist, prev_hist = hists[depth % 2], hists[(depth + 1) % 2]
            sub_args = (_ptr(prev_hist) if subtract and par_slot is not None else None,
                        _ptr(par_slot) if par_slot is not None else None)
            slot_cur = torch.empty(max(nt, 1), dtype=i32, device=dev)
            if _LEVEL_LOG is not None:   # tuning aid: per-level, per-class device times
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
                ev[0].record()
                for c, (a, b_, cnt) in enumerate(((lp, 0, n_s), (lp + 4 * cap, 1, n_m),
                                                  (lp + 8 * cap, 2, n_b))):
                    args_ = [lp, 0, lp + 4 * cap, 0, lp + 8 * cap, 0]
                    args_[2 * c + 1] = cnt
                    _check(L.gk_rf_split_level(
                        _ptr(D["Xb"]), _ptr(D["yfp"]), _ptr(D["y"]), _ptr(counts), n, F,
                        _ptr(tasks_d), *args_, big_chunks, _ptr(rows0), _ptr(rows1), _ptr(hist),
                        _ptr(split_d), *sub_args, _ptr(slot_cur), nt, st))
                    ev[c + 1].record()
            else:
                _check(L.gk_rf_split_level(
                    _ptr(D["Xb"]), _ptr(D["yfp"]), _ptr(D["y"]), _ptr(counts), n, F,
                    _ptr(tasks_d), lp, n_s, lp + 4 * cap, n_m, lp + 8 * cap, n_b, big_chunks,
                    _ptr(rows0), _ptr(rows1), _ptr(hist), _ptr(split_d), *sub_args,
                    _ptr(slot_cur), nt, st))
            if len(cursor) < 2 * nt:
                cursor = torch.empty(2 * nt, dtype=i32, device=dev)
            _check(L.gk_rf_partition_lists(
                _ptr(D["Xb"]), _ptr(counts), n, F, _ptr(tasks_d), nt, _ptr(split_d),
                lp, n_s, lp + 4 * cap, n_m, int(stats[4]), lp + 8 * cap, n_b, int(stats[5]),
                _ptr(rows0), _ptr(rows1), _ptr(cursor), st))
            lid_d = torch.empty(max(nt, 1), dtype=i32, device=dev)
            tasks_n = torch.empty(max(8 * nt, 4), dtype=i32, device=dev)
            node_n = torch.empty(max(2 * nt, 1), dtype=i32, device=dev)
            lists_n = torch.empty(max(6 * nt, 3), dtype=i32, device=dev)
            scratch = torch.empty(int(L.gk_rf_level_scratch_bytes(nt, TB)), dtype=torch.uint8,
                                  device=dev)
            par_next = torch.empty(max(2 * nt, 1), dtype=i32, device=dev)
            _check(L.gk_rf_next_level(
                _ptr(tasks_d), _ptr(node_d), _ptr(split_d), _ptr(cursor), nt, TB, depth + 1,
                max_depth,
                _ptr(next_id_d), _ptr(lid_d), _ptr(tasks_n), _ptr(node_n), _ptr(lists_n),
                2 * nt, _ptr(stats_d), _ptr(scratch), _ptr(slot_cur), _ptr(par_next), st))
            if _LEVEL_LOG is not None:
                ev[4].record()
            prev = stats
            rd = _Read(stats_d)
            yield rd
            stats = rd.get().astype(np.int64)  # the level's one host read
            if _LEVEL_LOG is not None:
                _LEVEL_LOG.append(dict(depth=depth, n_small=n_s, n_med=n_m, n_big=n_b,
                                       max_med=int(prev[4]), max_big=int(prev[5]),
                                       small_ms=ev[0].elapsed_time(ev[1]),
                                       med_ms=ev[1].elapsed_time(ev[2]),
                                       big_ms=ev[2].elapsed_time(ev[3]),
                                       part_next_ms=ev[3].elapsed_time(ev[4])))
            records.append((tasks_d, node_d, split_d, lid_d, nt, int(stats[0]) // 2))
            depth += 1
            if stats[0] == 0:
                break
            tasks_d, node_d, lists_d, cap = tasks_n, node_n, lists_n, 2 * nt
            par_slot = par_next

        if TB == 1:   # one tree: every node is a task of exactly one level
            next_id = np.array([sum(r[4] for r in records)], np.int64)
        else:
            rd = _Read(next_id_d)
            yield rd
            next_id = rd.get().astype(np.int64)
        return (yield from self._assemble_dev(counts, rows0, rows1, TB, records, next_id))

    def _assemble_dev(self, counts, rows0, rows1, TB, records, next_id):
        """_assemble on the device: node arrays by scatter from the level records,
        leaf statistics, bottom-up integer sums, then the sklearn-shaped arrays
        in two reads (the numpy form cost ~0.15 s per 16 deep trees)."""
        import torch

        from .runtime import _ptr, device

        L = _lib()
        dev = device()
        D = self._dev
        n = D["n"]
        st = torch.cuda.current_stream().cuda_stream
        i64 = torch.int64
        node_base = np.concatenate([[0], np.cumsum(next_id)[:-1]]).astype(np.int64)
        N = int(next_id.sum())
        nb_d = _h2d(node_base, dev)
        feat = torch.full((N,), TREE_UNDEFINED, dtype=i64, device=dev)
        nbin = torch.zeros(N, dtype=i64, device=dev)
        left = torch.full((N,), TREE_LEAF, dtype=i64, device=dev)
        depth_d = torch.zeros(TB, dtype=i64, device=dev)
        # all levels at once (level order kept); node arrays, leaf statistics and
        # the bottom-up sums in native kernels (include/gk.h gk_rf_assemble_*)
        tk = torch.cat([r[0][: 4 * r[4]].view(r[4], 4) for r in records])
        sp = torch.cat([r[2][: 6 * r[4]].view(r[4], 6) for r in records])
        nd = torch.cat([r[1][: r[4]] for r in records])
        lid_all = torch.cat([r[3][: r[4]] if r[3] is not None else
                             torch.full((r[4],), -1, dtype=torch.int32, device=dev)
                             for r in records])
        lvl_all = torch.cat([torch.full((r[4],), k, dtype=torch.int32, device=dev)
                             for k, r in enumerate(records)])
        n_all = int(tk.shape[0])
        _check(L.gk_rf_assemble_nodes(_ptr(tk), _ptr(sp), _ptr(nd), _ptr(lid_all), _ptr(lvl_all),
                                      n_all, _ptr(nb_d), _ptr(feat), _ptr(nbin), _ptr(left),
                                      _ptr(depth_d), st))
        # leaves: their tasks (level order) and node indices; sizes known on the
        # host (split counts from the level loop), so nothing synchronises
        n_split = int(sum(r[5] for r in records))
        li = torch.nonzero_static(sp[:, 0] < 0, size=n_all - n_split).squeeze(1)
        lv_d = tk[li].contiguous()
        gl = nb_d[lv_d[:, 0].long()] + nd[li].long()
        nl = int(lv_d.shape[0])
        if nl <= 256:   # few leaves (boosting stages): n bounds them, no read
            max_leaf = n
        else:
            rd = _Read((lv_d[:, 2] - lv_d[:, 1]).max())
            yield rd
            max_leaf = int(rd.get())
        stats_d = torch.empty(4 * max(nl, 1), dtype=i64, device=dev)
        _check(L.gk_rf_leaf_stats(_ptr(counts), n, D["F"], _ptr(D["yfp"]), _ptr(D["y2fp"]), _ptr(lv_d),
                                  nl, _ptr(rows0), _ptr(rows1), _ptr(stats_d), max_leaf, st))
        # exact integer sums bottom-up, one native launch per level
        ist = torch.zeros((N, 4), dtype=i64, device=dev)
        ist[gl] = stats_d[: 4 * nl].view(nl, 4)
        off = np.concatenate([[0], np.cumsum([r[4] for r in records])]).astype(np.int64)
        for k in range(len(records) - 1, -1, -1):
            if records[k][5] == 0:
                continue
            o, c = int(off[k]), int(records[k][4])
            _check(L.gk_rf_assemble_up(_ptr(tk[o:]), _ptr(sp[o:]), _ptr(nd[o:]), _ptr(lid_all[o:]),
                                       c, _ptr(nb_d), _ptr(ist), st))
        fl = torch.empty((4, N), dtype=torch.float64, device=dev)
        it = torch.empty((4, N), dtype=i64, device=dev)
        _check(L.gk_rf_assemble_final(N, _ptr(ist), _ptr(feat), _ptr(nbin), _ptr(left),
                                      _ptr(self._dev_thr), D["shift"], D["shift2"], _ptr(fl),
                                      _ptr(it), st))
        leaf_val_d = fl[1][gl]
        if TB == 1 and getattr(self, "_defer_reads", False):
            # boosting stages: nothing read here; the caller keeps the tree's
            # device arrays and reads every stage's depth once, after the loop
            return (fl, it, node_base, next_id, depth_d), (nl, lv_d, leaf_val_d)
        reads = [_Read(leaf_val_d), _Read(depth_d), _Read(lv_d)]
        yield reads[-1]
        leaf_value, tree_depth, lv = (r.get() for r in reads)
        lv = lv.view(TASK_DT).reshape(-1)
        # the trees stay in HBM (predict walks them there); host arrays on demand
        batch = TreeBatch(fl, it, node_base, next_id, tree_depth)
        trees = [Tree(node_count=int(next_id[k]), max_depth=int(tree_depth[k]), batch=batch,
                      start=int(node_base[k])) for k in range(TB)]
        return trees, (lv, lv_d, leaf_value)

    def _grow_host(self, counts, base, m, rows0, rows1, TB):
        import torch

        from .runtime import _ptr, device

        L = _lib()
        dev = device()
        D = self._dev
        n, F = D["n"], D["F"]
        st = torch.cuda.current_stream().cuda_stream
        max_depth = self.max_depth if self.max_depth is not None else 1 << 30

        # nodes get BFS ids per tree (children of one split adjacent); records are
        # kept per level and assembled into exactly-sized arrays at the end
        next_id = np.ones(TB, np.int64)
        tree_depth = np.zeros(TB, np.int32)
        leaves = []    # (tree, node, parity, begin, end) arrays per level
        splits = []    # (tree, node, feat, bin, left id) arrays per level

        # level 0 tasks: one root per tree
        t_tree = np.arange(TB, dtype=np.int32)
        t_node = np.zeros(TB, np.int64)
        t_begin = base.astype(np.int32)
        t_end = (base + m).astype(np.int32)
        t_par = np.zeros(TB, np.int32)
        t_depth = 0
        # a root with < 2 samples or max_depth 0 is a leaf right away
        elig = (t_end - t_begin >= 2) & (t_depth < max_depth)
        if (~elig).any():
            leaves.append((t_tree[~elig], t_node[~elig], t_par[~elig], t_begin[~elig], t_end[~elig]))
        t_tree, t_node, t_begin, t_end, t_par = (a[elig] for a in (t_tree, t_node, t_begin, t_end, t_par))
        cursor = torch.empty(2 * max(len(t_tree), 1), dtype=torch.int32, device=dev)
        while len(t_tree):
            nt = len(t_tree)
            tasks = np.zeros(nt, TASK_DT)
            tasks["tree"], tasks["begin"], tasks["end"], tasks["parity"] = t_tree, t_begin, t_end, t_par
            size = t_end - t_begin
            ids_small = np.nonzero(size <= SMALL)[0].astype(np.int32)
            ids_med = np.nonzero((size > SMALL) & (size <= MEDIUM))[0].astype(np.int32)
            ids_big = np.nonzero(size > MEDIUM)[0].astype(np.int32)
            tasks_d = torch.from_numpy(tasks.view(np.uint8)).to(dev)
            ids_d = {k: torch.from_numpy(v if len(v) else np.zeros(1, np.int32)).to(dev)
                     for k, v in (("s", ids_small), ("m", ids_med), ("b", ids_big))}
            split_d = torch.empty(nt * SPLIT_DT.itemsize, dtype=torch.uint8, device=dev)
            n_big = len(ids_big)
            big_chunks = int(((size[ids_big] + MEDIUM - 1) // MEDIUM).max()) if n_big else 0
            hist = torch.empty(max(int(L.gk_rf_hist_bytes(n_big, F)), 8), dtype=torch.uint8,
                               device=dev)
            _check(L.gk_rf_split_level(
                _ptr(D["Xb"]), _ptr(D["yfp"]), _ptr(D["y"]), _ptr(counts), n, F, _ptr(tasks_d),
                _ptr(ids_d["s"]), len(ids_small), _ptr(ids_d["m"]), len(ids_med), _ptr(ids_d["b"]),
                n_big, big_chunks, _ptr(rows0), _ptr(rows1), _ptr(hist), _ptr(split_d), None, None,
                None, 0, st))
            sp = split_d.cpu().numpy().view(SPLIT_DT)
            s = sp["feat"] >= 0
            # leaves of this level stay where they are
            if (~s).any():
                leaves.append((t_tree[~s], t_node[~s], t_par[~s], t_begin[~s], t_end[~s]))
            if not s.any():
                break
            ids_split = np.nonzero(s)[0].astype(np.int32)
            if len(cursor) < 2 * nt:
                cursor = torch.empty(2 * nt, dtype=torch.int32, device=dev)
            ids_split_d = torch.from_numpy(ids_split).to(dev)
            _check(L.gk_rf_partition(
                _ptr(D["Xb"]), _ptr(D["yfp"]), _ptr(D["y"]), _ptr(counts), n, F, _ptr(tasks_d), nt,
                _ptr(split_d), _ptr(ids_split_d), len(ids_split), int(size[ids_split].max()),
                _ptr(rows0), _ptr(rows1), _ptr(cursor), st))
            # children: adjacent BFS ids per tree, in task order
            pt, pn = t_tree[s], t_node[s]
            rank = np.zeros(len(pt), np.int64)
            if len(pt):
                starts = np.r_[0, np.nonzero(np.diff(pt))[0] + 1]
                run_len = np.diff(np.r_[starts, len(pt)])
                rank = np.arange(len(pt)) - np.repeat(starts, run_len)
            lid = next_id[pt] + 2 * rank
            next_id += 2 * np.bincount(pt, minlength=TB)
            splits.append((pt, pn, sp["feat"][s], sp["bin"][s], lid))
            nl = cursor[: 2 * nt].view(nt, 2)[:, 0].cpu().numpy()[s].astype(np.int32)
            # tasks partitioned inside their split search carry n_left (pad = 1)
            fused = sp["pad"][s] == 1
            nl = np.where(fused, sp["n_left"][s], nl).astype(np.int32)
            cb = np.empty(2 * len(pt), np.int32)
            ce = np.empty(2 * len(pt), np.int32)
            cb[0::2], ce[0::2] = t_begin[s], t_begin[s] + nl
            cb[1::2], ce[1::2] = t_begin[s] + nl, t_end[s]
            ct = np.repeat(pt, 2)
            cn = np.empty(2 * len(pt), np.int64)
            cn[0::2], cn[1::2] = lid, lid + 1
            cpar = np.repeat(1 - t_par[s], 2).astype(np.int32)
            t_depth += 1
            tree_depth[pt] = t_depth
            elig = (ce - cb >= 2) & (t_depth < max_depth)
            if (~elig).any():
                leaves.append((ct[~elig], cn[~elig], cpar[~elig], cb[~elig], ce[~elig]))
            t_tree, t_node, t_begin, t_end, t_par = ct[elig], cn[elig], cb[elig], ce[elig], cpar[elig]

        return self._assemble(counts, rows0, rows1, TB, leaves, splits, next_id, tree_depth)

    def _assemble(self, counts, rows0, rows1, TB, leaves, splits, next_id, tree_depth):
        """sklearn-shaped trees from the level records: leaves = [(tree, node,
        parity, begin, end)], splits = [(tree, node, feat, bin, left id)]."""
        import torch

        from .runtime import _ptr, device

        L = _lib()
        dev = device()
        D = self._dev
        n = D["n"]
        st = torch.cuda.current_stream().cuda_stream
        # leaf statistics (deterministic warp reductions), then bottom-up sums
        lt = np.concatenate([a[0] for a in leaves]).astype(np.int32)
        ln = np.concatenate([a[1] for a in leaves])
        lp = np.concatenate([a[2] for a in leaves]).astype(np.int32)
        lb = np.concatenate([a[3] for a in leaves]).astype(np.int32)
        le = np.concatenate([a[4] for a in leaves]).astype(np.int32)
        lv = np.zeros(len(lt), TASK_DT)
        lv["tree"], lv["begin"], lv["end"], lv["parity"] = lt, lb, le, lp
        lv_d = torch.from_numpy(lv.view(np.uint8)).to(dev)
        stats_d = torch.empty(4 * len(lt), dtype=torch.int64, device=dev)
        _check(L.gk_rf_leaf_stats(_ptr(counts), n, D["F"], _ptr(D["yfp"]), _ptr(D["y2fp"]), _ptr(lv_d),
                                  len(lt), _ptr(rows0), _ptr(rows1), _ptr(stats_d),
                                  int((le - lb).max()) if len(lt) else 0, st))
        # exactly-sized node arrays
        node_base = np.concatenate([[0], np.cumsum(next_id)[:-1]]).astype(np.int64)
        n_nodes_tot = int(next_id.sum())
        feat = np.full(n_nodes_tot, TREE_UNDEFINED, np.int32)
        nbin = np.zeros(n_nodes_tot, np.int32)
        left = np.full(n_nodes_tot, TREE_LEAF, np.int32)
        splits_by_level = []
        for pt, pn, fs, bs, lid in splits:
            gpar = node_base[pt] + pn
            feat[gpar] = fs
            nbin[gpar] = bs
            left[gpar] = lid
            splits_by_level.append((gpar, node_base[pt] + lid))
        # exact integer sums bottom-up, converted to float64 once per node
        istats = np.zeros((n_nodes_tot, 4), np.int64)
        istats[node_base[lt] + ln] = stats_d.cpu().numpy().reshape(-1, 4)
        for gpar, glid in reversed(splits_by_level):
            istats[gpar] = istats[glid] + istats[glid + 1]
        stats = np.empty((n_nodes_tot, 4))
        stats[:, 0] = istats[:, 0]
        stats[:, 1] = istats[:, 1]
        stats[:, 2] = np.ldexp(istats[:, 2].astype(np.float64), -D["shift"])
        stats[:, 3] = np.ldexp(istats[:, 3].astype(np.float64), -D["shift2"])

        trees = []
        for k in range(TB):
            cnt = int(next_id[k])
            g = slice(int(node_base[k]), int(node_base[k]) + cnt)
            f = feat[g].copy()
            cl = left[g].copy()
            is_split = cl >= 0
            cr = np.where(is_split, cl + 1, TREE_LEAF).astype(np.int64)
            thr = np.full(cnt, float(TREE_UNDEFINED))
            thr[is_split] = self._thr[f[is_split], nbin[g][is_split]]
            f = np.where(is_split, f, TREE_UNDEFINED).astype(np.int64)
            st_ = stats[g]
            w = st_[:, 1]
            val = st_[:, 2] / w
            imp = st_[:, 3] / w - val * val
            trees.append(Tree(node_count=cnt, children_left=cl.astype(np.int64), children_right=cr,
                              feature=f, threshold=thr, value=val.reshape(-1, 1, 1), impurity=imp,
                              n_node_samples=st_[:, 0].astype(np.int64), weighted_n_node_samples=w,
                              max_depth=int(tree_depth[k])))
        leaf_value = stats[node_base[lt] + ln, 2] / stats[node_base[lt] + ln, 1]
        return trees, (lv, lv_d, leaf_value)



class RandomForestRegressor(_LevelGrower):
    """GPU-trained random forest with scikit-learn's constructor/fit/predict."""

    _device_input = True   # fit / predict also take device tensors (trainer.train)

    def __init__(self, n_estimators: int = 100, *, max_depth: int | None = None,
                 random_state=None, n_bins: int = N_BINS, trees_per_batch: int | None = None,
                 shard: tuple[int, int] | None = None, concurrent: bool = True,
                 streams: int = 4):
        self.n_estimators = n_estimators
        self.max_depth = max_depth
        self.random_state = random_state
        self.n_bins = check_n_bins(n_bins)
        self.trees_per_batch = trees_per_batch
        self.shard = shard  # (rank, world): build trees t with t % world == rank
        self.concurrent = concurrent  # overlap tree batches (host work vs kernels)
        self.streams = streams        # batches in flight
        self.estimators_: list = []

    # ------------------------------------------------------------------ fit
    def fit(self, X, y, sample_weight=None):
        import torch

        from .runtime import _dev, _ptr, device, upload

        if sample_weight is not None:
            raise NotImplementedError("sample_weight is not supported (training.py never passes it)")
        from .errors import DeviceError

        if is_device_tensor(X):   # trainer.train's folds: no host copies at all
            dev = device()
            X = X.to(dev, torch.float64).contiguous()
            yd = torch.as_tensor(y).to(dev, torch.float64).reshape(-1).contiguous()
        else:
            X = np.ascontiguousarray(X, dtype=np.float64)
            y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
            if X.ndim != 2 or len(y) != len(X):
                raise ValueError("X and y have different lengths")
            try:
                dev = device()
            except DeviceError:
                check_finite(X, y)   # sklearn's input errors first, as on a GPU box
                raise
            # one upload; the input checks and the fixed-point targets run on
            # the device (np.isfinite over config #3's 64M values cost ~0.1 s)
            X = upload(X, dev)   # pinned staging ring (runtime.upload)
            yd = upload(y, dev)
        n, F = X.shape
        if n < 1 or F > 64 * 1024 or n >= 2 ** 31:
            raise ValueError("bad training table shape")
        if len(yd) != n:
            raise ValueError("X and y have different lengths")
        if not bool(torch.isfinite(X).all()):
            raise ValueError("Input X contains NaN or infinity.")
        if not bool(torch.isfinite(yd).all()):
            raise ValueError("Input y contains NaN or infinity.")
        check_n_bins(self.n_bins)
        self.n_features_in_ = F
        Xb = self._prepare_bins(X)
        # fixed-point targets: rint(ldexp(v, shift)) -- ldexp is an exact
        # power-of-two product, torch.round rounds half to even like np.rint
        ymax = float(yd.abs().max())
        shift = int(np.floor(62 - np.log2(max(ymax, 1e-300) * n + 1e-300)))
        shift = max(min(shift, 60), -60)
        yfp = torch.round(yd * (2.0 ** shift)).to(torch.int64)
        y2d = yd * yd
        y2max = float(y2d.max())
        shift2 = int(np.floor(62 - np.log2(max(y2max, 1e-300) * n + 1e-300)))
        shift2 = max(min(shift2, 60), -60)
        y2fp = torch.round(y2d * (2.0 ** shift2)).to(torch.int64)
        self._dev = dict(Xb=Xb, yfp=yfp, y2fp=y2fp, y=yd, n=n, F=F, shift=shift, shift2=shift2)

        seeds = tree_seeds(self.random_state, self.n_estimators)
        todo = list(range(self.n_estimators))
        if self.shard is not None:
            rank, world = self.shard
            todo = [t for t in todo if t % world == rank]
        self.estimators_ = [None] * self.n_estimators
        # trees grown level-wise together: <= 32 at 1M rows, more for small tables
        # (each level costs a few host round trips whatever the batch holds), and
        # at least `streams` batches when there are enough trees (measured on
        # B200 at 1M x 64: 4 batches in flight 18.7 ms/tree, 2: 24 ms/tree)
        tpb = self.trees_per_batch or max(16, min(int(32_000_000 // max(n, 1)),
                                                  -(-len(todo) // max(self.streams, 1))))
        # row-list positions are int32: a batch's bootstrap rows (~0.632 n per
        # tree) must stay below 2^31 (checked exactly after the bootstrap)
        tpb = max(1, min(tpb, int(0.9 * 2 ** 31 / (0.64 * n + 1))))
        batches = [todo[b0: b0 + tpb] for b0 in range(0, len(todo), tpb)]
        # `streams` batches in flight, each on its own stream, driven round-robin
        # from this thread: while one batch's level is read back, the others'
        # kernels run (concurrent=False: one batch at a time, one stream)
        n_str = max(1, min(self.streams, len(batches))) if self.concurrent else 1
        streams = _stream_pool(dev, n_str)
        main = torch.cuda.current_stream(dev)
        for st_ in streams:
            st_.wait_stream(main)
        results = _drive_many([self._grow_batch(seeds[b]) for b in batches], streams)
        for st_ in streams:
            main.wait_stream(st_)
        for batch, trees in zip(batches, results):
            for t, tree in zip(batch, trees):
                self.estimators_[t] = TreeEstimator(tree_=tree, random_state=int(seeds[t]))
        if self.shard is None:
            self._flat = None
        del self._dev, self._dev_thr
        return self

    def _grow_batch(self, seeds):
        """Generator (see _Read): bootstrap + compaction + level-wise growth +
        assembly of one batch of trees on the current stream."""
        import torch

        from .runtime import _ptr, device

        L = _lib()
        dev = device()
        D = self._dev
        n, F = D["n"], D["F"]
        st = torch.cuda.current_stream().cuda_stream
        TB = len(seeds)
        seeds_d = _h2d(seeds.astype(np.uint32), dev)
        counts = torch.empty(TB * n, dtype=torch.int32, device=dev)
        _check(L.gk_rf_bootstrap(_ptr(seeds_d), TB, n, _ptr(counts), st))
        rd = _Read((counts.view(TB, n) > 0).sum(dim=1))
        yield rd
        m = rd.get().astype(np.int64)
        base = np.concatenate([[0], np.cumsum(m)[:-1]]).astype(np.int64)
        total = int(m.sum())
        if total >= 2 ** 31:
            raise ValueError(f"forest: {TB} trees x {n} rows exceed the int32 row lists; "
                             "use a smaller trees_per_batch")
        # one up-front segment for this batch's row lists and level records, freed
        # into this stream's cache so the level loop's allocations split it
        # instead of each mapping fresh memory (cudaMalloc ~1 ms per level buffer)
        # (capped: a reservation only saves allocation calls, it must never be
        # what runs a large fit out of memory)
        try:
            torch.empty(min(total * 56 + (64 << 20), 4 << 30), dtype=torch.uint8, device=dev)
        except torch.OutOfMemoryError:
            pass
        base_d = _h2d(base, dev)
        # two ping-pong buffers of row records (include/gk.h gk_rf_record_bytes)
        rs = int(L.gk_rf_record_bytes(F))
        rows0 = torch.empty(max(total, 1) * rs, dtype=torch.uint8, device=dev)
        rows1 = torch.empty_like(rows0)
        fill = torch.empty(TB, dtype=torch.int32, device=dev)
        _check(L.gk_rf_compact(_ptr(counts), TB, n, _ptr(D["Xb"]), F, _ptr(D["yfp"]), _ptr(base_d),
                               _ptr(rows0), _ptr(fill), st))
        if os.environ.get("GK_RF_HOST_LEVELS", "0") == "1":
            return self._grow_host(counts, base, m, rows0, rows1, TB)[0]
        trees, _ = yield from self._grow_dev(counts, base, m, rows0, rows1, TB)
        return trees

    # -------------------------------------------------------------- predict
    def flat(self, leaf_scale: float = 1.0) -> FlatEnsemble:
        """The forest in the device node layout (leaves scaled by leaf_scale),
        as host arrays."""
        parts, offs, depths, off = [], [], [], 0
        for est in self.estimators_:
            t = est.tree_
            arr = np.zeros(t.node_count, NODE_DT)
            split = t.children_left >= 0
            arr["v"] = np.where(split, t.threshold, t.value[:, 0, 0] * leaf_scale)
            arr["feature"] = np.where(split, t.feature, -1)
            arr["left"] = np.where(split, t.children_left, np.arange(t.node_count) - 1)
            parts.append(arr)
            offs.append(off)
            depths.append(t.max_depth)
            off += t.node_count
        F = self.n_features_in_
        return FlatEnsemble(nodes=np.concatenate(parts).astype(NODE_DT),
                            tree_off=np.asarray(offs, np.int64), scale_lo=np.zeros(F),
                            scale_hi=np.ones(F), base_score=0.0, max_depth=max(depths),
                            manifest=tuple(f"f{i}" for i in range(F)),
                            tree_depth=np.asarray(depths, np.int32))

    def device_ensemble(self, leaf_scale: float = 1.0):
        """The forest as a DeviceEnsemble (16-byte nodes) without a host round
        trip when its trees are device-resident (TreeBatch.device_nodes);
        trees read back to the host go through flat()."""
        import torch

        from .runtime import DeviceEnsemble, _dev

        ests = [e.tree_ for e in self.estimators_]
        if not all(t.on_device for t in ests):
            return DeviceEnsemble.upload(self.flat(leaf_scale), layout="nodes")
        parts, offs, off = [], [], 0
        for t in ests:
            rec = t._batch.device_nodes(leaf_scale)
            parts.append(rec[t._start: t._start + t.node_count])
            offs.append(off)
            off += t.node_count
        nodes = torch.cat(parts).view(torch.uint8).view(-1)
        F = self.n_features_in_
        depths = np.asarray([t.max_depth for t in ests], np.int32)
        bufs = {"nodes": nodes, "off": _dev(np.asarray(offs, np.int64)), "depth": _dev(depths),
                "lo": _dev(np.zeros(F)), "hi": _dev(np.ones(F))}
        return DeviceEnsemble.from_buffers(bufs, base=0.0, n_trees=len(ests), n_feat=F,
                                           max_depth=int(depths.max()))

    def predict(self, X) -> np.ndarray:
        """Mean of the trees' predictions on float32-cast X (sklearn semantics),
        walked on the device."""
        import torch

        from .runtime import device, rf_predict, upload

        if getattr(self, "_flat", None) is None:
            self._flat = self.device_ensemble()
        if is_device_tensor(X):
            Xd = X.to(device(), torch.float64).to(torch.float32).to(torch.float64).contiguous()
        else:
            Xf = np.ascontiguousarray(np.asarray(X, dtype=np.float64).astype(np.float32),
                                      np.float64)
            Xd = upload(Xf, device())
        total, _ = rf_predict(self._flat, Xd)
        return total.cpu().numpy() / len(self.estimators_)
