"""Tree-ensemble documents (host side): load + validate, and flatten to the
16-byte device node layout of ``include/gk.h``.

Loading / validation restates the reference (``pkg/src/gpukalc/power.py:22-125``)
and keeps its error messages.  Flattening renumbers each tree breadth-first so
that every split's children are adjacent (``right == left + 1``) and the top
levels of every tree are contiguous -- the layout the traversal kernel gathers
from.  Leaves keep the reference's values; traversal order and the x <= thr
rule are unchanged (``power.py:156-168``).
"""

from __future__ import annotations

import json
from collections.abc import Mapping
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .errors import EnsembleError

ENSEMBLE_SCHEMA_VERSION = 1
NODE_DT = np.dtype({"names": ["v", "feature", "left"], "formats": ["<f8", "<i4", "<i4"],
                    "offsets": [0, 8, 12], "itemsize": 16})


@dataclass(frozen=True)
class TreeEnsemble:
    """Reference ``power.py:22-33`` (same fields)."""

    base_score: float
    feature_manifest: tuple
    scale_min: tuple
    scale_max: tuple
    trees: tuple
    gains: tuple
    _flat: dict = field(default_factory=dict, compare=False, repr=False)

    @property
    def n_features(self) -> int:
        return len(self.feature_manifest)


def _check_tree(nodes, n_features: int, t: int) -> None:
    """Reference ``power.py:36-70``: field checks, then exactly-once reachability."""
    if not nodes:
        raise EnsembleError(f"tree {t} has no nodes")
    n = len(nodes)
    for i, nd in enumerate(nodes):
        at = f"tree {t} node {i}"
        if "value" in nd:
            if not isinstance(nd["value"], (int, float)):
                raise EnsembleError(f"{at}: leaf value must be a number")
            continue
        for key in ("feature", "threshold", "left", "right"):
            if key not in nd:
                raise EnsembleError(f"{at}: missing '{key}'")
        f = nd["feature"]
        if not isinstance(f, int) or not 0 <= f < n_features:
            raise EnsembleError(f"{at}: feature index {f} out of range")
        for ch in (nd["left"], nd["right"]):
            if not isinstance(ch, int) or not 0 <= ch < n:
                raise EnsembleError(f"{at}: child index {ch} out of range")
    seen = bytearray(n)
    todo = [0]
    while todo:
        i = todo.pop()
        if seen[i]:
            raise EnsembleError(f"tree {t}: node {i} reached twice")
        seen[i] = 1
        nd = nodes[i]
        if "value" not in nd:
            todo.append(nd["left"])
            todo.append(nd["right"])
    if not all(seen):
        raise EnsembleError(f"tree {t}: node {seen.index(0)} unreachable")


def load_ensemble(source) -> TreeEnsemble:
    """JSON path or parsed mapping -> TreeEnsemble (reference ``power.py:73-125``).

    A path goes through the native loader (libgkhost, ``include/gk_ensio.h``:
    parse + validate + breadth-first flatten, trees in parallel) when it is
    built; the returned ensemble then carries its device layout already and
    materialises the reference's node dicts only if ``trees`` is read.
    Documents the native loader declines (any validation error, or constructs
    it does not model) take this Python path, which raises the reference's
    exception with its message."""
    if not isinstance(source, Mapping):
        fast = _load_native(source)
        if fast is not None:
            return fast
    return _load_python(source)


def _load_python(source) -> TreeEnsemble:
    if isinstance(source, Mapping):
        doc = source
    else:
        try:
            doc = json.loads(Path(source).read_text())
        except (OSError, json.JSONDecodeError) as exc:
            raise EnsembleError(f"cannot read ensemble: {exc}") from exc
    if doc.get("schema_version") != ENSEMBLE_SCHEMA_VERSION:
        raise EnsembleError(f"unsupported ensemble schema_version {doc.get('schema_version')!r}, "
                            f"expected {ENSEMBLE_SCHEMA_VERSION}")
    man = doc.get("feature_manifest")
    if not isinstance(man, list) or not man:
        raise EnsembleError("feature_manifest must be a non-empty list")
    if any(not isinstance(m, str) for m in man):
        raise EnsembleError("feature_manifest entries must be strings")
    if len(set(man)) != len(man):
        raise EnsembleError("feature_manifest has duplicate names")
    k = len(man)
    sc = doc.get("scaling")
    if not isinstance(sc, Mapping) or "min" not in sc or "max" not in sc:
        raise EnsembleError("scaling must provide 'min' and 'max' arrays")
    lo, hi = list(sc["min"]), list(sc["max"])
    if len(lo) != k or len(hi) != k:
        raise EnsembleError(f"scaling arrays must have {k} entries to match the manifest")
    for i, (a, b) in enumerate(zip(lo, hi)):
        if b < a:
            raise EnsembleError(f"scaling for '{man[i]}' has max < min")
    trees = doc.get("trees")
    if not isinstance(trees, list):
        raise EnsembleError("trees must be a list")
    for t, tree in enumerate(trees):
        if not isinstance(tree, Mapping) or "nodes" not in tree:
            raise EnsembleError(f"tree {t} must be an object with 'nodes'")
        _check_tree(tree["nodes"], k, t)
    gains = doc.get("gains", [0.0] * k)
    if len(gains) != k:
        raise EnsembleError(f"gains must have {k} entries to match the manifest")
    if any(g < 0 for g in gains):
        raise EnsembleError("gains must be >= 0")
    return TreeEnsemble(base_score=float(doc.get("base_score", 0.0)),
                        feature_manifest=tuple(man), scale_min=tuple(float(v) for v in lo),
                        scale_max=tuple(float(v) for v in hi),
                        trees=tuple(tuple(dict(n) for n in tr["nodes"]) for tr in trees),
                        gains=tuple(float(g) for g in gains))


class _LazyTrees(tuple):
    """The reference's ``trees`` (a tuple of tuples of node dicts, document
    order) materialised from the native loader's arrays on first use."""

    def __new__(cls, arrays):
        obj = super().__new__(cls)
        obj._arrays = arrays
        obj._cache = None
        return obj

    def _get(self):
        if self._cache is None:
            off, feat, val, left, right, kind = self._arrays
            ends = list(off[1:]) + [len(feat)]
            trees = []
            for o, e in zip(off, ends):
                nodes = []
                for i in range(int(o), int(e)):
                    v = val[i]
                    v = int(v) if kind[i] & 2 else float(v)
                    if kind[i] & 1:
                        nodes.append({"value": v})
                    else:
                        nodes.append({"feature": int(feat[i]), "threshold": v,
                                      "left": int(left[i]), "right": int(right[i])})
                trees.append(tuple(nodes))
            self._cache = tuple(trees)
        return self._cache

    def __len__(self):
        return len(self._arrays[0])

    def __iter__(self):
        return iter(self._get())

    def __getitem__(self, i):
        return self._get()[i]

    def __eq__(self, other):
        return tuple(self._get()) == tuple(other)

    def __ne__(self, other):
        return not self == other

    __hash__ = None

    def __repr__(self):
        return f"<{len(self)} trees>"


def _load_native(path):
    """Native parse of an ensemble file; None when the caller must take the
    Python path (library missing, unreadable file, or a declined document)."""
    import ctypes as C

    try:
        from .ptx_native import load_library
        L = load_library()
    except (OSError, RuntimeError):
        return None
    if not getattr(L, "_ens_bound", False):
        vp = C.c_void_p
        L.gk_ens_parse.restype = vp
        L.gk_ens_parse.argtypes = [C.c_char_p, C.c_size_t, C.c_int, vp, C.c_char_p, C.c_size_t]
        L.gk_ens_sizes_of.argtypes = [vp, vp]
        L.gk_ens_copy.restype = C.c_int
        L.gk_ens_copy.argtypes = [vp] * 14
        L.gk_ens_free.argtypes = [vp]
        L._ens_bound = True
    try:
        text = Path(path).read_bytes()
    except OSError:
        return None

    class Sizes(C.Structure):
        _fields_ = [("n_trees", C.c_uint64), ("n_nodes", C.c_uint64), ("n_feat", C.c_uint64),
                    ("manifest_bytes", C.c_uint64), ("max_depth", C.c_uint32),
                    ("pad_", C.c_uint32), ("base_score", C.c_double)]

    status = C.c_int(0)
    why = C.create_string_buffer(128)
    h = L.gk_ens_parse(text, len(text), 0, C.byref(status), why, len(why))
    if not h:
        return None
    try:
        if status.value != 0:
            return None
        sz = Sizes()
        L.gk_ens_sizes_of(h, C.byref(sz))
        nt, nn, k = int(sz.n_trees), int(sz.n_nodes), int(sz.n_feat)
        nodes = np.zeros(max(nn, 1), NODE_DT)
        off = np.zeros(nt, np.int64)
        depth = np.zeros(nt, np.int32)
        lo, hi, gains = np.zeros(k), np.zeros(k), np.zeros(k)
        man = np.zeros(max(int(sz.manifest_bytes), 1), np.uint8)
        man_off = np.zeros(k + 1, np.int64)
        of = np.zeros(nn, np.int32)
        ov = np.zeros(nn)
        ol = np.zeros(nn, np.int32)
        orr = np.zeros(nn, np.int32)
        ok = np.zeros(nn, np.uint8)
        p = [a.ctypes.data for a in (nodes, off, depth, lo, hi, gains, man, man_off, of, ov, ol,
                                     orr, ok)]
        if L.gk_ens_copy(h, *p):
            return None
    finally:
        L.gk_ens_free(h)
    raw = man.tobytes()
    manifest = tuple(raw[man_off[i]:man_off[i + 1]].decode("utf-8") for i in range(k))
    ens = TreeEnsemble(base_score=float(sz.base_score), feature_manifest=manifest,
                       scale_min=tuple(float(v) for v in lo), scale_max=tuple(float(v) for v in hi),
                       trees=_LazyTrees((off, of, ov, ol, orr, ok)),
                       gains=tuple(float(g) for g in gains))
    ens._flat["flat"] = FlatEnsemble(nodes=nodes, tree_off=off, scale_lo=lo.copy(),
                                     scale_hi=hi.copy(), base_score=float(sz.base_score),
                                     max_depth=int(sz.max_depth), manifest=manifest,
                                     tree_depth=depth)
    return ens


@dataclass
class FlatEnsemble:
    """Device layout of one ensemble (host numpy arrays)."""

    nodes: np.ndarray      # NODE_DT; a leaf is {value, -1, own index - 1} (absorbing)
    tree_off: np.ndarray   # int64 [n_trees]
    scale_lo: np.ndarray   # f64 [n_feat]
    scale_hi: np.ndarray
    base_score: float
    max_depth: int
    manifest: tuple
    tree_depth: np.ndarray | None = None   # int32 [n_trees]

    def __post_init__(self):
        if self.tree_depth is None:
            self.tree_depth = np.full(len(self.tree_off), self.max_depth, dtype=np.int32)

    @property
    def n_trees(self) -> int:
        return len(self.tree_off)

    @property
    def n_feat(self) -> int:
        return len(self.scale_lo)


def _flatten_tree(nodes) -> tuple[np.ndarray, int]:
    out = np.zeros(len(nodes), NODE_DT)
    order = [0]           # old ids in new order (BFS, children adjacent)
    depth = [0]
    k = 0
    max_d = 0
    while k < len(order):
        nd = nodes[order[k]]
        if "value" in nd:
            out[k] = (float(nd["value"]), -1, k - 1)   # absorbing leaf: right = self
        else:
            left = len(order)
            order.append(nd["left"])
            order.append(nd["right"])
            depth += [depth[k] + 1, depth[k] + 1]
            max_d = max(max_d, depth[k] + 1)
            out[k] = (float(nd["threshold"]), int(nd["feature"]), left)
        k += 1
    return out, max_d


def flatten(ens: TreeEnsemble) -> FlatEnsemble:
    """TreeEnsemble -> FlatEnsemble (cached on the ensemble object)."""
    cached = ens._flat.get("flat")
    if cached is not None:
        return cached
    parts, offs, depths, off = [], [], [], 0
    for tree in ens.trees:
        arr, d = _flatten_tree(tree)
        parts.append(arr)
        offs.append(off)
        depths.append(d)
        off += len(arr)
    nodes = np.concatenate(parts).astype(NODE_DT) if parts else np.zeros(1, NODE_DT)
    flat = FlatEnsemble(nodes=nodes, tree_off=np.asarray(offs, dtype=np.int64),
                        scale_lo=np.asarray(ens.scale_min, dtype=np.float64),
                        scale_hi=np.asarray(ens.scale_max, dtype=np.float64),
                        base_score=float(ens.base_score), max_depth=max(depths, default=0),
                        manifest=tuple(ens.feature_manifest),
                        tree_depth=np.asarray(depths, dtype=np.int32))
    ens._flat["flat"] = flat
    return flat


def random_forest_flat(n_trees: int, depth: int, manifest, scale_lo, scale_hi, seed: int,
                       split_p: float = 0.985, leaf_scale: float | None = None) -> FlatEnsemble:
    """A declared synthetic ensemble for throughput runs (BASELINE config #4/#5):
    n_trees trees of max depth `depth`, each node below the max depth splitting
    with probability split_p (0.985 at depth 16 gives ~110k nodes/tree, the size
    sklearn grows at 1M rows x depth 16 -- SURVEY §7.3.4).  Thresholds are uniform
    in scaled space; leaves are RF-style (mean value / n_trees)."""
    rng = np.random.default_rng(seed)
    nf = len(manifest)
    scale = (1.0 / n_trees) if leaf_scale is None else leaf_scale
    parts, offs, depths, off = [], [], [], 0
    for _ in range(n_trees):
        level_n = 1
        levels = []
        for d in range(depth + 1):
            split = rng.random(level_n) < (split_p if d > 0 else 1.0)
            if d == depth:
                split[:] = False
            levels.append(split)
            level_n = int(split.sum()) * 2
            if level_n == 0:
                break
        n_nodes = sum(len(s) for s in levels)
        arr = np.zeros(n_nodes, NODE_DT)
        base = 0
        for d, split in enumerate(levels):
            cnt = len(split)
            nxt = base + cnt
            idx = np.arange(base, base + cnt)
            sp = idx[split]
            arr["feature"][sp] = rng.integers(0, nf, len(sp))
            arr["v"][sp] = rng.random(len(sp))
            arr["left"][sp] = nxt + 2 * np.arange(len(sp))
            lf = idx[~split]
            arr["feature"][lf] = -1
            arr["left"][lf] = lf - 1                  # absorbing leaf: right = self
            arr["v"][lf] = (30.0 + 120.0 * rng.random(len(lf))) * scale
            base = nxt
        parts.append(arr)
        offs.append(off)
        depths.append(len(levels) - 1)
        off += n_nodes
    return FlatEnsemble(nodes=np.concatenate(parts).astype(NODE_DT),
                        tree_off=np.asarray(offs, dtype=np.int64),
                        scale_lo=np.asarray(scale_lo, dtype=np.float64),
                        scale_hi=np.asarray(scale_hi, dtype=np.float64), base_score=0.0,
                        max_depth=max(depths), manifest=tuple(manifest),
                        tree_depth=np.asarray(depths, dtype=np.int32))


BLOCK2_DT = np.dtype([("t", "<u4", (3,)), ("f", "<u4"), ("e", "<u4", (4,))])
GK_LEAF = 0x80000000
BLOCK2_MAX_FEAT = 255


def f32_round_down(v: np.ndarray) -> np.ndarray:
    """Largest float32 <= v, elementwise (NaN stays NaN; v > FLT_MAX -> FLT_MAX)."""
    v = np.asarray(v, dtype=np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        f = v.astype(np.float32)
        up = f.astype(np.float64) > v
    f[up] = np.nextafter(f[up], np.float32(-np.inf))
    return f


NODE8_DT = np.dtype([("t", "<u4"), ("meta", "<u4")])
NODE8_MAX_FEAT = 127          # feature index lives in the signed top byte (0xFF = leaf)
NODE8_MAX_RIGHT = (1 << 24) - 1


def nodes8(flat: FlatEnsemble) -> np.ndarray | None:
    """gk_node8 form of `flat` (same index space), or None when the ensemble does
    not fit it (>127 features, >16M nodes per tree).  Splits:
    {round-down-f32(threshold), feature << 24 | left + 1}; leaves {0, 0xFF << 24 | self}."""
    nd = flat.nodes
    if flat.n_feat > NODE8_MAX_FEAT or len(nd) == 0:
        return None
    leaf = nd["feature"] < 0
    right = nd["left"].astype(np.int64) + 1          # leaf: left = self - 1 -> right = self
    if (right < 0).any() or (right > NODE8_MAX_RIGHT).any():
        return None
    out = np.zeros(len(nd), NODE8_DT)
    out["t"][~leaf] = f32_round_down(nd["v"][~leaf]).view(np.uint32)
    feat = np.where(leaf, 0xFF, nd["feature"]).astype(np.uint32)
    out["meta"] = (feat << 24) | right.astype(np.uint32)
    return out


@dataclass
class Blocked:
    """Two-level blocked walk form of a FlatEnsemble (gk_block2, include/gk.h)."""

    blocks: np.ndarray     # BLOCK2_DT [n_blocks]
    thr64: np.ndarray      # f64 [3 * n_blocks]
    leaf_val: np.ndarray   # f64 [n_leaves]
    root: np.ndarray       # u32 [n_trees]


def blocked(flat: FlatEnsemble) -> Blocked | None:
    """Depth-2 blocks of every tree (vectorised over all nodes): a block per
    internal node at even depth holding it and its two children; exits are the
    grandchildren (a block id, or GK_LEAF | leaf id).  None if the ensemble does
    not fit the format (>255 features, >= 2^31 blocks or leaves)."""
    nd = flat.nodes
    N = len(nd)
    if flat.n_feat > BLOCK2_MAX_FEAT or N == 0 or flat.n_trees == 0:
        return None
    sizes = np.diff(np.append(flat.tree_off, N))
    base = np.repeat(flat.tree_off, sizes)
    leaf = nd["feature"] < 0
    left = np.where(leaf, 0, base + nd["left"].astype(np.int64))
    depth = np.full(N, -1, np.int64)
    frontier = flat.tree_off.astype(np.int64)
    d = 0
    while len(frontier):
        depth[frontier] = d
        inner = frontier[~leaf[frontier]]
        frontier = np.concatenate([left[inner], left[inner] + 1])
        d += 1
    is_blk = ~leaf & (depth % 2 == 0)
    blk_id = np.cumsum(is_blk) - 1
    leaf_id = np.cumsum(leaf) - 1
    if is_blk.sum() >= GK_LEAF or leaf.sum() >= GK_LEAF:
        return None

    def ref(nodes):
        return np.where(leaf[nodes], GK_LEAF | leaf_id[nodes], blk_id[nodes]).astype(np.uint32)

    r = np.flatnonzero(is_blk)
    slots = np.stack([r, left[r], left[r] + 1], axis=1)            # [nb, 3]
    inner = ~leaf[slots]
    out = np.zeros(len(r), BLOCK2_DT)
    thr = np.where(inner, nd["v"][slots], 0.0)
    out["t"] = np.where(inner, f32_round_down(thr).view(np.uint32), 0)
    feat = np.where(inner, nd["feature"][slots], 0).astype(np.uint32)
    out["f"] = feat[:, 0] | (feat[:, 1] << 8) | (feat[:, 2] << 16)
    for k in (1, 2):
        s_k = slots[:, k]
        c = left[s_k]
        lf = leaf[s_k]
        own = ref(s_k)
        out["e"][:, 2 * (k - 1)] = np.where(lf, own, ref(np.where(lf, s_k, c)))
        out["e"][:, 2 * (k - 1) + 1] = np.where(lf, own, ref(np.where(lf, s_k, c + 1)))
    if len(r) == 0:  # all trees are single leaves: keep block 0 (the walk's sink) addressable
        out, thr = np.zeros(1, BLOCK2_DT), np.zeros((1, 3))
    return Blocked(blocks=out, thr64=np.ascontiguousarray(thr.reshape(-1)),
                   leaf_val=np.ascontiguousarray(nd["v"][leaf]),
                   root=ref(flat.tree_off.astype(np.int64)))


# ---------------------------------------------------------------- gk_block3
# Three-level blocks with 16-bit keys (include/gk.h gk_block3): one 32-byte load
# per three levels, the last split level's leaves inline ("terminal" blocks),
# so a depth-16 path costs 6 scattered 32-byte loads instead of the 2-level
# blocks' 8 + a leaf-value load (the walks are bound by one distinct L1 line per
# lane per load, tools/ubench/gather.cu).
BLOCK3_DT = np.dtype([("w", "<u4", (8,))])
B3_TERMINAL = 1
BLOCK3_MAX_FEAT = 255


def key16(v: np.ndarray) -> np.ndarray:
    """16-bit order key of round-down-f32(v): the top half of the f32's
    order-preserving bits, -0.0 taken as +0.0, NaN -> 0xFFFF (above +inf).
    a = key16(x) vs t = key16(thr): a < t -> x < thr, a > t -> x > thr (or x
    NaN), a == t -> the exact fp64 test decides (gk_block3 walk)."""
    f = f32_round_down(np.asarray(v, dtype=np.float64))
    f = np.where(f == 0, np.float32(0.0), f).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    o = np.where(u & 0x80000000, ~u & 0xFFFFFFFF, u | 0x80000000) >> 16
    return np.where(np.isnan(f), 0xFFFF, o).astype(np.uint16)


@dataclass
class Blocked3:
    """Three-level blocked walk form of a FlatEnsemble (gk_block3, include/gk.h)."""

    blocks: np.ndarray     # BLOCK3_DT [n_blocks]
    thr64: np.ndarray      # f64 [7 * n_blocks]
    leaf_val: np.ndarray   # f64 [n_leaf_slots]
    root: np.ndarray       # u32 [n_trees]: block id, or GK_LEAF | leaf id


def blocked3(flat: FlatEnsemble) -> Blocked3 | None:
    """gk_block3 form of `flat`: a block per internal node at depth 0, 3, 6, ...
    A node whose two children are leaves becomes a terminal block {key,
    feature, both leaf values}; any other holds its 3-level subtree (7 nodes;
    a leaf above the third level is padded: its subtree's nodes route
    anywhere and all of its slots name that leaf) and 8 exit slots, each a
    child block (contiguous from block_base in slot order) or a leaf
    (contiguous from leaf_base).  Blocks are numbered level by level in (parent,
    slot) order.  None if the ensemble does not fit (> 255 features, >= 2^31
    blocks or leaf slots)."""
    nd = flat.nodes
    N = len(nd)
    if flat.n_feat > BLOCK3_MAX_FEAT or N == 0 or flat.n_trees == 0:
        return None
    sizes = np.diff(np.append(flat.tree_off, N))
    base = np.repeat(flat.tree_off, sizes)
    leaf = nd["feature"] < 0
    left = np.where(leaf, 0, base + nd["left"].astype(np.int64))
    # height (0 for leaves): children follow their parent in a tree's BFS order
    depth = np.full(N, -1, np.int64)
    frontier = flat.tree_off.astype(np.int64)
    levels = []
    d = 0
    while len(frontier):
        depth[frontier] = d
        levels.append(frontier)
        inner = frontier[~leaf[frontier]]
        frontier = np.concatenate([left[inner], left[inner] + 1])
        d += 1
    height = np.zeros(N, np.int64)
    for fr in reversed(levels):
        inner = fr[~leaf[fr]]
        height[inner] = 1 + np.maximum(height[left[inner]], height[left[inner] + 1])
    # a NaN threshold (x <= NaN is always false) takes key 0, below every
    # row's key (-inf is 0x007F, a NaN row 0xFFFF): always right, never a tie
    K = np.where(np.isnan(nd["v"]), 0, key16(nd["v"])).astype(np.uint32)
    F = np.where(leaf, 0, nd["feature"]).astype(np.uint32)
    THR = np.where(leaf, np.inf, nd["v"])

    blocks, thr64, leaf_vals = [], [], []
    n_blocks = 0
    n_leaves = 0
    root = np.zeros(flat.n_trees, np.uint32)
    roots = flat.tree_off.astype(np.int64)
    rl = leaf[roots]
    # single-leaf trees: their leaf slots first
    root[rl] = GK_LEAF | (np.arange(int(rl.sum()), dtype=np.uint32))
    leaf_vals.append(nd["v"][roots[rl]])
    n_leaves += int(rl.sum())
    cur = roots[~rl]                                       # this level's block roots, id order
    root[~rl] = np.arange(len(cur), dtype=np.uint32)
    while len(cur):
        nb = len(cur)
        w = np.zeros((nb, 8), np.uint32)
        t64 = np.full((nb, 7), np.inf)
        term = height[cur] == 1
        # terminal blocks: key and feature where a 3-level block keeps node 0's
        # (halfword 0, byte 14), the left / right leaf values in w[1..2] / w[6..7]
        tc = cur[term]
        w[term, 0] = K[tc]
        w[term, 3] = F[tc] << 16
        lv = nd["v"][left[tc]].view(np.uint64)
        rv = nd["v"][left[tc] + 1].view(np.uint64)
        w[term, 1], w[term, 2] = (lv & 0xFFFFFFFF).astype(np.uint32), (lv >> 32).astype(np.uint32)
        w[term, 6], w[term, 7] = (rv & 0xFFFFFFFF).astype(np.uint32), (rv >> 32).astype(np.uint32)
        w[term, 5] = B3_TERMINAL << 16
        t64[term, 0] = THR[tc]
        # three-level blocks
        full = ~term
        r = cur[full]
        n = np.empty((len(r), 7), np.int64)
        n[:, 0] = r
        n[:, 1], n[:, 2] = left[r], left[r] + 1
        for k in (1, 2):                                  # block-depth 2 (padded under leaves)
            c = n[:, k]
            lf = leaf[c]
            n[:, 3 + 2 * (k - 1)] = np.where(lf, c, left[c])
            n[:, 4 + 2 * (k - 1)] = np.where(lf, c, left[c] + 1)
        slots = np.empty((len(r), 8), np.int64)
        for j in range(4):
            c = n[:, 3 + j]
            lf = leaf[c]
            slots[:, 2 * j] = np.where(lf, c, left[c])
            slots[:, 2 * j + 1] = np.where(lf, c, left[c] + 1)
        kk = np.where(leaf[n], 0xFFFF, K[n])              # padded / leaf entries never decide
        ff = np.where(leaf[n], 0, F[n])
        t64[full] = np.where(leaf[n], np.inf, THR[n])
        wf = np.zeros((len(r), 8), np.uint32)
        wf[:, 0] = kk[:, 0] | (kk[:, 1] << 16)
        wf[:, 1] = kk[:, 2] | (kk[:, 3] << 16)
        wf[:, 2] = kk[:, 4] | (kk[:, 5] << 16)
        wf[:, 3] = kk[:, 6] | (ff[:, 0] << 16) | (ff[:, 1] << 24)
        wf[:, 4] = ff[:, 2] | (ff[:, 3] << 8) | (ff[:, 4] << 16) | (ff[:, 5] << 24)
        sl = leaf[slots]                                  # [nb_full, 8]
        mask = (sl.astype(np.uint32) << np.arange(8, dtype=np.uint32)).sum(axis=1).astype(np.uint32)
        wf[:, 5] = ff[:, 6] | (mask << 8)
        n_child = (~sl).sum(axis=1)
        n_lf = sl.sum(axis=1)
        wf[:, 6] = (n_blocks + nb + np.concatenate([[0], np.cumsum(n_child)[:-1]])).astype(np.uint32)
        wf[:, 7] = (n_leaves + np.concatenate([[0], np.cumsum(n_lf)[:-1]])).astype(np.uint32)
        w[full] = wf
        blocks.append(w)
        thr64.append(t64)
        leaf_vals.append(nd["v"][slots[sl]])             # (parent, slot) order
        n_leaves += int(n_lf.sum())
        n_blocks += nb
        cur = slots[~sl]                                  # next level's roots, (parent, slot) order
        if n_blocks + len(cur) >= GK_LEAF or n_leaves >= GK_LEAF >> 1:
            return None
    out = np.zeros(max(n_blocks, 1), BLOCK3_DT)
    if n_blocks:
        out["w"] = np.concatenate(blocks)
        t = np.concatenate(thr64).reshape(-1)
    else:   # all trees are single leaves: keep block 0 addressable
        t = np.full(7, np.inf)
    return Blocked3(blocks=out, thr64=np.ascontiguousarray(t),
                    leaf_val=np.ascontiguousarray(np.concatenate(leaf_vals) if leaf_vals
                                                  else np.zeros(1)),
                    root=root)


def flat_to_document(flat: FlatEnsemble) -> dict:
    """FlatEnsemble -> reference JSON document (for cross-checks on small ensembles)."""
    trees = []
    ends = list(flat.tree_off[1:]) + [len(flat.nodes)]
    for o, e in zip(flat.tree_off, ends):
        nodes = []
        for nd in flat.nodes[o:e]:
            if nd["feature"] < 0:
                nodes.append({"value": float(nd["v"])})
            else:
                nodes.append({"feature": int(nd["feature"]), "threshold": float(nd["v"]),
                              "left": int(nd["left"]), "right": int(nd["left"]) + 1})
        trees.append({"nodes": nodes})
    return {"schema_version": 1, "base_score": flat.base_score,
            "feature_manifest": list(flat.manifest),
            "scaling": {"min": [float(v) for v in flat.scale_lo],
                        "max": [float(v) for v in flat.scale_hi]},
            "trees": trees, "gains": [0.0] * len(flat.manifest)}


# ---------------------------------------------------------------- native writer


def _writer():
    import ctypes as C

    from .ptx_native import load_library

    L = load_library()
    if not getattr(L, "_ensw_bound", False):
        vp = C.c_void_p
        L.gk_ens_write.restype = C.c_int
        L.gk_ens_write.argtypes = [C.c_int64, C.c_double, vp, vp, C.c_uint64, vp, vp, vp,
                                   C.c_uint64, vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, vp, vp]
        L.gk_ens_float_repr.restype = C.c_int
        L.gk_ens_float_repr.argtypes = [vp, C.c_uint64, vp, vp]
        L.gk_ens_buf_free.argtypes = [vp]
        L._ensw_bound = True
    return L


def _take(L, fn, *args) -> bytes:
    import ctypes as C

    out, n = C.c_void_p(), C.c_size_t()
    if fn(*args, C.byref(out), C.byref(n)):
        raise MemoryError("gk_ens_write: allocation failed")
    try:
        return C.string_at(out.value, n.value)
    finally:
        L.gk_ens_buf_free(out)


def float_reprs(x) -> list:
    """CPython repr() of each double, computed by the native writer (test hook)."""
    L = _writer()
    x = np.ascontiguousarray(x, dtype=np.float64)
    if len(x) == 0:
        return []
    return _take(L, L.gk_ens_float_repr, x.ctypes.data, len(x)).decode().split(" ")


def document_text(*, base_score: float, manifest, scale_lo, scale_hi, gains, trees,
                  schema_version: int = ENSEMBLE_SCHEMA_VERSION, indent: int | None = 2) -> str:
    """``json.dumps(doc, indent=indent)`` of an ensemble document, formatted
    natively (libgkhost ``gk_ens_write``) and byte-identical to CPython's json.
    `trees`: per tree a dict of document-order arrays ``is_leaf``, ``feature``,
    ``value`` (leaf value or threshold), ``left``, ``right`` (what
    ``export._tree_nodes`` reads from sklearn's tree arrays)."""
    L = _writer()
    enc = [m.encode("utf-8") for m in manifest]
    blob = b"".join(enc) or b"\0"
    moff = np.zeros(len(enc) + 1, np.int64)
    moff[1:] = np.cumsum([len(e) for e in enc]) if enc else []
    sizes = [len(t["is_leaf"]) for t in trees]
    noff = np.zeros(len(trees) + 1, np.int64)
    noff[1:] = np.cumsum(sizes) if sizes else []

    def cat(key, dt):
        if not trees:
            return np.zeros(1, dt)
        return np.ascontiguousarray(np.concatenate([np.asarray(t[key]) for t in trees]).astype(dt))

    leaf, feat, val = cat("is_leaf", np.uint8), cat("feature", np.int32), cat("value", np.float64)
    left, right = cat("left", np.int32), cat("right", np.int32)
    lo, hi, g = (np.ascontiguousarray(a, dtype=np.float64) for a in (scale_lo, scale_hi, gains))
    if not (len(lo) == len(hi) == len(g) == len(enc)):
        raise ValueError("manifest, scaling and gains must have the same length")
    p = [a.ctypes.data for a in (moff, lo, hi, g, noff, leaf, feat, val, left, right)]
    text = _take(L, L.gk_ens_write, int(schema_version), float(base_score), blob, p[0], len(enc),
                 p[1], p[2], p[3], len(trees), p[4], p[5], p[6], p[7], p[8], p[9],
                 -1 if indent is None else int(indent), 0)
    return text.decode("ascii")
