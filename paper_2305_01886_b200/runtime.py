"""Device runtime: loads ``libgk.so`` (sm_100a) and drives its C-ABI with
torch-owned device buffers.

PyTorch is plumbing here -- device memory, streams, host<->device copies.  All
arithmetic of the hot path runs inside libgk's kernels.  There is no CPU
fallback: if the library or a CUDA device is missing, every entry point raises
:class:`DeviceError`.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import abi
from .errors import DeviceError
from .pack import KSTAT_DT, Corpus, arch_records, config_array, latency_table

LIB_PATH = Path(__file__).resolve().parent / "libgk.so"
EXPORTS = ("gk_abi_version", "gk_last_error", "gk_device_sm_count", "gk_static_features",
           "gk_schedule_features", "gk_rf_predict", "gk_sweep_workspace_bytes",
           "gk_predict_energy_sweep", "gk_set_stage_timing", "gk_get_stage_ms")
_lib = None


def load_library(path: Path | None = None):
    """ctypes handle of libgk with argtypes set.  Does not touch the GPU."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path or LIB_PATH)
    if not p.exists():
        raise DeviceError(f"{p} is missing: build it with `python -m paper_2305_01886_b200.build` "
                          "(there is no CPU fallback)")
    try:
        L = C.CDLL(str(p))
    except OSError as exc:
        raise DeviceError(f"cannot load {p}: {exc}") from exc
    vp, u32, i64 = C.c_void_p, C.c_uint32, C.c_int64
    L.gk_abi_version.restype = C.c_int
    L.gk_last_error.restype = C.c_char_p
    L.gk_device_sm_count.restype = C.c_int
    L.gk_static_features.argtypes = [vp, vp, vp, vp, vp]
    L.gk_schedule_features.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, u32, vp, vp, vp]
    L.gk_rf_predict.argtypes = [vp, vp, i64, i64, vp, vp, vp, vp, vp]
    L.gk_sweep_workspace_bytes.argtypes = [vp, vp, u32]
    L.gk_sweep_workspace_bytes.restype = C.c_size_t
    L.gk_predict_energy_sweep.argtypes = [vp, vp, vp, vp, u32, vp, vp, vp, vp, vp, vp]
    L.gk_set_stage_timing.argtypes = [C.c_int]
    L.gk_get_stage_ms.argtypes = [vp]
    if L.gk_abi_version() != 5:
        raise DeviceError("libgk ABI version mismatch")
    if path is None:
        _lib = L
    return L


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the sm_100a path has no CPU fallback")
    return torch


def device():
    return _torch().device("cuda", _torch().cuda.current_device())


def _check(rc: int) -> None:
    if rc != 0:
        raise DeviceError(load_library().gk_last_error().decode() or f"libgk error {rc}")


def _stream(stream=None) -> int:
    t = _torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return s.cuda_stream


def _dev(a: np.ndarray, dev=None):
    """numpy -> device tensor of raw bytes (structured dtypes go as uint8).
    Large arrays go through the pinned staging ring (upload())."""
    t = _torch()
    a = np.ascontiguousarray(a)
    if a.nbytes >= _STAGE_MIN:
        return upload(a.view(np.uint8).reshape(-1) if a.dtype.fields else a, dev)
    if not a.flags.writeable:      # torch.from_numpy wants a writable buffer
        a = a.copy()
    host = t.from_numpy(a.view(np.uint8).reshape(-1) if a.dtype.fields else a)
    return host.to(dev or device(), non_blocking=False)


_STAGE_CHUNK = 8 << 20     # bytes per pinned staging buffer
_STAGE_N = 4               # buffers in the ring
_STAGE_MIN = 4 * _STAGE_CHUNK
_stage = {"bufs": None, "events": None}
_stage_lock = threading.Lock()


def upload(a: np.ndarray, dev=None):
    """Pageable host array -> new device tensor, staged through a ring of
    pinned buffers: torch's multi-threaded CPU copy fills one buffer while
    the DMA of the previous ones runs (B200 box, 512 MB fp64 table: 10 ms /
    52 GB/s vs 46 ms / 11 GB/s for a pageable .to(), tools/upload_probe.py).
    The copies run on the current stream; the result is ready for work
    queued after them."""
    import warnings

    import torch as t   # (not _torch(): a gloo group's CPU device needs no GPU)

    a = np.ascontiguousarray(a)
    dev = dev if dev is not None else device()
    with warnings.catch_warnings():   # read-only arrays: only read here
        warnings.simplefilter("ignore", UserWarning)
        src = t.from_numpy(a)
    if t.device(dev).type != "cuda":   # e.g. a gloo group's CPU tensors
        return src.to(dev, copy=True)
    if a.nbytes < _STAGE_MIN:
        return src.to(dev)
    flat = src.reshape(-1).view(t.uint8)
    out = t.empty(a.nbytes, dtype=t.uint8, device=dev)
    st = t.cuda.current_stream(dev)
    with _stage_lock:
        if _stage["bufs"] is None:
            _stage["bufs"] = [t.empty(_STAGE_CHUNK, dtype=t.uint8, pin_memory=True)
                              for _ in range(_STAGE_N)]
            _stage["events"] = [None] * _STAGE_N
        bufs, evs = _stage["bufs"], _stage["events"]
        for i, o in enumerate(range(0, a.nbytes, _STAGE_CHUNK)):
            k = i % _STAGE_N
            if evs[k] is not None:
                evs[k].synchronize()          # the buffer's previous DMA is done
            c = min(_STAGE_CHUNK, a.nbytes - o)
            bufs[k][:c].copy_(flat[o:o + c])
            out[o:o + c].copy_(bufs[k][:c], non_blocking=True)
            evs[k] = t.cuda.Event()
            evs[k].record(st)
    return out.view(src.dtype).view(src.shape)


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


@dataclass
class DeviceCorpus:
    """A packed corpus resident in HBM."""

    corpus: Corpus
    bufs: dict = field(default_factory=dict)
    desc: abi.GkCorpus | None = None

    @classmethod
    def upload(cls, corpus: Corpus) -> "DeviceCorpus":
        dc = cls(corpus.check())
        for k in ("tok", "preds", "blk", "fpreds", "topo", "ker"):
            arr = getattr(corpus, k)
            if len(arr) == 0:
                arr = np.zeros(1, arr.dtype)
            dc.bufs[k] = _dev(arr)
        b = dc.bufs
        dc.desc = abi.GkCorpus(_ptr(b["tok"]), _ptr(b["preds"]), _ptr(b["blk"]), _ptr(b["fpreds"]),
                               _ptr(b["topo"]), _ptr(b["ker"]), corpus.n_tok, len(corpus.blk),
                               corpus.n_ker, max(len(corpus.sigs), 1), corpus.max_n,
                               corpus.max_blk)
        return dc

    @property
    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.bufs.values())


@dataclass
class DeviceGrid:
    """kernels x archs x configs, resident in HBM."""

    n_k: int
    n_arch: int
    n_cfg: int
    bufs: dict = field(default_factory=dict)
    desc: abi.GkGrid | None = None

    @classmethod
    def build(cls, dcorpus: DeviceCorpus, profiles, configs, kernel_ids=None, n_tw=None,
              gm=None) -> "DeviceGrid":
        """n_tw / gm: optional per-config overrides (schedule_block/_cfg faces)."""
        corpus = dcorpus.corpus
        kid = (np.arange(corpus.n_ker, dtype=np.uint32) if kernel_ids is None
               else np.asarray(kernel_ids, dtype=np.uint32))
        if len(kid) and int(kid.max()) >= corpus.n_ker:
            raise ValueError("kernel id out of range")
        cfg = config_array(configs)
        arch = arch_records(profiles)
        lat = np.ascontiguousarray(latency_table(profiles, corpus.sigs))
        g = cls(len(kid), len(arch), len(cfg))
        g.bufs = {"kid": _dev(kid if len(kid) else np.zeros(1, np.uint32)), "cfg": _dev(cfg),
                  "arch": _dev(arch), "lat": _dev(lat),
                  # this grid's mem_throughput clamp counter (gk_grid.tp_clamps)
                  "clamps": _dev(np.zeros(1, np.int64))}
        if n_tw is not None:
            g.bufs["n_tw"] = _dev(np.asarray(n_tw, dtype=np.int64))
        if gm is not None:
            g.bufs["gm"] = _dev(np.asarray(gm, dtype=np.float64))
        if len(kid) > 1:
            # largest-first processing order for the device work queue: a
            # kernel's scheduling cost grows with sum over blocks of n^2
            blk = corpus.blk
            n = blk["n"].astype(np.int64)
            per_block = n * n + n
            cost_all = np.add.reduceat(per_block, corpus.ker["blk0"].astype(np.int64)) \
                if len(blk) else np.zeros(corpus.n_ker, np.int64)
            cost_all = np.where(corpus.ker["n_blk"] > 0, cost_all, 0)
            order = np.argsort(-cost_all[kid], kind="stable").astype(np.uint32)
            g.bufs["order"] = _dev(order)
        g.desc = abi.GkGrid(_ptr(g.bufs["kid"]), _ptr(g.bufs["cfg"]), _ptr(g.bufs["arch"]),
                            _ptr(g.bufs["lat"]), _ptr(g.bufs.get("n_tw")),
                            _ptr(g.bufs.get("gm")), _ptr(g.bufs.get("order")),
                            _ptr(g.bufs["clamps"]), len(kid),
                            len(cfg), len(arch), 0)
        return g

    @property
    def n_points(self) -> int:
        return self.n_k * self.n_arch * self.n_cfg


@dataclass
class DeviceEnsemble:
    flat: object
    bufs: dict = field(default_factory=dict)
    desc: abi.GkEnsemble | None = None

    LAYOUTS = ("nodes", "nodes8", "blocks", "blocks3")

    @classmethod
    def upload(cls, flat, layout: str | None = None) -> "DeviceEnsemble":
        """Copy a FlatEnsemble to the device in walk layout `layout`:
        "nodes" (16-byte gk_node only), "nodes8" (+ gk_node8: 8-byte nodes) or
        "blocks" (+ gk_block2: one 256-bit load per two levels).  Measured on
        B200: K4 (gk_rf_predict) is fastest on blocks (1.43x on config #4's
        random rows, which are L2/DRAM-latency bound; 7 % on the sweep's rows);
        the fused sweep walks the 16-byte nodes unless GK_FUSED_COMPACT=1.
        Default: $GK_WALK_LAYOUT or "blocks".  A layout the ensemble does not
        fit falls back to "nodes"; the 16-byte nodes stay resident in every
        layout (leaf values, exact tie thresholds)."""
        import os

        from .ensemble import blocked, blocked3, nodes8

        layout = layout or os.environ.get("GK_WALK_LAYOUT", "blocks")
        if layout not in cls.LAYOUTS:
            raise ValueError(f"walk layout must be one of {cls.LAYOUTS}, got {layout!r}")
        de = cls(flat)
        de.bufs = {"nodes": _dev(flat.nodes),
                   "off": _dev(flat.tree_off if flat.n_trees else np.zeros(1, np.int64)),
                   "depth": _dev(flat.tree_depth if flat.n_trees else np.zeros(1, np.int32)),
                   "lo": _dev(flat.scale_lo), "hi": _dev(flat.scale_hi)}
        if layout == "nodes8":
            n8 = nodes8(flat)
            if n8 is not None:
                de.bufs["nodes8"] = _dev(n8)
        elif layout == "blocks":
            bl = blocked(flat)
            if bl is not None:
                de.bufs.update(blocks=_dev(bl.blocks), thr64=_dev(bl.thr64),
                               leaf_val=_dev(bl.leaf_val), root=_dev(bl.root))
        elif layout == "blocks3":
            b3 = blocked3(flat)
            if b3 is not None:
                de.bufs.update(blocks3=_dev(b3.blocks), thr64=_dev(b3.thr64),
                               leaf_val=_dev(b3.leaf_val), root=_dev(b3.root))
        de.desc = cls._desc(de.bufs, float(flat.base_score), flat.n_trees, flat.n_feat,
                            flat.max_depth)
        return de

    @staticmethod
    def _desc(b: dict, base: float, n_trees: int, n_feat: int, max_depth: int):
        return abi.GkEnsemble(_ptr(b["nodes"]), _ptr(b["off"]), _ptr(b["depth"]),
                              _ptr(b["lo"]), _ptr(b["hi"]), float(base), int(n_trees),
                              int(n_feat), int(max_depth), _ptr(b.get("nodes8")),
                              _ptr(b.get("blocks")), _ptr(b.get("thr64")),
                              _ptr(b.get("leaf_val")), _ptr(b.get("root")),
                              _ptr(b.get("blocks3")))

    @classmethod
    def from_buffers(cls, bufs: dict, *, base: float, n_trees: int, n_feat: int,
                     max_depth: int) -> "DeviceEnsemble":
        """An ensemble over device buffers that are already in walk layout
        (e.g. received by dist.broadcast_device_ensemble)."""
        de = cls(None)
        de.bufs = dict(bufs)
        de.desc = cls._desc(de.bufs, base, n_trees, n_feat, max_depth)
        return de

    @property
    def layout(self) -> str:
        for name in ("blocks3", "blocks", "nodes8"):
            if name in self.bufs:
                return name
        return "nodes"


# ------------------------------------------------------------------ calls


def static_features(dc: DeviceCorpus, dg: DeviceGrid, stream=None):
    t = _torch()
    dev = device()
    ks = t.empty(dg.n_k * KSTAT_DT.itemsize, dtype=t.uint8, device=dev)
    ls = t.empty((dg.n_arch, dg.n_k, 3), dtype=t.float64, device=dev)
    _check(load_library().gk_static_features(C.byref(dc.desc), C.byref(dg.desc), _ptr(ks),
                                             _ptr(ls), _stream(stream)))
    return ks, ls


def schedule_features(dc: DeviceCorpus, dg: DeviceGrid, *, si=True, sf=True, feat=True,
                      sel_idx=None, trace=False, stream=None) -> dict:
    """K1 + K2/K3 over a grid; returns device tensors keyed like the oracle."""
    t = _torch()
    dev = device()
    n = dg.n_points
    ks, ls = static_features(dc, dg, stream)
    out = {"status": t.empty(n, dtype=t.uint8, device=dev)}
    if si:
        out["si"] = t.empty((n, abi.NSI), dtype=t.int64, device=dev)
    if sf:
        out["sf"] = t.empty((n, abi.NSF), dtype=t.float64, device=dev)
    if feat:
        out["feat"] = t.empty((n, abi.NFEAT), dtype=t.float64, device=dev)
    sel_t = None
    if sel_idx is not None:
        sel_t = _dev(np.asarray(sel_idx, dtype=np.int32))
        out["sel"] = t.empty((n, len(sel_idx)), dtype=t.float64, device=dev)
    tr = None
    if trace:
        if dg.n_k != 1:
            raise ValueError("trace needs a single-kernel grid")
        k = dc.corpus.ker[int(dg.bufs["kid"][0].item())]
        nt, nb = int(k["n_tok"]), int(k["n_blk"])
        for key, shape, dt in (("start", (n, nt), t.float64), ("duration", (n, nt), t.float64),
                               ("latency", (n, nt), t.float64), ("n_batches", (n, nt), t.int64),
                               ("blk_delay", (n, nb), t.float64),
                               ("blk_finish", (n, nb), t.float64)):
            out["tr_" + key] = t.zeros(shape, dtype=dt, device=dev)
        tr = abi.GkTrace(*[_ptr(out["tr_" + k]) for k in ("start", "duration", "latency",
                                                          "n_batches", "blk_delay", "blk_finish")])
    _check(load_library().gk_schedule_features(
        C.byref(dc.desc), C.byref(dg.desc), _ptr(ks), _ptr(ls), _ptr(out["status"]),
        _ptr(out.get("si")), _ptr(out.get("sf")), _ptr(out.get("feat")), _ptr(sel_t),
        0 if sel_idx is None else len(sel_idx), _ptr(out.get("sel")),
        C.byref(tr) if tr is not None else None, _stream(stream)))
    out["kstat"], out["latsum"] = ks, ls
    return out


def throughput_clamps(dg: "DeviceGrid", reset: bool = True, stream=None) -> int:
    """How often the throughput model was clamped to tp_floor on the device
    for grid `dg` since its last reset (the reference logs a warning per
    clamped call, profiles.py:173-181).  The counter belongs to the grid
    (gk_grid.tp_clamps), so concurrent sweeps keep separate counts.
    Synchronises `stream`."""
    t = _torch()
    c = dg.bufs["clamps"]
    s = t.cuda.current_stream() if stream is None else stream
    with t.cuda.stream(s):
        v = int(c.item())
        if reset:
            c.zero_()
    return v


def rf_predict(de: DeviceEnsemble, X, *, status=None, time_us=None, stream=None):
    """K4 (+K6) over device rows X [n, >= n_feat] float64."""
    t = _torch()
    if X.dtype != t.float64 or not X.is_cuda or X.dim() != 2:
        raise ValueError("X must be a 2-D float64 CUDA tensor")
    X = X.contiguous()
    n = X.shape[0]
    power = t.empty(n, dtype=t.float64, device=X.device)
    energy = t.empty(n, dtype=t.float64, device=X.device) if time_us is not None else None
    _check(load_library().gk_rf_predict(C.byref(de.desc), _ptr(X), X.shape[1], n, _ptr(status),
                                        _ptr(time_us), _ptr(power), _ptr(energy),
                                        _stream(stream)))
    return power, energy


class Sweep:
    """Preallocated fused energy sweep (K1 -> K2/K3 -> K4 -> K6) over one grid."""

    def __init__(self, dc: DeviceCorpus, dg: DeviceGrid, ensembles, sel_idx):
        t = _torch()
        if len(ensembles) != dg.n_arch:
            raise ValueError("one ensemble per arch")
        self.dc, self.dg, self.ens = dc, dg, list(ensembles)
        self.sel = _dev(np.asarray(sel_idx, dtype=np.int32))
        self.n_sel = len(sel_idx)
        arr = (abi.GkEnsemble * len(ensembles))(*[e.desc for e in ensembles])
        self.ens_arr = arr
        L = load_library()
        ws = L.gk_sweep_workspace_bytes(C.byref(dc.desc), C.byref(dg.desc), self.n_sel)
        dev = device()
        self.work = t.empty(max(ws, 256), dtype=t.uint8, device=dev)
        n = dg.n_points
        self.status = t.empty(n, dtype=t.uint8, device=dev)
        self.time_us = t.empty(n, dtype=t.float64, device=dev)
        self.power = t.empty(n, dtype=t.float64, device=dev)
        self.energy = t.empty(n, dtype=t.float64, device=dev)

    def stage_ms(self, stream=None) -> dict:
        """Run one sweep with per-stage CUDA events (synchronises); ms per stage."""
        L = load_library()
        L.gk_set_stage_timing(1)
        try:
            self.run(stream)
            out = (C.c_float * 3)()
            _check(L.gk_get_stage_ms(out))
        finally:
            L.gk_set_stage_timing(0)
        if self.fused:
            return {"k1_static": out[0], "k23_schedule<fused>": out[1]}
        return {"k1_static": out[0], "k23_schedule": out[1], "k4_rf_predict": out[2]}

    @property
    def fused(self) -> bool:
        """libgk runs the sweep as one fused kernel unless GK_SWEEP_FUSED=0."""
        import os

        return os.environ.get("GK_SWEEP_FUSED", "1")[:1] != "0"

    def run(self, stream=None):
        _check(load_library().gk_predict_energy_sweep(
            C.byref(self.dc.desc), C.byref(self.dg.desc), self.ens_arr, _ptr(self.sel),
            self.n_sel, _ptr(self.work), _ptr(self.status), _ptr(self.time_us), _ptr(self.power),
            _ptr(self.energy), _stream(stream)))
        return self.status, self.time_us, self.power, self.energy


class HostSweep:
    """The energy sweep from HOST buffers to HOST results -- the reference-facing
    batch call (cli.py:184-197's per-launch loop as one call).

    Every `submit()` is one full step: the packed corpus is copied from pinned
    host memory to the device (copy stream 1), the fused sweep runs (compute
    stream), and (status, time_us, power_w, energy_uj) are copied back to
    pinned host memory (copy stream 2).  Device inputs and host outputs are
    multi-buffered (`depth` slots), so successive steps pipeline: step s + 1's
    H2D and step s - 1's D2H run on the B200's copy engines while step s
    computes.  `run()` = one submitted step, synchronised.

    `n_chunks` > 1 additionally splits one step into kernel chunks (each a
    self-contained sub-corpus); measured on B200 this does NOT pay for a
    single step, because one fused launch cannot finish faster than its
    longest work item (~2.5 ms on config #2), so it is off by default."""

    def __init__(self, corpus: Corpus, profiles, configs, ensembles, sel_idx, n_chunks: int = 1,
                 depth: int = 2):
        t = _torch()
        dev = device()
        n_k = corpus.n_ker
        n_chunks = max(1, min(n_chunks, n_k)) if n_k else 1
        blk = corpus.blk
        n = blk["n"].astype(np.int64)
        if n_k and n_chunks > 1:
            kc = np.add.reduceat(n * n + n + 1, corpus.ker["blk0"].astype(np.int64)) \
                if len(blk) else np.ones(n_k, np.int64)
            kc = np.where(corpus.ker["n_blk"] > 0, kc, 1)
            cum = np.cumsum(kc)
            cuts = [0] + [int(np.searchsorted(cum, cum[-1] * i / n_chunks)) + 1
                          for i in range(1, n_chunks)] + [n_k]
            cuts = sorted(set(min(max(c, 0), n_k) for c in cuts))
        else:
            cuts = [0, n_k]
        self.n_cfg, self.n_arch = len(configs), len(profiles)
        P_k = self.n_cfg * self.n_arch
        self.n_points = n_k * P_k
        self.depth = max(1, depth)
        # host inputs (pinned, shared by every slot) and per-slot device state
        self.chunks = []
        for k0, k1 in zip(cuts[:-1], cuts[1:]):
            if k1 <= k0 and n_k:
                continue
            sub = corpus.slice(k0, k1) if (k0, k1) != (0, n_k) else corpus
            host = {}
            for k in ("tok", "preds", "blk", "fpreds", "topo", "ker"):
                a = np.ascontiguousarray(getattr(sub, k))
                if len(a) == 0:
                    a = np.zeros(1, a.dtype)
                host[k] = t.from_numpy(a.view(np.uint8).reshape(-1) if a.dtype.fields else a) \
                    .pin_memory()
            slots = []
            for _ in range(self.depth):
                dc = DeviceCorpus.upload(sub)
                dg = DeviceGrid.build(dc, profiles, configs)
                slots.append({"dc": dc, "sweep": Sweep(dc, dg, ensembles, sel_idx)})
            self.chunks.append({"host": host, "slots": slots, "p0": k0 * P_k, "p1": k1 * P_k})
        self.h2d_bytes = sum(h.numel() * h.element_size() for c in self.chunks
                             for h in c["host"].values())
        self.d2h_bytes = self.n_points * (1 + 3 * 8)
        self.outs = [{"status": t.empty(self.n_points, dtype=t.uint8).pin_memory(),
                      "time_us": t.empty(self.n_points, dtype=t.float64).pin_memory(),
                      "power_w": t.empty(self.n_points, dtype=t.float64).pin_memory(),
                      "energy_uj": t.empty(self.n_points, dtype=t.float64).pin_memory()}
                     for _ in range(self.depth)]
        self.s_h2d = t.cuda.Stream(device=dev)
        self.s_d2h = t.cuda.Stream(device=dev)
        self.ev_free = [t.cuda.Event() for _ in range(self.depth)]   # slot's D2H done
        self.n_submitted = 0

    @property
    def out(self) -> dict:
        """Host results of the most recently submitted step."""
        return self.outs[(self.n_submitted - 1) % self.depth]

    def submit(self, stream=None) -> dict:
        """Enqueue one step (H2D -> sweep -> D2H) on `stream` (default: the
        current stream) and the two copy streams; returns that step's host
        output dict (valid after synchronisation)."""
        t = _torch()
        cs = stream or t.cuda.current_stream()
        k = self.n_submitted % self.depth
        first = self.n_submitted < self.depth
        self.n_submitted += 1
        # the slot's previous step must have finished its D2H (which follows its compute)
        if first:
            self.s_h2d.wait_stream(cs)
        else:
            self.s_h2d.wait_event(self.ev_free[k])
        ev_in = []
        with t.cuda.stream(self.s_h2d):
            for c in self.chunks:
                dc = c["slots"][k]["dc"]
                for name, h in c["host"].items():
                    dc.bufs[name].copy_(h, non_blocking=True)
                e = t.cuda.Event()
                e.record(self.s_h2d)
                ev_in.append(e)
        ev_done = []
        for c, e in zip(self.chunks, ev_in):
            cs.wait_event(e)
            c["slots"][k]["sweep"].run(cs)
            d = t.cuda.Event()
            d.record(cs)
            ev_done.append(d)
        out = self.outs[k]
        with t.cuda.stream(self.s_d2h):
            for c, d in zip(self.chunks, ev_done):
                self.s_d2h.wait_event(d)
                sw, p0, p1 = c["slots"][k]["sweep"], c["p0"], c["p1"]
                out["status"][p0:p1].copy_(sw.status, non_blocking=True)
                out["time_us"][p0:p1].copy_(sw.time_us, non_blocking=True)
                out["power_w"][p0:p1].copy_(sw.power, non_blocking=True)
                out["energy_uj"][p0:p1].copy_(sw.energy, non_blocking=True)
            self.ev_free[k].record(self.s_d2h)
        return out

    def finish(self, stream=None):
        """Make `stream` (default: current) wait for every submitted step."""
        t = _torch()
        cs = stream or t.cuda.current_stream()
        cs.wait_stream(self.s_d2h)
        cs.wait_stream(self.s_h2d)

    def run(self, stream=None) -> dict:
        out = self.submit(stream)
        self.finish(stream)
        return out


class HostRowsPredictor:
    """Batched power (+ energy) for a HOST row table (the reference-facing
    `predict_power` over many rows), streamed through the device in chunks:
    chunk k + 1's H2D copy and chunk k - 1's D2H copy run on their own
    streams while K4 walks chunk k (two device slots).  X_host / out_host
    should be pinned (torch `pin_memory()`) for the copies to be asynchronous."""

    def __init__(self, ensemble: "DeviceEnsemble", n_cols: int, chunk_rows: int = 8 << 20):
        t = _torch()
        dev = device()
        self.de, self.n_cols, self.chunk = ensemble, int(n_cols), int(chunk_rows)
        self.x = [t.empty((self.chunk, self.n_cols), dtype=t.float64, device=dev) for _ in range(2)]
        self.p = [t.empty(self.chunk, dtype=t.float64, device=dev) for _ in range(2)]
        self.s_h2d = t.cuda.Stream(device=dev)
        self.s_d2h = t.cuda.Stream(device=dev)
        self.ev_free = [t.cuda.Event() for _ in range(2)]   # slot's D2H done
        self.used = [False, False]

    def run(self, X_host, out_host, stream=None):
        """Enqueue power for every row of X_host [n, n_cols] into out_host [n];
        returns after enqueueing (synchronise before reading out_host)."""
        t = _torch()
        cs = stream or t.cuda.current_stream()
        n = X_host.shape[0]
        L = load_library()
        self.s_h2d.wait_stream(cs)
        self.s_d2h.wait_stream(cs)
        for k, r0 in enumerate(range(0, n, self.chunk)):
            r1 = min(n, r0 + self.chunk)
            slot = k % 2
            with t.cuda.stream(self.s_h2d):
                if self.used[slot]:
                    self.s_h2d.wait_event(self.ev_free[slot])
                self.x[slot][: r1 - r0].copy_(X_host[r0:r1], non_blocking=True)
                ev_in = t.cuda.Event()
                ev_in.record(self.s_h2d)
            cs.wait_event(ev_in)
            _check(L.gk_rf_predict(C.byref(self.de.desc), _ptr(self.x[slot]), self.n_cols, r1 - r0,
                                   None, None, _ptr(self.p[slot]), None, cs.cuda_stream))
            ev_done = t.cuda.Event()
            ev_done.record(cs)
            with t.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(ev_done)
                out_host[r0:r1].copy_(self.p[slot][: r1 - r0], non_blocking=True)
                self.ev_free[slot].record(self.s_d2h)
            self.used[slot] = True
        cs.wait_stream(self.s_d2h)
        return out_host
