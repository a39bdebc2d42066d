"""Correlation-based feature pruning with the statistics on the GPU.

Same interface and decisions as the reference trainer
(``gpukalc_trainer/dataset.py:128-193``): ``prune_correlated(dataset, method,
threshold)`` drops constant columns first, then walks the surviving columns in
order and, for every pair whose |correlation| exceeds the threshold, drops the
less preferred one (``PREFERRED_FEATURES`` first, then the earlier column);
``prune_two_stage`` runs Pearson then Kendall.  Only the correlation matrix
moves to the device (``gk_corr_*`` in ``include/gk.h``):

* Kendall (pandas -> ``scipy.stats.kendalltau`` per pair, tau-b): the device
  computes the exact integer counts (discordant pairs, x / y / joint ties), and
  tau follows scipy's own expression on them, so every coefficient is
  bit-identical to pandas';
* Pearson: centred co-moments by deterministic fixed-order fp64 sums.  pandas'
  nancorr accumulates differently (a streaming update per pair), so a
  coefficient may differ in the last bits; a decision can only differ when
  |r| is within ~1e-12 of the threshold.

Frames with non-finite values (pandas masks them pair by pair) take pandas'
own corr -- host preprocessing, not the prediction path.
"""

from __future__ import annotations

import ctypes as C
import logging
from dataclasses import dataclass, replace

import numpy as np

from .errors import TrainerError

log = logging.getLogger(__name__)

PRUNE_METHODS = ("pearson", "kendall")
PREFERRED_FEATURES = frozenset({       # reference dataset.py:24-40
    "avg_comp_lat", "avg_glob_lat", "avg_shar_lat", "branch", "comp_inst_kernel",
    "glob_inst_kernel", "glob_load_sm", "glob_store_sm", "misc_inst_kernel",
    "inst_issue_cycles", "cache_penalty", "occupancy", "reg_thread", "shmem_block", "block_size",
})
PAIR_BATCH_ELEMS = 1 << 27             # rows x pairs per Kendall launch (workspace ~6 GB)


@dataclass(frozen=True)
class Dataset:
    """Reference ``dataset.py:45-66``: feature frame, target, provenance."""

    X: object            # pandas.DataFrame
    y: object            # pandas.Series
    provenance: object = None
    source: str | None = None

    def __post_init__(self):
        if self.X.shape[0] != self.y.shape[0]:
            raise TrainerError("feature matrix and target have different lengths")
        if self.X.isna().any().any() or self.y.isna().any():
            raise TrainerError("dataset contains missing values")

    @property
    def manifest(self) -> tuple:
        return tuple(self.X.columns)

    @property
    def n_rows(self) -> int:
        return int(self.X.shape[0])


@dataclass(frozen=True)
class DropEntry:
    """Reference ``dataset.py:69-84``: one pruning decision."""

    dropped: str
    kept: str | None
    method: str
    coefficient: float | None

    def as_dict(self) -> dict:
        return {"dropped": self.dropped, "kept": self.kept, "method": self.method,
                "coefficient": self.coefficient}


def _lib():
    from .runtime import load_library

    L = load_library()
    if not getattr(L, "_corr_bound", False):
        vp, i64, i32, sz = C.c_void_p, C.c_int64, C.c_int32, C.c_size_t
        L.gk_corr_ranks_workspace.restype = sz
        L.gk_corr_ranks_workspace.argtypes = [i64]
        L.gk_corr_ranks.argtypes = [vp, i64, i32, i64, vp, vp, vp, vp, sz, vp]
        L.gk_corr_kendall_workspace.restype = sz
        L.gk_corr_kendall_workspace.argtypes = [i64, i32]
        L.gk_corr_kendall.argtypes = [vp, i64, i32, vp, vp, vp, vp, vp, i32, vp, vp, vp, sz, vp]
        L.gk_corr_pearson_workspace.restype = sz
        L.gk_corr_pearson_workspace.argtypes = [i64, i32]
        L.gk_corr_pearson.argtypes = [vp, i64, i32, i64, vp, vp, vp, sz, vp]
        L._corr_bound = True
    return L


def kendall_counts(X: np.ndarray):
    """Exact tau-b ingredients on the device: per column (n_unique, ties) and
    per pair a < b (discordant, joint ties).  X: [n, K] finite float64."""
    import torch

    from .runtime import _check, _dev, _ptr, device

    X = np.ascontiguousarray(X, dtype=np.float64)
    n, K = X.shape
    L = _lib()
    dev = device()
    st = torch.cuda.current_stream().cuda_stream
    Xd = _dev(X, dev)
    ranks = torch.empty(K * n, dtype=torch.int32, device=dev)
    nu = torch.empty(K, dtype=torch.int32, device=dev)
    ties = torch.empty(K, dtype=torch.int64, device=dev)
    wsb = L.gk_corr_ranks_workspace(n)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _check(L.gk_corr_ranks(_ptr(Xd), n, K, K, _ptr(ranks), _ptr(nu), _ptr(ties), _ptr(ws), wsb, st))
    del Xd, ws
    nu_h = nu.cpu().numpy().astype(np.uint32)
    ties_h = ties.cpu().numpy()
    pairs = [(a, b) for a in range(K) for b in range(a + 1, K)]
    dis = np.zeros(len(pairs), np.int64)
    ntie = np.zeros(len(pairs), np.int64)
    per = max(1, min(len(pairs), PAIR_BATCH_ELEMS // max(n, 1)))
    if pairs:
        wsb = L.gk_corr_kendall_workspace(n, per)
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        for s in range(0, len(pairs), per):
            pa = np.array([p[0] for p in pairs[s:s + per]], np.int32)
            pb = np.array([p[1] for p in pairs[s:s + per]], np.int32)
            pa_d, pb_d = torch.from_numpy(pa).to(dev), torch.from_numpy(pb).to(dev)
            d = torch.empty(len(pa), dtype=torch.int64, device=dev)
            t = torch.empty(len(pa), dtype=torch.int64, device=dev)
            _check(L.gk_corr_kendall(_ptr(ranks), n, K, nu_h.ctypes.data, pa.ctypes.data,
                                     pb.ctypes.data, _ptr(pa_d), _ptr(pb_d), len(pa), _ptr(d),
                                     _ptr(t), _ptr(ws), wsb, st))
            dis[s:s + len(pa)] = d.cpu().numpy()
            ntie[s:s + len(pa)] = t.cpu().numpy()
    return nu_h, ties_h, pairs, dis, ntie


def kendall_matrix(X: np.ndarray) -> np.ndarray:
    """DataFrame.corr("kendall") for a finite matrix: tau-b per pair from the
    device's exact counts, with scipy's expression (``_stats_py._kendalltau``)."""
    n, K = np.shape(X)
    nu, ties, pairs, dis, ntie = kendall_counts(X)
    out = np.eye(K)
    tot = (n * (n - 1)) // 2
    for (a, b), d, nt in zip(pairs, dis, ntie):
        xtie, ytie = int(ties[a]), int(ties[b])
        if xtie == tot or ytie == tot:
            tau = np.nan
        else:
            cmd = tot - xtie - ytie + int(nt) - 2 * int(d)
            tau = cmd / np.sqrt(tot - xtie) / np.sqrt(tot - ytie)
            tau = float(np.minimum(1., max(-1., tau)))
        out[a, b] = out[b, a] = tau
    return out


def pearson_matrix(X: np.ndarray) -> np.ndarray:
    """DataFrame.corr("pearson") for a finite matrix: r = C_ab / sqrt(C_aa C_bb)
    from the device's centred co-moments (NaN for a zero-variance column)."""
    import torch

    from .runtime import _check, _dev, _ptr, device

    X = np.ascontiguousarray(X, dtype=np.float64)
    n, K = X.shape
    L = _lib()
    dev = device()
    Xd = _dev(X, dev)
    mean = torch.empty(K, dtype=torch.float64, device=dev)
    co = torch.empty(K * (K + 1) // 2, dtype=torch.float64, device=dev)
    wsb = L.gk_corr_pearson_workspace(n, K)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _check(L.gk_corr_pearson(_ptr(Xd), n, K, K, _ptr(mean), _ptr(co), _ptr(ws), wsb,
                             torch.cuda.current_stream().cuda_stream))
    c = co.cpu().numpy()
    C_ = np.zeros((K, K))
    iu = np.triu_indices(K)
    C_[iu] = c
    C_ = C_ + np.triu(C_, 1).T
    d = np.diag(C_)
    with np.errstate(invalid="ignore", divide="ignore"):
        r = C_ / np.sqrt(np.outer(d, d))
    r = np.clip(r, -1.0, 1.0)
    np.fill_diagonal(r, np.where(d > 0, 1.0, np.nan))
    return r


def _corr(frame, method: str) -> np.ndarray:
    X = frame.to_numpy(dtype=float)
    if not np.isfinite(X).all():   # pandas masks non-finite values per pair
        return frame.corr(method=method).to_numpy()
    return kendall_matrix(X) if method == "kendall" else pearson_matrix(X)


def _prefer(a: str, b: str, order: dict) -> tuple:
    def rank(name):
        return (0 if name in PREFERRED_FEATURES else 1, order[name])

    return (a, b) if rank(a) <= rank(b) else (b, a)


def prune_correlated(dataset, method: str = "pearson", threshold: float = 0.85):
    """Reference ``dataset.py:138-183`` with the correlation matrix on the GPU.
    `dataset`: this module's Dataset or the reference's (any frozen dataclass
    with an ``X`` DataFrame)."""
    if method not in PRUNE_METHODS:
        raise TrainerError(f"unknown correlation method '{method}'")
    if not 0.0 < threshold < 1.0:
        raise TrainerError("correlation threshold must be in (0, 1)")
    drops, survivors = [], []
    for col in dataset.X.columns:
        if dataset.X[col].nunique(dropna=False) <= 1:
            drops.append(DropEntry(col, None, "constant", None))
            log.info("dropping constant column %s", col)
        else:
            survivors.append(col)
    corr = _corr(dataset.X[survivors], method) if survivors else np.zeros((0, 0))
    pos = {c: i for i, c in enumerate(survivors)}
    order = {name: i for i, name in enumerate(dataset.X.columns)}
    alive = dict.fromkeys(survivors, True)
    for i, a in enumerate(survivors):
        if not alive[a]:
            continue
        for b in survivors[i + 1:]:
            if not alive[b]:
                continue
            coef = float(corr[pos[a], pos[b]])
            if abs(coef) > threshold:
                kept, dropped = _prefer(a, b, order)
                alive[dropped] = False
                drops.append(DropEntry(dropped, kept, method, coef))
                log.info("dropping %s (|%s|=%.4f with %s)", dropped, method, abs(coef), kept)
                if dropped == a:
                    break
    kept_cols = [c for c in survivors if alive[c]]
    if not kept_cols:
        raise TrainerError("pruning removed every feature column")
    return replace(dataset, X=dataset.X[kept_cols]), drops


def prune_two_stage(dataset, pearson: float = 0.85, kendall: float = 0.85):
    """Reference ``dataset.py:186-193``: Pearson pass, then Kendall on the survivors."""
    after_pearson, log1 = prune_correlated(dataset, "pearson", pearson)
    after_kendall, log2 = prune_correlated(after_pearson, "kendall", kendall)
    return after_kendall, log1 + log2


__all__ = ["Dataset", "DropEntry", "prune_correlated", "prune_two_stage", "kendall_matrix", "pearson_matrix",
           "kendall_counts", "PREFERRED_FEATURES"]
