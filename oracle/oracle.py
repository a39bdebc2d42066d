"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper around the CPU oracle
(``oracle/gk_oracle.c``).  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs as the checker; the product
package never imports this module.

Same inputs as the device path (packed corpus, arch records, configs) and the
same output arrays, so parity tests compare them with ``np.array_equal`` on
float64 bit patterns.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2305_01886_b200 import abi
from paper_2305_01886_b200.pack import KSTAT_DT, arch_records, config_array, latency_table

HERE = Path(__file__).resolve().parent
LIB = HERE / "libgk_oracle.so"
_lib = None


def build(force: bool = False) -> Path:
    deps = [HERE / "gk_oracle.c", HERE.parent / "include" / "gk.h"]
    if force or not LIB.exists() or any(LIB.stat().st_mtime < d.stat().st_mtime for d in deps):
        subprocess.run(["make", "-C", str(HERE), "-B" if force else "libgk_oracle.so"],
                       check=True, capture_output=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        vp = C.c_void_p
        L.gko_static_features.argtypes = [vp, vp, vp, vp]
        L.gko_schedule_features.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_uint32, vp,
                                            vp, C.c_int]
        L.gko_rf_predict.argtypes = [vp, vp, C.c_int64, C.c_int64, vp, vp, vp, vp, C.c_int]
        L.gko_bootstrap_counts.argtypes = [C.c_uint32, C.c_int64, vp]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def default_threads() -> int:
    return int(os.environ.get("GK_ORACLE_THREADS", os.cpu_count() or 1))


class HostGrid:
    """Host-side descriptors for one (corpus, kernels x archs x configs) grid."""

    def __init__(self, corpus, profiles, configs, kernel_ids=None, n_tw=None, gm=None):
        self.corpus = corpus.check()
        self.n_tw = None if n_tw is None else np.ascontiguousarray(n_tw, dtype=np.int64)
        self.gm = None if gm is None else np.ascontiguousarray(gm, dtype=np.float64)
        self.kernel_ids = np.ascontiguousarray(
            np.arange(corpus.n_ker, dtype=np.uint32) if kernel_ids is None
            else np.asarray(kernel_ids, dtype=np.uint32))
        self.cfg = config_array(configs)
        self.arch = arch_records(profiles)
        self.lat = np.ascontiguousarray(latency_table(profiles, corpus.sigs))
        self.c = abi.GkCorpus(_p(corpus.tok), _p(corpus.preds), _p(corpus.blk), _p(corpus.fpreds),
                              _p(corpus.topo), _p(corpus.ker), corpus.n_tok, len(corpus.blk),
                              corpus.n_ker, max(len(corpus.sigs), 1), corpus.max_n,
                              corpus.max_blk)
        self.g = abi.GkGrid(_p(self.kernel_ids), _p(self.cfg), _p(self.arch), _p(self.lat),
                            _p(self.n_tw), _p(self.gm), None, None, len(self.kernel_ids),
                            len(self.cfg), len(self.arch), 0)

    @property
    def n_points(self) -> int:
        return len(self.kernel_ids) * len(self.arch) * len(self.cfg)


def static_features(hg: HostGrid):
    ks = np.zeros(len(hg.kernel_ids), KSTAT_DT)
    ls = np.zeros((len(hg.arch), len(hg.kernel_ids), 3))
    lib().gko_static_features(C.byref(hg.c), C.byref(hg.g), _p(ks), _p(ls))
    return ks, ls


def schedule_features(hg: HostGrid, *, sel_idx=None, trace: bool = False, threads=None) -> dict:
    n = hg.n_points
    ks, ls = static_features(hg)
    out = {"status": np.zeros(n, np.uint8), "si": np.zeros((n, abi.NSI), np.int64),
           "sf": np.zeros((n, abi.NSF)), "feat": np.zeros((n, abi.NFEAT))}
    sel = None
    if sel_idx is not None:
        sel_idx = np.ascontiguousarray(sel_idx, dtype=np.int32)
        sel = out["sel"] = np.zeros((n, len(sel_idx)))
    tr = None
    if trace:
        if len(hg.kernel_ids) != 1:
            raise ValueError("trace needs a single-kernel grid")
        k = hg.corpus.ker[hg.kernel_ids[0]]
        nt, nb = int(k["n_tok"]), int(k["n_blk"])
        for key, shape, dt in (("start", (n, nt), np.float64), ("duration", (n, nt), np.float64),
                               ("latency", (n, nt), np.float64), ("n_batches", (n, nt), np.int64),
                               ("blk_delay", (n, nb), np.float64),
                               ("blk_finish", (n, nb), np.float64)):
            out["tr_" + key] = np.zeros(shape, dt)
        tr = abi.GkTrace(*[_p(out["tr_" + k]) for k in ("start", "duration", "latency",
                                                        "n_batches", "blk_delay", "blk_finish")])
    lib().gko_schedule_features(C.byref(hg.c), C.byref(hg.g), _p(ks), _p(ls), _p(out["status"]),
                                _p(out["si"]), _p(out["sf"]), _p(out["feat"]), _p(sel_idx),
                                0 if sel_idx is None else len(sel_idx), _p(sel),
                                C.byref(tr) if tr is not None else None,
                                default_threads() if threads is None else threads)
    out["kstat"], out["latsum"] = ks, ls
    return out


def rf_predict(flat, X, *, status=None, time_us=None, threads=None):
    X = np.ascontiguousarray(X, dtype=np.float64)
    n = X.shape[0]
    keep = [flat.nodes, flat.tree_off, np.ascontiguousarray(flat.tree_depth, dtype=np.int32),
            flat.scale_lo, flat.scale_hi]
    e = abi.GkEnsemble(*[_p(a) for a in keep], flat.base_score, flat.n_trees, flat.n_feat,
                       flat.max_depth)
    power = np.zeros(n)
    energy = np.zeros(n) if time_us is not None else None
    st = None if status is None else np.ascontiguousarray(status, dtype=np.uint8)
    tu = None if time_us is None else np.ascontiguousarray(time_us, dtype=np.float64)
    rc = lib().gko_rf_predict(C.byref(e), _p(X), X.shape[1], n, _p(st), _p(tu), _p(power),
                              _p(energy), default_threads() if threads is None else threads)
    if rc:
        raise ValueError("oracle rf_predict: too many features")
    return power, energy


def bootstrap_counts(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.uint8)
    lib().gko_bootstrap_counts(seed & 0xFFFFFFFF, n, _p(out))
    return out
