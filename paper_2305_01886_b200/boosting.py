"""GPU gradient boosting behind scikit-learn's estimator shape.

Drop-in for the estimator the reference trainer builds for its DEFAULT family
(``gpukalc_trainer.training._make_model("gradient_boosted")``,
``training.py:67-72``): ``GradientBoostingRegressor(n_estimators,
learning_rate, random_state[, max_depth])`` with ``fit(X, y)``,
``predict(X)``, ``estimators_[k][0].tree_`` and ``init_.predict`` -- what
``gpukalc_trainer.export.ensemble_document`` reads (``export.py:55-59``: leaves
x learning_rate, base_score = init prediction).

Semantics kept from scikit-learn's squared-error boosting: the initial
prediction is mean(y) (DummyRegressor); stage k fits a regression tree
(max_depth 3 by default, min_samples_split 2, min_samples_leaf 1, all
features) to the negative gradient y - F and adds learning_rate * leaf mean
to F.  The friedman_mse criterion ranks splits exactly like the MSE proxy the
K5 split search uses (both are W_l W_r (m_l - m_r)^2 up to the node's constant
weight).  Trees are grown by the K5 kernels (histogram split search over
<= 256 bins per feature, thresholds at sklearn's midpoints); the stage update
and the next residual run in one kernel (gk_gb_step) on rows grouped by leaf,
so F never leaves the device.  Parity bar: R^2 / MAPE (BASELINE.json).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .ensemble import NODE_DT, FlatEnsemble
from .errors import DeviceError
from .forest import (Tree, TreeBatch, TreeEstimator, _check, _LevelGrower, _lib, check_finite,
                     check_n_bins, is_device_tensor)


def _shifts(bound: float, n: int) -> tuple[int, int]:
    """Fixed-point exponents so that n * |r| and n * r^2 stay below 2^62."""
    def one(b):
        s = int(np.floor(62 - np.log2(max(b, 1e-300) * n + 1e-300)))
        return max(min(s, 60), -60)

    return one(bound), one(bound * bound)


class _Init:
    """The fitted initial estimator (sklearn's DummyRegressor(strategy='mean'))."""

    def __init__(self, value: float):
        self.constant_ = np.array([[value]])
        self.value = value

    def predict(self, X):
        return np.full(len(X), self.value)


class GradientBoostingRegressor(_LevelGrower):
    """GPU-trained gradient boosting (squared error) with sklearn's face."""

    _device_input = True   # fit / predict also take device tensors (trainer.train)

    def __init__(self, n_estimators: int = 100, *, learning_rate: float = 0.1,
                 max_depth: int | None = 3, random_state=None, n_bins: int = 256):
        self.n_estimators = n_estimators
        self.learning_rate = learning_rate
        self.max_depth = max_depth
        self.random_state = random_state
        self.n_bins = check_n_bins(n_bins)
        self.estimators_: list = []

    def fit(self, X, y, sample_weight=None):
        import torch

        from .runtime import _dev, _ptr, device, upload

        if sample_weight is not None:
            raise NotImplementedError("sample_weight is not supported (training.py never passes it)")
        if not self.learning_rate > 0.0:
            raise ValueError("learning_rate must be > 0")
        on_dev = is_device_tensor(X)
        if on_dev:   # trainer.train's device folds: X stays on the device
            X = X.to(device(), torch.float64).contiguous()
            y = (y.detach().to("cpu", torch.float64).numpy() if is_device_tensor(y)
                 else np.asarray(y, dtype=np.float64))
            y = np.ascontiguousarray(y).reshape(-1)   # the init mean is numpy's (sklearn's)
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
            # one upload; the finite check and the bin edges run on the device
            # (host isfinite + edges cost ~0.1 s of a 100-stage fit at 1M x 64)
            X = upload(X, dev)   # pinned staging ring (runtime.upload)
        n, F = X.shape
        if n < 1 or F > 64 * 1024 or n >= 2 ** 31:
            raise ValueError("bad training table shape")
        if len(y) != n:
            raise ValueError("X and y have different lengths")
        if not bool(torch.isfinite(X).all()):
            raise ValueError("Input X contains NaN or infinity.")
        check_finite(np.zeros((1, 1)), y)
        check_n_bins(self.n_bins)
        self.n_features_in_ = F
        L = _lib()
        if not getattr(L, "_gb_bound", False):
            vp, i32 = C.c_void_p, C.c_int32
            L.gk_gb_step.argtypes = [vp, i32, vp, vp, vp, i32, vp, vp, vp, vp, i32, i32, vp, i32,
                                     vp]
            L._gb_bound = True
        dev = device()
        st = torch.cuda.current_stream().cuda_stream
        Xb = self._prepare_bins(X)
        f0 = float(np.mean(y))                        # DummyRegressor(strategy="mean")
        self.init_ = _Init(f0)
        r0 = y - f0
        rmax = float(np.max(np.abs(r0)))
        shift, shift2 = _shifts(rmax, n)
        yfp = torch.from_numpy(np.rint(np.ldexp(r0, shift)).astype(np.int64)).to(dev)
        y2fp = torch.from_numpy(np.rint(np.ldexp(r0 * r0, shift2)).astype(np.int64)).to(dev)
        yd = _dev(y, dev)
        Fd = torch.full((n,), f0, dtype=torch.float64, device=dev)
        self._dev = dict(Xb=Xb, yfp=yfp, y2fp=y2fp, y=yd, n=n, F=F, shift=shift, shift2=shift2)
        counts = torch.ones(n, dtype=torch.int32, device=dev)
        # row records (include/gk.h gk_rf_record_bytes), rebuilt every stage from
        # the stage's targets; two ping-pong buffers
        rs = int(L.gk_rf_record_bytes(F))
        rows0 = torch.empty(n * rs, dtype=torch.uint8, device=dev)
        rows1 = torch.empty_like(rows0)
        base_d = torch.zeros(1, dtype=torch.int64, device=dev)
        fill = torch.empty(1, dtype=torch.int32, device=dev)
        absmax = torch.zeros(1, dtype=torch.int64, device=dev)
        base, m = np.zeros(1, np.int64), np.array([n], np.int64)
        seeds = np.random.RandomState(self.random_state).randint(np.iinfo(np.int32).max,
                                                                   size=self.n_estimators)
        # a stage reads only its three level sizes: the tree stays on the device
        # (depths read once after the loop), the leaf values feed the residual
        # update on the device, and max |y - F| comes back asynchronously --
        # the next stage's levels run before it is needed
        absmax_h = torch.zeros(1, dtype=torch.int64, pin_memory=True)
        absmax_ev = None
        pending = []
        self._defer_reads = True
        try:
            for k in range(self.n_estimators):
                _check(L.gk_rf_compact(_ptr(counts), 1, n, _ptr(Xb), F, _ptr(yfp), _ptr(base_d),
                                       _ptr(rows0), _ptr(fill), st))
                tree_d, leaves = self._grow(counts, base, m, rows0, rows1, 1)
                if isinstance(tree_d, list):   # GK_RF_HOST_LEVELS=1: host trees, host leaves
                    lv, lv_d, leaf_value = leaves
                    nl, leaf_val_d = len(lv), torch.from_numpy(leaf_value).to(dev)
                else:
                    nl, lv_d, leaf_val_d = leaves
                pending.append(tree_d)
                if k + 1 == self.n_estimators:
                    break
                if absmax_ev is not None:   # max |y - F| after the previous stage
                    absmax_ev.synchronize()
                    rmax = float(absmax_h.numpy().view(np.float64)[0])
                # next stage's fixed point: |y - F_new| <= (1 + lr) max |y - F| (leaf
                # means are averages of the current residuals)
                shift, shift2 = _shifts(rmax * (1.0 + self.learning_rate) * (1.0 + 1e-9)
                                        + 1e-300, n)
                lvals = leaf_val_d * self.learning_rate   # the fp64 product numpy formed
                absmax.zero_()
                # n bounds the leaf sizes (the launcher caps CTAs per leaf by the
                # leaf count, so deep unbounded stages stay small grids)
                _check(L.gk_gb_step(_ptr(lv_d), nl, _ptr(lvals), _ptr(rows0), _ptr(rows1), F,
                                    _ptr(yd), _ptr(Fd), _ptr(yfp), _ptr(y2fp), shift, shift2,
                                    _ptr(absmax), n, st))
                absmax_h.copy_(absmax, non_blocking=True)
                absmax_ev = torch.cuda.Event()
                absmax_ev.record()
                self._dev["shift"], self._dev["shift2"] = shift, shift2
        finally:
            self._defer_reads = False
        dev_trees = [p for p in pending if not isinstance(p, list)]
        depths = (torch.cat([p[4] for p in dev_trees]).cpu().numpy() if dev_trees
                  else np.zeros(0, np.int64))
        self.estimators_, j = [], 0
        for k, p in enumerate(pending):
            if isinstance(p, list):
                tree = p[0]
            else:
                fl, it, node_base, next_id, _ = p
                batch = TreeBatch(fl, it, node_base, next_id, depths[j: j + 1])
                tree = Tree(node_count=int(next_id[0]), max_depth=int(depths[j]), batch=batch,
                            start=0)
                j += 1
            self.estimators_.append([TreeEstimator(tree_=tree, random_state=int(seeds[k]))])
        self.n_estimators_ = len(self.estimators_)
        self._flat = None
        del self._dev, self._dev_thr
        return self

    # -------------------------------------------------------------- predict
    def flat(self) -> FlatEnsemble:
        """The model as one device ensemble: base = init prediction, leaves x
        learning_rate (what export.py writes, ``export.py:55-59``)."""
        parts, offs, depths, off = [], [], [], 0
        lr = float(self.learning_rate)
        for (est,) in self.estimators_:
            t = est.tree_
            arr = np.zeros(t.node_count, NODE_DT)
            split = t.children_left >= 0
            arr["v"] = np.where(split, t.threshold, t.value[:, 0, 0] * lr)
            arr["feature"] = np.where(split, t.feature, -1)
            arr["left"] = np.where(split, t.children_left, np.arange(t.node_count) - 1)
            parts.append(arr)
            offs.append(off)
            depths.append(t.max_depth)
            off += t.node_count
        F = self.n_features_in_
        return FlatEnsemble(nodes=np.concatenate(parts).astype(NODE_DT),
                            tree_off=np.asarray(offs, np.int64), scale_lo=np.zeros(F),
                            scale_hi=np.ones(F), base_score=float(self.init_.value),
                            max_depth=max(depths), manifest=tuple(f"f{i}" for i in range(F)),
                            tree_depth=np.asarray(depths, np.int32))

    def predict(self, X) -> np.ndarray:
        """init + sum over stages of learning_rate * leaf value, on float32-cast X
        (sklearn's predict_stages order)."""
        import torch

        from .runtime import DeviceEnsemble, device, rf_predict, upload

        if getattr(self, "_flat", None) is None:
            self._flat = DeviceEnsemble.upload(self.flat())
        if is_device_tensor(X):
            Xd = X.to(device(), torch.float64).to(torch.float32).to(torch.float64).contiguous()
        else:
            Xf = np.ascontiguousarray(np.asarray(X, dtype=np.float64).astype(np.float32),
                                      np.float64)
            Xd = upload(Xf, device())
        total, _ = rf_predict(self._flat, Xd)
        return total.cpu().numpy()


__all__ = ["GradientBoostingRegressor"]
