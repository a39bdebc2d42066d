"""Trainer face: ``train(dataset, family, ...)`` with the GPU forest / GPU boosting.

Mirrors ``gpukalc_trainer.training.train`` (``training.py:94-160``): canonical
row order (mergesort by every feature, then the target; ``:82-91``), 5-fold
``KFold(shuffle=True, random_state=seed)``, a ``MinMaxScaler`` fit per training
fold, fold metrics (R^2, RMSE, MAE), then a final fit on all rows.  The forest
(``_make_model``'s RandomForestRegressor, ``:73-76``) is
:class:`paper_2305_01886_b200.forest.RandomForestRegressor` (GPU, K5); the
default family's GradientBoostingRegressor (``:67-72``) is
:class:`paper_2305_01886_b200.boosting.GradientBoostingRegressor` (GPU, K5 +
gk_gb_step).  Export
follows ``export.py:26-83`` so the document loads in the reference's
``load_ensemble`` and in this package's.

Host glue here uses pandas / scikit-learn's KFold, MinMaxScaler and metrics
exactly as the reference trainer does; tree fitting and prediction run on the
device.  Like the reference, this module never imports the predictor face.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path
from typing import Any

import numpy as np

from .boosting import GradientBoostingRegressor
from .errors import TrainerError
from .forest import RandomForestRegressor

FAMILIES = ("random_forest", "gradient_boosted")
N_FOLDS = 5
MIN_ROWS = 50


@dataclass(frozen=True)
class FoldMetrics:
    r2: float
    rmse: float
    mae: float

    def as_dict(self) -> dict:
        return {"r2": self.r2, "rmse": self.rmse, "mae": self.mae}


@dataclass
class TrainResult:
    family: str
    seed: int
    hyperparameters: dict[str, Any]
    manifest: tuple
    model: Any
    scaler: Any
    fold_metrics: list
    mean_metrics: FoldMetrics
    X: np.ndarray = field(repr=False)
    y: np.ndarray = field(repr=False)
    holdout_indices: np.ndarray = field(repr=False)
    fold_mape_pct: list = field(default_factory=list)   # harness metric (not in the reference)

    def metrics_doc(self) -> dict:
        return {"family": self.family, "seed": self.seed,
                "hyperparameters": self.hyperparameters, "n_rows": int(self.X.shape[0]),
                "n_features": len(self.manifest), "feature_manifest": list(self.manifest),
                "folds": [m.as_dict() for m in self.fold_metrics],
                "mean": self.mean_metrics.as_dict()}


def _make_model(family: str, n_estimators: int, learning_rate: float, max_depth, seed: int):
    if family == "random_forest":
        return RandomForestRegressor(n_estimators=n_estimators, max_depth=max_depth,
                                     random_state=seed)
    if family == "gradient_boosted":   # training.py:67-72 (GPU boosting, boosting.py)
        kwargs = {} if max_depth is None else {"max_depth": max_depth}
        return GradientBoostingRegressor(n_estimators=n_estimators, learning_rate=learning_rate,
                                         random_state=seed, **kwargs)
    raise TrainerError(f"unsupported model family '{family}'; choose from {', '.join(FAMILIES)}")


def canonical_order(X: np.ndarray, y: np.ndarray) -> np.ndarray:
    """The row order of ``training.py:82-91``: a stable lexicographic sort by
    every feature column, then the target (pandas ``sort_values(by=manifest +
    [target], kind="mergesort")``), computed most-significant key first: one
    stable argsort of the first column, then only the runs of rows still tied
    on all keys so far are re-sorted by the next key (continuous features
    leave no ties after the first pass: one argsort instead of pandas' 65-key
    factorisation, ~15 s at 1M x 64).  Values compare like pandas' (-0.0 ==
    0.0; the Dataset forbids NaN)."""
    F = X.shape[1]

    def key(j):   # column j (the target after the features), no up-front copies
        return X[:, j] if j < F else y

    n = len(y)
    order = np.argsort(key(0), kind="stable")
    tied = np.ones(n, bool)     # position i tied with i - 1 on every key so far
    tied[0] = False
    for k in range(1, F + 1):
        v = key(k - 1)[order]
        tied[1:] &= v[1:] == v[:-1]
        if not tied.any():
            break
        grp = np.cumsum(~tied)                  # group id per sorted position
        multi = tied | np.r_[tied[1:], False]   # members of groups of size > 1
        pos = np.flatnonzero(multi)
        sub = order[pos]
        # stable sort of those rows by (group, key k): lexsort's last key is primary
        perm = np.lexsort((key(k)[sub], grp[pos]))
        order[pos] = sub[perm]
    return order


def canonical_rows(X, y, manifest) -> tuple[np.ndarray, np.ndarray]:
    """Reference ``training.py:82-91``: stable sort by all features then target."""
    X = np.asarray(X, dtype=float)
    y = np.asarray(y, dtype=float)
    if X.ndim != 2 or X.shape[1] != len(manifest) or len(y) != len(X):
        raise TrainerError("feature matrix and target have different lengths")
    order = canonical_order(X, y)
    return X[order], y[order]


def _minmax_on_device(Xd):
    """A fitted sklearn MinMaxScaler for the device table Xd: the column minima
    and maxima are reduced on the device (exact), and the scaler is fitted on
    that 2-row summary -- data_min_ / data_max_ / scale_ / min_ come out of
    sklearn's own code, identical to fitting on the rows."""
    from sklearn.preprocessing import MinMaxScaler

    summary = np.stack([Xd.amin(dim=0).cpu().numpy(), Xd.amax(dim=0).cpu().numpy()])
    sc = MinMaxScaler().fit(summary)
    sc.n_samples_seen_ = int(Xd.shape[0])
    return sc


def _scale_on_device(sc, Xd):
    """MinMaxScaler.transform on the device: X * scale_, then + min_ (sklearn's
    in-place `X *= scale_; X += min_`, the same two roundings)."""
    import torch

    scale = torch.from_numpy(np.asarray(sc.scale_, np.float64)).to(Xd.device)
    shift = torch.from_numpy(np.asarray(sc.min_, np.float64)).to(Xd.device)
    return torch.add(torch.mul(Xd, scale), shift)


def train(dataset, family: str = "gradient_boosted", *, n_estimators: int = 500,
          learning_rate: float = 0.05, max_depth: int | None = None, seed: int = 0) -> TrainResult:
    """5-fold CV, then a final fit on all rows (reference ``training.py:94-160``).

    `dataset` is the reference's Dataset (X DataFrame, y Series) or any object
    with ``X``, ``y`` and ``manifest``; or an (X, y, manifest) tuple.
    """
    from sklearn.metrics import mean_absolute_error, mean_squared_error, r2_score
    from sklearn.model_selection import KFold
    from sklearn.preprocessing import MinMaxScaler

    if family not in FAMILIES:
        raise TrainerError(f"unsupported model family '{family}'; choose from " + ", ".join(FAMILIES))
    if isinstance(dataset, tuple):
        Xraw, yraw, manifest = dataset
    else:
        Xraw, yraw = dataset.X, dataset.y
        manifest = tuple(getattr(dataset, "manifest", None) or list(dataset.X.columns))
    n_rows = len(yraw)
    if n_rows < MIN_ROWS:
        raise TrainerError(f"need at least {MIN_ROWS} rows for {N_FOLDS}-fold CV, got {n_rows}")
    X, y = canonical_rows(Xraw, yraw, manifest)
    if np.ptp(y) == 0.0:
        raise TrainerError("degenerate target: every row has the same value")
    probe = _make_model(family, n_estimators, learning_rate, max_depth, seed)  # family check
    # models that take device tensors get every fold scaled on the device from
    # one upload of the canonical table: the same float64 values as
    # MinMaxScaler.transform (X * scale_ then + min_, two IEEE roundings), no
    # host copies of the folds (they were ~40 % of a config #3 train())
    dev_folds = getattr(probe, "_device_input", False)
    if dev_folds:
        import torch

        from .runtime import device, upload

        Xd = upload(np.ascontiguousarray(X, dtype=np.float64), device())
        yd = upload(np.ascontiguousarray(y, dtype=np.float64), device())
    folds, mapes = [], []
    holdout = np.empty(0, dtype=int)
    for tr, te in KFold(n_splits=N_FOLDS, shuffle=True, random_state=seed).split(X):
        model = _make_model(family, n_estimators, learning_rate, max_depth, seed)
        if dev_folds:
            tr_d, te_d = (torch.from_numpy(i).to(Xd.device) for i in (tr, te))
            Xtr = Xd.index_select(0, tr_d)
            scaler = _minmax_on_device(Xtr)
            model.fit(_scale_on_device(scaler, Xtr), yd.index_select(0, tr_d))
            del Xtr
            pred = model.predict(_scale_on_device(scaler, Xd.index_select(0, te_d)))
        else:
            scaler = MinMaxScaler().fit(X[tr])
            model.fit(scaler.transform(X[tr]), y[tr])
            pred = model.predict(scaler.transform(X[te]))
        folds.append(FoldMetrics(r2=float(r2_score(y[te], pred)),
                                 rmse=float(np.sqrt(mean_squared_error(y[te], pred))),
                                 mae=float(mean_absolute_error(y[te], pred))))
        mapes.append(float(np.mean(np.abs((y[te] - pred) / y[te])) * 100.0))
        holdout = te
    mean = FoldMetrics(r2=float(np.mean([m.r2 for m in folds])),
                       rmse=float(np.mean([m.rmse for m in folds])),
                       mae=float(np.mean([m.mae for m in folds])))
    final_model = _make_model(family, n_estimators, learning_rate, max_depth, seed)
    if dev_folds:
        final_scaler = _minmax_on_device(Xd)
        final_model.fit(_scale_on_device(final_scaler, Xd), yd)
        del Xd, yd
    else:
        final_scaler = MinMaxScaler().fit(X)
        final_model.fit(final_scaler.transform(X), y)
    return TrainResult(family=family, seed=seed,
                       hyperparameters={"n_estimators": n_estimators,
                                        "learning_rate": learning_rate, "max_depth": max_depth},
                       manifest=tuple(manifest), model=final_model, scaler=final_scaler,
                       fold_metrics=folds, mean_metrics=mean, X=X, y=y, holdout_indices=holdout,
                       fold_mape_pct=mapes)


# ------------------------------------------------------------------ export


def _tree_nodes(tree, leaf_scale: float) -> list:
    """sklearn-style tree arrays -> node dicts (``export.py:26-39``)."""
    nodes = []
    for i in range(tree.node_count):
        if tree.children_left[i] == -1:
            nodes.append({"value": float(tree.value[i][0][0]) * leaf_scale})
        else:
            nodes.append({"feature": int(tree.feature[i]), "threshold": float(tree.threshold[i]),
                          "left": int(tree.children_left[i]),
                          "right": int(tree.children_right[i])})
    return nodes


def _accumulate_gains(tree, gains: np.ndarray) -> None:
    """Weighted impurity decrease per feature (``export.py:42-50``)."""
    w, imp = tree.weighted_n_node_samples, tree.impurity
    for i in range(tree.node_count):
        left, right = tree.children_left[i], tree.children_right[i]
        if left == -1:
            continue
        dec = w[i] * imp[i] - w[left] * imp[left] - w[right] * imp[right]
        gains[tree.feature[i]] += max(float(dec), 0.0)


def ensemble_document(result: TrainResult) -> dict:
    """Portable ensemble JSON (``export.py:53-83``): RF leaves x 1/n_trees,
    boosted leaves x learning_rate with base_score = the init prediction."""
    estimators, leaf_scale, base_score = _doc_parts(result)
    gains = np.zeros(len(result.manifest))
    trees = []
    for est in estimators:
        trees.append({"nodes": _tree_nodes(est.tree_, leaf_scale)})
        _accumulate_gains(est.tree_, gains)
    return {"schema_version": 1, "base_score": base_score, "feature_manifest": list(result.manifest),
            "scaling": {"min": [float(v) for v in result.scaler.data_min_],
                        "max": [float(v) for v in result.scaler.data_max_]},
            "trees": trees, "gains": [float(g) for g in gains]}


def _doc_parts(result: TrainResult):
    if result.family == "gradient_boosted":
        estimators = [est[0] for est in result.model.estimators_]
        leaf_scale = float(result.model.learning_rate)
        base_score = float(result.model.init_.predict(np.zeros((1, len(result.manifest))))[0])
    elif result.family == "random_forest":
        estimators = list(result.model.estimators_)
        leaf_scale = 1.0 / len(estimators)
        base_score = 0.0
    else:
        raise TrainerError(f"unsupported model family '{result.family}'")
    return estimators, leaf_scale, base_score


def ensemble_document_text(result: TrainResult) -> str:
    """``json.dumps(ensemble_document(result), indent=2)`` without building the
    per-node dicts: the tree arrays go straight to the native writer
    (libgkhost ``gk_ens_write``, byte-identical text).  Gains
    accumulate in the same order as ``_accumulate_gains`` (np.add.at is
    sequential)."""
    from .ensemble import document_text

    estimators, leaf_scale, base_score = _doc_parts(result)
    gains = np.zeros(len(result.manifest))
    trees = []
    for est in estimators:
        t = est.tree_
        cl, cr = np.asarray(t.children_left), np.asarray(t.children_right)
        leaf = cl == -1
        vals = np.asarray(t.value)[:, 0, 0].astype(np.float64) * leaf_scale
        trees.append({"is_leaf": leaf, "feature": np.where(leaf, 0, t.feature),
                      "value": np.where(leaf, vals, np.asarray(t.threshold, np.float64)),
                      "left": np.where(leaf, 0, cl), "right": np.where(leaf, 0, cr)})
        w, imp = np.asarray(t.weighted_n_node_samples), np.asarray(t.impurity)
        sp = np.flatnonzero(~leaf)
        dec = w[sp] * imp[sp] - w[cl[sp]] * imp[cl[sp]] - w[cr[sp]] * imp[cr[sp]]
        np.add.at(gains, np.asarray(t.feature)[sp], np.maximum(dec, 0.0))
    return document_text(base_score=base_score, manifest=list(result.manifest),
                         scale_lo=np.asarray(result.scaler.data_min_, np.float64),
                         scale_hi=np.asarray(result.scaler.data_max_, np.float64),
                         gains=gains, trees=trees, indent=2)


VECTOR_SCHEMA_VERSION = 1  # export.py:23


def _sample_rows(result: TrainResult, n_vectors: int) -> np.ndarray:
    """Rows of the test vectors as ``export.py:128-134`` picks them: the last
    CV fold's held-out rows (all rows when that pool is too small), sampled
    without replacement by ``default_rng(seed)``, in row order."""
    pool = np.asarray(result.holdout_indices)
    if pool.size < n_vectors:
        pool = np.arange(result.X.shape[0])
    rng = np.random.default_rng(result.seed)
    return np.sort(rng.choice(pool, size=min(n_vectors, pool.size), replace=False))


def export_ensemble(result: TrainResult, out_dir, *, n_vectors: int = 20) -> tuple[Path, Path]:
    """Write ensemble.json and test_vectors.json; return both paths
    (``export.py:150-175``).  The ensemble text comes from the native writer
    (the bytes of ``json.dumps(doc, indent=2)``); each vector's prediction is
    the exported document walked on the device (K4: min-max scaling, then
    base + leaves in tree order -- the reference walker's arithmetic,
    ``export.py:101-125``) after loading the file back, so the vectors check
    the file, not the in-memory model."""
    import torch

    from .ensemble import flatten, load_ensemble
    from .runtime import DeviceEnsemble, device, rf_predict, upload

    if n_vectors < 1:
        raise TrainerError("need at least one test vector")
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    ensemble_path = out / "ensemble.json"
    ensemble_path.write_text(ensemble_document_text(result) + "\n")
    picked = _sample_rows(result, n_vectors)
    rows = np.ascontiguousarray(np.asarray(result.X, np.float64)[picked])
    de = DeviceEnsemble.upload(flatten(load_ensemble(ensemble_path)))
    power, _ = rf_predict(de, upload(rows, device()))
    pred = power.cpu().numpy()
    vectors = [{"inputs": {name: float(v) for name, v in zip(result.manifest, row)},
                "prediction": float(p)} for row, p in zip(rows, pred)]
    vectors_path = out / "test_vectors.json"
    vectors_path.write_text(json.dumps({
        "schema_version": VECTOR_SCHEMA_VERSION,
        "ensemble_file": ensemble_path.name,
        "vectors": vectors,
    }, indent=2) + "\n")
    return ensemble_path, vectors_path
