"""Gradient-boosted family: the trainer's DEFAULT family
(reference training.py:67-72, sklearn GradientBoostingRegressor) on the GPU.

Parity bar (BASELINE.json): trained-model R^2 / MAPE within 0.5 points of the
reference train(..., "gradient_boosted") over the same KFold folds
(tests/golden/trainer_gbt.json, produced by the reference with sklearn 1.9.0).
On features with <= 256 distinct values the histogram split search is exact,
so the GPU trees follow sklearn's own trees."""

import json

import numpy as np
import pytest

from goldens import G
from test_forest import power_frame


def test_make_model_builds_the_gpu_booster_with_sklearn_defaults():
    from paper_2305_01886_b200.boosting import GradientBoostingRegressor
    from paper_2305_01886_b200.trainer import _make_model

    m = _make_model("gradient_boosted", 500, 0.05, None, 7)
    assert isinstance(m, GradientBoostingRegressor)
    assert (m.n_estimators, m.learning_rate, m.max_depth, m.random_state) == (500, 0.05, 3, 7)
    assert _make_model("gradient_boosted", 10, 0.1, 5, 0).max_depth == 5


def test_reference_golden_present():
    ref = json.loads((G / "trainer_gbt.json").read_text())
    assert ref["sklearn_version"] and len([k for k in ref if k.startswith("n")]) == 3


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["n600_seed3_est200_lr0.05_depthNone",
                                 "n2000_seed5_est150_lr0.1_depth4",
                                 "n3000_seed7_est100_lr0.1_depthNone"])
def test_train_gbt_r2_mape_parity_with_reference(key):
    from paper_2305_01886_b200.trainer import train

    ref = json.loads((G / "trainer_gbt.json").read_text())[key]
    fr = power_frame(ref["n_rows"], ref["frame_seed"])
    feats = ref["features"]
    res = train((fr[feats].to_numpy(), fr["power_w"].to_numpy(), tuple(feats)), "gradient_boosted",
                n_estimators=ref["n_estimators"], learning_rate=ref["learning_rate"],
                max_depth=ref["max_depth"], seed=0)
    r2 = res.mean_metrics.r2
    mape = float(np.mean(res.fold_mape_pct))
    assert abs(r2 - ref["mean"]["r2"]) <= 0.005, (r2, ref["mean"]["r2"])
    assert abs(mape - ref["mean_mape_pct"]) <= 0.5, (mape, ref["mean_mape_pct"])
    assert res.model.init_.value == pytest.approx(ref["init"], rel=1e-12)


@pytest.mark.gpu
def test_gbt_export_walks_to_model_predictions():
    import oracle as O
    from paper_2305_01886_b200.ensemble import flatten, load_ensemble
    from paper_2305_01886_b200.trainer import ensemble_document, train

    fr = power_frame(900, 13)
    feats = [c for c in fr.columns if c not in ("kernel", "power_w")]
    res = train((fr[feats].to_numpy(), fr["power_w"].to_numpy(), tuple(feats)), "gradient_boosted",
                n_estimators=60, learning_rate=0.1, seed=2)
    model = res.model
    assert len(model.estimators_) == 60 and all(len(e) == 1 for e in model.estimators_)
    for (est,) in model.estimators_:
        t = est.tree_
        assert t.max_depth <= 3
        leaf = t.children_left == -1
        assert (t.children_right[~leaf] == t.children_left[~leaf] + 1).all()
    doc = ensemble_document(res)
    assert doc["base_score"] == float(np.mean(res.y))
    flat = flatten(load_ensemble(doc))
    pw, _ = O.rf_predict(flat, res.X[:300])
    np.testing.assert_allclose(pw, model.predict(res.scaler.transform(res.X[:300])), rtol=1e-9)


@pytest.mark.gpu
def test_gbt_follows_sklearn_when_bins_are_exact():
    """<= 256 distinct values per feature: one bin per value, so every split the
    GPU search can choose is one sklearn's exhaustive search considers."""
    from sklearn.ensemble import GradientBoostingRegressor as SkGBR

    from paper_2305_01886_b200.boosting import GradientBoostingRegressor

    rng = np.random.default_rng(0)
    n = 4000
    X = np.stack([rng.integers(0, 50, n), rng.integers(0, 200, n), rng.integers(0, 7, n),
                  rng.integers(0, 120, n)], axis=1).astype(np.float64)
    y = 3.0 * X[:, 0] + 0.1 * X[:, 1] ** 1.5 + 20.0 * (X[:, 2] > 3) + rng.normal(0, 1, n)
    ours = GradientBoostingRegressor(40, learning_rate=0.1, random_state=0).fit(X, y)
    sk = SkGBR(n_estimators=40, learning_rate=0.1, random_state=0).fit(X, y)

    def canon(t, i=0):  # node-order independent (ours BFS, sklearn DFS)
        if t.children_left[i] == -1:
            return ("leaf", round(float(t.value[i][0][0]), 6))
        return (int(t.feature[i]), float(t.threshold[i]), canon(t, t.children_left[i]),
                canon(t, t.children_right[i]))

    same = sum(canon(a.tree_) == canon(b.tree_)
               for (a,), b in zip(ours.estimators_, sk.estimators_[:, 0]))
    assert same >= 30, same   # near-ties in the proxy may order a few splits differently
    p_ours, p_sk = ours.predict(X), sk.predict(X)
    assert np.max(np.abs(p_ours - p_sk)) < 0.05 * np.std(y)


@pytest.mark.gpu
def test_train_gbt_device_folds_equal_host_folds(monkeypatch):
    """trainer.train's device folds for the boosted family: fold metrics and
    the final model's trees equal the host-fold path bit for bit."""
    from paper_2305_01886_b200 import trainer as T
    from paper_2305_01886_b200.boosting import GradientBoostingRegressor

    rng = np.random.default_rng(8)
    X = rng.random((30_000, 10)) * 7.0
    y = 10 + 3 * X[:, 0] + np.cos(X[:, 1]) + rng.normal(0, 0.3, 30_000)
    names = tuple(f"f{i}" for i in range(10))
    res = {}
    for dev in (True, False):
        monkeypatch.setattr(GradientBoostingRegressor, "_device_input", dev)
        res[dev] = T.train((X, y, names), "gradient_boosted", n_estimators=12, max_depth=3, seed=1)
    a, b = res[True], res[False]
    assert [m.r2 for m in a.fold_metrics] == [m.r2 for m in b.fold_metrics]
    assert a.model.init_.value == b.model.init_.value
    for (ea,), (eb,) in zip(a.model.estimators_, b.model.estimators_):
        for f in ("children_left", "feature", "threshold", "value"):
            assert np.array_equal(getattr(ea.tree_, f), getattr(eb.tree_, f))
