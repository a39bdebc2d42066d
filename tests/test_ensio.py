"""Native ensemble JSON loader (libgkhost, include/gk_ensio.h) -- SURVEY §8(f)#3.

CPU tests (host code): every document of tests/golden/ensio_cases.json (edge
cases + seeded mutations, outcomes recorded from the reference's
load_ensemble) loads to the reference's result or raises its exception and
message; accepted documents give flat device arrays byte-identical to the
Python loader + flatten, and the lazily materialised node dicts equal the
reference's."""

import json
import re

import numpy as np
import pytest

from goldens import G
from paper_2305_01886_b200 import ensemble as E
from paper_2305_01886_b200.errors import EnsembleError


def _outcome(path):
    try:
        e = E.load_ensemble(path)
    except EnsembleError as exc:
        return {"error": "EnsembleError", "message": str(exc)}, None
    return ({"base_score": repr(e.base_score), "manifest": list(e.feature_manifest),
             "min": [repr(v) for v in e.scale_min], "max": [repr(v) for v in e.scale_max],
             "gains": [repr(v) for v in e.gains],
             "trees": [[{k: repr(v) for k, v in n.items()} for n in t] for t in e.trees]}, e)


def test_library_exports_every_declared_symbol():
    from paper_2305_01886_b200.ptx_native import load_library

    L = load_library()
    hdr = (G.parents[1] / "include" / "gk_ensio.h").read_text()
    for name in set(re.findall(r"\b(gk_ens_\w+)\s*\(", hdr)):
        assert getattr(L, name) is not None


def test_reference_outcomes(tmp_path):
    cases = json.loads((G / "ensio_cases.json").read_text())["cases"]
    bad, native_ok = [], 0
    for c in cases:
        p = tmp_path / "e.json"
        p.write_text(c["text"], encoding="utf-8")
        got, ens = _outcome(p)
        if got != c["ref"]:
            bad.append((c["name"], got, c["ref"]))
        if ens is not None:
            native_ok += isinstance(ens.trees, E._LazyTrees)
            want = E.flatten(E._load_python(p))
            assert E.flatten(ens).nodes.tobytes() == want.nodes.tobytes(), c["name"]
    assert not bad, bad[:3]
    assert native_ok >= 12  # the common documents took the native path


def _docs():
    from paper_2305_01886_b200.ensemble import flat_to_document, random_forest_flat

    yield json.loads((G / "power_ensemble.json").read_text())
    for seed, (nt, d, nf) in enumerate([(3, 5, 4), (40, 9, 15), (7, 12, 64)]):
        flat = random_forest_flat(nt, d, [f"x{i}" for i in range(nf)], np.zeros(nf),
                                  np.arange(1, nf + 1, dtype=float), seed=seed, split_p=0.8)
        doc = flat_to_document(flat)
        doc["base_score"] = 12.5 + seed
        yield doc


@pytest.mark.parametrize("indent", [None, 2])
def test_native_equals_python_loader(tmp_path, indent):
    for k, doc in enumerate(_docs()):
        p = tmp_path / f"d{k}.json"
        p.write_text(json.dumps(doc, indent=indent))
        fast = E.load_ensemble(p)
        slow = E._load_python(p)
        assert isinstance(fast.trees, E._LazyTrees)
        a, b = E.flatten(fast), E.flatten(slow)
        assert a.nodes.tobytes() == b.nodes.tobytes()
        assert np.array_equal(a.tree_off, b.tree_off) and np.array_equal(a.tree_depth, b.tree_depth)
        assert a.max_depth == b.max_depth and a.base_score == b.base_score
        assert np.array_equal(a.scale_lo, b.scale_lo) and np.array_equal(a.scale_hi, b.scale_hi)
        assert fast == slow   # incl. the materialised node dicts


def test_unreadable_path_raises_reference_error(tmp_path):
    with pytest.raises(EnsembleError, match="cannot read ensemble"):
        E.load_ensemble(tmp_path / "missing.json")


# ------------------------------------------------------------------ writer


def test_float_repr_matches_cpython():
    import math

    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100_000) * 10.0 ** rng.integers(-300, 300, 100_000),
                        rng.random(50_000), np.ldexp(1.0, np.arange(-1074, 1024)),
                        -np.nextafter(np.ldexp(1.0, np.arange(-1000, 1000)), np.inf),
                        rng.integers(-2 ** 62, 2 ** 62, 20_000).astype(np.float64),
                        [0.0, -0.0, 1e16, 1e15, 0.0001, 0.00001, 5e-324, math.pi, 1 / 3]])
    assert E.float_reprs(x) == [repr(float(v)) for v in x]


def _sk_result(family):
    from sklearn.ensemble import GradientBoostingRegressor, RandomForestRegressor
    from sklearn.preprocessing import MinMaxScaler

    from paper_2305_01886_b200.trainer import FoldMetrics, TrainResult
    from test_forest import power_frame

    fr = power_frame(400, 21)
    feats = [c for c in fr.columns if c not in ("kernel", "power_w")]
    X, y = fr[feats].to_numpy(), fr["power_w"].to_numpy()
    sc = MinMaxScaler().fit(X)
    m = (RandomForestRegressor(7, max_depth=6, random_state=0) if family == "random_forest"
         else GradientBoostingRegressor(n_estimators=9, learning_rate=0.05, random_state=0))
    m.fit(sc.transform(X), y)
    fm = FoldMetrics(1.0, 0.0, 0.0)
    return TrainResult(family=family, seed=0, hyperparameters={}, manifest=tuple(feats) + (),
                       model=m, scaler=sc, fold_metrics=[fm], mean_metrics=fm, X=X, y=y,
                       holdout_indices=np.arange(10))


@pytest.mark.parametrize("family", ["random_forest", "gradient_boosted"])
def test_export_text_is_json_dumps_of_the_document(family):
    from paper_2305_01886_b200.trainer import ensemble_document, ensemble_document_text

    res = _sk_result(family)
    assert ensemble_document_text(res) == json.dumps(ensemble_document(res), indent=2)


def test_document_text_compact_and_escapes():
    trees = [{"is_leaf": np.array([0, 1, 1]), "feature": np.array([1, 0, 0]),
              "value": np.array([0.5, -1e-7, np.inf]), "left": np.array([1, 0, 0]),
              "right": np.array([2, 0, 0])}, {"is_leaf": np.array([1]), "feature": [0],
                                               "value": [float("nan")], "left": [0], "right": [0]}]
    man = ["a\"b\\c\n", "café \U0001F600 \x7f\x01"]
    kw = dict(base_score=-0.0, manifest=man, scale_lo=[0.0, -2.5], scale_hi=[1e300, 3.0],
              gains=[0.0, 7.25], trees=trees)
    doc = {"schema_version": 1, "base_score": -0.0, "feature_manifest": man,
           "scaling": {"min": [0.0, -2.5], "max": [1e300, 3.0]},
           "trees": [{"nodes": [{"feature": 1, "threshold": 0.5, "left": 1, "right": 2},
                                {"value": -1e-7}, {"value": float("inf")}]},
                     {"nodes": [{"value": float("nan")}]}], "gains": [0.0, 7.25]}
    assert E.document_text(**kw, indent=None) == json.dumps(doc)
    assert E.document_text(**kw, indent=2) == json.dumps(doc, indent=2)
    assert E.document_text(**kw, indent=0) == json.dumps(doc, indent=0)
    empty = dict(kw, trees=[])
    assert E.document_text(**empty) == json.dumps(dict(doc, trees=[]), indent=2)


def _walk_document(doc, inputs):
    """export.py:101-125 restated (the reference's test-vector walker)."""
    raw = [float(inputs[n]) for n in doc["feature_manifest"]]
    lo, hi = doc["scaling"]["min"], doc["scaling"]["max"]
    x = [(v - a) / (b - a) if b > a else 0.0 for v, a, b in zip(raw, lo, hi)]
    total = float(doc.get("base_score", 0.0))
    for tree in doc["trees"]:
        nodes = tree["nodes"]
        node = nodes[0]
        while "value" not in node:
            node = nodes[node["left"] if x[node["feature"]] <= node["threshold"] else node["right"]]
        total += node["value"]
    return total


@pytest.mark.gpu
@pytest.mark.parametrize("family", ["random_forest", "gradient_boosted"])
@pytest.mark.parametrize("n_vectors", [1, 7, 20, 500])
def test_export_ensemble_writes_reference_test_vectors(tmp_path, family, n_vectors):
    """export_ensemble mirrors export.py:150-175: returns (ensemble_path,
    vectors_path); vectors are holdout rows (all rows when the holdout is too
    small) drawn by default_rng(seed), predictions bit-equal to the reference
    walker over the written file."""
    from paper_2305_01886_b200.errors import TrainerError
    from paper_2305_01886_b200.trainer import export_ensemble

    res = _sk_result(family)
    ep, vp = export_ensemble(res, tmp_path / "out", n_vectors=n_vectors)
    assert ep.name == "ensemble.json" and vp.name == "test_vectors.json"
    doc = json.loads(ep.read_text())
    vec = json.loads(vp.read_text())
    assert vec["schema_version"] == 1 and vec["ensemble_file"] == "ensemble.json"
    pool = res.holdout_indices if res.holdout_indices.size >= n_vectors else np.arange(len(res.X))
    want_rows = np.sort(np.random.default_rng(res.seed).choice(
        pool, size=min(n_vectors, pool.size), replace=False))
    assert len(vec["vectors"]) == len(want_rows)
    for v, i in zip(vec["vectors"], want_rows):
        assert list(v["inputs"]) == list(res.manifest)
        assert [v["inputs"][n] for n in res.manifest] == [float(a) for a in res.X[i]]
        assert v["prediction"] == _walk_document(doc, v["inputs"])
    assert vp.read_text().endswith("}\n")
    with pytest.raises(TrainerError, match="at least one test vector"):
        export_ensemble(res, tmp_path / "x", n_vectors=0)
