"""Golden outcomes of the REFERENCE ensemble loader (gpukalc.load_ensemble,
power.py:73-125) on edge-case documents and seeded random mutations of valid
ones (pins the native loader in libgkhost and this package's Python loader).

Run in the build container only (imports /root/reference):

    python tests/golden/make_ensio_golden.py

Writes tests/golden/ensio_cases.json: per case the document TEXT and the
reference outcome -- the exception type + message, or the loaded ensemble
(base score, manifest, scaling, gains, trees as node dicts).
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path[:0] = [str(REF / "src"), str(ROOT)]

import gpukalc as R  # noqa: E402


def doc(trees, k=2, **kw):
    d = {"schema_version": 1, "base_score": 0.5,
         "feature_manifest": [f"f{i}" for i in range(k)],
         "scaling": {"min": [0.0] * k, "max": [1.0] * k}, "trees": trees,
         "gains": [0.0] * k}
    d.update(kw)
    return d


STUMP = [{"nodes": [{"feature": 0, "threshold": 0.5, "left": 1, "right": 2},
                    {"value": 1.0}, {"value": 2.0}]}]
DEEP = [{"nodes": [{"feature": 1, "threshold": 0.25, "left": 2, "right": 1},
                   {"feature": 0, "threshold": 0.75, "left": 4, "right": 3},
                   {"value": -1.5}, {"value": 7}, {"value": 3.25}]}]

EDGE = {
    "stump": json.dumps(doc(STUMP)),
    "deep_unordered": json.dumps(doc(DEEP + STUMP)),
    "ints_everywhere": json.dumps(doc([{"nodes": [{"feature": 0, "threshold": 1, "left": 1,
                                                   "right": 2}, {"value": 3}, {"value": -4}]}],
                                      base_score=2)),
    "no_trees": json.dumps(doc([])),
    "no_gains_no_base": json.dumps({k: v for k, v in doc(STUMP).items()
                                    if k not in ("gains", "base_score")}),
    "schema_float": json.dumps(doc(STUMP, schema_version=1.0)),
    "schema_2": json.dumps(doc(STUMP, schema_version=2)),
    "schema_true": json.dumps(doc(STUMP, schema_version=True)),
    "schema_missing": json.dumps({k: v for k, v in doc(STUMP).items() if k != "schema_version"}),
    "manifest_empty": json.dumps(doc(STUMP, feature_manifest=[])),
    "manifest_dup": json.dumps(doc(STUMP, feature_manifest=["a", "a"])),
    "manifest_nonstr": json.dumps(doc(STUMP, feature_manifest=["a", 3])),
    "manifest_unicode": json.dumps(doc(STUMP, feature_manifest=["café", "über\U0001F600"])),
    "manifest_escapes": '{"schema_version": 1, "feature_manifest": ["a\\"b", "\\u0041"], '
                        '"scaling": {"min": [0, 0], "max": [1, 1]}, "trees": []}',
    "scaling_missing": json.dumps({k: v for k, v in doc(STUMP).items() if k != "scaling"}),
    "scaling_short": json.dumps(doc(STUMP, scaling={"min": [0.0], "max": [1.0, 1.0]})),
    "scaling_inverted": json.dumps(doc(STUMP, scaling={"min": [0.0, 2.0], "max": [1.0, 1.0]})),
    "scaling_equal": json.dumps(doc(STUMP, scaling={"min": [0.5, 1.0], "max": [0.5, 1.0]})),
    "trees_not_list": json.dumps(doc({"nodes": []})),
    "tree_no_nodes": json.dumps(doc([{"n": []}])),
    "tree_empty": json.dumps(doc([{"nodes": []}])),
    "leaf_string": json.dumps(doc([{"nodes": [{"value": "1"}]}])),
    "leaf_bool": json.dumps(doc([{"nodes": [{"value": True}]}])),
    "split_missing_left": json.dumps(doc([{"nodes": [{"feature": 0, "threshold": 0.5,
                                                      "right": 1}, {"value": 1}]}])),
    "feature_range": json.dumps(doc([{"nodes": [{"feature": 2, "threshold": 0.5, "left": 1,
                                                 "right": 2}, {"value": 1}, {"value": 2}]}])),
    "feature_float": json.dumps(doc([{"nodes": [{"feature": 1.0, "threshold": 0.5, "left": 1,
                                                 "right": 2}, {"value": 1}, {"value": 2}]}])),
    "child_range": json.dumps(doc([{"nodes": [{"feature": 0, "threshold": 0.5, "left": 1,
                                               "right": 3}, {"value": 1}, {"value": 2}]}])),
    "cycle": json.dumps(doc([{"nodes": [{"feature": 0, "threshold": 0.5, "left": 1, "right": 0},
                                        {"value": 1}]}])),
    "twice": json.dumps(doc([{"nodes": [{"feature": 0, "threshold": 0.5, "left": 1, "right": 1},
                                        {"value": 1}]}])),
    "orphan": json.dumps(doc([{"nodes": [{"value": 1}, {"value": 2}]}])),
    "gains_short": json.dumps(doc(STUMP, gains=[0.0])),
    "gains_negative": json.dumps(doc(STUMP, gains=[0.0, -1.0])),
    "nan_inf": '{"schema_version": 1, "base_score": NaN, "feature_manifest": ["a"], '
               '"scaling": {"min": [-Infinity], "max": [Infinity]}, "trees": [{"nodes": '
               '[{"feature": 0, "threshold": NaN, "left": 1, "right": 2}, {"value": Infinity}, '
               '{"value": -0.0}]}]}',
    "dup_keys": '{"schema_version": 2, "schema_version": 1, "feature_manifest": ["a"], '
                '"scaling": {"min": [0], "max": [1]}, "trees": [{"nodes": [{"value": 1, '
                '"value": 2.5}]}, {"nodes": [{"value": 9}], "nodes": [{"value": 3}]}]}',
    "extra_keys": '{"schema_version": 1, "x": {"y": [1, 2, {"z": null}]}, "feature_manifest": '
                  '["a"], "scaling": {"min": [0], "max": [1], "note": "s"}, "trees": '
                  '[{"id": 7, "nodes": [{"value": 1}]}]}',
    "node_extra_key": '{"schema_version": 1, "feature_manifest": ["a"], "scaling": {"min": [0], '
                      '"max": [1]}, "trees": [{"nodes": [{"value": 1, "cover": 3}]}]}',
    "big_int": '{"schema_version": 1, "feature_manifest": ["a"], "scaling": {"min": [0], '
               '"max": [1]}, "trees": [{"nodes": [{"value": 123456789012345678901}]}]}',
    "exp_numbers": '{"schema_version": 1, "feature_manifest": ["a"], "scaling": {"min": [-1e-3], '
                   '"max": [2E+2]}, "trees": [{"nodes": [{"feature": 0, "threshold": 1.5e-1, '
                   '"left": 1, "right": 2}, {"value": 1e308}, {"value": -2.5E-308}]}]}',
    "bad_json": '{"schema_version": 1, "feature_manifest": ["a"],}',
    "leading_zero": '{"schema_version": 01}',
    "trailing_data": json.dumps(doc(STUMP)) + " x",
    "whitespace": "\n\t " + json.dumps(doc(STUMP), indent=3) + " \r\n",
}


def outcome(text: str, tmp: Path) -> dict:
    tmp.write_text(text, encoding="utf-8")
    try:
        e = R.load_ensemble(tmp)
    except Exception as exc:  # noqa: BLE001 - the outcome IS the exception
        return {"error": type(exc).__name__, "message": str(exc)}
    return {"base_score": repr(e.base_score), "manifest": list(e.feature_manifest),
            "min": [repr(v) for v in e.scale_min], "max": [repr(v) for v in e.scale_max],
            "gains": [repr(v) for v in e.gains],
            "trees": [[{k: repr(v) for k, v in n.items()} for n in t] for t in e.trees]}


NOISE = ["{", "}", "[", "]", ",", ":", '"', "1", "-", ".5", "e9", "true", "null", "NaN",
         '"value": 2', '"left": 0', '"feature": 7', " ", "\\", "0", "9e999"]


def main() -> None:
    tmp = HERE / "_ensio_tmp.json"
    cases = []
    for name, text in EDGE.items():
        cases.append({"name": name, "text": text, "ref": outcome(text, tmp)})
    rng = random.Random(1017)
    base = json.dumps(doc(DEEP + STUMP + DEEP, k=2))
    for i in range(160):
        t = base
        for _ in range(rng.randint(1, 3)):
            j = rng.randrange(len(t))
            if rng.random() < 0.4:
                t = t[:j] + t[j + rng.randint(1, 4):]
            else:
                t = t[:j] + rng.choice(NOISE) + t[j:]
        cases.append({"name": f"mut{i}", "text": t, "ref": outcome(t, tmp)})
    tmp.unlink()
    (HERE / "ensio_cases.json").write_text(json.dumps({"source": "gpukalc.load_ensemble",
                                                       "cases": cases}))
    kinds: dict = {}
    for c in cases:
        k = c["ref"].get("error", "ok")
        kinds[k] = kinds.get(k, 0) + 1
    print(len(cases), kinds)


if __name__ == "__main__":
    main()
