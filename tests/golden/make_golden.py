"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
(gpukalc / gpukalc-trainer, imported from /root/reference) on seeded inputs.

Run in the build container only (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py

Outputs (all small, committed):
  ref_fixtures.json   reference test fixtures (PTX, profile, ensembles) + KAT values
  sched_<set>.npz     schedule_kernel + extract_features outputs per point
  trace_k20.npz       per-instruction schedule rows (schedule_block rows)
  power.json/.npz     a reference-trained RF ensemble document, predict_power and
                      predict_energy outputs on real feature rows
  rf_bootstrap.npz    sklearn RandomForestRegressor per-tree seeds + bootstrap counts
  trainer_rf.json     reference train(random_forest) fold metrics (+ harness MAPE)
  trainer_gbt.json    reference train(gradient_boosted) fold metrics (+ harness MAPE),
                      and the exported ensemble's test vectors of one final model
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path[:0] = [str(REF / "src"), str(REF / "trainer" / "src"), str(ROOT)]

import gpukalc as R  # noqa: E402
from gpukalc.scheduler import LaunchConfig  # noqa: E402

from paper_2305_01886_b200 import corpus as CG  # noqa: E402
from paper_2305_01886_b200 import pack  # noqa: E402

ARCHS = ["tesla_k20", "tesla_m60", "gtx1050", "quadro_k4200"]
SETS = {
    # name: (n_kernels, seed, configs, archs)
    "c1": (100, 0, CG.CONFIG1, ARCHS),
    "c2": (16, 1, CG.config2_grid(), ["tesla_k20"]),
    "rnd": (24, 7, CG.random_configs(random.Random(99), 40), ARCHS),
    "c5": (6, 5, CG.config5_grid(), ["tesla_k20", "tesla_m60", "gtx1050"]),
}


def corpus_digest(c) -> str:
    """Digest of the packed corpus's semantic fields (independent of record padding
    and of derived fields), so a layout change does not invalidate the goldens."""
    h = hashlib.sha256()
    t = c.tok
    for f in ("res", "cls", "sig", "pred0"):
        h.update(np.ascontiguousarray(t[f]).astype(np.int64).tobytes())
    b = c.blk
    for f in ("mult", "tok0", "n", "fpred0", "n_fpred", "n_glob", "res_cnt", "is_exit"):
        h.update(np.ascontiguousarray(b[f]).astype(np.int64).tobytes())
    k = c.ker
    for f in ("blk0", "n_blk", "topo0", "max_n", "tok0", "n_tok"):
        h.update(np.ascontiguousarray(k[f]).astype(np.int64).tobytes())
    for a in (c.preds, c.fpreds, c.topo):
        h.update(np.ascontiguousarray(a).astype(np.int64).tobytes())
    h.update(json.dumps([list(s) for s in c.sigs]).encode())
    return h.hexdigest()


def ref_point(p, g, cfg):
    """Reference outputs for one point: status, si[6], sf[9], feat[32]."""
    si = np.zeros(6, np.int64)
    sf = np.full(9, np.nan)
    feat = np.full(32, np.nan)
    try:
        L = LaunchConfig(*cfg)
        ks = R.schedule_kernel(p, g, L)
    except R.ScheduleError as exc:
        assert "does not fit" in str(exc), exc
        return 1, si, sf, feat
    si[:] = [ks.threads_scheduled, ks.threads_per_sm, ks.blocks_per_sm, ks.waves,
             ks.n_global, ks.n_shared]
    sf[:] = [ks.gm_latency, ks.d_kernel, ks.overhead_cycles, ks.gm_penalty, ks.sm_penalty,
             ks.cm_penalty, ks.d_total, ks.time_us(p), ks.cfg.delay]
    try:
        feat[:] = R.extract_features(p, g, L).as_row()
    except R.ScheduleError:
        return 2, si, sf, feat
    return 0, si, sf, feat


def make_set(name, n_k, seed, configs, archs):
    kernels = CG.synth_corpus(n_k, seed)
    graphs = [R.parse_ptx(t, n, loop_counts=l) for n, t, l in kernels]
    profs = [R.resolve_profile(a) for a in archs]
    n = n_k * len(archs) * len(configs)
    st = np.zeros(n, np.uint8)
    si = np.zeros((n, 6), np.int64)
    sf = np.zeros((n, 9))
    ft = np.zeros((n, 32))
    p_i = 0
    for g in graphs:
        for p in profs:
            for c in configs:
                st[p_i], si[p_i], sf[p_i], ft[p_i] = ref_point(p, g, c)
                p_i += 1
    digest = corpus_digest(pack.pack_corpus(graphs))
    np.savez_compressed(HERE / f"sched_{name}.npz", status=st, si=si, sf=sf, feat=ft,
                        configs=np.asarray(configs, np.int64), archs=np.asarray(archs),
                        seed=seed, n_kernels=n_k, corpus_sha256=digest)
    print(f"{name}: {n} points, status {np.bincount(st, minlength=3)}, "
          f"gm<0 {(sf[:, 0] < 0).sum()}")


def make_trace():
    kernels = CG.synth_corpus(6, 21)
    configs = [(64, 256, 32, 0), (65535, 1024, 0, 0), (5, 96, 0, 4096)]
    p = R.resolve_profile("tesla_k20")
    out = {}
    for ki, (n, t, l) in enumerate(kernels):
        g = R.parse_ptx(t, n, loop_counts=l)
        for ci, c in enumerate(configs):
            ks = R.schedule_kernel(p, g, LaunchConfig(*c))
            rows = [r for b in ks.cfg.blocks for r in b.rows]
            out[f"k{ki}c{ci}_start"] = np.array([r.start for r in rows])
            out[f"k{ki}c{ci}_duration"] = np.array([r.duration for r in rows])
            out[f"k{ki}c{ci}_latency"] = np.array([r.latency for r in rows])
            out[f"k{ki}c{ci}_n_batches"] = np.array([r.n_batches for r in rows], np.int64)
            out[f"k{ki}c{ci}_blk_delay"] = np.array([b.delay for b in ks.cfg.blocks])
            out[f"k{ki}c{ci}_blk_finish"] = np.array(ks.cfg.finish)
    np.savez_compressed(HERE / "trace_k20.npz", configs=np.asarray(configs), seed=21,
                        n_kernels=6, **out)
    print("trace: 18 points")


def make_fixtures():
    fx = REF / "tests" / "fixtures"
    doc = {
        "ptx": {k: (fx / f"{k}.ptx").read_text() for k in ("worked_example", "vecadd", "nn_euclid")},
        "fixture_profile": json.loads((fx / "fixture_profile.json").read_text()),
        "ensembles": {k: json.loads((fx / f"ensemble_{k}.json").read_text())
                      for k in ("stump", "constant")},
        "source": "pkg/tests/fixtures (reference test fixtures, copied as data)",
    }
    # known-answer values as the reference computes them (pkg/tests/*)
    fp = R.profiles.profile_from_dict(doc["fixture_profile"])
    wg = R.parse_ptx(doc["ptx"]["worked_example"], "pair_load_add")
    bs = R.schedule_block(fp, wg.blocks[0], 256)
    vg = R.parse_ptx(doc["ptx"]["vecadd"], "vecadd")
    k20 = R.resolve_profile("k20")
    ks = R.schedule_kernel(k20, vg, LaunchConfig(64, 256))
    ng = R.parse_ptx(doc["ptx"]["nn_euclid"], "nn_euclid")
    nn = R.extract_features(k20, ng, LaunchConfig(256, 256, reg_per_thread=32))
    doc["kat"] = {
        "worked_starts": [r.start for r in bs.rows], "worked_delay": bs.delay,
        "vecadd_64x256": {"gm_latency": ks.gm_latency, "d_total": ks.d_total,
                          "time_us": ks.time_us(k20), "waves": ks.waves,
                          "blocks_per_sm": ks.blocks_per_sm},
        "nn_256x256_r32": nn.as_dict(),
        "energy_cells": [[5689.25, 83.28, R.predict_energy(5689.25, 83.28)],
                         [8945.25, 138.16, R.predict_energy(8945.25, 138.16)]],
    }
    (HERE / "ref_fixtures.json").write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")
    print("fixtures + KATs")


def make_power():
    """Reference-trained RF over the 15 selected features of set c1 (k20 rows)."""
    import pandas as pd
    from gpukalc_trainer import ensemble_document, train
    from gpukalc_trainer.dataset import Dataset

    d = np.load(HERE / "sched_c1.npz")
    ok = d["status"] == 0
    feat = d["feat"][ok]
    sel = [R.FEATURE_ORDER.index(f) for f in R.SELECTED_FEATURES]
    X = feat[:, sel]
    rng = np.random.default_rng(2026)
    # generative power in the style of trainer/tests/conftest.py:8-32
    y = (30.0 + 40.0 * X[:, R.SELECTED_FEATURES.index("occupancy")]
         + 0.003 * np.minimum(X[:, R.SELECTED_FEATURES.index("inst_issue_cycles")], 2e4)
         + 12.0 * (X[:, R.SELECTED_FEATURES.index("glob_load_sm")] > 50)
         + rng.normal(0.0, 1.0, len(X)))
    frame = pd.DataFrame(X, columns=list(R.SELECTED_FEATURES))
    ds = Dataset(X=frame, y=pd.Series(y), provenance=pd.DataFrame(index=frame.index))
    res = train(ds, "random_forest", n_estimators=16, max_depth=7, seed=0)
    doc = ensemble_document(res)
    (HERE / "power_ensemble.json").write_text(json.dumps(doc) + "\n")
    ens = R.load_ensemble(doc)
    rows = d["feat"][:, sel]
    power = np.array([R.predict_power(ens, [float(v) for v in r]) if s == 0 else np.nan
                      for r, s in zip(rows, d["status"])])
    t_us = d["sf"][:, 7]
    energy = np.array([R.predict_energy(float(pw), float(t)) if s == 0 and pw >= 0 and t >= 0 else np.nan
                       for pw, t, s in zip(power, t_us, d["status"])])
    np.savez_compressed(HERE / "power.npz", power=power, energy=energy,
                        sel=np.asarray(sel, np.int32))
    print("power: RF", len(doc["trees"]), "trees;", int(np.isfinite(power).sum()), "rows")


def make_bootstrap():
    from sklearn.ensemble import RandomForestRegressor
    from sklearn.ensemble._forest import _generate_sample_indices

    out = {}
    for n in (1000, 4097):
        X = np.random.default_rng(n).random((n, 3))
        y = X[:, 0]
        for seed in (0, 1, 42):
            rf = RandomForestRegressor(n_estimators=5, max_depth=2, random_state=seed).fit(X, y)
            seeds = [int(e.random_state) for e in rf.estimators_]
            cnt = np.stack([np.bincount(_generate_sample_indices(s, n, n, None), minlength=n)
                            for s in seeds]).astype(np.uint8)
            out[f"n{n}_s{seed}_seeds"] = np.asarray(seeds, np.int64)
            out[f"n{n}_s{seed}_counts"] = cnt
    import sklearn

    np.savez_compressed(HERE / "rf_bootstrap.npz", sklearn_version=sklearn.__version__, **out)
    print("bootstrap: sklearn", sklearn.__version__)


def make_trainer_metrics():
    """Reference train(..., 'random_forest') on the trainer's synthetic frame."""
    import pandas as pd
    from gpukalc_trainer import train
    from gpukalc_trainer.dataset import Dataset

    sys.path.insert(0, str(REF / "trainer" / "tests"))
    from conftest import power_frame  # the reference trainer's own generator

    out = {}
    for n, seed, depth in ((600, 3, 16), (2000, 5, 12)):
        fr = power_frame(n, seed=seed)
        feats = [c for c in fr.columns if c not in ("kernel", "power_w")]
        ds = Dataset(X=fr[feats].astype(float), y=fr["power_w"].astype(float),
                     provenance=fr[["kernel"]])
        res = train(ds, "random_forest", n_estimators=40, max_depth=depth, seed=0)
        from sklearn.model_selection import KFold

        mapes = []
        for (tr, te), _m in zip(KFold(5, shuffle=True, random_state=0).split(res.X),
                                res.fold_metrics):
            from sklearn.preprocessing import MinMaxScaler

            sc = MinMaxScaler().fit(res.X[tr])
            from sklearn.ensemble import RandomForestRegressor

            m = RandomForestRegressor(n_estimators=40, max_depth=depth, random_state=0)
            m.fit(sc.transform(res.X[tr]), res.y[tr])
            pred = m.predict(sc.transform(res.X[te]))
            mapes.append(float(np.mean(np.abs((res.y[te] - pred) / res.y[te])) * 100))
        out[f"n{n}_seed{seed}_depth{depth}"] = {
            "n_rows": n, "frame_seed": seed, "max_depth": depth, "n_estimators": 40,
            "folds": [m.as_dict() for m in res.fold_metrics], "mean": res.mean_metrics.as_dict(),
            "fold_mape_pct": mapes, "mean_mape_pct": float(np.mean(mapes)),
            "features": feats,
        }
    import sklearn

    out["sklearn_version"] = sklearn.__version__
    (HERE / "trainer_rf.json").write_text(json.dumps(out, indent=1) + "\n")
    print("trainer metrics")


def make_trainer_gbt():
    """Reference train(..., 'gradient_boosted') -- the trainer's DEFAULT family
    (training.py:67-72, sklearn GradientBoostingRegressor) -- on its own
    synthetic frame, with the same harness MAPE over the same KFold folds."""
    from gpukalc_trainer import train
    from gpukalc_trainer.dataset import Dataset
    from sklearn.ensemble import GradientBoostingRegressor
    from sklearn.model_selection import KFold
    from sklearn.preprocessing import MinMaxScaler

    sys.path.insert(0, str(REF / "trainer" / "tests"))
    from conftest import power_frame  # the reference trainer's own generator

    out = {}
    for n, seed, n_est, lr, depth in ((600, 3, 200, 0.05, None), (2000, 5, 150, 0.1, 4),
                                      (3000, 7, 100, 0.1, None)):
        fr = power_frame(n, seed=seed)
        feats = [c for c in fr.columns if c not in ("kernel", "power_w")]
        ds = Dataset(X=fr[feats].astype(float), y=fr["power_w"].astype(float),
                     provenance=fr[["kernel"]])
        res = train(ds, "gradient_boosted", n_estimators=n_est, learning_rate=lr,
                    max_depth=depth, seed=0)
        kw = {} if depth is None else {"max_depth": depth}
        mapes = []
        for tr, te in KFold(5, shuffle=True, random_state=0).split(res.X):
            sc = MinMaxScaler().fit(res.X[tr])
            m = GradientBoostingRegressor(n_estimators=n_est, learning_rate=lr, random_state=0, **kw)
            m.fit(sc.transform(res.X[tr]), res.y[tr])
            pred = m.predict(sc.transform(res.X[te]))
            mapes.append(float(np.mean(np.abs((res.y[te] - pred) / res.y[te])) * 100))
        out[f"n{n}_seed{seed}_est{n_est}_lr{lr}_depth{depth}"] = {
            "n_rows": n, "frame_seed": seed, "n_estimators": n_est, "learning_rate": lr,
            "max_depth": depth, "folds": [m.as_dict() for m in res.fold_metrics],
            "mean": res.mean_metrics.as_dict(), "fold_mape_pct": mapes,
            "mean_mape_pct": float(np.mean(mapes)), "features": feats,
            "init": float(res.model.init_.predict(np.zeros((1, len(feats))))[0]),
        }
    import sklearn

    out["sklearn_version"] = sklearn.__version__
    (HERE / "trainer_gbt.json").write_text(json.dumps(out, indent=1) + "\n")
    print("trainer gbt metrics")


if __name__ == "__main__":
    only = set(sys.argv[1:])
    if not only or "sched" in only:
        make_fixtures()
        for name, args in SETS.items():
            make_set(name, *args)
        make_trace()
    if not only:
        make_power()
        make_bootstrap()
        make_trainer_metrics()
    if not only or "gbt" in only:
        make_trainer_gbt()
