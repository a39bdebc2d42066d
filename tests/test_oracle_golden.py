"""CPU: the oracle (oracle/gk_oracle.c) pinned against golden vectors produced
by the reference itself, and against the reference tests' known answers.
This is what makes the oracle trustworthy as the checker of the GPU path."""

import numpy as np
import pytest

import oracle as O
from goldens import bits_equal, fixture_profile, fixtures, load_set, mismatch_report
from paper_2305_01886_b200 import abi, pack, ptx
from paper_2305_01886_b200.ensemble import flatten, load_ensemble
from paper_2305_01886_b200.profiles import resolve_profile


@pytest.mark.parametrize("name", ["c1", "c2", "rnd", "c5"])
def test_oracle_matches_reference_goldens(golden, name):
    d, gs, c, profs, cfgs = load_set(name)
    assert golden.corpus_digest(c) == str(d["corpus_sha256"]), "parser/packer drifted"
    out = O.schedule_features(O.HostGrid(c, profs, cfgs))
    assert np.array_equal(out["status"], d["status"])
    ok = d["status"] != 1
    assert np.array_equal(out["si"][ok], d["si"][ok])
    assert bits_equal(out["sf"][ok], d["sf"][ok]), mismatch_report(out["sf"][ok], d["sf"][ok],
                                                                   abi.SF_NAMES)
    ok0 = d["status"] == 0
    assert bits_equal(out["feat"][ok0], d["feat"][ok0]), mismatch_report(
        out["feat"][ok0], d["feat"][ok0], pack.FEATURE_ORDER)


def test_goldens_cover_negative_latency_and_infeasible(golden):
    d, *_ = load_set("c5")
    assert (d["sf"][:, 0] < 0).sum() > 100          # SURVEY §7.3.9 region
    d, *_ = load_set("rnd")
    assert (d["status"] == 1).sum() > 100           # infeasible launches flagged


def test_oracle_trace_matches_reference_rows(golden):
    import goldens

    t = np.load(goldens.G / "trace_k20.npz")
    gs = goldens.graphs(int(t["n_kernels"]), int(t["seed"]))
    c = pack.pack_corpus(gs)
    cfgs = [tuple(int(v) for v in r) for r in t["configs"]]
    for ki in range(len(gs)):
        out = O.schedule_features(O.HostGrid(c, [resolve_profile("k20")], cfgs, [ki]), trace=True)
        for ci in range(len(cfgs)):
            for key in ("start", "duration", "latency", "blk_delay", "blk_finish"):
                assert bits_equal(out["tr_" + key][ci], t[f"k{ki}c{ci}_{key}"]), (ki, ci, key)
            assert np.array_equal(out["tr_n_batches"][ci], t[f"k{ki}c{ci}_n_batches"])


def test_worked_example_kat():
    """pkg/tests/test_scheduler.py:34-40: starts [0,10,20,10,333,655,0], delay 665."""
    fx = fixtures()
    g = ptx.parse_ptx(fx["ptx"]["worked_example"], "pair_load_add")
    c = pack.pack_corpus([g])
    # schedule_block(profile, block, 256) with gm_latency=None -> table "global" = 315
    fp = fixture_profile()
    out = O.schedule_features(O.HostGrid(c, [fp], [(1, 256, 0, 0)], n_tw=[256],
                                         gm=[fp.latency.instructions["global"]]), trace=True)
    assert list(out["tr_start"][0]) == [0.0, 10.0, 20.0, 10.0, 333.0, 655.0, 0.0]
    assert list(out["tr_duration"][0][:6]) == [10, 10, 34, 322, 322, 10]
    assert out["tr_blk_delay"][0][0] == 665.0 == fx["kat"]["worked_delay"]
    assert list(out["tr_n_batches"][0][[0, 3, 6]]) == [2, 8, 64]
    # strict variant (no issue gap): pkg/tests/test_scheduler.py:43-46
    doc = dict(fx["fixture_profile"])
    doc["latencies"] = dict(doc["latencies"], issue_gap={})
    from paper_2305_01886_b200.profiles import profile_from_dict

    sp = profile_from_dict(doc)
    out = O.schedule_features(O.HostGrid(c, [sp], [(1, 256, 0, 0)], n_tw=[256], gm=[315.0]),
                              trace=True)
    assert list(out["tr_start"][0]) == [0.0, 10.0, 20.0, 10.0, 332.0, 654.0, 0.0]


def test_vecadd_and_nn_kats():
    fx = fixtures()
    k20 = resolve_profile("k20")
    g = ptx.parse_ptx(fx["ptx"]["vecadd"], "vecadd")
    out = O.schedule_features(O.HostGrid(pack.pack_corpus([g]), [k20], [(64, 256, 0, 0)]))
    sf = out["sf"][0]
    kat = fx["kat"]["vecadd_64x256"]
    assert sf[0] == kat["gm_latency"] and sf[6] == kat["d_total"] and sf[7] == kat["time_us"]
    # pkg/tests/test_cli.py:42-53 values
    assert sf[0] == pytest.approx(330.01552, rel=1e-12)
    assert sf[6] == pytest.approx(4022.367353605568, rel=1e-12)
    assert sf[7] == pytest.approx(5.130570604088735, rel=1e-12)
    g = ptx.parse_ptx(fx["ptx"]["nn_euclid"], "nn_euclid")
    out = O.schedule_features(O.HostGrid(pack.pack_corpus([g]), [k20], [(256, 256, 32, 0)]))
    want = fx["kat"]["nn_256x256_r32"]
    got = dict(zip(pack.FEATURE_ORDER, out["feat"][0]))
    assert got == want
    assert got["waves"] == 3 and got["comp_inst_sm"] == 57 and got["inst_issue_cycles"] == 6720.0


def test_oracle_power_matches_reference():
    import json

    import goldens

    doc = json.loads((goldens.G / "power_ensemble.json").read_text())
    p = np.load(goldens.G / "power.npz")
    d, *_ = load_set("c1")
    X = np.nan_to_num(d["feat"][:, p["sel"]])
    power, energy = O.rf_predict(flatten(load_ensemble(doc)), X, status=d["status"],
                                 time_us=np.nan_to_num(d["sf"][:, 7]))
    ok = d["status"] == 0
    assert bits_equal(power[ok], p["power"][ok])
    # batched energy is the fp64 product; reference is a decimal product (<= 1 ulp)
    np.testing.assert_allclose(energy[ok], p["energy"][ok], rtol=1e-15)


def test_oracle_fixture_ensembles():
    fx = fixtures()
    stump = flatten(load_ensemble(fx["ensembles"]["stump"]))
    pw, _ = O.rf_predict(stump, np.array([[256.0], [513.0], [512.0]]))
    assert list(pw) == [45.0, 55.0, 45.0]   # pkg/tests/test_power.py:67-71
    const = flatten(load_ensemble(fx["ensembles"]["constant"]))
    pw, _ = O.rf_predict(const, np.array([[1024.0, 1.0]]))
    assert list(pw) == [42.5]


def test_bootstrap_counts_match_sklearn():
    import goldens

    b = np.load(goldens.G / "rf_bootstrap.npz")
    for n in (1000, 4097):
        for seed in (0, 1, 42):
            seeds = b[f"n{n}_s{seed}_seeds"]
            want = b[f"n{n}_s{seed}_counts"]
            for t, s in enumerate(seeds):
                assert np.array_equal(O.bootstrap_counts(int(s), n), want[t]), (n, seed, t)
