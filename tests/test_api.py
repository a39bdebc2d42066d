"""The drop-in predictor face (reference names, signatures, exceptions).

KAT values are the reference tests' (pkg/tests/test_scheduler.py,
test_features.py, test_power.py, test_cli.py); CPU tests cover validation
that happens before any device call, GPU tests the device-backed results."""

import json

import pytest

from goldens import G, fixtures
import paper_2305_01886_b200 as gk
from paper_2305_01886_b200 import EnsembleError, LaunchConfig, ScheduleError


def _two_tree_doc():
    # pkg/tests/test_power.py:31-56 (same values, restated)
    return {"schema_version": 1, "base_score": 10.0,
            "feature_manifest": ["occupancy", "block_size"],
            "scaling": {"min": [0.0, 0.0], "max": [1.0, 1024.0]},
            "trees": [{"nodes": [{"feature": 0, "threshold": 0.5, "left": 1, "right": 2},
                                 {"value": 1.0},
                                 {"feature": 1, "threshold": 0.25, "left": 3, "right": 4},
                                 {"value": 2.0}, {"value": 3.0}]},
                      {"nodes": [{"feature": 1, "threshold": 0.75, "left": 1, "right": 2},
                                 {"value": 10.0}, {"value": 20.0}]}],
            "gains": [0.25, 0.75]}


# ------------------------------------------------------------------ CPU


def test_import_is_light():
    import subprocess
    import sys

    probe = ("import sys, paper_2305_01886_b200;"
             "m = {k.split('.')[0] for k in sys.modules};"
             "sys.exit(1 if m & {'sklearn', 'pandas', 'scipy', 'torch'} else 0)")
    assert subprocess.run([sys.executable, "-c", probe]).returncode == 0


def test_launch_config_validation():
    with pytest.raises(ScheduleError):
        LaunchConfig(0, 256)
    with pytest.raises(ScheduleError):
        LaunchConfig(1, 0)
    with pytest.raises(ScheduleError):
        LaunchConfig(1, 32, reg_per_thread=-1)
    assert LaunchConfig(64, 256).total_threads == 16384


def test_energy_is_decimal_exact():
    assert gk.predict_energy(5689.25, 83.28) == 473800.74
    assert gk.predict_energy(8945.25, 138.16) == 1235875.74
    with pytest.raises(EnsembleError):
        gk.predict_energy(-1.0, 1.0)
    with pytest.raises(EnsembleError):
        gk.predict_energy(1.0, -1.0)
    rep = gk.EnergyReport.build("vecadd", time_us=83.28, power_w=5689.25)
    assert rep.energy_uj == 473800.74


@pytest.mark.parametrize("mutate,match", [
    (lambda d: d.update(schema_version=2), "schema_version"),
    (lambda d: d.update(feature_manifest=[]), "non-empty"),
    (lambda d: d.update(feature_manifest=["a", "a"]), "duplicate"),
    (lambda d: d["scaling"].update(min=[0.0]), "2 entries"),
    (lambda d: d["scaling"].update(max=[-1.0, 1024.0]), "max < min"),
    (lambda d: d["trees"][0]["nodes"][0].update(left=99), "out of range"),
    (lambda d: d["trees"][0]["nodes"][0].update(feature=5), "feature index"),
    (lambda d: d["trees"][0]["nodes"][2].update(left=0), "reached twice"),
    (lambda d: d["trees"][1].update(nodes=[{"value": 1.0}, {"value": 2.0}]), "unreachable"),
    (lambda d: d["trees"][0]["nodes"][0].pop("threshold"), "threshold"),
    (lambda d: d["trees"][0].update(nodes=[]), "no nodes"),
    (lambda d: d.update(gains=[1.0]), "gains"),
    (lambda d: d.update(gains=[-0.1, 0.2]), ">= 0"),
])
def test_ensemble_validation_messages(mutate, match):
    doc = _two_tree_doc()
    mutate(doc)
    with pytest.raises(EnsembleError, match=match):
        gk.load_ensemble(doc)


def test_predict_power_input_validation_before_device():
    ens = gk.load_ensemble(_two_tree_doc())
    with pytest.raises(EnsembleError, match="2 feature values"):
        gk.predict_power(ens, [0.9])
    with pytest.raises(EnsembleError, match="block_size"):
        gk.predict_power(ens, {"occupancy": 1.0})


def test_shipped_profiles_resolve():
    assert gk.list_shipped_profiles() == ["gtx1050", "quadro_k4200", "tesla_k20", "tesla_m60"]
    p = gk.resolve_profile("k20")
    assert p.nSM == 13 and p.nu_gpu == 784.0
    with pytest.raises(gk.ProfileError, match="not found"):
        gk.resolve_profile("nope")


def test_c_abi_library_exports_every_header_symbol():
    """libgk.so loads (no GPU needed) and exports every function gk.h declares."""
    import ctypes
    import re
    from pathlib import Path

    from paper_2305_01886_b200 import runtime

    hdr = (Path(__file__).resolve().parents[1] / "include" / "gk.h").read_text()
    names = set(re.findall(r"^\s*(?:int|size_t|const char \*)\s*(gk_\w+)\(", hdr, re.M))
    assert len(names) >= 15
    lib = ctypes.CDLL(str(runtime.LIB_PATH))
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert runtime.load_library().gk_abi_version() == 5


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
def test_schedule_kernel_vecadd_golden():
    fx = fixtures()
    g = gk.parse_ptx(fx["ptx"]["vecadd"], "vecadd")
    k20 = gk.resolve_profile("k20")
    ks = gk.schedule_kernel(k20, g, LaunchConfig(64, 256))
    assert ks.waves == 1 and ks.blocks_per_sm == 8
    assert ks.gm_latency == pytest.approx(330.01552, rel=1e-12)       # test_cli.py:51
    assert ks.d_total == pytest.approx(4022.367353605568, rel=1e-12)  # test_cli.py:52
    assert ks.time_us(k20) == pytest.approx(5.130570604088735, rel=1e-12)
    assert ks.d_total == fx["kat"]["vecadd_64x256"]["d_total"]
    # per-instruction rows (the --trace face) are populated and consistent
    rows = [r for b in ks.cfg.blocks for r in b.rows]
    assert len(rows) == sum(len(b.instructions) for b in g.blocks)
    assert all(r.finish == r.start + r.duration for r in rows)
    assert ks.cfg.delay == max(ks.cfg.finish[i] for i in g.exit_blocks)


@pytest.mark.gpu
def test_schedule_kernel_infeasible_raises_reference_message():
    fx = fixtures()
    g = gk.parse_ptx(fx["ptx"]["vecadd"], "vecadd")
    with pytest.raises(ScheduleError, match="does not fit"):
        gk.schedule_kernel(gk.resolve_profile("k20"), g, LaunchConfig(1, 2048, reg_per_thread=64))


@pytest.mark.gpu
def test_extract_features_nn_euclid():
    fx = fixtures()
    g = gk.parse_ptx(fx["ptx"]["nn_euclid"], "nn_euclid")
    vec = gk.extract_features(gk.resolve_profile("k20"), g, LaunchConfig(256, 256, reg_per_thread=32))
    assert vec.as_dict() == fx["kat"]["nn_256x256_r32"]
    assert vec.waves == 3 and vec.comp_inst_sm == 57 and vec.glob_inst_sm == 12   # test_features.py:42-53
    assert vec.inst_issue_cycles == 6720.0 and vec.occupancy == 1.0


@pytest.mark.gpu
def test_predict_power_reference_cases():
    fx = fixtures()
    stump = gk.load_ensemble(fx["ensembles"]["stump"])
    assert gk.predict_power(stump, {"block_size": 256}) == 45.0     # test_power.py:67-71
    assert gk.predict_power(stump, {"block_size": 513}) == 55.0
    assert gk.predict_power(stump, {"block_size": 512}) == 45.0     # boundary goes left
    const = gk.load_ensemble(fx["ensembles"]["constant"])
    assert gk.predict_power(const, {"block_size": 256, "occupancy": 0.5}) == 42.5
    ens = gk.load_ensemble(_two_tree_doc())
    assert gk.predict_power(ens, {"occupancy": 0.4, "block_size": 900.0}) == 31.0
    assert gk.predict_power(ens, {"occupancy": 0.9, "block_size": 128.0}) == 22.0
    assert gk.predict_power(ens, [0.9, 128.0]) == 22.0
    doc = _two_tree_doc()
    doc["scaling"]["min"] = [0.7, 0.0]
    doc["scaling"]["max"] = [0.7, 1024.0]   # constant column scales to 0
    ens = gk.load_ensemble(doc)
    for occ in (0.0, 0.7, 1.0):
        assert gk.predict_power(ens, {"occupancy": occ, "block_size": 0.0}) == 21.0


@pytest.mark.gpu
def test_predict_launches_matches_scalar_faces():
    fx = fixtures()
    g = gk.parse_ptx(fx["ptx"]["vecadd"], "vecadd")
    k20 = gk.resolve_profile("k20")
    ens = gk.load_ensemble(json.loads((G / "power_ensemble.json").read_text()))
    launches = [LaunchConfig(64, 256), LaunchConfig(128, 256), LaunchConfig(65535, 1024)]
    rows = gk.predict_launches(k20, g, launches, ens)
    for L, row in zip(launches, rows):
        ks = gk.schedule_kernel(k20, g, L)
        assert row["d_total_cycles"] == ks.d_total and row["time_us"] == ks.time_us(k20)
        vec = gk.extract_features(k20, g, L)
        pw = gk.predict_power(ens, vec.as_dict())
        assert row["power_w"] == pw
        assert row["energy_uj"] == gk.predict_energy(pw, row["time_us"])


@pytest.mark.gpu
def test_staged_upload_equals_the_host_array():
    """runtime.upload (pinned staging ring): sizes below / at / above the
    staging threshold, a tail shorter than a chunk, read-only and structured
    arrays (through _dev), back-to-back calls reusing the ring."""
    import torch

    import numpy as np

    from paper_2305_01886_b200 import runtime as R

    rng = np.random.default_rng(0)
    ch = R._STAGE_CHUNK
    for nbytes in (8, R._STAGE_MIN - 8, R._STAGE_MIN, 5 * ch + 24, 13 * ch + 8):
        a = rng.random(nbytes // 8)
        d = R.upload(a)
        assert d.dtype == torch.float64 and d.shape == a.shape
        assert np.array_equal(d.cpu().numpy(), a)
    b = rng.integers(0, 255, (3 * ch, 3), dtype=np.uint8)
    b.setflags(write=False)
    assert np.array_equal(R.upload(b).cpu().numpy(), b)
    s = np.zeros(R._STAGE_MIN // 16 + 3, dtype=[("v", "<f8"), ("f", "<i4"), ("l", "<i4")])
    s["v"] = rng.random(len(s))
    s["f"] = np.arange(len(s))
    got = R._dev(s).cpu().numpy()
    assert np.array_equal(got, s.view(np.uint8).reshape(-1))
