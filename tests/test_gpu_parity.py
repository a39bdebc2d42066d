"""GPU parity: libgk (sm_100a) through its C-ABI vs the reference's golden
vectors and vs the CPU oracle on the same seeded inputs.

Bar (BASELINE.json): features and cycles bit-exact (float64 bit patterns),
power/energy within 1e-5 relative given identical trees (here: bit-exact
power -- leaves are summed in tree order -- and energy within 1 ulp-scale
rtol 1e-15 of the reference's decimal product)."""

import json
import random

import numpy as np
import pytest

import oracle as O
from goldens import G, bits_equal, fixture_profile, fixtures, graphs, load_set, mismatch_report
from paper_2305_01886_b200 import abi, corpus, pack, ptx
from paper_2305_01886_b200.ensemble import flatten, load_ensemble, random_forest_flat
from paper_2305_01886_b200.profiles import resolve_profile

pytestmark = pytest.mark.gpu


def _rt():
    from paper_2305_01886_b200 import runtime

    return runtime


def _run(c, profs, cfgs, kernel_ids=None, trace=False, sel_idx=None, n_tw=None, gm=None):
    rt = _rt()
    dc = rt.DeviceCorpus.upload(c)
    dg = rt.DeviceGrid.build(dc, profs, cfgs, kernel_ids, n_tw=n_tw, gm=gm)
    out = rt.schedule_features(dc, dg, trace=trace, sel_idx=sel_idx)
    return {k: v.cpu().numpy() for k, v in out.items()}


def _assert_same(got, want, status_ref):
    assert np.array_equal(got["status"], status_ref)
    ok = status_ref != 1
    assert np.array_equal(got["si"][ok], want["si"][ok])
    assert bits_equal(got["sf"][ok], want["sf"][ok]), mismatch_report(
        got["sf"][ok], want["sf"][ok], abi.SF_NAMES)
    ok0 = status_ref == 0
    assert bits_equal(got["feat"][ok0], want["feat"][ok0]), mismatch_report(
        got["feat"][ok0], want["feat"][ok0], pack.FEATURE_ORDER)


@pytest.mark.parametrize("name", ["c1", "c2", "rnd", "c5"])
def test_device_matches_reference_goldens(name):
    d, gs, c, profs, cfgs = load_set(name)
    got = _run(c, profs, cfgs)
    _assert_same(got, d, d["status"])
    ks = got["kstat"].view(pack.KSTAT_DT)
    assert len(ks) == len(gs)


def test_device_static_features_match_oracle():
    d, gs, c, profs, cfgs = load_set("c1")
    got = _run(c, profs, cfgs)
    ks, ls = O.static_features(O.HostGrid(c, profs, cfgs))
    assert np.array_equal(got["kstat"].view(pack.KSTAT_DT), ks)
    assert bits_equal(got["latsum"], ls)


def test_device_trace_matches_reference_rows():
    t = np.load(G / "trace_k20.npz")
    gs = graphs(int(t["n_kernels"]), int(t["seed"]))
    c = pack.pack_corpus(gs)
    cfgs = [tuple(int(v) for v in r) for r in t["configs"]]
    for ki in range(len(gs)):
        out = _run(c, [resolve_profile("k20")], cfgs, [ki], trace=True)
        for ci in range(len(cfgs)):
            for key in ("start", "duration", "latency", "blk_delay", "blk_finish"):
                assert bits_equal(out["tr_" + key][ci], t[f"k{ki}c{ci}_{key}"]), (ki, ci, key)
            assert np.array_equal(out["tr_n_batches"][ci], t[f"k{ki}c{ci}_n_batches"])


def test_worked_example_on_device():
    """pkg/tests/test_scheduler.py:34-46 through the block-level override face."""
    fx = fixtures()
    g = ptx.parse_ptx(fx["ptx"]["worked_example"], "pair_load_add")
    c = pack.pack_corpus([g])
    fp = fixture_profile()
    out = _run(c, [fp], [(1, 256, 0, 0)], trace=True, n_tw=[256], gm=[315.0])
    assert list(out["tr_start"][0]) == [0.0, 10.0, 20.0, 10.0, 333.0, 655.0, 0.0]
    assert out["tr_blk_delay"][0][0] == 665.0


@pytest.mark.parametrize("seed,n_k,n_cfg", [(101, 300, 37), (102, 64, 256)])
def test_device_matches_oracle_random_grids(seed, n_k, n_cfg):
    rng = random.Random(seed)
    gs = [ptx.parse_ptx(t, n, loop_counts=l) for n, t, l in corpus.synth_corpus(n_k, seed)]
    c = pack.pack_corpus(gs)
    profs = [resolve_profile(a) for a in ("k20", "m60", "1050", "k4200")]
    cfgs = corpus.random_configs(rng, n_cfg)
    got = _run(c, profs, cfgs)
    want = O.schedule_features(O.HostGrid(c, profs, cfgs))
    _assert_same(got, want, want["status"])


def test_device_long_blocks_use_global_scratch():
    """Blocks longer than the shared-memory slab (48 instructions) and kernels
    with many blocks take the global-scratch path; results must not change."""
    rng = random.Random(5)
    texts = []
    for k in range(12):
        n = rng.choice([60, 130, 400, 900])
        body = []
        for i in range(n):
            body.append(rng.choice([
                f"add.s32 %r{i + 10}, %r{rng.randint(1, i + 9)}, %r{rng.randint(1, i + 9)};",
                f"ld.global.f32 %f{i + 10}, [%rd{rng.randint(1, 3)}];",
                f"st.shared.f32 [%rd2], %f{rng.randint(1, i + 9)};",
                f"fma.rn.f64 %fd{i + 10}, %fd1, %fd2, %fd{rng.randint(1, i + 9)};",
                f"sqrt.rn.f32 %f{i + 10}, %f{rng.randint(1, i + 9)};",
                "bar.sync 0;"]))
        texts.append((f"long{k}", ".entry long%d() {\n%s\nret;\n}" % (k, "\n".join(body))))
    # a kernel with 40 small blocks
    blocks = []
    for b in range(40):
        blocks.append(f"$L{b}:\n add.s32 %r{b + 2}, %r{b + 1}, 1;\n setp.lt.s32 %p1, %r{b + 2}, 7;\n"
                      f" @%p1 bra $L{b + 1};")
    texts.append(("many", ".entry many() {\n%s\n$L40:\nret;\n}" % "\n".join(blocks)))
    gs = [ptx.parse_ptx(t, n) for n, t in texts]
    c = pack.pack_corpus(gs)
    assert c.max_n > 48 and c.max_blk >= 40
    profs = [resolve_profile("k20"), resolve_profile("m60")]
    cfgs = corpus.CONFIG1 + [(65535, 1024, 0, 0), (7, 96, 0, 0)]
    got = _run(c, profs, cfgs)
    want = O.schedule_features(O.HostGrid(c, profs, cfgs))
    _assert_same(got, want, want["status"])


def test_selected_feature_output():
    d, gs, c, profs, cfgs = load_set("c1")
    sel = pack.manifest_indices(pack.SELECTED_FEATURES)
    got = _run(c, profs, cfgs, sel_idx=sel)
    ok = d["status"] == 0
    assert bits_equal(got["sel"][ok], d["feat"][ok][:, sel])


# ------------------------------------------------------------- inference


def test_rf_predict_matches_reference_power():
    rt = _rt()
    import torch

    doc = json.loads((G / "power_ensemble.json").read_text())
    p = np.load(G / "power.npz")
    d, *_ = load_set("c1")
    X = torch.tensor(np.nan_to_num(d["feat"][:, p["sel"]]), device="cuda")
    de = rt.DeviceEnsemble.upload(flatten(load_ensemble(doc)))
    st = torch.tensor(d["status"], device="cuda")
    tu = torch.tensor(np.nan_to_num(d["sf"][:, 7]), device="cuda")
    power, energy = rt.rf_predict(de, X, status=st, time_us=tu)
    power, energy = power.cpu().numpy(), energy.cpu().numpy()
    ok = d["status"] == 0
    assert bits_equal(power[ok], p["power"][ok])
    np.testing.assert_allclose(energy[ok], p["energy"][ok], rtol=1e-15)


@pytest.mark.parametrize("n_rows,ld", [(1, 15), (1000, 15), (4099, 64), (777, 20)])
def test_rf_predict_random_forest_matches_oracle(n_rows, ld):
    rt = _rt()
    import torch

    rng = np.random.default_rng(n_rows)
    nf = 15 if ld == 20 else ld
    flat = random_forest_flat(37, 10, [f"f{i}" for i in range(nf)], np.zeros(nf), np.ones(nf),
                              seed=n_rows)
    X = rng.random((n_rows, ld)) * 1.2 - 0.1
    X[: min(5, n_rows), 0] = 0.5  # exact-threshold-ish values
    de = rt.DeviceEnsemble.upload(flat)
    p_dev, _ = rt.rf_predict(de, torch.tensor(X, device="cuda"))
    p_ref, _ = O.rf_predict(flat, X[:, :nf] if ld == 20 else X)
    assert bits_equal(p_dev.cpu().numpy(), p_ref)


def test_rf_fixture_ensembles_on_device():
    rt = _rt()
    import torch

    fx = fixtures()
    st = rt.DeviceEnsemble.upload(flatten(load_ensemble(fx["ensembles"]["stump"])))
    p, _ = rt.rf_predict(st, torch.tensor([[256.0], [513.0], [512.0], [768.0]], dtype=torch.float64, device="cuda"))
    assert p.cpu().tolist() == [45.0, 55.0, 45.0, 55.0]
    cst = rt.DeviceEnsemble.upload(flatten(load_ensemble(fx["ensembles"]["constant"])))
    p, _ = rt.rf_predict(cst, torch.tensor([[1024.0, 1.0]], dtype=torch.float64, device="cuda"))
    assert p.cpu().tolist() == [42.5]


def test_fused_sweep_matches_oracle_pipeline():
    rt = _rt()
    d, gs, c, profs, cfgs = load_set("c5")
    sel = pack.manifest_indices(pack.SELECTED_FEATURES)
    flats = [random_forest_flat(24, 9, pack.SELECTED_FEATURES, np.zeros(15),
                                np.nanmax(np.nan_to_num(d["feat"][:, sel]), axis=0) + 1.0, seed=a)
             for a in range(len(profs))]
    dc = rt.DeviceCorpus.upload(c)
    dg = rt.DeviceGrid.build(dc, profs, cfgs)
    sw = rt.Sweep(dc, dg, [rt.DeviceEnsemble.upload(f) for f in flats], sel)
    status, t_us, power, energy = [x.cpu().numpy() for x in sw.run()]
    assert np.array_equal(status, d["status"])
    ok = status == 0
    assert bits_equal(t_us[ok], d["sf"][ok, 7])
    n_cfg, n_arch = len(cfgs), len(profs)
    arch_of = (np.arange(len(status)) // n_cfg) % n_arch
    for a in range(n_arch):
        m = ok & (arch_of == a)
        pw, en = O.rf_predict(flats[a], d["feat"][m][:, sel], time_us=d["sf"][m, 7])
        assert bits_equal(power[m], pw)
        assert bits_equal(energy[m], en)


def test_config5_first_1000_kernels_every_point():
    """SURVEY §8(d) #5 parity bar: all points of the first 1,000 kernels of
    config #5 (seed 5; 256 configs x {k20, m60, gtx1050} = 768,000 points)
    bit-exact against the oracle -- cycles, schedule scalars, all 32 features --
    and the fused sweep's time / power / energy on the same grid."""
    from paper_2305_01886_b200 import workloads

    rt = _rt()
    c = workloads.synth_packed(1000, seed=5)
    profs = [resolve_profile(a) for a in ("tesla_k20", "tesla_m60", "gtx1050")]
    cfgs = corpus.config5_grid()
    got = _run(c, profs, cfgs)
    want = O.schedule_features(O.HostGrid(c, profs, cfgs))
    assert len(want["status"]) == 768_000
    _assert_same(got, want, want["status"])
    assert (want["status"] == 0).sum() > 700_000
    sel = pack.manifest_indices(pack.SELECTED_FEATURES)
    ok = want["status"] == 0
    hi = np.nanmax(np.where(ok[:, None], want["feat"][:, sel], np.nan), axis=0) + 1.0
    flats = [random_forest_flat(32, 12, pack.SELECTED_FEATURES, np.zeros(15), hi, seed=50 + a)
             for a in range(3)]
    dc = rt.DeviceCorpus.upload(c)
    dg = rt.DeviceGrid.build(dc, profs, cfgs)
    sw = rt.Sweep(dc, dg, [rt.DeviceEnsemble.upload(f) for f in flats], sel)
    status, t_us, power, energy = [x.cpu().numpy() for x in sw.run()]
    assert np.array_equal(status, want["status"])
    assert bits_equal(t_us[ok], want["sf"][ok, 7])
    arch_of = (np.arange(len(status)) // len(cfgs)) % 3
    for a in range(3):
        m = ok & (arch_of == a)
        pw, en = O.rf_predict(flats[a], want["feat"][m][:, sel], time_us=want["sf"][m, 7])
        assert bits_equal(power[m], pw)
        assert bits_equal(energy[m], en)


def test_throughput_clamps_counted_and_logged(caplog):
    """A throughput model that goes non-positive is clamped to tp_floor
    (profiles.py:173-181, the reference warns per call): the device counts the
    clamps, the batched face logs them once, results equal the oracle's."""
    import logging

    from paper_2305_01886_b200 import api
    from paper_2305_01886_b200.profiles import profile_from_dict, profile_to_dict

    doc = profile_to_dict(resolve_profile("k20"))
    doc["throughput_models"]["global"]["b"] = 0.5   # a (b - exp(-c n)) < 0 for small n
    prof = profile_from_dict(doc)
    gs = graphs(6, 41)
    cfgs = [(1, 32, 0, 0), (4, 64, 0, 0), (64, 256, 0, 0)]
    with caplog.at_level(logging.WARNING):
        got = api.schedule_batch([prof], gs, cfgs)
    msgs = [r.getMessage() for r in caplog.records if "clamped to tp_floor" in r.getMessage()]
    assert len(msgs) == 1 and int(msgs[0].split(" times")[0].rsplit(" ", 1)[1]) > 0
    want = O.schedule_features(O.HostGrid(pack.pack_corpus(gs), [prof], cfgs))
    assert np.array_equal(got["status"], want["status"])
    ok = want["status"] == 0
    assert bits_equal(got["sf"][ok], want["sf"][ok]) and bits_equal(got["feat"][ok], want["feat"][ok])


def test_throughput_clamp_counters_are_per_grid():
    """Reentrancy: two grids swept concurrently on two streams
    count their own clamps (gk_grid.tp_clamps; no library-global counter)."""
    import torch

    from paper_2305_01886_b200 import runtime as rt
    from paper_2305_01886_b200.profiles import profile_from_dict, profile_to_dict

    doc = profile_to_dict(resolve_profile("k20"))
    doc["throughput_models"]["global"]["b"] = 0.5
    bad = profile_from_dict(doc)
    gs = graphs(6, 41)
    cfgs = [(1, 32, 0, 0), (4, 64, 0, 0), (64, 256, 0, 0)]
    dc = rt.DeviceCorpus.upload(pack.pack_corpus(gs))
    g_bad = rt.DeviceGrid.build(dc, [bad], cfgs)
    g_ok = rt.DeviceGrid.build(dc, [resolve_profile("k20")], cfgs)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s1):
            rt.schedule_features(dc, g_bad, stream=s1)
        with torch.cuda.stream(s2):
            rt.schedule_features(dc, g_ok, stream=s2)
    torch.cuda.synchronize()
    n_bad = rt.throughput_clamps(g_bad, reset=False)
    assert n_bad > 0 and n_bad % 3 == 0
    assert rt.throughput_clamps(g_ok) == 0
    assert rt.throughput_clamps(g_bad, reset=True) == n_bad
    assert rt.throughput_clamps(g_bad) == 0


def test_many_archs_and_single_point_grids():
    """n_arch > 4 takes K1's wide latency-sum path; a 1 x 1 x 1 grid; the
    per-arch tables of duplicated profiles stay independent."""
    from paper_2305_01886_b200.profiles import profile_from_dict, profile_to_dict

    gs = [ptx.parse_ptx(t, n, loop_counts=l) for n, t, l in corpus.synth_corpus(40, 77)]
    c = pack.pack_corpus(gs)
    base = [resolve_profile(a) for a in ("k20", "m60", "1050", "k4200")]
    doc = profile_to_dict(base[0])
    doc["latencies"]["issue_gap"] = {}
    doc["name"] = "k20_nogap"
    profs = base + [profile_from_dict(doc), fixture_profile(), base[2]]
    cfgs = corpus.random_configs(random.Random(7), 9)
    got = _run(c, profs, cfgs)
    want = O.schedule_features(O.HostGrid(c, profs, cfgs))
    _assert_same(got, want, want["status"])
    one = pack.pack_corpus(gs[:1])
    got1 = _run(one, base[:1], [(13, 128, 32, 0)])
    want1 = O.schedule_features(O.HostGrid(one, base[:1], [(13, 128, 32, 0)]))
    _assert_same(got1, want1, want1["status"])


def test_empty_inputs():
    """Zero kernels and zero rows are valid batches: empty outputs, no launch errors."""
    rt = _rt()
    import torch

    got = _run(pack.pack_corpus([]), [resolve_profile("k20")], corpus.config2_grid())
    assert got["status"].shape == (0,) and got["feat"].shape[0] == 0
    flat = random_forest_flat(5, 6, ["a", "b"], np.zeros(2), np.ones(2), seed=3)
    de = rt.DeviceEnsemble.upload(flat)
    p, e = rt.rf_predict(de, torch.zeros((0, 2), dtype=torch.float64, device="cuda"),
                         time_us=torch.zeros(0, dtype=torch.float64, device="cuda"))
    assert p.shape == (0,) and e.shape == (0,)
    torch.cuda.synchronize()
