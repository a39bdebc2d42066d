"""Host-buffer energy sweep (runtime.HostSweep): corpus slices are
self-contained (CPU, oracle), and the pipelined host path returns the same
bits as the device-resident sweep over the whole grid (GPU)."""

import numpy as np
import pytest

import oracle as O
from paper_2305_01886_b200 import corpus as CG
from paper_2305_01886_b200 import pack, workloads
from paper_2305_01886_b200.ensemble import random_forest_flat
from paper_2305_01886_b200.profiles import resolve_profile


def test_corpus_slices_schedule_like_the_whole():
    c = workloads.synth_packed(60, seed=3)
    profs = [resolve_profile("k20"), resolve_profile("gtx1050")]
    cfgs = CG.CONFIG1 + [(65535, 1024, 0, 0)]
    full = O.schedule_features(O.HostGrid(c, profs, cfgs))
    parts = [c.slice(a, b) for a, b in ((0, 1), (1, 17), (17, 40), (40, 60))]
    outs = [O.schedule_features(O.HostGrid(p, profs, cfgs)) for p in parts]
    for k in ("status", "si", "sf", "feat"):
        got = np.concatenate([o[k] for o in outs])
        assert np.array_equal(full[k].view(np.uint8), got.view(np.uint8)), k
    assert c.slice(5, 5).n_ker == 0 and [n for p in parts for n in p.names] == c.names


@pytest.mark.gpu
@pytest.mark.parametrize("chunks,depth", [(1, 2), (3, 2), (7, 3), (1, 1)])
def test_host_sweep_matches_device_sweep(chunks, depth):
    import torch

    from paper_2305_01886_b200 import runtime as rt

    c = workloads.synth_packed(120, seed=9)
    profs = [resolve_profile("k20"), resolve_profile("m60")]
    cfgs = CG.config2_grid()[:20]
    sel = pack.manifest_indices(pack.SELECTED_FEATURES)
    ens = [rt.DeviceEnsemble.upload(random_forest_flat(16, 8, pack.SELECTED_FEATURES,
                                                       np.zeros(15), np.full(15, 1e4), seed=a))
           for a in range(2)]
    dc = rt.DeviceCorpus.upload(c)
    dg = rt.DeviceGrid.build(dc, profs, cfgs)
    want = [x.cpu().numpy() for x in rt.Sweep(dc, dg, ens, sel).run()]
    hs = rt.HostSweep(c, profs, cfgs, ens, sel, n_chunks=chunks, depth=depth)
    outs = [hs.submit() for _ in range(5)]   # pipelined steps reuse the slots
    hs.finish()
    torch.cuda.synchronize()
    for out in outs[-depth:]:
        got = [out[k].numpy() for k in ("status", "time_us", "power_w", "energy_uj")]
        assert np.array_equal(got[0], want[0])
        for g, w in zip(got[1:], want[1:]):
            assert np.array_equal(g.view(np.uint64), w.view(np.uint64))
    out = hs.run()
    torch.cuda.synchronize()
    assert np.array_equal(out["energy_uj"].numpy().view(np.uint64), want[3].view(np.uint64))


@pytest.mark.gpu
def test_host_rows_predictor_matches_device_walk():
    import torch

    from paper_2305_01886_b200 import runtime as rt

    rng = np.random.default_rng(4)
    n, F = 10_007, 12
    X = rng.random((n, F))
    flat = random_forest_flat(23, 7, [f"f{i}" for i in range(F)], np.zeros(F), np.ones(F), seed=2)
    de = rt.DeviceEnsemble.upload(flat)
    want, _ = rt.rf_predict(de, torch.tensor(X, device="cuda"))
    Xh = torch.from_numpy(X).pin_memory()
    out = torch.empty(n, dtype=torch.float64).pin_memory()
    hp = rt.HostRowsPredictor(de, F, chunk_rows=3000)   # 4 chunks over 2 device slots
    for _ in range(2):
        hp.run(Xh, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.numpy().view(np.uint64), want.cpu().numpy().view(np.uint64))
