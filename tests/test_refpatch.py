"""tools/refpatch.py (the reference suites on the device path) binds every
hot-path name it documents -- checked here in the build container, where the
reference is importable; the suites themselves run on a GPU box
(tools/refsuite.sh, results in profiles/r1/refsuite_*.txt)."""

import importlib
import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference sources absent (GPU box)")


def test_plugin_rebinds_hot_path_names(monkeypatch):
    monkeypatch.syspath_prepend(str(REF / "src"))
    monkeypatch.syspath_prepend(str(REF / "trainer" / "src"))
    for m in [m for m in sys.modules if m.startswith(("gpukalc", "tools.refpatch"))]:
        monkeypatch.delitem(sys.modules, m)
    rp = importlib.import_module("tools.refpatch")
    rp.install(warm=False)
    import gpukalc
    import gpukalc.features as F
    import gpukalc.power as P
    import gpukalc.scheduler as S
    import gpukalc_trainer.dataset as D
    import gpukalc_trainer.training as T

    assert S.schedule_kernel is rp.schedule_kernel and gpukalc.schedule_kernel is rp.schedule_kernel
    assert S.schedule_block is rp.schedule_block and S.schedule_cfg is rp.schedule_cfg
    assert F.extract_features is rp.extract_features and F.features_to_csv is rp.features_to_csv
    assert F.features_from_csv is rp.features_from_csv
    assert P.load_ensemble is rp.load_ensemble and P.predict_power is rp.predict_power
    assert T._make_model is rp._make_model and D.prune_correlated is rp.prune_correlated
    assert len(rp.PATCHED) >= 20
    # the estimators it hands the trainer are this package's, sklearn-shaped
    m = rp._make_model("random_forest", 3, 0.1, 4, 0)
    assert type(m).__module__ == "paper_2305_01886_b200.forest" and m.n_estimators == 3
    # the CSV adapters run on the host library (no GPU needed)
    text = F.features_to_csv([])
    assert text.startswith("kernel,avg_comp_lat,")
    assert F.features_from_csv(text) == []
