"""Time each stage (K1, K2/K3, K4) of the c2 workload on the GPU with CUDA
events, no host work between launches.  Tuning aid; not the bench."""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2305_01886_b200 import corpus as CG  # noqa: E402
from paper_2305_01886_b200 import pack, runtime as rt, workloads  # noqa: E402
from paper_2305_01886_b200.ensemble import random_forest_flat  # noqa: E402
from paper_2305_01886_b200.profiles import resolve_profile  # noqa: E402

n_k = int(os.environ.get("NK", 10000))
c = workloads.synth_packed(n_k, seed=1000)
dc = rt.DeviceCorpus.upload(c)
dg = rt.DeviceGrid.build(dc, [resolve_profile("tesla_k20")], CG.config2_grid())
sel = pack.manifest_indices(pack.SELECTED_FEATURES)
out = rt.schedule_features(dc, dg, si=False, sf=True, feat=False, sel_idx=sel)
torch.cuda.synchronize()
res = {}
for name, fn in (("k23", lambda: rt.schedule_features(dc, dg, si=False, sf=True, feat=False,
                                                        sel_idx=sel)),):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / 5
if os.environ.get("RF", "1") == "1":
    X = out["sel"]
    ok = out["status"] == 0
    lo = torch.nan_to_num(X[ok].min(0).values).cpu().numpy()
    hi = torch.nan_to_num(X[ok].max(0).values).cpu().numpy()
    flat = random_forest_flat(500, 16, pack.SELECTED_FEATURES, lo, hi, seed=7)
    de = rt.DeviceEnsemble.upload(flat)
    for _ in range(2):
        rt.rf_predict(de, X, status=out["status"], time_us=out["sf"][:, 7])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        rt.rf_predict(de, X, status=out["status"], time_us=out["sf"][:, 7])
    e1.record()
    torch.cuda.synchronize()
    res["k4"] = e0.elapsed_time(e1) / 5
    sw = rt.Sweep(dc, dg, [de], sel)
    for _ in range(2):
        sw.run()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        sw.run()
    e1.record()
    torch.cuda.synchronize()
    res["sweep"] = e0.elapsed_time(e1) / 5
    res["fused"] = os.environ.get("GK_SWEEP_FUSED", "1")
res["smem_rows"] = os.environ.get("GK_SMEM_ROWS", "default")
res["points"] = dg.n_points
print(json.dumps(res))
