"""Run K4 (standalone ensemble walk) on the c2 sweep's selected features, a few
launches, for ncu captures of the walk formats (GK_BLOCKED=0/1).  Not a bench."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

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
X = out["sel"]
ok = out["status"] == 0
lo = torch.nan_to_num(X[ok].min(0).values).cpu().numpy()
hi = torch.nan_to_num(X[ok].max(0).values).cpu().numpy()
de = rt.DeviceEnsemble.upload(random_forest_flat(500, 16, pack.SELECTED_FEATURES, lo, hi, seed=7))
for _ in range(3):
    rt.rf_predict(de, X, status=out["status"], time_us=out["sf"][:, 7])
torch.cuda.synchronize()
print("ok", de.compact)
