"""Small invocations of every libgk kernel family, for compute-sanitizer
(memcheck / racecheck / initcheck).  Not a test of results (the parity tests
do that) -- a target for the sanitizers."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as G  # noqa: E402
from paper_2305_01886_b200 import corpus as CG  # noqa: E402
from paper_2305_01886_b200 import pack, runtime as rt, workloads  # noqa: E402
from paper_2305_01886_b200.boosting import GradientBoostingRegressor  # noqa: E402
from paper_2305_01886_b200.ensemble import random_forest_flat  # noqa: E402
from paper_2305_01886_b200.forest import RandomForestRegressor  # noqa: E402
from paper_2305_01886_b200.profiles import resolve_profile  # noqa: E402
from paper_2305_01886_b200.pruning import kendall_matrix, pearson_matrix  # noqa: E402

G.smoke()                                                  # K1, K3 (+trace off), fused sweep
c = workloads.synth_packed(40, seed=2)
profs = [resolve_profile("k20"), resolve_profile("m60"), resolve_profile("gtx1050"),
         resolve_profile("k4200"), resolve_profile("k20")]     # 5 archs: K1 wide path
dc = rt.DeviceCorpus.upload(c)
dg = rt.DeviceGrid.build(dc, profs, CG.config2_grid()[:10])
sel = pack.manifest_indices(pack.SELECTED_FEATURES)
rt.schedule_features(dc, dg, sel_idx=sel)                  # K3 non-fused
dg1 = rt.DeviceGrid.build(dc, profs[:1], CG.config2_grid()[:4], kernel_ids=[3])
rt.schedule_features(dc, dg1, sel_idx=sel, trace=True)     # K3 with the trace rows
rng = np.random.default_rng(0)
X = rng.random((5000, 15))
for layout in ("nodes", "nodes8", "blocks"):
    flat = random_forest_flat(11, 8, pack.SELECTED_FEATURES, np.zeros(15), np.ones(15), seed=1)
    de = rt.DeviceEnsemble.upload(flat, layout=layout)
    rt.rf_predict(de, torch.tensor(X, device="cuda"))      # K4 (+ compact walks)
Xf, y = rng.random((3000, 8)), rng.random(3000)
RandomForestRegressor(5, max_depth=6, random_state=0).fit(Xf, y)   # K5 (medium / mid / small / tiny)
X64, y64 = rng.random((20000, 64)), rng.random(20000)
RandomForestRegressor(3, max_depth=14, random_state=0).fit(X64, y64)  # K5 F = 64: vector paths, fused partitions
Xb, yb = rng.random((60000, 8)), rng.random(60000)
RandomForestRegressor(2, max_depth=2, random_state=0).fit(Xb, yb)  # K5 big-node path
GradientBoostingRegressor(5, random_state=0).fit(Xf, y)            # K5 + gb_step
GradientBoostingRegressor(3, max_depth=3, random_state=0).fit(Xb, yb)  # gb_step CTA reduction, big leaves
GradientBoostingRegressor(2, max_depth=None, random_state=0).fit(Xf, y)  # many leaves (bounded grids)
RandomForestRegressor(2, max_depth=6, random_state=0).fit(np.tile(Xb, (2, 1)),
                                                          np.tile(yb, 2))  # sibling subtraction
Xw = rng.random((600, 300))
mw = RandomForestRegressor(2, max_depth=5, random_state=0).fit(Xw, rng.random(600))
mw.predict(Xw[:200])                                               # K4 fp64 nodes, 32-row tiles
flat3 = random_forest_flat(7, 9, pack.SELECTED_FEATURES, np.zeros(15), np.ones(15), seed=3)
rt.rf_predict(rt.DeviceEnsemble.upload(flat3, layout="blocks3"), torch.tensor(X, device="cuda"))
rt.upload(rng.random(5 * rt._STAGE_CHUNK // 8 + 3))                # staged upload ring
Xk = np.round(rng.random((2000, 5)) * 10)
kendall_matrix(Xk)
pearson_matrix(Xk)                                                 # correlation kernels
hs = rt.HostSweep(c, profs[:2], CG.config2_grid()[:8],
                  [rt.DeviceEnsemble.upload(random_forest_flat(6, 5, pack.SELECTED_FEATURES,
                                                               np.zeros(15), np.ones(15), seed=a))
                   for a in range(2)], sel)
hs.run()
torch.cuda.synchronize()
print("sanitize target done")
