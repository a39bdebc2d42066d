"""Per-kernel device time of a Python workload via torch.profiler (CUPTI),
for host-orchestrated paths (forest / boosting fits).  Tuning aid.

    python tools/kernel_profile.py rf [rows] [trees] [top] [serial] | gbt [rows] [stages]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import torch  # noqa: E402

from paper_2305_01886_b200.workloads import config3_table  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "rf"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
k = int(sys.argv[3]) if len(sys.argv) > 3 else 32
X, y = config3_table(rows)
X = (X - X.min(0)) / (X.max(0) - X.min(0))
TOP = int(sys.argv[4]) if len(sys.argv) > 4 else 40
KW = {} if len(sys.argv) <= 5 else {"concurrent": False}
if what == "rf":
    from paper_2305_01886_b200.forest import RandomForestRegressor as M

    def run():
        M(k, max_depth=16, random_state=0, **KW).fit(X, y)
else:
    from paper_2305_01886_b200.boosting import GradientBoostingRegressor as M

    def run():
        M(k, learning_rate=0.1, random_state=0).fit(X, y)
run()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    run()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
tot = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name.split("(")[0][:60]
        d = tot.setdefault(name, [0, 0.0])
        d[0] += 1
        d[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
gpu = sum(v[1] for v in tot.values()) / 1e3
print(f"wall {wall * 1e3:.1f} ms, summed device time {gpu:.1f} ms")
for name, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:TOP]:
    print(f"{name:60s} {n:6d} {us / 1e3:9.2f} ms")
