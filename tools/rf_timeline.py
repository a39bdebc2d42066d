"""Where does a forest fit's wall time go?  torch.profiler (CPU + CUDA) over
one fit; prints the GPU-busy fraction (union of kernel / memcpy intervals),
the fit's phases and the largest GPU-idle gaps with the host ops running in
them.  Tuning aid.

    python tools/rf_timeline.py [rows] [trees]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import torch  # noqa: E402

from paper_2305_01886_b200.forest import RandomForestRegressor as M  # noqa: E402
from paper_2305_01886_b200.workloads import config3_table  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 500
X, y = config3_table(rows)
X = (X - X.min(0)) / (X.max(0) - X.min(0))
if "cold" not in sys.argv[3:]:   # `cold`: profile the process's first fit
    M(8, max_depth=16, random_state=0).fit(X, y)
torch.cuda.synchronize()
acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=acts) as prof:
    t0 = time.perf_counter()
    M(k, max_depth=16, random_state=0).fit(X, y)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ev = prof.events()
gpu = sorted((e.time_range.start, e.time_range.end) for e in ev
             if e.device_type == torch.autograd.DeviceType.CUDA)
cpu = [e for e in ev if e.device_type == torch.autograd.DeviceType.CPU]
t_lo = min(e.time_range.start for e in cpu)
t_hi = max(e.time_range.end for e in cpu)
busy, cur_s, cur_e, gaps = 0.0, None, None, []
for s, e in gpu:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, cur_e, s))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
print(f"wall {wall * 1e3:.0f} ms; profiled span {(t_hi - t_lo) / 1e3:.0f} ms; GPU busy "
      f"{busy / 1e3:.0f} ms; first GPU op at +{(gpu[0][0] - t_lo) / 1e3:.0f} ms, last ends "
      f"{(t_hi - gpu[-1][1]) / 1e3:.0f} ms before the end")
gaps.sort(reverse=True)
print(f"idle gaps: {len(gaps)}, total {sum(g[0] for g in gaps) / 1e3:.0f} ms; largest:")
for d, a, b in gaps[:12]:
    ops = {}
    for e in cpu:
        ov = min(b, e.time_range.end) - max(a, e.time_range.start)
        if ov > 0.2 * d and e.name.startswith(("aten::", "cuda", "Memcpy")) is False:
            ops[e.name] = max(ops.get(e.name, 0), ov)
    top = sorted(ops.items(), key=lambda kv: -kv[1])[:4]
    print(f"  {d / 1e3:7.2f} ms at +{(a - t_lo) / 1e3:7.1f} ms: " +
          ", ".join(f"{n[:40]} {v / 1e3:.1f}" for n, v in top))
tot = {}
for e in cpu:
    tot[e.name] = tot.get(e.name, 0) + e.self_cpu_time_total
print("top host self time:")
for n, v in sorted(tot.items(), key=lambda kv: -kv[1])[:15]:
    print(f"  {n[:60]:60s} {v / 1e3:8.1f} ms")
