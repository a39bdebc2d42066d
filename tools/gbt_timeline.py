"""Where does a gradient-boosting fit's wall time go?  torch.profiler over one
100-stage fit at 1M x 64 (bench.py's gbt_fit): GPU-busy fraction, device time
by kernel and the host calls that wait.  Tuning aid.

    python tools/gbt_timeline.py [rows] [stages]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]

import torch  # noqa: E402

from paper_2305_01886_b200.boosting import GradientBoostingRegressor as G  # noqa: E402
from paper_2305_01886_b200.workloads import config3_table  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 100
X, y = config3_table(rows)
X = (X - X.min(0)) / (X.max(0) - X.min(0))
G(5, max_depth=3, random_state=0).fit(X, y)
torch.cuda.synchronize()
t0 = time.perf_counter()
G(k, max_depth=3, random_state=0).fit(X, y)
torch.cuda.synchronize()
print(f"unprofiled fit {time.perf_counter() - t0:.3f} s")
acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=acts) as prof:
    t0 = time.perf_counter()
    G(k, max_depth=3, random_state=0).fit(X, y)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ev = prof.events()
gpu = [e for e in ev if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end) for e in gpu)
busy, cs, ce = 0.0, None, None
for s, e in iv:
    if ce is None or s > ce:
        if ce is not None:
            busy += ce - cs
        cs, ce = s, e
    else:
        ce = max(ce, e)
busy += ce - cs
print(f"profiled wall {wall * 1e3:.0f} ms, GPU busy {busy / 1e3:.0f} ms")
by = {}
for e in gpu:
    n = e.name[:60]
    d, c = by.get(n, (0.0, 0))
    by[n] = (d + e.time_range.end - e.time_range.start, c + 1)
print("device time by kernel / copy:")
for n, (d, c) in sorted(by.items(), key=lambda kv: -kv[1][0])[:14]:
    print(f"  {n:60s} {d / 1e3:8.2f} ms  x{c}")
tot = {}
for e in ev:
    if e.device_type == torch.autograd.DeviceType.CPU:
        tot[e.name] = tot.get(e.name, 0) + e.self_cpu_time_total
print("top host self time:")
for n, v in sorted(tot.items(), key=lambda kv: -kv[1])[:12]:
    print(f"  {n[:60]:60s} {v / 1e3:8.1f} ms")
# GPU idle gaps and the host ops running in them (summed by op name)
cpu = [e for e in ev if e.device_type == torch.autograd.DeviceType.CPU]
gaps, ce = [], None
for s_, e_ in iv:
    if ce is not None and s_ > ce:
        gaps.append((ce, s_))
    ce = e_ if ce is None else max(ce, e_)
print(f"idle gaps: {len(gaps)}, total {sum(b - a for a, b in gaps) / 1e3:.1f} ms")
inside = {}
for e in cpu:
    for a, b in gaps:
        ov = min(b, e.time_range.end) - max(a, e.time_range.start)
        if ov > 0:
            inside[e.name] = inside.get(e.name, 0) + ov
print("host ops overlapping the gaps (us, summed):")
for n_, v in sorted(inside.items(), key=lambda kv: -kv[1])[:16]:
    print(f"  {n_[:60]:60s} {v / 1e3:8.2f} ms")
