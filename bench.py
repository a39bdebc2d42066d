"""bench.py -- batched energy-prediction throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c5s] [--kernels N_KERNELS]

Workload (default "c2"): BASELINE.json configs[1] -- 10k synthetic kernels x the
64-config launch grid on the tesla_k20 profile (640k points per GPU) -- run
through the FULL energy pipeline (static features K1 -> cycle estimator +
features K2/K3 -> 500-tree depth-16 ensemble K4 -> energy K6), because the
metric is energy-prediction points/s.  "c5s" is one GPU's slice of configs[4]
(256 configs x 3 archs, one ensemble per arch) with the kernel count chosen by
--kernels.  A step = one sweep over the GPU's points with inputs resident in
HBM.  Multi-GPU (torchrun): every rank sweeps its own kernel shard (weak
scaling, no data-path collective); time = max over ranks.

One JSON line on rank 0.  See DESIGN.md §Measurement for the byte accounting.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]

PEAKS = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0


TRAFFIC = ROOT / "profiles" / "r1" / "traffic.json"


def ncu_traffic(workload: str, kernel: str, units: int):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/r1/traffic.json), scaled per unit to this launch's size."""
    try:
        rec = json.loads(TRAFFIC.read_text())[workload][kernel]
    except Exception:
        return None, None
    per_unit = (rec["read"] + rec["write"]) / rec["units"]
    src = f"ncu --set full, {rec['capture']}"
    if rec["units"] != units:
        src += f"; scaled from {rec['units']} to {units} {rec['unit']}s"
    if rec.get("binding"):
        src += f"; binding unit (ncu): {rec['binding']}"
    return per_unit * units, src


def hbm_peak():
    try:
        return float(json.loads(PEAKS.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append([time.perf_counter()] + parts)

    def window(self, t0: float, t1: float):
        """Keep the samples taken inside [t0, t1] (the timed region); if the
        region is shorter than the sampling period keep the busy samples around it."""
        inside = [r for r in self.rows if t0 <= r[0] <= t1]
        self.scope = "timed region"
        if not inside:
            inside = [r for r in self.rows if r[0] >= t0 - 1.0]
            self.scope = "timed region +/- 1 s (region shorter than the 100 ms period)"
        self.rows = inside

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        rows = [r[1:] for r in self.rows]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[4:8]) if v == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "scope": getattr(self, "scope", "all")}


# --------------------------------------------------------------- workload


def build_workload(args, rank: int):
    from paper_2305_01886_b200 import corpus as CG
    from paper_2305_01886_b200 import pack, workloads
    from paper_2305_01886_b200.profiles import resolve_profile

    if args.workload == "c2":
        n_k = args.kernels or 10000
        cfgs = CG.config2_grid()
        archs = ["tesla_k20"]
    elif args.workload == "c5s":
        n_k = args.kernels or 2000
        cfgs = CG.config5_grid()
        archs = ["tesla_k20", "tesla_m60", "gtx1050"]
    else:
        raise SystemExit(f"unknown workload {args.workload}")
    t0 = time.time()
    c = workloads.synth_packed(n_k, seed=1000 + rank)
    profs = [resolve_profile(a) for a in archs]
    sel = pack.manifest_indices(pack.SELECTED_FEATURES)
    return {"corpus": c, "profiles": profs, "configs": cfgs, "archs": archs, "sel": sel,
            "n_k": n_k, "build_s": time.time() - t0}


def make_ensembles(W, dc, dg, rt, n_trees, depth):
    """Declared synthetic ensembles: n_trees random trees of
    depth `depth` (~109k nodes each at depth 16), scaling bounds = min/max of the
    workload's own features (what MinMaxScaler would fit)."""
    import torch

    from paper_2305_01886_b200 import pack
    from paper_2305_01886_b200.ensemble import random_forest_flat

    if dg.n_points > 100_000_000:   # bounds from a kernel subset (the full selection would be ~92 GB at config #5)
        sub = rt.DeviceGrid.build(dc, W["profiles"], W["configs"],
                                  kernel_ids=np.arange(min(dg.n_k, 100_000_000 // (dg.n_points // dg.n_k))))
        out = rt.schedule_features(dc, sub, si=False, sf=False, feat=False, sel_idx=W["sel"])
    else:
        out = rt.schedule_features(dc, dg, si=False, sf=False, feat=False, sel_idx=W["sel"])
    X = out["sel"]
    ok = out["status"] == 0
    Xo = X[ok]
    lo = torch.nan_to_num(Xo.min(dim=0).values).cpu().numpy()
    hi = torch.nan_to_num(Xo.max(dim=0).values).cpu().numpy()
    flats = [random_forest_flat(n_trees, depth, pack.SELECTED_FEATURES, lo, hi, seed=7 + a)
             for a in range(len(W["profiles"]))]
    return flats


# ----------------------------------------------------------------- ours


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2305_01886_b200 import runtime as rt

    torch.cuda.set_device(local_rank)
    W = build_workload(args, rank)
    c = W["corpus"]
    dc = rt.DeviceCorpus.upload(c)
    dg = rt.DeviceGrid.build(dc, W["profiles"], W["configs"])
    n_pts = dg.n_points
    flats = make_ensembles(W, dc, dg, rt, args.trees, args.depth)
    ens = [rt.DeviceEnsemble.upload(f, layout=os.environ.get("GK_WALK_LAYOUT")) for f in flats]
    sweep = rt.Sweep(dc, dg, ens, W["sel"])
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    # ---- timed: K steps, device events per step, L2 flushed (untimed) between steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        t_w = time.perf_counter()
        while True:  # warm-up (>= W steps, and >= 1 s so the clock sampler is running)
            for _ in range(args.warmup):
                sweep.run()
            torch.cuda.synchronize()
            if time.perf_counter() - t_w > 1.0:
                break
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(args.steps):
            flush.zero_()
            evs[k][0].record(stream)
            sweep.run()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        time.sleep(0.25)
    clk.window(t0, t1)
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(sum(step_ms))

    # ---- per-kernel split (same stream, events between launches)
    split = per_kernel_split(rt, dc, dg, sweep, W, flush, args.steps)

    # ---- config #2 as BASELINE words it: the cycle estimator alone (K1 + K3,
    # every KernelSchedule scalar out, no features / power), same grid
    cyc = cycle_sweep(rt, dc, dg, flush, args.steps, world)

    # ---- e2e: host buffers in, results out, through the C-ABI per step
    e2e = run_e2e(rt, W, ens, args.steps, flush)
    # the host-buffer path returns the same bits as the device-resident sweep
    st_d, tu_d, pw_d, en_d = (x.cpu().numpy() for x in sweep.run())
    torch.cuda.synchronize()
    o = e2e.pop("out")
    assert np.array_equal(o["status"].numpy(), st_d)
    assert np.array_equal(o["energy_uj"].numpy().view(np.uint64), en_d.view(np.uint64))

    # ---- reductions across ranks (max time, sum of points)
    t = torch.tensor([total_ms, e2e["ms"]], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, e2e_ms = float(t[0]), float(t[1])
    st = sweep.status.cpu().numpy()
    return {"W": W, "n_pts": n_pts, "total_ms": total_ms, "step_ms": step_ms, "split": split,
            "e2e_ms": e2e_ms, "e2e": e2e, "clk": clk.summary(), "flats": flats, "cycle": cyc,
            "infeasible": int((st != 0).sum()), "dc_bytes": dc.nbytes}


def cycle_sweep(rt, dc, dg, flush, steps, world):
    """K1 + K3 over the grid writing status + the 6 int64 / 9 fp64 schedule
    outputs per point (schedule_kernel's KernelSchedule scalars), no features,
    no ensemble: BASELINE configs[1]'s "cycle-estimator-only sweep"."""
    import torch
    import torch.distributed as dist

    for _ in range(3):
        rt.schedule_features(dc, dg, feat=False)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for k in range(steps):
        flush.zero_()
        evs[k][0].record(stream)
        rt.schedule_features(dc, dg, feat=False)
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([sum(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    return {"value": dg.n_points * world * steps / (ms / 1e3), "unit": "points/s",
            "ms_per_step": ms / steps, "kernels": "k1_static + k23_schedule (status, si[6], sf[9])",
            "gpu_launches": 2 * steps}


def per_kernel_split(rt, dc, dg, sweep, W, flush, steps):
    """Average device time of each stage of the sweep: CUDA events recorded by
    libgk between its launches on the launching stream (no host work between)."""
    acc = {}
    n = max(steps, 1)
    for _ in range(n):
        flush.zero_()
        for k, v in sweep.stage_ms().items():
            acc[k] = acc.get(k, 0.0) + v / n
    return acc


def run_e2e(rt, W, ens, steps, flush):
    """Reference-facing call with HOST buffers (runtime.HostSweep): every step
    copies the pinned host corpus to the device, sweeps, and copies (status,
    time, power, energy) back to pinned host memory -- all inside the timing.
    Steps are submitted back to back (double-buffered), so step s + 1's H2D and
    step s - 1's D2H overlap step s's sweep on the copy engines."""
    import os

    import torch

    hs = rt.HostSweep(W["corpus"], W["profiles"], W["configs"], ens, W["sel"],
                      n_chunks=int(os.environ.get("GK_E2E_CHUNKS", "1")))
    stream = torch.cuda.current_stream()
    for _ in range(2):
        hs.submit()
    hs.finish()
    torch.cuda.synchronize()
    flush.zero_()  # inputs come from host memory every step; L2 starts cold once
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        hs.submit()
    hs.finish()
    b.record(stream)
    torch.cuda.synchronize()
    return {"ms": a.elapsed_time(b), "h2d": hs.h2d_bytes, "d2h": hs.d2h_bytes,
            "chunks": len(hs.chunks), "out": hs.out}


# ------------------------------------------------------------ CPU legs


def cpu_sample(args, W, flats, n_kernels: int, threads: int):
    """Oracle (CPU restatement, `kind: port`) over the first n_kernels kernels of
    the workload: schedule + features + ensemble + energy.  Returns (points, s)."""
    import oracle as O

    c = W["corpus"]
    hg = O.HostGrid(c, W["profiles"], W["configs"], kernel_ids=np.arange(n_kernels))
    t0 = time.perf_counter()
    out = O.schedule_features(hg, sel_idx=W["sel"], threads=threads)
    n_cfg, n_arch = len(W["configs"]), len(W["profiles"])
    arch_of = (np.arange(hg.n_points) // n_cfg) % n_arch
    for a in range(n_arch):
        m = arch_of == a
        O.rf_predict(flats[a], out["sel"][m], status=out["status"][m],
                     time_us=np.nan_to_num(out["sf"][m, 7]), threads=threads)
    return hg.n_points, time.perf_counter() - t0


def cpu_flats(args, W):
    """Ensembles for CPU-only runs (no device): bounds from oracle features."""
    import oracle as O

    from paper_2305_01886_b200 import pack
    from paper_2305_01886_b200.ensemble import random_forest_flat

    hg = O.HostGrid(W["corpus"], W["profiles"], W["configs"],
                    kernel_ids=np.arange(min(200, W["n_k"])))
    out = O.schedule_features(hg, sel_idx=W["sel"])
    X = out["sel"][out["status"] == 0]
    lo, hi = np.nanmin(X, axis=0), np.nanmax(X, axis=0)
    return [random_forest_flat(args.trees, args.depth, pack.SELECTED_FEATURES, lo, hi, seed=7 + a)
            for a in range(len(W["profiles"]))]


def sample_kernels(W, target_s: float, threads: int, flats) -> int:
    pts, dt = cpu_sample(None, W, flats, 2, threads)
    per_kernel = dt / 2
    return int(max(2, min(W["n_k"], target_s / max(per_kernel, 1e-6))))


# ------------------------------------------------------------------ main


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c4", "c5s"])
    ap.add_argument("--kernels", type=int, default=0)
    ap.add_argument("--rows", type=int, default=0, help="c4: total rows (default 100M)")
    ap.add_argument("--trees", type=int, default=500)
    ap.add_argument("--depth", type=int, default=16)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline (profiling)")
    ap.add_argument("--no-rf", action="store_true", help="skip the config #3 forest fit")
    ap.add_argument("--no-e2e", action="store_true", help="c4: skip the host-row e2e leg")
    ap.add_argument("--rf-rows", type=int, default=1_000_000)
    ap.add_argument("--rf-trees", type=int, default=500)  # config #3 in full
    ap.add_argument("--gbt-stages", type=int, default=100)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    threads = os.cpu_count() or 1
    metric = "energy-prediction points/sec"

    if args.impl == "reference":
        if rank != 0:
            return
        W = build_workload(args, 0)
        flats = cpu_flats(args, W)
        nk = sample_kernels(W, args.cpu_seconds / max(args.steps + args.warmup, 1), threads, flats)
        for _ in range(1):
            cpu_sample(args, W, flats, min(nk, 2), threads)
        pts = sec = 0.0
        for _ in range(args.steps):
            p, s = cpu_sample(args, W, flats, nk, threads)
            pts += p
            sec += s
        v = pts / sec
        sample = (f"first {nk} kernels x {len(W['configs'])} configs x {len(W['archs'])} arch "
                  f"per step ({int(pts / args.steps)} points), oracle port, {threads} threads")
        print(json.dumps({
            "impl": "reference", "metric": metric, "value": v, "unit": "points/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args), "kernels": W["n_k"],
                       "configs": len(W["configs"]), "archs": W["archs"],
                       "ensemble": f"{args.trees} trees depth {args.depth} (declared random)"},
            "cpu_baseline": {"value": v, "unit": "points/s", "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}))
        return

    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.workload == "c1":
        if rank == 0:
            run_c1(args, threads)
        if world > 1:
            dist.destroy_process_group()
        return
    if args.workload == "c4":
        run_c4(args, rank, world, local_rank, threads)
        if world > 1:
            dist.destroy_process_group()
        return
    R = run_ours(args, rank, world, local_rank)
    if not args.no_rf:
        R["rf"] = rf_fit_measure(args, rank, world, threads)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    W = R["W"]
    n_total = R["n_pts"] * world
    value = n_total * args.steps / (R["total_ms"] / 1e3)
    e2e_value = n_total * args.steps / (R["e2e_ms"] / 1e3)
    # roofline of the dominant kernel
    split = R["split"]
    dom = max(split, key=split.get)
    n_pts = R["n_pts"]
    flat = R["flats"][0]
    ens_bytes = int(flat.nodes.nbytes)
    nsel = len(W["sel"])
    alg = {
        # tokens + preds + blocks + kernels read once, config + outputs per point
        "k1_static": R["dc_bytes"] + W["n_k"] * (64 + 24),
        "k23_schedule": R["dc_bytes"] + W["n_k"] * (64 + 24) + n_pts * (1 + 8 * 9 + 8 * nsel),
        "k4_rf_predict": ens_bytes * len(R["flats"]) + n_pts * (8 * nsel + 1 + 8 + 16),
        # fused: corpus + configs once, ensemble once, status + time + power + energy out
        "k23_schedule<fused>": R["dc_bytes"] + W["n_k"] * (64 + 24)
        + ens_bytes * len(R["flats"]) + n_pts * (1 + 8 * 3),
    }
    peak, peak_kind = hbm_peak()
    achieved = alg[dom] / (split[dom] / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(args.workload, dom, n_pts if dom != "k1_static" else W["n_k"])
    # CPU baseline on rank 0 (bounded sample)
    nk, cp, cs = 0, 0, 1.0
    if not args.no_cpu:
        nk = sample_kernels(W, args.cpu_seconds, threads, R["flats"])
        cp, cs = cpu_sample(args, W, R["flats"], nk, threads)
    line = {
        "metric": metric, "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": R["total_ms"] / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args), "kernels_per_gpu": W["n_k"],
                   "configs": len(W["configs"]), "archs": W["archs"],
                   "points_per_gpu": n_pts, "tokens_per_gpu": W["corpus"].n_tok,
                   "ensemble": f"{args.trees} trees depth {args.depth} "
                               f"({flat.nodes.shape[0] // max(flat.n_trees, 1)} nodes/tree, "
                               "declared random)",
                   "l2": "256 MB flush between timed steps (untimed); ensemble > L2",
                   "infeasible_points": R["infeasible"], "parallelism": f"dp{world} (kernel shards)"},
        "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": R["e2e"]["h2d"],
                "d2h_bytes_per_step": R["e2e"]["d2h"],
                "path": "runtime.HostSweep: per step pinned host corpus -> H2D -> fused sweep -> "
                        "D2H of (status, time, power, energy) to pinned host; steps double-buffered "
                        "on 3 streams (copies overlap the neighbouring steps' sweeps)"},
        "gpu_launches": len(split) * args.steps,
        "kernel_ms": split,
        "cycle_sweep": R["cycle"],
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "algorithmic_bytes": alg[dom], "traffic": traffic,
                     "traffic_source": traffic_src},
        "cpu_baseline": {"value": cp / cs, "unit": "points/s", "cores": threads, "kind": "port",
                         "sample": f"first {nk} kernels of the workload ({cp} points), oracle "
                                   f"schedule+features+ensemble+energy"},
        "clocks": R["clk"],
        "setup_s": round(W["build_s"], 2),
    }
    if "rf" in R:
        line["rf_fit"] = R["rf"]
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_c4(args, rank, world, local_rank, threads):
    """BASELINE configs[3]: batched inference of a 500-tree depth-16 ensemble over
    100M feature rows x 64 (fp64, 51 GB resident in HBM), rows sharded over ranks.
    Rows are generated on the device (U[0,1) like config #3's table); the ensemble
    is the declared random one (~110k nodes/tree).  A step = one pass of K4 over
    the GPU's rows; metric rows/s (+ HBM GB/s of the row stream)."""
    import torch
    import torch.distributed as dist

    from paper_2305_01886_b200 import runtime as rt
    from paper_2305_01886_b200.ensemble import random_forest_flat

    torch.cuda.set_device(local_rank)
    n = (args.rows or 100_000_000) // world
    F = 64
    g = torch.Generator(device="cuda").manual_seed(4 + rank)
    X = torch.rand((n, F), dtype=torch.float64, device="cuda", generator=g)
    flat = random_forest_flat(args.trees, args.depth, [f"f{i}" for i in range(F)], np.zeros(F),
                              np.ones(F), seed=11)
    # random independent rows: the walk is bound by L2/DRAM latency, so the
    # two-level block layout (half the dependent loads) is the default here
    de = rt.DeviceEnsemble.upload(flat, layout=os.environ.get("GK_WALK_LAYOUT", "blocks"))
    power = torch.empty(n, dtype=torch.float64, device="cuda")
    L = rt.load_library()
    import ctypes

    def step():
        rt._check(L.gk_rf_predict(ctypes.byref(de.desc), X.data_ptr(), F, n, None, None,
                                  power.data_ptr(), None, torch.cuda.current_stream().cuda_stream))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    with ClockSampler(local_rank) as clk:
        t0 = time.perf_counter()
        for k in range(args.steps):
            evs[k][0].record()
            step()
            evs[k][1].record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        time.sleep(0.25)
    clk.window(t0, t1)
    ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    if rank != 0:
        return
    rows_total = n * world
    value = rows_total * args.steps / (ms / 1e3)
    alg = n * (8 * F + 8) + flat.nodes.nbytes  # rows in + power out + ensemble once
    achieved = alg / (ms / args.steps / 1e3) / 1e9
    peak, peak_kind = hbm_peak()
    traffic, traffic_src = ncu_traffic("c4", "k4_rf_predict", n)
    line = {"metric": "RF inference rows/sec", "value": value, "unit": "rows/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "BASELINE configs[3]: 500-tree depth-16 ensemble over "
                                   f"{rows_total} rows x 64 fp64",
                       "ensemble": f"{args.trees} trees depth {args.depth} "
                                   f"({len(flat.nodes) // flat.n_trees} nodes/tree, declared random)",
                       "rows_per_gpu": n, "l2": "rows (51 GB) >> L2", "walk_layout": de.layout},
            "gpu_launches": args.steps,
            "roofline": {"bound": "hbm", "kernel": "k4_rf_predict", "achieved": achieved,
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak, "algorithmic_bytes": alg, "traffic": traffic,
                         "traffic_source": traffic_src},
            "clocks": clk.summary()}
    # e2e: the same rows from pinned HOST memory, streamed in chunks through
    # runtime.HostRowsPredictor (H2D / K4 / D2H on three streams), power back
    # to pinned host memory -- all inside the timing
    if not args.no_e2e:
        Xh = torch.empty((n, F), dtype=torch.float64).pin_memory()
        Xh.copy_(X)
        ph = torch.empty(n, dtype=torch.float64).pin_memory()
        hp = rt.HostRowsPredictor(de, F)
        hp.run(Xh, ph)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            hp.run(Xh, ph)
        b.record()
        torch.cuda.synchronize()
        e2e_ms = a.elapsed_time(b)
        assert torch.equal(ph[:100000].to(power.device), power[:100000])
        line["e2e"] = {"value": rows_total * args.steps / (e2e_ms / 1e3), "unit": "rows/s",
                       "h2d_bytes_per_step": n * F * 8, "d2h_bytes_per_step": n * 8,
                       "path": "runtime.HostRowsPredictor: pinned host rows -> 8M-row chunks "
                               "(H2D / K4 / D2H on 3 streams) -> pinned host power"}
        del Xh, ph, hp
    if not args.no_cpu:
        import oracle as O

        ns = 20000
        Xs = X[:ns].cpu().numpy()
        t0 = time.perf_counter()
        O.rf_predict(flat, Xs, threads=threads)
        cs = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": ns / cs, "unit": "rows/s", "cores": threads,
                                "kind": "port", "sample": f"{ns} rows, oracle walk"}
    print(json.dumps(line))


def run_c1(args, threads):
    """BASELINE configs[0], the reference's own CPU-runnable case, end to end
    through this package's public API: 100 synthetic PTX kernels x the 4
    config #1 launches on tesla_k20 -> parse + pack (native front-end) ->
    cycles + features (K1/K3) -> power labels from the trainer tests'
    generative form (seed 2026) -> train(..., "random_forest", 500 trees,
    seed 0: 5-fold CV + final fit, GPU forest) -> export (native writer) + load
    (native loader) -> energy for every point (fused sweep).  Metric: seconds
    (lower is better).  CPU leg (same run, this host): the same pipeline
    through the oracle port (C, all threads), scikit-learn's forest and the
    Python JSON path."""
    import tempfile

    import torch

    from paper_2305_01886_b200 import corpus as CG
    from paper_2305_01886_b200 import pack
    from paper_2305_01886_b200 import runtime as rt
    from paper_2305_01886_b200.ensemble import flatten, load_ensemble
    from paper_2305_01886_b200.profiles import resolve_profile
    from paper_2305_01886_b200.ptx_native import pack_ptx
    from paper_2305_01886_b200.trainer import ensemble_document_text, train

    items = CG.synth_corpus(100, 0)
    prof = [resolve_profile("tesla_k20")]
    sel = pack.manifest_indices(pack.SELECTED_FEATURES)
    names = pack.SELECTED_FEATURES

    def labels(feat):
        rng = np.random.default_rng(2026)
        F = pack.FEATURE_ORDER
        occ, iic, ld = (feat[:, F.index(n)] for n in ("occupancy", "inst_issue_cycles",
                                                      "glob_load_sm"))
        return 30.0 + 40.0 * occ + 0.003 * iic + 12.0 * (ld > 50) + rng.normal(0, 1, len(feat))

    def gpu_once():
        t = {}
        t0 = time.perf_counter()
        c = pack_ptx(items)
        t["parse"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        dc = rt.DeviceCorpus.upload(c)
        dg = rt.DeviceGrid.build(dc, prof, CG.CONFIG1)
        out = {k: v.cpu().numpy() for k, v in rt.schedule_features(dc, dg, sel_idx=sel).items()}
        t["schedule_features"] = time.perf_counter() - t0
        ok = out["status"] == 0
        X, y = out["feat"][ok][:, sel], labels(out["feat"][ok])
        t0 = time.perf_counter()
        res = train((X, y, names), "random_forest", n_estimators=500, seed=0)
        torch.cuda.synchronize()
        t["train_rf"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        with tempfile.TemporaryDirectory() as d:
            path = Path(d) / "ensemble.json"
            path.write_text(ensemble_document_text(res) + "\n")
            ens = load_ensemble(path)
        t["export_load"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        sw = rt.Sweep(dc, dg, [rt.DeviceEnsemble.upload(flatten(ens))], sel)
        st, tu, pw, en = (x.cpu().numpy() for x in sw.run())
        t["predict_energy"] = time.perf_counter() - t0
        return t, int(ok.sum()), res.mean_metrics.r2

    gpu_once()  # warm-up (library load, first-touch allocations)
    torch.cuda.synchronize()
    runs = [gpu_once() for _ in range(args.steps)]
    tot = [sum(r[0].values()) for r in runs]
    best = runs[int(np.argmin(tot))]
    line = {"metric": "config #1 end-to-end pipeline seconds", "value": float(np.median(tot)),
            "unit": "s", "n_gpus": 1, "steps": args.steps, "warmup": 1,
            "ms_per_step": float(np.median(tot)) * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "BASELINE configs[0]: 100 synthetic PTX kernels x 4 launch "
                                   "configs (tesla_k20): parse, cycles + features, "
                                   "train RF (500 trees, 5-fold CV + final), export + load, "
                                   "energy", "feasible_points": best[1],
                       "cv_r2": best[2]},
            "stages_s": best[0]}
    if not args.no_cpu:
        import oracle as O
        from sklearn.ensemble import RandomForestRegressor as SkRF

        from paper_2305_01886_b200 import ptx
        from paper_2305_01886_b200 import trainer as T
        from paper_2305_01886_b200.ensemble import _load_python
        from paper_2305_01886_b200.ensemble import random_forest_flat  # noqa: F401

        t = {}
        t0 = time.perf_counter()
        c = pack.pack_corpus(ptx.parse_ptx(tx, n, loop_counts=lp) for n, tx, lp in items)
        t["parse"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        o = O.schedule_features(O.HostGrid(c, prof, CG.CONFIG1), sel_idx=sel, threads=threads)
        t["schedule_features"] = time.perf_counter() - t0
        ok = o["status"] == 0
        X, y = o["feat"][ok][:, sel], labels(o["feat"][ok])
        orig = T._make_model
        T._make_model = lambda fam, n_est, lr, md, seed: SkRF(n_estimators=n_est, max_depth=md,
                                                              random_state=seed)
        try:
            t0 = time.perf_counter()
            res = T.train((X, y, names), "random_forest", n_estimators=500, seed=0)
            t["train_rf"] = time.perf_counter() - t0
        finally:
            T._make_model = orig
        t0 = time.perf_counter()
        with tempfile.TemporaryDirectory() as d:
            path = Path(d) / "ensemble.json"
            path.write_text(json.dumps(T.ensemble_document(res), indent=2) + "\n")
            flat = flatten(_load_python(path))
        t["export_load"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        O.rf_predict(flat, o["feat"][ok][:, sel], time_us=o["sf"][ok, 7], threads=threads)
        t["predict_energy"] = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": sum(t.values()), "unit": "s", "cores": threads,
                                "kind": "port", "stages_s": t,
                                "sample": "the whole workload: Python parser + oracle port (C, "
                                          "all threads) + scikit-learn RandomForestRegressor "
                                          "(the reference trainer's model, n_jobs=None) + "
                                          "Python JSON export / load"}
    print(json.dumps(line))


def rf_table(rows: int, seed: int = 3):
    """BASELINE config #3 table: 64 U[0,1) columns (8 rounded to integers),
    y = 30 + 40 x0 + 20 x1^2 + 12 [x2 > 0.5] + 0.003*20000 x3 + N(0,1)."""
    rng = np.random.default_rng(seed)
    X = rng.random((rows, 64))
    X[:, 56:] = np.floor(X[:, 56:] * 20)
    y = (30 + 40 * X[:, 0] + 20 * X[:, 1] ** 2 + 12 * (X[:, 2] > 0.5) + 0.003 * 20000 * X[:, 3]
         + rng.normal(0, 1, rows))
    X = (X - X.min(0)) / (X.max(0) - X.min(0))  # what MinMaxScaler hands the model
    return X, y


def rf_fit_measure(args, rank, world, threads):
    """Config #3: GPU forest fit on 1M x 64, depth 16, `--rf-trees` trees sharded
    by tree across ranks (time = max over ranks), extrapolated to 500 trees; plus
    scikit-learn (the reference's own RF) and the GPU on the same bounded sample."""
    import torch
    import torch.distributed as dist

    from paper_2305_01886_b200.forest import RandomForestRegressor

    X, y = rf_table(args.rf_rows)
    RandomForestRegressor(2, max_depth=4, random_state=0).fit(X[:4096], y[:4096])  # warm-up
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    m = RandomForestRegressor(args.rf_trees, max_depth=16, random_state=0,
                              shard=(rank, world) if world > 1 else None).fit(X, y)
    if world > 1:   # every rank ends with the whole forest (NCCL all-gather of the trees)
        from paper_2305_01886_b200.dist import allgather_forest

        allgather_forest(m)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt = float(t[0])
    nodes = float(np.mean([e.tree_.node_count for e in m.estimators_ if e is not None]))
    out = {"workload": f"BASELINE configs[2]: {args.rf_rows} x 64 table, depth 16, "
                       f"{args.rf_trees} trees measured (tree-sharded over {world} GPU)",
           "fit_s": dt, "s_per_tree": dt / args.rf_trees,
           "nodes_per_tree": nodes,
           "timing": "host wall clock around fit() (+ the tree all-gather at N > 1), device synced"}
    if args.rf_trees != 500:
        out["fit_s_500_trees_extrapolated"] = dt * 500 / args.rf_trees
    if rank == 0 and not args.no_cpu:
        from sklearn.ensemble import RandomForestRegressor as SkRF

        ns, ts = 100_000, 16
        # GPU first: scikit-learn's worker threads keep spinning on the host
        # cores for a while after its fit returns
        t0 = time.perf_counter()
        RandomForestRegressor(ts, max_depth=16, random_state=0).fit(X[:ns], y[:ns])
        torch.cuda.synchronize()
        gs = time.perf_counter() - t0
        t0 = time.perf_counter()
        SkRF(ts, max_depth=16, random_state=0, n_jobs=threads).fit(X[:ns].astype(np.float32), y[:ns])
        cs = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": cs, "unit": "s", "cores": threads, "kind": "reference",
                               "sample": f"scikit-learn {ts}-tree RandomForestRegressor fit, "
                                         f"{ns} rows x 64, depth 16, n_jobs={threads}",
                               "gpu_same_sample_s": gs}
    out["gbt_fit"] = gbt_fit_measure(args, X, y, rank, world, threads)
    return out


def gbt_fit_measure(args, X, y, rank, world, threads):
    """The trainer's default family (gradient boosting, training.py:67-72) on
    the same 1M x 64 table: `--gbt-stages` depth-3 stages on the GPU (stages
    are sequential; replicas only under torchrun), next to scikit-learn's
    GradientBoostingRegressor (single-threaded by design) on a bounded sample."""
    import torch

    from paper_2305_01886_b200.boosting import GradientBoostingRegressor

    GradientBoostingRegressor(2, random_state=0).fit(X[:4096], y[:4096])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    GradientBoostingRegressor(args.gbt_stages, learning_rate=0.1, random_state=0).fit(X, y)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out = {"workload": f"{len(y)} x {X.shape[1]} table, {args.gbt_stages} stages, depth 3, lr 0.1",
           "fit_s": dt, "ms_per_stage": dt / args.gbt_stages * 1e3,
           "timing": "host wall clock around fit(), device synced"}
    if rank == 0 and not args.no_cpu:
        from sklearn.ensemble import GradientBoostingRegressor as SkGBR

        ns, ss = 50_000, 4
        t0 = time.perf_counter()
        SkGBR(n_estimators=ss, learning_rate=0.1, random_state=0).fit(X[:ns].astype(np.float32), y[:ns])
        cs = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": cs / ss * 1e3, "unit": "ms/stage", "cores": 1,
                               "kind": "reference",
                               "sample": f"scikit-learn GradientBoostingRegressor, {ns} rows x "
                                         f"{X.shape[1]}, {ss} stages (sklearn boosting is "
                                         "single-threaded)"}
    return out


def workload_name(args) -> str:
    if args.workload == "c2":
        return ("BASELINE configs[1]: 10k kernels x 64 launch configs, tesla_k20, full energy "
                "pipeline (K1+K2/K3+K4+K6)")
    return "BASELINE configs[4] per-GPU slice: kernels x 256 configs x 3 archs"


if __name__ == "__main__":
    main()
