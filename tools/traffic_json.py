"""profiles/r2/traffic.json from the ncu captures of tools/profile_round.sh:
DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) and the
binding unit's utilisation, per unit of work, for bench.py's roofline block.

    python tools/traffic_json.py gpurun_out/prof
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
from ncu_summary import summary  # noqa: E402

prof = Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof")
CAPS = {
    # capture, workload key, kernel key, units per launch, unit, description
    "k23_fused_c5.ncu-rep": ("c5", "k23_schedule<fused>", 100_000 * 256 * 3, "point",
                             "bench.py --kernels 100000 (c5 grid, 76.8M points; launch 4)"),
    "k1_static_c5.ncu-rep": ("c5", "k1_static", 100_000, "kernel",
                             "bench.py --kernels 100000 (c5 grid; launch 4)"),
    "k4_c4.ncu-rep": ("c4", "k4_rf_predict", 10_000_000, "row",
                      "bench.py --workload c4 --rows 10000000 (k4_rf_predict_rounds, blocks)"),
}


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9,
         "nsecond": 1}


def num(v):
    """(value, unit) from ncu_summary -> float in bytes / ns / plain units."""
    if not v or v[0] in (None, "", "n/a"):
        return None
    return float(str(v[0]).replace(",", "")) * SCALE.get(v[1], 1)


OUT = ROOT / "profiles" / "r2" / "traffic.json"
old = json.loads(OUT.read_text()) if OUT.exists() else {}
out = {"_doc": "dram__bytes_read.sum + dram__bytes_write.sum per launch and the binding "
               "unit's utilisation from one `ncu --set full --clock-control none` capture "
               "(tools/profile_round.sh) of the command named; bench.py reports it as "
               "roofline.traffic / roofline.binding when the workload and kernel match. "
               "Per-unit values scale the capture to the bench launch (stated)."}
for f, (wl, kern, units, unit, cap) in CAPS.items():
    p = prof / f
    if not p.exists():
        continue
    rec = summary(str(p))[0]
    l1 = num(rec.get("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"))
    issue = num(rec.get("smsp__issue_active.avg.pct_of_peak_sustained_active"))
    out.setdefault(wl, {})[kern] = {
        "read": num(rec["dram__bytes_read.sum"]), "write": num(rec["dram__bytes_write.sum"]),
        "units": units, "unit": unit, "capture": cap,
        "duration_ns": num(rec.get("gpu__time_duration.sum")),
        "l1tex_pct_of_peak": l1, "lts_pct_of_peak": num(
            rec.get("lts__throughput.avg.pct_of_peak_sustained_elapsed")),
        "issue_active_pct": issue,
        "warps_active_pct": num(rec.get("sm__warps_active.avg.pct_of_peak_sustained_active")),
        "l2_hit_pct": num(rec.get("lts__t_sector_hit_rate.pct")),
    }
for wl, kerns in old.items():   # entries whose capture is not in this pass stay
    if wl.startswith("_"):
        continue
    for kern, rec in kerns.items():
        out.setdefault(wl, {}).setdefault(kern, rec)
dst = OUT
dst.write_text(json.dumps(out, indent=1) + "\n")
print(dst.read_text())
