"""Binding-unit summary of ncu --set full captures (tuning aid, runs here).

    python tools/ncu_binding.py REP...

Per capture: duration, issue-active, the busiest units' throughput fractions
(L1/TEX, shared-memory pipe, L2, DRAM, FMA / ALU / FP64 pipes) and the DRAM
bytes -- the unit with the largest fraction is the kernel's binding unit."""
import csv
import io
import subprocess
import sys

M = {
    "gpu__time_duration.sum": "ms",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1tex",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wf",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum.pct_of_peak_sustained_elapsed": "smem_atom",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
}


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    r = {}
    for k, name in M.items():
        if k in hdr:
            i = hdr.index(k)
            v = float(vals[i].replace(",", ""))
            u = units[i]
            if name == "ms":
                v = v / 1e6 if u == "ns" else v / 1e3 if u == "us" else v
            if name.startswith("dram_"):
                v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            r[name] = v
    r["kernel"] = vals[hdr.index("Kernel Name")][:40]
    return r


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        r = summary(rep)
        units = {k: r.get(k, 0.0) for k in ("l1tex", "smem_wf", "smem_atom", "l2", "dram", "alu",
                                            "fma", "fp64", "lsu_pipe")}
        top = max(units, key=units.get)
        print(f"{rep.split('/')[-1]:<22} {r['kernel']:<40} {r['ms']:8.3f} ms  issue {r['issue']:5.1f}%  "
              + "  ".join(f"{k} {v:5.1f}%" for k, v in units.items())
              + f"  dram {(r.get('dram_rd', 0) + r.get('dram_wr', 0)) / 1e9:6.3f} GB  -> {top}")
