#!/bin/bash
# per-kernel device time of one 32-tree K5 batch (ncu launch list; run on a GPU box)
O=${1:-gpurun_out/k5l}; mkdir -p $O
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python tools/k5_ncu.py > $O/l.log 2>&1
python - $O/launches.csv <<'PY'
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]; data = rows[i + 1:]
ix = {n: h.index(n) for n in ("Kernel Name", "Metric Name", "Metric Value", "ID")}
per = collections.OrderedDict()
for r in data:
    if len(r) < len(h): continue
    per.setdefault((int(r[ix["ID"]]), r[ix["Kernel Name"]][:48]), {})[r[ix["Metric Name"]]] = r[ix["Metric Value"]]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
units = {r[ix["Metric Name"]]: r[h.index("Metric Unit")] for r in data if len(r) >= len(h)}
dram = 0.0
for (_, k), m in per.items():
    a = agg[k]; a[0] += 1; a[1] += float(m["gpu__time_duration.sum"].replace(",", ""))
    a[2] += float(m["smsp__inst_executed.sum"].replace(",", ""))
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        dram += float(m.get(key, "0").replace(",", "")) * SC.get(units.get(key, "byte"), 1)
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
    print(f"{k:50s} n={a[0]:4d} {a[1]/1e6:8.2f} ms {100*a[1]/tot:5.1f}%  {a[2]/1e9:7.2f} G inst")
print(f"total {tot/1e6:.2f} ms")
print(f"dram_bytes {dram:.6e}")
PY
