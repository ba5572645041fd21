#!/bin/bash
# Per-launch time and DRAM bytes of every kernel in two fused 512^3 multires coarse steps.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/mres_launches.csv python tools/prof_mres.py 512 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/mres_launches.csv")))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hd = rows[h]; data = rows[h + 1:]
K, M, V, U = hd.index("Kernel Name"), hd.index("Metric Name"), hd.index("Metric Value"), hd.index("Metric Unit")
ids = collections.OrderedDict()
for r in data:
    d = ids.setdefault(r[0], {"k": r[K]})
    d[r[M]] = (float(r[V].replace(",", "")), r[U])
for i, d in list(ids.items())[-40:]:
    t = d.get("gpu__time_duration.sum", (0, ""))
    rd = d.get("dram__bytes_read.sum", (0, "")); wr = d.get("dram__bytes_write.sum", (0, ""))
    print(i, d["k"][:60], t, rd, wr)
PY
