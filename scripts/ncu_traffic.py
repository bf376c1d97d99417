"""Per-launch DRAM traffic of the main kernel from an ncu metrics CSV
(dram__bytes_read.sum + dram__bytes_write.sum, one launch per sweep point) ->
profiles/ncu_main_kernel.json, which bench.py reports as roofline.traffic.
  python scripts/ncu_traffic.py gpurun_out/dram_r01b.csv fa3-sweep-causal-hd128-16384tok-hidden2048 [source-note]
"""
import csv
import json
import os
import sys

src, workload = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
rows = [r for r in csv.reader(l for l in open(src) if not l.startswith("=="))]
h = rows[0]
per = {}
for r in rows[1:]:
    d = dict(zip(h, r))
    if "dash_bwd_kernel" not in d["Kernel Name"] and "dash_bwd_pair_kernel" not in d["Kernel Name"]:
        continue
    per.setdefault(d["ID"], {})[d["Metric Name"]] = float(d["Metric Value"])
launches = [v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in per.values()]
out_p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                     "ncu_main_kernel.json")
j = json.load(open(out_p)) if os.path.exists(out_p) else {}
j[workload] = {"dram_bytes_per_launch": sum(launches) / len(launches),
               "per_launch": launches, "launches": len(launches),
               "source": os.path.basename(src), "note": note}
json.dump(j, open(out_p, "w"), indent=1)
print(json.dumps(j[workload]))
