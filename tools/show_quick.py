"""Print the results of tools/gpu_quick.sh (run from the repo root)."""
import collections
import csv
import json

print(open("gpurun_out/pytest_gpu.log").read().strip().splitlines()[-2:])
print(open("gpurun_out/passes.log").read().strip())
try:
    rows = list(csv.reader(open("gpurun_out/quick_inst.csv")))
    h, agg = None, collections.defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            agg[(r[h.index("Kernel Name")].split("(")[0][-40:], r[h.index("Metric Name")])].append(
                float(r[h.index("Metric Value")]))
    for k, v in sorted(agg.items()):
        print(f"{sum(v) / len(v):14.1f}  {k}")
except FileNotFoundError:
    pass
d = json.loads(open("gpurun_out/bench_quick.log").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", (d.get("e2e") or {}).get("value"), "seq", d["roofline"]["pass_ms_in_sequence"])
