"""Per-SASS-region stall attribution from an ncu source-page CSV (--print-source sass).

    ncu -i rep.ncu-rep --page source --csv --print-source sass --kernel-name regex:k_row > x.csv
    python tools/ncu_sass_hot.py x.csv [--reason stall_long_sb] [--top 30] [--context 3]
"""
import argparse
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--reason", default="Warp Stall Sampling (All Samples)")
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--context", type=int, default=0)
ap.add_argument("--kernel", type=int, default=0, help="which kernel section of the CSV")
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
# the CSV may hold several kernels, each a "Kernel Name" row then a header row
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
k = min(a.kernel, len(starts) - 1)
end = starts[k + 1] if k + 1 < len(starts) else len(rows)
print(rows[starts[k]][1][:140])
hdr = rows[starts[k] + 1]
data = [dict(zip(hdr, r)) for r in rows[starts[k] + 2:end]]
num = lambda d, k: float(d.get(k) or 0)  # noqa: E731
tot = sum(num(d, a.reason) for d in data)
reasons = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
print(f"{a.reason}: {tot:.0f} samples, {sum(num(d, 'Instructions Executed') for d in data):.0f} warp instructions")
print({r: int(sum(num(d, r) for d in data)) for r in reasons if sum(num(d, r) for d in data) > 0})
top = sorted(range(len(data)), key=lambda i: -num(data[i], a.reason))[: a.top]
shown = set()
for i in sorted(top):
    for j in range(max(0, i - a.context), min(len(data), i + 1)):
        if j in shown:
            continue
        shown.add(j)
        d = data[j]
        why = ",".join(f"{r[6:]}={int(num(d, r))}" for r in reasons if num(d, r) > 0)
        print(f"{j:5d} {d['Source'][:64]:64s} {num(d, a.reason):5.0f} x{int(num(d, 'Instructions Executed')):6d} {why}")
