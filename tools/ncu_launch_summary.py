"""Per-kernel totals from an ncu launch list (--metrics gpu__time_duration.sum
--csv): launches, total and mean duration, share of the profiled time.
python tools/ncu_launch_summary.py LAUNCHES.csv [top]"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
with open(path) as f:
    lines = [ln for ln in f if ln.startswith('"')]
agg = collections.defaultdict(lambda: [0, 0.0])
for row in csv.DictReader(lines):
    if row.get("Metric Name") != "gpu__time_duration.sum":
        continue
    us = float(row["Metric Value"].replace(",", "")) * SCALE.get(row["Metric Unit"], 1.0)
    name = row["Kernel Name"].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += us
total = sum(v[1] for v in agg.values())
print(f"# {path}: {sum(v[0] for v in agg.values())} launches, {total / 1e3:.1f} ms profiled "
      "(ncu: serialised, cold-cache per launch; shares, not absolute step times)")
print(f"{'launches':>8} {'total_us':>12} {'mean_us':>10} {'share':>6}  kernel")
for name, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{n:8d} {us:12.1f} {us / n:10.2f} {100 * us / total:5.1f}%  {name}")
