"""Summarise an ncu --csv launch list: per-kernel count, total and mean
device time, share of the listed time.  Usage: ncu_summary.py launches.csv [skip_regex]"""
import csv, re, sys, collections
path = sys.argv[1]
skip = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
    if skip and skip.search(name):
        continue
    v = float(r["Metric Value"]); unit = r["Metric Unit"]
    ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
    rows.append((name, ns, r["Grid Size"], r["Block Size"]))
agg = collections.OrderedDict()
for n, ns, g, b in rows:
    a = agg.setdefault(n, [0, 0.0, g, b]); a[0] += 1; a[1] += ns
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':42s} {'count':>6s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}  grid/block")
for n, (c, ns, g, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n[:42]:42s} {c:6d} {ns/1e3:10.1f} {ns/1e3/c:9.2f} {100*ns/tot:5.1f}%  {g} {b}")
print(f"total listed: {tot/1e3:.1f} us over {sum(a[0] for a in agg.values())} launches")
