"""Sum per-kernel DRAM bytes and time of ONE decode step from an ncu CSV
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum)
of tools/profile_step.py: the step's kernels are those from the last
embed launch (the first kernel of a decode step) on."""
import csv, sys, json
rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
recs = {}
for r in csv.DictReader(rows):
    k = (r["ID"], r["Kernel Name"])
    recs.setdefault(k, {})[r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
items = sorted(recs.items(), key=lambda kv: int(kv[0][0]))
starts = [i for i, ((_, n), _) in enumerate(items) if "embed_kernel" in n]
step = items[starts[-1]:] if starts else []
def b(m):
    v, u = m
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
def t(m):
    v, u = m
    return v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1)
tot_b = sum(b(m["dram__bytes_read.sum"]) + b(m["dram__bytes_write.sum"]) for _, m in step)
tot_t = sum(t(m["gpu__time_duration.sum"]) for _, m in step)
print(json.dumps({"kernels": len(step), "dram_bytes": tot_b, "serialized_us": tot_t}))
