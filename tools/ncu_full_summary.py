"""Key metrics of an `ncu --set full` report (.ncu-rep) as text, one block per
captured launch.  Usage: ncu_full_summary.py report.ncu-rep > profiles/x.txt"""
import csv
import io
import subprocess
import sys

DETAILS = ["Duration", "Grid Size", "Block Size", "Cluster Size", "Registers Per Thread",
           "Dynamic Shared Memory Per Block", "DRAM Throughput", "Memory Throughput",
           "Compute (SM) Throughput", "L2 Hit Rate", "Achieved Occupancy",
           "Issue Slots Busy", "No Eligible", "Warp Cycles Per Issued Instruction"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
       "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
       "smsp__pcsamp_warps_issue_stalled_barrier",
       "smsp__pcsamp_warps_issue_stalled_wait",
       "smsp__pcsamp_warps_issue_stalled_sleeping",
       "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
       "smsp__pcsamp_warps_issue_stalled_mio_throttle",
       "smsp__pcsamp_warps_issue_stalled_lg_throttle",
       "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
       "smsp__pcsamp_warps_issue_stalled_selected",
       "lts__throughput.avg.pct_of_peak_sustained_elapsed",
       "lts__t_bytes.sum"]


def page(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    det = {}
    rows = page(rep, "details")
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if "ID" not in d or "Kernel Name" not in d:
            continue
        key = (d["ID"], d["Kernel Name"].split("(")[0])
        if d["Metric Name"] in DETAILS:
            det.setdefault(key, []).append(f"{d['Metric Name']}: {d['Metric Value']} {d['Metric Unit']}")
    raw = page(rep, "raw")
    rh, units = raw[0], raw[1]
    for i, r in enumerate(raw[2:]):
        d = dict(zip(rh, r))
        key = (d.get("ID", str(i)), d.get("Kernel Name", "?").split("(")[0])
        for m in RAW:
            if m in d:
                det.setdefault(key, []).append(f"{m}: {d[m]} {units[rh.index(m)]}")
    print(f"# {rep}")
    for (i, name), lines in det.items():
        print(f"\n## launch {i}: {name}")
        for line in lines:
            print("  " + line)


if __name__ == "__main__":
    main()
