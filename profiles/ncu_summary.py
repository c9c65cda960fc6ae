"""Key metrics of an `ncu --set full` report (one kernel launch), read with
`ncu -i <rep> --page raw --csv`.  Usage: python ncu_summary.py prof.ncu-rep [algo_bytes]"""
import csv
import io
import subprocess
import sys

WANT = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, vals = rows[0], rows[1], rows[2]
get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
for w in WANT:
    if w in get:
        v, u = get[w]
        print(f"{w:70s} {v[:90]} {u}")


def to_bytes(v, u):
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


tr = to_bytes(*get["dram__bytes_read.sum"]) + to_bytes(*get["dram__bytes_write.sum"])
print(f"{'traffic_bytes (dram read + write)':70s} {tr:.0f}")
if len(sys.argv) > 2:
    print(f"{'algorithmic_bytes':70s} {float(sys.argv[2]):.0f}  traffic/algo = {tr / float(sys.argv[2]):.2f}")
