"""Key metrics of launches in an `ncu --set full` report, read with
`ncu -i <rep> --page raw --csv`.

  python ncu_summary.py prof.ncu-rep [--kernel REGEX] [--index K] [--algo BYTES]
      metrics of the K-th launch whose name matches REGEX (default: first launch)
  python ncu_summary.py prof.ncu-rep --kernel REGEX --traffic-json out.json --config NAME
      average DRAM bytes (read + write) per matching launch -> the `traffic`
      figure bench.py reports for that kernel
"""
import argparse
import csv
import io
import json
import re
import subprocess

WANT = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def to_bytes(v, u):
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{h: (v, u) for h, u, v in zip(hdr, units, r)} for r in rows[2:]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel", default=".")
    ap.add_argument("--index", type=int, default=0)
    ap.add_argument("--algo", type=float, default=None)
    ap.add_argument("--traffic-json", default=None)
    ap.add_argument("--config", default="powerlaw_1m_10m")
    a = ap.parse_args()
    sel = [L for L in launches(a.rep) if re.search(a.kernel, L["Kernel Name"][0])]
    if not sel:
        raise SystemExit(f"no launch matches {a.kernel!r}")
    if a.traffic_json:
        per = [to_bytes(*L["dram__bytes_read.sum"]) + to_bytes(*L["dram__bytes_write.sum"]) for L in sel]
        json.dump({"kernel": a.kernel, "config": a.config, "bytes_per_launch": sum(per) / len(per),
                   "launches": len(per), "per_launch": per,
                   "source": f"{a.rep} (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum)"},
                  open(a.traffic_json, "w"), indent=1)
        print(f"{len(per)} launches, mean traffic {sum(per) / len(per):.0f} B")
        return
    get = sel[a.index]
    for w in WANT:
        if w in get:
            v, u = get[w]
            print(f"{w:78s} {v[:90]} {u}")
    tr = to_bytes(*get["dram__bytes_read.sum"]) + to_bytes(*get["dram__bytes_write.sum"])
    print(f"{'traffic_bytes (dram read + write)':78s} {tr:.0f}")
    if a.algo:
        print(f"{'algorithmic_bytes':78s} {a.algo:.0f}  traffic/algo = {tr / a.algo:.2f}")


if __name__ == "__main__":
    main()
