"""Summarise ncu output into small JSON files under profiles/.

  python tools/ncu_summary.py full   <report.ncu-rep> <out.json> [algorithmic_bytes]
  python tools/ncu_summary.py launch <launches.csv>   <out.json>

`full` keeps the SOL / DRAM / occupancy / pipe counters of each profiled kernel
and the hottest source lines (warp-stall samples); `launch` aggregates a
`--metrics gpu__time_duration.sum` launch list into per-kernel counts, mean
duration and share of the captured time.
"""
import collections
import csv
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
    "smsp__average_warp_latency_issue_stalled_barrier", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]


def full(rep, out, alg=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = {"kernel": d.get("Kernel Name", "")[:120]}
        for key in KEYS:
            if key in d and d[key] != "":
                k[key] = [d[key], units[hdr.index(key)]]
        try:
            rd = float(d["dram__bytes_read.sum"]) * _scale(units[hdr.index("dram__bytes_read.sum")])
            wr = float(d["dram__bytes_write.sum"]) * _scale(units[hdr.index("dram__bytes_write.sum")])
            us = float(d["gpu__time_duration.sum"]) * _tscale(units[hdr.index("gpu__time_duration.sum")])
            k["dram_bytes"] = rd + wr
            k["dram_gbs"] = (rd + wr) / us / 1e3
            if alg:
                k["algorithmic_bytes"] = alg
                k["traffic_over_algorithmic"] = (rd + wr) / alg
        except (KeyError, ValueError):
            pass
        kernels.append(k)
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    agg, total, path = {}, 0.0, None
    for r in csv.reader(src.splitlines()):
        if len(r) >= 2 and r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if len(r) > 4 and r[0].isdigit():
            try:
                v = float(r[4])
            except ValueError:
                continue
            key = f"{path}:{r[0]}  {r[1].strip()[:90]}"
            agg[key] = agg.get(key, 0.0) + v
            total += v
    hot = [[round(100 * v / max(total, 1), 1), k] for k, v in sorted(agg.items(), key=lambda x: -x[1])[:20]]
    json.dump({"report": rep.split("/")[-1], "kernels": kernels, "hot_lines_pct_of_stall_samples": hot},
              open(out, "w"), indent=1)


def _scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def _tscale(u):
    return {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(u, 1.0)


def launch(csv_path, out):
    rows = list(csv.reader(open(csv_path)))
    hdr, agg = None, collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                u = d.get("Metric Unit", "")
                v = float(d["Metric Value"].replace(",", "")) * (1e-3 if u in ("ns", "nsecond") else
                                                                  1e3 if u in ("ms", "msecond") else 1.0)
                agg[d["Kernel Name"].split("(")[0][:90]].append(v)
    tot = sum(sum(v) for v in agg.values())
    res = [{"kernel": k, "launches": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / tot}
           for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))]
    json.dump({"source": csv_path.split("/")[-1], "total_us": tot, "kernels": res}, open(out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
    else:
        launch(sys.argv[2], sys.argv[3])
