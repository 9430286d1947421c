"""Summarise one kernel of an `ncu --set full` report (.ncu-rep) into the JSON
kept under profiles/: duration, DRAM bytes, throughput, pipe utilisation,
occupancy, top stall reasons.

    python tools/ncu_summary.py report.ncu-rep out.json [alg_bytes_per_launch]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "sm__cycles_active.avg": "sm_cycles_active_avg",
    "sm__cycles_elapsed.avg": "sm_cycles_elapsed_avg",
}


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
            "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}.get(u, 1)


def main():
    rep, out = sys.argv[1], sys.argv[2]
    alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    res = {"report": rep.split("/")[-1], "kernel": v[h.index("Kernel Name")][:120]}
    for k, name in KEYS.items():
        if k in h:
            i = h.index(k)
            try:
                res[name] = float(v[i].replace(",", "")) * unit_scale(u[i])
            except ValueError:
                res[name] = v[i]
    stalls = []
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    res["top_stalls_per_issue"] = {n: round(x, 3) for x, n in sorted(stalls, reverse=True)[:6]}
    if "dram_bytes_read" in res:
        res["dram_bytes_per_launch"] = res["dram_bytes_read"] + res.get("dram_bytes_write", 0.0)
    if alg:
        res["alg_bytes_per_launch"] = alg
        res["dram_over_alg"] = res["dram_bytes_per_launch"] / alg
    res["note"] = ("ncu replay: cold caches, serialised, clocks unlocked (--clock-control none); "
                   "durations here are not bench values")
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
