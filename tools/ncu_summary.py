"""Summarise an `ncu --set full` report of one kernel launch into profiles/r02.

    python tools/ncu_summary.py REPORT.ncu-rep CONFIG KERNEL [--launch I]

Writes profiles/r02/ncu_<KERNEL>_<CONFIG>.json (duration, DRAM bytes, throughput, IPC,
occupancy, shared-memory wavefronts and bank conflicts, the fp64 pipe, the
stall reasons per issued instruction) and records the launch's DRAM bytes
(read + write) in profiles/r02/traffic.json under CONFIG / KERNEL, which
bench.py reports as roofline.traffic. Runs here (ncu reads reports without a
GPU)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "r02")

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "inst_executed": "warp_instructions",
    "sm__inst_executed.avg.per_cycle_active": "ipc_per_sm",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.per_cycle_active": "warps_active_per_sm",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "dynamic_smem",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sass__inst_executed_shared_loads": "lds_instructions",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "sm__inst_executed_pipe_fp64.sum": "fp64_pipe_instructions",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    report, config, key = sys.argv[1:4]
    launch = int(sys.argv[sys.argv.index("--launch") + 1]) if "--launch" in sys.argv else 0
    head, units, vals = raw(report)
    v = vals[launch]
    kname = v[head.index("Kernel Name")] if "Kernel Name" in head else key
    res = {"report": os.path.basename(report), "kernel": kname, "config": config,
           "how": "ncu --set full --clock-control none (one launch, cold L2, serialised); tools/ncu_summary.py"}
    for m, field in METRICS.items():
        if m in head:
            i = head.index(m)
            try:
                res[field] = {"value": float(v[i].replace(",", "")), "unit": units[i]}
            except ValueError:
                pass
    stalls = {}
    for i, m in enumerate(head):
        if m.startswith("smsp__average_warps_issue_stalled_") and m.endswith("_per_issue_active.ratio"):
            try:
                x = float(v[i])
            except ValueError:
                continue
            if x >= 0.02:
                stalls[m[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(x, 3)
    res["stalls_per_issued_instruction"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd, wr = res.get("dram_read"), res.get("dram_write")
    if rd and wr:
        res["dram_bytes"] = rd["value"] * scale.get(rd["unit"], 1) + wr["value"] * scale.get(wr["unit"], 1)
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"ncu_{key}_{config}.json"), "w") as f:
        json.dump(res, f, indent=1)
    tp = os.path.join(OUT, "traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    if "dram_bytes" in res:
        traffic.setdefault(config, {})[key] = res["dram_bytes"]
    traffic["how"] = "dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu --set full, tools/ncu_summary.py)"
    with open(tp, "w") as f:
        json.dump(traffic, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
