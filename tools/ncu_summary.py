"""Summarise an ncu --set full report into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_C5.ncu-rep profiles/r1_ncu_C5_v3

Writes <dir>/full_summary.json (the metrics the roofline discussion cites, per
kernel, averaged over the captured launches) and refreshes
profiles/ncu_kernel_metrics.json (per short kernel name bench.py uses: DRAM
bytes read + written per launch and the pipe utilisations of the capture).  Reads the report with `ncu -i --page raw`.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "sm__cycles_elapsed.avg.per_second",
]

SHORT = {"mr1_kernel": "mr1", "mr2_kernel": "mr2", "classify_kernel": "classify", "sieve_kernel": "sieve",
         "qscatter_kernel": "sort", "plan_kernel": "plan", "dense_kernel": "dense", "small_kernel": "small",
         "small_warp_kernel": "small"}

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def short_name(full):
    base = full.split("(")[0].split("<")[0].replace("void ", "").strip()
    return SHORT.get(base, base), base


def main():
    rep, outdir = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    per = {}
    for d in data:
        sname, base = short_name(d[col["Kernel Name"]])
        ent = per.setdefault(base, {"short": sname, "launches": 0, "sum": {}, "unit": {}})
        ent["launches"] += 1
        for k in KEYS:
            if k not in col:
                continue
            try:
                v = float(d[col[k]].replace(",", ""))
            except ValueError:
                continue
            ent["sum"][k] = ent["sum"].get(k, 0.0) + v
            ent["unit"][k] = units[col[k]]
    summary = {}
    for base, ent in per.items():
        n = ent["launches"]
        s = {"short": ent["short"], "launches_captured": n}
        for k, v in ent["sum"].items():
            s[k] = f"{v / n:.6g} {ent['unit'][k]}".strip()
        rb = ent["sum"].get("dram__bytes_read.sum", 0.0) / n * SCALE.get(ent["unit"].get("dram__bytes_read.sum", "byte"), 1)
        wb = ent["sum"].get("dram__bytes_write.sum", 0.0) / n * SCALE.get(ent["unit"].get("dram__bytes_write.sum", "byte"), 1)
        s["dram_bytes_per_launch"] = rb + wb
        summary[base] = s
    os.makedirs(outdir, exist_ok=True)
    with open(os.path.join(outdir, "full_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_kernel_metrics.json")
    old = json.load(open(tpath)) if os.path.exists(tpath) else {}
    # named as it is committed: profiles/<dir>/full_summary.json
    src = os.path.basename(os.path.normpath(outdir)) + "/full_summary.json"
    # entries are keyed "<short>@<config>" when the output directory names the
    # configuration (r1_ncu_C5_v11 -> C5), which bench.py looks up per config;
    # the plain "<short>" key is refreshed only by launches that did work (a
    # no-op launch, e.g. classify on a dense chunk, must not stand for the kernel)
    m = re.search(r"_(C\d)_", os.path.basename(os.path.normpath(outdir)) + "_")
    cfg = m.group(1) if m else None
    for base, s in summary.items():
        def pct(k):
            v = s.get(k)
            return float(v.split()[0]) if v else None
        dur = s.get("gpu__time_duration.sum", "0 ms").split()
        dur_ms = float(dur[0]) * (1e-3 if len(dur) > 1 and dur[1] == "us" else 1.0)
        ent = {
            "dram_bytes_per_launch": s["dram_bytes_per_launch"],
            "fmaheavy_pipe_pct": pct("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            "fp64_pipe_pct": pct("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": pct("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "dram_pct": pct("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "source": src,
        }
        if cfg:
            old[f"{s['short']}@{cfg}"] = ent
        if dur_ms >= 0.05:
            old[s["short"]] = ent
    with open(tpath, "w") as f:
        json.dump(old, f, indent=1)
    print(json.dumps({k: {kk: vv for kk, vv in v.items() if kk in ("short", "gpu__time_duration.sum",
                      "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "dram_bytes_per_launch")}
                      for k, v in summary.items()}, indent=1))


if __name__ == "__main__":
    main()
