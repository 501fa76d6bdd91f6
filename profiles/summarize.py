#!/usr/bin/env python
"""Summaries of the ncu outputs of profiles/profile_round.sh (run here, on the files that
gpurun brought back into gpurun_out/):

    python profiles/summarize.py TAG [--launches gpurun_out/prof_launches.csv]
                                     [--full gpurun_out/prof_full.ncu-rep]

writes profiles/rNN_TAG_ncu_launch_list_summary.txt (per-kernel shares of the launch list),
profiles/rNN_TAG_ncu_full_summary.txt (time, DRAM, registers, occupancy, issue, FMA pipe and
the top stall reasons per kernel of the --set full capture) and refreshes
profiles/ncu_traffic.json (DRAM bytes per launch, read by bench.py's roofline)."""
import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROUND = os.environ.get("PROFILE_ROUND", "r02")  # file prefix of the summaries
ROOT = os.path.dirname(HERE)
# bench.py profile names of the kernels (tac_profile_kernel_name)
PROFILE_NAME = {"k_elem_grad_cells": "elem_grad", "k_elem_grad_rows": "elem_grad", "k_elem_curv_cells": "elem_curv", "k_vert_pre": "vert_pre",
                "k_dir_reduce": "dir_reduce", "k_dir_apply": "dir_apply", "k_contact_classify_staged": "contact_classify",
                "k_contact_curv_staged": "contact_curv", "k_contact_curv_direct": "contact_curv", "k_contact_friction": "contact_friction",
                "k_contact_near<2>": "contact_near_ee", "k_contact_near<0>": "contact_near_gi",
                "k_contact_near<1>": "contact_near_ig", "k_broadphase_list": "broadphase_rebuild"}


def short(name):
    n = name.replace("void ", "").replace("(int)", "").replace("(bool)", "")
    n = n.split("(")[0].replace("tac::", "")
    # template arguments that only select an instantiation (axis-aligned cells, body frame,
    # tolerance-mode remapping) are dropped; k_dir_reduce keeps SURF, k_contact_near its KIND
    if n.startswith(("k_elem", "k_contact_classify", "k_vert_pre", "k_dir_apply")):
        n = n.split("<")[0]
    if n.startswith("k_dir_reduce<"):  # k_dir_reduce<SURF, TOL> -> k_dir_reduce<SURF>
        n = n.split(",")[0].rstrip(">") + ">"
    if n.startswith("k_contact_near<"):  # k_contact_near<KIND, MOLL> -> k_contact_near<KIND>
        n = n.split(",")[0].rstrip(">") + ">"
    return n


def launches(path, tag):
    rows = [l for l in open(path) if l.startswith('"')]
    r = list(csv.reader(io.StringIO("".join(rows))))
    h = r[0]
    kn, mv, un = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    unit = None
    for row in r[1:]:
        k = short(row[kn])
        tot[k] += float(row[mv].replace(",", ""))
        cnt[k] += 1
        unit = row[un]
    s = sum(tot.values())
    out = [f"ncu --metrics gpu__time_duration.sum --clock-control none (profiles/profile_round.sh launch list, bench.py "
           f"--steps 1 --warmup 3, C3 1,024 envs): {sum(cnt.values())} launches, {unit}",
           "cold-cache, serialised per-launch times: compare SHARES with bench.py's live CUDA-event profile, not absolutes",
           f"{'kernel':32s} {'launches':>8s} {'total':>12s} {'mean':>10s} {'share':>7s}"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        out.append(f"{k:32s} {cnt[k]:8d} {tot[k]:12.1f} {tot[k] / cnt[k]:10.2f} {100 * tot[k] / s:6.1f}%")
    p = os.path.join(HERE, f"{ROUND}_{tag}_ncu_launch_list_summary.txt")
    open(p, "w").write("\n".join(out) + "\n")
    print(p)


def full(path, tag):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h = r[0]
    cols = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
            "sm__maximum_warps_per_active_cycle_pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "smsp__thread_inst_executed_per_inst_executed.ratio"]
    idx = [h.index(c) for c in cols]
    stall = [i for i, c in enumerate(h) if c.startswith("smsp__average_warps_issue_stalled_")
             and c.endswith("_per_issue_active.ratio")]
    ki = h.index("Kernel Name")
    units = r[1]
    out = [f"ncu --set full --clock-control none --import-source on (profiles/profile_round.sh), one launch per kernel "
           f"mid-trajectory, C3 1,024 envs; units: " + ", ".join(f"{c}={units[i]}" for c, i in zip(cols, idx) if units[i]),
           "kernel, " + ", ".join(cols) + ", top stall reasons (warps per issue)"]
    traffic = {}
    for row in r[2:]:
        k = short(row[ki])
        vals = sorted(((float(row[i] or 0), h[i].replace("smsp__average_warps_issue_stalled_", "")
                        .replace("_per_issue_active.ratio", "")) for i in stall), reverse=True)[:5]
        out.append(f"{k}, " + ", ".join(row[i] for i in idx) + ", " + " ".join(f"{n}={v:.2f}" for v, n in vals))
        if k in PROFILE_NAME:
            mb = float(row[idx[1]]) + float(row[idx[2]])
            scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}.get(units[idx[1]], 1e6)
            traffic[PROFILE_NAME[k]] = int(round(mb * scale))
    p = os.path.join(HERE, f"{ROUND}_{tag}_ncu_full_summary.txt")
    open(p, "w").write("\n".join(out) + "\n")
    print(p)
    if traffic:
        traffic = {"_source": f"ncu --set full --clock-control none (profiles/profile_round.sh), dram__bytes_read.sum + "
                              f"dram__bytes_write.sum per launch, C3 1,024 envs; see profiles/{ROUND}_{tag}_ncu_full_summary.txt",
                   **dict(sorted(traffic.items()))}
        json.dump(traffic, open(os.path.join(HERE, "ncu_traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches", default=os.path.join(ROOT, "gpurun_out", "prof_launches.csv"))
    ap.add_argument("--full", default=os.path.join(ROOT, "gpurun_out", "prof_full.ncu-rep"))
    a = ap.parse_args()
    if os.path.exists(a.launches):
        launches(a.launches, a.tag)
    if os.path.exists(a.full):
        full(a.full, a.tag)
    sys.exit(0)
