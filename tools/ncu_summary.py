"""Summarise ncu reports / launch lists into profiles/ (markdown + traffic.json).

python tools/ncu_summary.py report <rep.ncu-rep> [<rep2> ...]   -> markdown on stdout
python tools/ncu_summary.py launches <launches.csv>             -> per-kernel time share
python tools/ncu_summary.py traffic <key>=<rep> ...              -> profiles/traffic.json
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Block Size", "Grid Size", "Theoretical Occupancy", "Achieved Occupancy", "Block Limit Registers",
        "Block Limit Shared Mem", "Executed Instructions", "Executed Ipc Active", "Issue Slots Busy",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput", "Memory Throughput"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed_pipe_fma.sum", "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
       "smsp__inst_executed.sum"]


def short(name):
    name = name.replace("void ", "").replace("dmpc::", "").replace("(int)", "").replace("(bool)", "")
    depth = 0
    for i, ch in enumerate(name):
        depth += ch == "<"
        depth -= ch == ">"
        if ch == "(" and depth == 0:
            return name[:i]
    return name


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def report(paths):
    for rep in paths:
        print(f"### {os.path.basename(rep)}\n")
        rows = ncu_csv(["-i", rep, "--page", "details", "--csv"])
        h = rows[0]
        ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
        per = defaultdict(dict)
        order = []
        for r in rows[1:]:
            k = short(r[ki])
            if k not in order:
                order.append(k)
            if r[mi] in KEYS and r[mi] not in per[k]:
                per[k][r[mi]] = f"{r[vi]} {r[ui]}".strip()
        raw = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
        rh = raw[0]
        stall = []
        for i, name in enumerate(rh):
            if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
                stall.append((i, name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        rk = rh.index("Kernel Name")
        byname = {short(x[rk]): x for x in raw[2:] if len(x) > rk}
        for k in order:
            if k not in byname:
                continue
            r = byname[k]
            print(f"**{k}**\n")
            print("| metric | value |\n|---|---|")
            for m in KEYS:
                if m in per[k]:
                    print(f"| {m} | {per[k][m]} |")
            for m in RAW:
                if m in rh:
                    print(f"| {m} | {r[rh.index(m)]} {raw[1][rh.index(m)]} |")
            vals = sorted(((float(r[i] or 0), n) for i, n in stall), reverse=True)
            tot = sum(v for v, _ in vals) or 1
            print("| top stall reasons | " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in vals[:6]) + " |\n")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            k = short(r[ki])
            v = float(r[vi].replace(",", ""))
            tot[k] += v
            cnt[k] += 1
    s = sum(tot.values())
    print("| kernel | launches | total time | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| {k} | {cnt[k]} | {v:.0f} | {100 * v / s:.1f}% |")


def traffic(pairs):
    out = {}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    if os.path.exists(path):
        out = json.load(open(path))
    for p in pairs:
        key, rep = p.split("=", 1)
        raw = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
        h = raw[0]
        units = raw[1]
        r = raw[2]  # first kernel in the report (the forward)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(r[h.index("dram__bytes_read.sum")]) * scale[units[h.index("dram__bytes_read.sum")]]
        wr = float(r[h.index("dram__bytes_write.sum")]) * scale[units[h.index("dram__bytes_write.sum")]]
        out[key] = rd + wr
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "report":
        report(sys.argv[2:])
    elif cmd == "launches":
        launches(sys.argv[2])
    else:
        traffic(sys.argv[2:])
