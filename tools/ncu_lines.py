"""Attribute ncu SASS-level metrics (instructions executed, stall samples) to CUDA
source lines, using nvdisasm -g line info of the same cubin.

usage: python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> <object.o> <mangled-fn> [top]
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def sass_lines(obj, fn):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
    start = txt.index(f".text.{fn}:")
    end = txt.find("//---------------------", start)
    body = txt[start:end]
    cur = ("?", 0)
    m = {}
    for ln in body.splitlines():
        mm = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if mm:
            cur = (os.path.basename(mm.group(1)), int(mm.group(2)))
            continue
        mm = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if mm:
            m[int(mm.group(1), 16)] = cur
    return m


def main():
    rep, kre, obj, fn = sys.argv[1:5]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    h = rows[hi]
    ai, ii, wi = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    si = h.index("Source")
    recs = []
    for r in rows[hi + 1:]:
        if len(r) <= wi or not r[ai].startswith("0x"):
            if recs:
                break
            continue
        recs.append((int(r[ai], 16), int(r[ii] or 0), int(r[wi] or 0), r[si]))
    base = recs[0][0]
    lm = sass_lines(obj, fn)
    agg = defaultdict(lambda: [0, 0])
    op = defaultdict(lambda: [0, 0])
    for a, n, w, s in recs:
        key = lm.get(a - base, ("?", 0))
        agg[key][0] += n
        agg[key][1] += w
        opc = s.split()[0] if s.split() else "?"
        if opc.startswith("@"):
            opc = s.split()[1]
        opc = opc.split(".")[0]
        op[opc][0] += n
        op[opc][1] += w
    tn = sum(v[0] for v in agg.values()) or 1
    tw = sum(v[1] for v in agg.values()) or 1
    print(f"total warp-instructions {tn:,}  stall samples {tw:,}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{100 * v[1] / tw:5.1f}% stall {100 * v[0] / tn:5.1f}% inst  {k[0]}:{k[1]}")
    print("--- by opcode (inst%, stall%)")
    for k, v in sorted(op.items(), key=lambda kv: -kv[1][0])[:25]:
        print(f"{k:10s} {100 * v[0] / tn:5.1f}% {100 * v[1] / tw:5.1f}%")


if __name__ == "__main__":
    main()
