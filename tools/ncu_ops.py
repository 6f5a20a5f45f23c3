"""Executed warp-instructions by opcode for source lines matching a filter (development aid).

python tools/ncu_ops.py <report> <kernel-regex> <object.o> <mangled-fn> <file:lo-hi> [<file:lo-hi> ...]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

sys.path.insert(0, "tools")
from ncu_lines import sass_lines  # noqa: E402

rep, kre, obj, fn = sys.argv[1:5]
ranges = []
for a in sys.argv[5:]:
    f, r = a.split(":")
    lo, hi = r.split("-")
    ranges.append((f, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi_ = next(i for i, r in enumerate(rows) if "Address" in r)
h = rows[hi_]
ai, ii, si = h.index("Address"), h.index("Instructions Executed"), h.index("Source")
recs = []
for r in rows[hi_ + 1:]:
    if len(r) <= si or not r[ai].startswith("0x"):
        if recs:
            break
        continue
    recs.append((int(r[ai], 16), int(r[ii] or 0), r[si]))
base = recs[0][0]
lm = sass_lines(obj, fn)
c = Counter()
tot = 0
for a, n, s in recs:
    f, l = lm.get(a - base, ("?", 0))
    if any(f == rf and lo <= l <= hi for rf, lo, hi in ranges) or (not ranges):
        op = s.split()[0] if s.split() else "?"
        if op.startswith("@"):
            op = s.split()[1]
        c[op.split(".")[0]] += n
        tot += n
print(f"total {tot:,}")
for k, v in c.most_common(30):
    print(f"{k:10s} {v:14,} {100 * v / tot:5.1f}%")
