"""Per-source-line stall-reason breakdown of an ncu report (development aid).

python tools/ncu_stalls.py <report> <kernel-regex> <object.o> <mangled-fn> [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

sys.path.insert(0, "tools")
from ncu_lines import sass_lines  # noqa: E402

rep, kre, obj, fn = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r)
h = rows[hi]
ai = h.index("Address")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ri = [h.index(c) for c in reasons]
recs = []
for r in rows[hi + 1:]:
    if len(r) <= max(ri) or not r[ai].startswith("0x"):
        if recs:
            break
        continue
    recs.append((int(r[ai], 16), [int(r[i] or 0) for i in ri]))
base = recs[0][0]
lm = sass_lines(obj, fn)
agg = defaultdict(lambda: [0] * len(reasons))
for a, v in recs:
    k = lm.get(a - base, ("?", 0))
    agg[k] = [x + y for x, y in zip(agg[k], v)]
tot = sum(sum(v) for v in agg.values()) or 1
colt = [sum(v[i] for v in agg.values()) for i in range(len(reasons))]
print("overall:", ", ".join(f"{reasons[i][6:]} {100 * colt[i] / tot:.1f}%" for i in
                            sorted(range(len(reasons)), key=lambda i: -colt[i])[:8]))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:top]:
    s = sum(v)
    parts = sorted(range(len(reasons)), key=lambda i: -v[i])[:4]
    print(f"{100 * s / tot:5.1f}% {k[0]}:{k[1]}  " + ", ".join(f"{reasons[i][6:]} {100 * v[i] / s:.0f}%" for i in parts))
