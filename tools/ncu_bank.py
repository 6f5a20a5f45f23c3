"""Shared-memory bank conflicts by source line: ncu's per-SASS "L1 Wavefronts Shared
Excessive" / "L1 Wavefronts Shared" attributed with nvdisasm line info (development aid).

usage: python tools/ncu_bank.py <report.ncu-rep> <kernel-regex> <object.o> <mangled-fn> [top]
"""
import csv
import io
import os
import subprocess
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_lines import sass_lines  # noqa: E402


def num(v):
    try:
        return float(v.replace(",", "")) if v else 0.0
    except ValueError:
        return 0.0


def main():
    rep, kre, obj, fn = sys.argv[1:5]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    h = rows[hi]
    ai, si = h.index("Address"), h.index("Source")
    xi, wi = h.index("L1 Wavefronts Shared Excessive"), h.index("L1 Wavefronts Shared")
    recs = []
    for r in rows[hi + 1:]:
        if len(r) <= wi or not r[ai].startswith("0x"):
            if recs:
                break
            continue
        recs.append((int(r[ai], 16), num(r[xi]), num(r[wi]), r[si]))
    base = recs[0][0]
    lm = sass_lines(obj, fn)
    agg = defaultdict(lambda: [0.0, 0.0, set()])
    for a, x, w, s in recs:
        key = lm.get(a - base, ("?", 0))
        agg[key][0] += x
        agg[key][1] += w
        if x > 0:
            agg[key][2].add(s.split()[0] if not s.startswith("@") else s.split()[1])
    tx = sum(v[0] for v in agg.values()) or 1
    tw = sum(v[1] for v in agg.values()) or 1
    print(f"shared wavefronts {tw:,.0f}  excessive {tx:,.0f} ({100 * tx / tw:.1f}%)")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        if v[0] <= 0:
            break
        print(f"  {100 * v[0] / tx:5.1f}% of excess  {v[0]:12,.0f} / {v[1]:12,.0f} wavefronts  {k[0]}:{k[1]}  "
              f"{' '.join(sorted(v[2]))}")


if __name__ == "__main__":
    main()
