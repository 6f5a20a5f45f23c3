"""List local-memory (spill) instructions of one kernel by source line (development aid).

python tools/spills.py <object.o> <mangled-fn>
"""
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

obj, fn = sys.argv[1:3]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
s = txt.index(f".text.{fn}:")
e = txt.find("\n\t.section", s + 10)
body = txt[s:e if e > 0 else len(txt)]
cur = ("?", 0)
c = Counter()
for ln in body.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    mm = re.search(r"\b(LDL|STL)(\.\w+)*\b", ln)
    if mm:
        c[(cur, mm.group(1))] += 1
for (k, op), v in sorted(c.items(), key=lambda kv: (kv[0][0][0], kv[0][0][1])):
    print(f"{k[0]}:{k[1]} {op} x{v}")
