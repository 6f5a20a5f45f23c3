"""Instruction count per source region of one kernel (nvdisasm -g line info)."""
import os, re, subprocess, sys, tempfile
from collections import Counter
obj, fn = sys.argv[1], sys.argv[2]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
s = txt.index(f".text.{fn}:"); e = txt.find("//---------------------", s); body = txt[s:e]
cur = ("?", 0); cnt = Counter()
for ln in body.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m: cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
    if re.search(r"/\*[0-9a-f]{4,}\*/", ln): cnt[cur] += 1
src = {}
def region(f, l):
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2605_29155_b200", "csrc", f)
    if f not in src:
        src[f] = open(p).read().splitlines() if os.path.exists(p) else []
    lines = src[f]
    for k in range(min(l, len(lines)) - 1, -1, -1):
        t = lines[k]
        if f.startswith("ilqr") and ("// ====" in t or "// ----" in t or "auto stage_cost" in t):
            return t.strip()[:70]
        if not f.startswith("ilqr") and re.match(r"^(template|DMPC_DEV|struct|__global__)", t):
            return (lines[k + 1] if t.startswith("template") else t).strip()[:70]
    return "?"
reg = Counter()
for (f, l), n in cnt.items(): reg[(f, region(f, l))] += n
tot = sum(cnt.values())
print("total", tot)
for (f, r), n in reg.most_common(25): print(f"{n:6d} {100*n/tot:5.1f}%  {f}: {r}")
