"""Aggregate ncu_lines.py output of the forward kernel into phases (development aid).

python tools/ncu_phases.py <report> [kernel-regex] [object] [mangled]
"""
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "ilqr_forward"
obj = sys.argv[3] if len(sys.argv) > 3 else "paper_2605_29155_b200/build/inst_Quad13_float.o"
fn = sys.argv[4] if len(sys.argv) > 4 else "_ZN4dmpc19ilqr_forward_kernelINS_6Quad13ELi16ELb0EfLb0EEEvNS_7FwdArgsE"
out = subprocess.run([sys.executable, "tools/ncu_lines.py", rep, kre, obj, fn, "2000"], capture_output=True,
                     text=True).stdout
src = open("paper_2605_29155_b200/csrc/ilqr_forward.cuh").read().splitlines()
marks = [(i + 1, re.sub(r"[^a-z0-9 ]", "", l.lower()).strip()[:40]) for i, l in enumerate(src)
         if "// ====" in l or "// ----" in l or "PHASE:" in l]
ph = {}
for l in out.splitlines():
    m = re.match(r"\s*([\d.]+)% stall\s+([\d.]+)% inst\s+(\S+):(\d+)", l)
    if not m:
        continue
    st, ins, f, ln = float(m[1]), float(m[2]), m[3], int(m[4])
    if f == "ilqr_forward.cuh":
        name = "prologue"
        for mk, nm in marks:
            if ln >= mk:
                name = f"fwd:{nm}"
    else:
        name = f
    a = ph.setdefault(name, [0.0, 0.0])
    a[0] += st
    a[1] += ins
print(out.splitlines()[0])
for k, v in sorted(ph.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:50s} stall {v[0]:5.1f}  inst {v[1]:5.1f}")
