"""Flag SASS memory instructions whose L2-policy descriptor register (desc[URn]) is never
written in the kernel (development aid, "A code-generation hazard").

python tools/sass_desc_check.py [libdiffmpc.so]
"""
import os
import re
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                        "paper_2605_29155_b200", "libdiffmpc.so")
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
def disasm(cub):
    return cub, subprocess.run(["nvdisasm", os.path.join(d, cub)], capture_output=True, text=True).stdout


bad = 0
kernels = 0
with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as pool:
    texts = list(pool.map(disasm, sorted(f for f in os.listdir(d) if f.endswith(".cubin"))))
for cub, txt in texts:
    for m in re.finditer(r"\.text\.(\S+):\n(.*?)(?=\n\s*\.section|\Z)", txt, re.S):
        fn, body = m.group(1), m.group(2)
        kernels += 1
        written = set()
        for ln in body.splitlines():
            mm = re.match(r"\s*/\*[0-9a-f]+\*/\s*(?:@!?U?P\w+\s+)?(\S+)\s+([^;]*);", ln)
            if not mm:
                continue
            dst = mm.group(2).split(",")[0].strip()
            for r in re.findall(r"UR(\d+)", dst):
                n = int(r)
                written.add(n)
                if ".64" in mm.group(1) or "CS2UR" in mm.group(1) or "LDCU.64" in mm.group(1):
                    written.add(n + 1)
        for ln in body.splitlines():
            for r in re.findall(r"desc\[UR(\d+)\]", ln):
                if int(r) not in written:
                    bad += 1
                    print(f"{cub} {fn[:90]}: {ln.strip()[:110]}")
print(f"{kernels} kernels checked, {bad} instructions with an unwritten descriptor register")
sys.exit(1 if bad else 0)
