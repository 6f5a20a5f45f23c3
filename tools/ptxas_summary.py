import re, sys, subprocess
log = open(sys.argv[1]).read().splitlines()
cur = None; rows = {}
for ln in log:
    m = re.search(r"Compiling entry function '([^']+)'", ln)
    if m: cur = m.group(1); rows[cur] = {}; continue
    if cur is None: continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m: rows[cur].update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
    m = re.search(r"Used (\d+) registers", ln)
    if m: rows[cur]['regs'] = int(m.group(1))
names = list(rows)
dem = subprocess.run(['c++filt'], input='\n'.join(names), capture_output=True, text=True).stdout.splitlines()
for n, d in zip(names, dem):
    if len(sys.argv) > 2 and not re.search(sys.argv[2], d): continue
    r = rows[n]
    d = re.sub(r'\(anonymous namespace\)::|dmpc::', '', d)
    print(f"{r.get('regs','?'):>4} regs  stack {r.get('stack','?'):>4}  spill st/ld {r.get('spill_st','?')}/{r.get('spill_ld','?')}  {d[:110]}")
