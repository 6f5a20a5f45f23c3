import os, subprocess, statistics, torch, json, sys
print(subprocess.run(["nvidia-smi","topo","-m"],capture_output=True,text=True).stdout)
print(subprocess.run(["lscpu"],capture_output=True,text=True).stdout[:1500])
def probe(tag, mb=200, nstream=1, reps=8):
    dev=torch.device("cuda"); n=mb<<20
    h_in=torch.empty(n,dtype=torch.uint8).pin_memory(); h_out=torch.empty(n,dtype=torch.uint8).pin_memory()
    h_in.fill_(1); h_out.fill_(1)
    d_in=torch.empty(n,dtype=torch.uint8,device=dev); d_out=torch.empty(n,dtype=torch.uint8,device=dev)
    ss=[torch.cuda.Stream() for _ in range(2*nstream)]
    ch=n//nstream
    ts=[]
    for i in range(reps+2):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for s in ss: s.wait_event(e0)
        for k in range(nstream):
            with torch.cuda.stream(ss[k]): d_in[k*ch:(k+1)*ch].copy_(h_in[k*ch:(k+1)*ch],non_blocking=True)
            with torch.cuda.stream(ss[nstream+k]): h_out[k*ch:(k+1)*ch].copy_(d_out[k*ch:(k+1)*ch],non_blocking=True)
        for s in ss:
            ev=torch.cuda.Event(); ev.record(s); torch.cuda.current_stream().wait_event(ev)
        e1.record(); torch.cuda.synchronize()
        if i>=2: ts.append(e0.elapsed_time(e1))
    t=statistics.median(ts)
    print(tag, f"mb={mb} streams/dir={nstream} bidir GB/s={2*n/t/1e6:.1f}", flush=True)
probe("default")
probe("default", nstream=4)
probe("default", mb=64)
# GPU-local cpus
out=subprocess.run(["nvidia-smi","topo","-m"],capture_output=True,text=True).stdout
line=[l for l in out.splitlines() if l.startswith("GPU0")][0].split()
print("GPU0 row", line)
cpus=None
for tok in line:
    if "-" in tok and tok.replace("-","").replace(",","").isdigit():
        cpus=tok; break
if cpus:
    s=set()
    for part in cpus.split(","):
        a,b=part.split("-"); s|=set(range(int(a),int(b)+1))
    os.sched_setaffinity(0,s); print("affinity", cpus)
    probe("local")
    probe("local", nstream=4)
