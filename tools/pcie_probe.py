"""Host<->device copy bandwidth of this box (the bound of bench.py's e2e leg).

    python tools/pcie_probe.py [--mb 200] [--reps 10]

Pinned host buffers, one copy engine per direction: H2D alone, D2H alone, and both
directions at once on two streams (what the e2e pipeline sustains at best). CUDA-event
timed, median of reps. Prints one JSON line.
"""
import argparse
import json
import statistics

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=200)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda")
    n = a.mb << 20
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device=dev)
    d_out = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        ts = []
        for i in range(a.reps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            s1.wait_event(e0)
            s2.wait_event(e0)
            fn()
            for s in (s1, s2):
                ev = torch.cuda.Event()
                ev.record(s)
                torch.cuda.current_stream().wait_event(ev)
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    t_h, t_d, t_b = timed(h2d), timed(d2h), timed(both)
    r = {"bytes": n, "h2d_gbs": n / t_h / 1e6, "d2h_gbs": n / t_d / 1e6,
         "bidir_gbs": 2 * n / t_b / 1e6, "bidir_ms": t_b}
    print(json.dumps(r))


if __name__ == "__main__":
    main()
