"""PCIe copy rates on this box (pinned host memory, CUDA events): H2D alone,
D2H alone, and both directions at once on two streams -- the ceiling of the
e2e (host-buffer) SpMV, which moves x in and y out every step.

    python tools/pcie_probe.py [--mb 32] [--reps 20]
"""
import argparse
import json

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--mb", type=int, default=32)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
nb = a.mb << 20
h_in = torch.empty(nb, dtype=torch.uint8).pin_memory()
h_out = torch.empty(nb, dtype=torch.uint8).pin_memory()
d_in = torch.empty(nb, dtype=torch.uint8, device="cuda")
d_out = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps * 1e-3


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


s1.wait_stream(torch.cuda.current_stream())
s2.wait_stream(torch.cuda.current_stream())
t_in, t_out, t_both = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"mb": a.mb, "h2d_GBps": nb / t_in / 1e9, "d2h_GBps": nb / t_out / 1e9,
                  "duplex_ms_per_pair": t_both * 1e3,
                  "duplex_GBps_each": nb / t_both / 1e9}))
