"""Pinned host <-> device copy bandwidth (the ceiling of bench.py's e2e leg): H2D alone, D2H alone,
and both directions at once on two streams, 1 GiB each, CUDA events."""
import json

import torch

N = 1 << 30
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_in = torch.empty(N, dtype=torch.uint8, device="cuda")
d_out = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))
bi = timed(both)
print(json.dumps({"h2d_GBps": N / h2d / 1e6, "d2h_GBps": N / d2h / 1e6, "bidir_each_GBps": N / bi / 1e6}))
