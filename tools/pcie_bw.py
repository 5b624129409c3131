"""Pinned host<->device copy bandwidth on this box: H2D alone, D2H alone, both
directions at once (separate streams). Used to bound the host-path (e2e) numbers."""
import json
import torch

n = 64 << 20  # bytes per copy
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=20):
    for _ in range(3):
        if h2d:
            with torch.cuda.stream(s1):
                d.copy_(h, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s1.wait_event(a)
    s2.wait_event(a)
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d.copy_(h, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
    e1.record(s1)
    e2.record(s2)
    torch.cuda.current_stream().wait_event(e1)
    torch.cuda.current_stream().wait_event(e2)
    b.record()
    torch.cuda.synchronize()
    return n * reps / (a.elapsed_time(b) / 1e3) / 1e9


print(json.dumps({"h2d_gbs": run(True, False), "d2h_gbs": run(False, True), "both_each_gbs": run(True, True)}))
