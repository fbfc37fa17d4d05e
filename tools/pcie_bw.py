"""Host<->device copy bandwidth on this box (pinned memory), for the e2e
pipeline's bound: one 240 MB H2D, the same split over 2 streams, one D2H,
and H2D + D2H concurrently."""
import json
import torch

n = 240 * 2**20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n // 6, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n // 6, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        for s in (s1, s2):
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


out = {}
out["h2d_1stream_GBs"] = n / timed(lambda: d.copy_(h, non_blocking=True)) / 1e6
def two():
    with torch.cuda.stream(s1):
        d[: n // 2].copy_(h[: n // 2], non_blocking=True)
    with torch.cuda.stream(s2):
        d[n // 2:].copy_(h[n // 2:], non_blocking=True)
out["h2d_2streams_GBs"] = n / timed(two) / 1e6
out["d2h_1stream_GBs"] = n / timed(lambda: h.copy_(d, non_blocking=True)) / 1e6
def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
out["h2d_240MB_plus_d2h_40MB_ms"] = timed(both)
out["h2d_240MB_alone_ms"] = timed(lambda: d.copy_(h, non_blocking=True))
print(json.dumps(out))
