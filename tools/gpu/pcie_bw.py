"""Host<->device copy bandwidth from pinned memory (the ceiling of bench.py's e2e leg):
1 GiB H2D alone, D2H alone, and both at once on two streams."""
import json
import torch

N = 1 << 30
h_a = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h_b = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(N, dtype=torch.uint8, device="cuda")
d_b = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    a.record(cur)
    for _ in range(reps):
        fn()
    s1.wait_stream(cur)
    cur.wait_stream(s1)
    cur.wait_stream(s2)
    b.record(cur)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    d_a.copy_(h_a, non_blocking=True)


def d2h():
    h_b.copy_(d_b, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_a, non_blocking=True)
    with torch.cuda.stream(s2):
        h_b.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"h2d_GBps": round(N / t1 / 1e6, 1), "d2h_GBps": round(N / t2 / 1e6, 1),
                  "duplex_GBps_total": round(2 * N / t3 / 1e6, 1)}))
