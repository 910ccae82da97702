"""PCIe bound of the e2e leg: pinned H2D, D2H and both at once (full duplex), CUDA events."""
import json

import torch

n = 25_557_032
dev = torch.device("cuda", 0)
h_in = torch.randn(n).pin_memory()
h_out = torch.empty(n).pin_memory()
d_a = torch.empty(n, device=dev)
d_b = torch.randn(n, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    a.record(cur)
    for _ in range(reps):
        fn()
    for s in (s1, s2):
        cur.wait_stream(s)
    b.record(cur)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(s1):
        s1.wait_stream(torch.cuda.current_stream())
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        s2.wait_stream(torch.cuda.current_stream())
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


def both_chunked(chunk=1 << 21):
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        with torch.cuda.stream(s1):
            d_a[a:b].copy_(h_in[a:b], non_blocking=True)
        with torch.cuda.stream(s2):
            h_out[a:b].copy_(d_b[a:b], non_blocking=True)


B = 4 * n
r = {}
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both), ("both_chunked_8MB", both_chunked),
                 ("both_chunked_2MB", lambda: both_chunked(1 << 19))):
    ms = timed(fn)
    r[name] = {"ms": ms, "GBps_each_way": B / ms / 1e6}
r["e2e_bound_fp32_GBps"] = B / r["both"]["ms"] / 1e6
print(json.dumps(r))
