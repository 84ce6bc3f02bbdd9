#!/usr/bin/env python
"""Does the host link carry both directions at once? Times a host->device
copy (8 n bytes), a device->host copy (16 n bytes), and both together on two
streams (pinned memory), n = config 2's K0 rows."""
import json
import torch

n = 2356227
dev = torch.device("cuda", 0)
xh = torch.empty(n, dtype=torch.float64).pin_memory()
oh = torch.empty(2 * n, dtype=torch.float64).pin_memory()
xd = torch.empty(n, dtype=torch.float64, device=dev)
od = torch.empty(2 * n, dtype=torch.float64, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, k=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / k


def h2d():
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    s1.synchronize()


def d2h():
    with torch.cuda.stream(s2):
        oh.copy_(od, non_blocking=True)
    s2.synchronize()


def both():
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        oh.copy_(od, non_blocking=True)
    s1.synchronize()
    s2.synchronize()


def both_chunked(c=8):
    m = n // c
    for q in range(c):
        with torch.cuda.stream(s1):
            xd[q * m:(q + 1) * m].copy_(xh[q * m:(q + 1) * m], non_blocking=True)
        with torch.cuda.stream(s2):
            oh[2 * q * m:2 * (q + 1) * m].copy_(od[2 * q * m:2 * (q + 1) * m], non_blocking=True)
    s1.synchronize()
    s2.synchronize()


r = {"h2d_ms": timed(h2d), "d2h_ms": timed(d2h), "both_ms": timed(both),
     "both_8chunks_ms": timed(both_chunked)}
r["h2d_gbs"] = 8 * n / r["h2d_ms"] / 1e6
r["d2h_gbs"] = 16 * n / r["d2h_ms"] / 1e6
print(json.dumps(r))
