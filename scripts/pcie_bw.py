"""Raw pinned host<->device copy bandwidth (the e2e bound): each direction
alone, then both directions at once on two streams (full duplex)."""
import json
import time

import torch

for gb in (1, 5):
    n = gb * (1 << 30) // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    h2 = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    d2 = torch.empty(n, dtype=torch.float32, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(json.dumps({"dir": name, "GB": gb * 1.073741824, "GBps": round(gb * 1.073741824 / dt, 1)}))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    both(); torch.cuda.synchronize()
    t = time.perf_counter(); both(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(json.dumps({"dir": "h2d+d2h concurrent", "GB_each": gb * 1.073741824,
                      "GBps_each": round(gb * 1.073741824 / dt, 1), "GBps_total": round(2 * gb * 1.073741824 / dt, 1)}))
