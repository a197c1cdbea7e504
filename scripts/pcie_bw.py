"""Raw pinned host<->device copy bandwidth (the e2e bound)."""
import time, torch, json
for gb in (1, 5):
    n = gb * (1 << 30) // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(json.dumps({"dir": name, "GB": gb * 1.073741824, "GBps": round(gb * 1.073741824 / dt, 1)}))
