"""PCIe probe (development tool): pinned H2D, D2H and both at once on two streams, the bound of
the e2e leg (bench.py e2e moves x in and y out every product).  One JSON line per size."""
import json, sys
import torch

for mb in [int(s) for s in (sys.argv[1:] or ["456", "228", "64"])]:
    n = mb << 20
    hx = torch.empty(n, dtype=torch.uint8, pin_memory=True).fill_(1)
    hy = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dx = torch.empty(n, dtype=torch.uint8, device="cuda")
    dy = torch.empty(n, dtype=torch.uint8, device="cuda").fill_(2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def run(h2d, d2h, reps=10):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in (s1, s2):
            s.wait_event(e0)
        for _ in range(reps):
            if h2d:
                with torch.cuda.stream(s1):
                    dx.copy_(hx, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    hy.copy_(dy, non_blocking=True)
        cur = torch.cuda.current_stream()
        cur.wait_stream(s1)
        cur.wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3

    run(True, True, 2)
    th, td, tb = run(True, False), run(False, True), run(True, True)
    print(json.dumps({"MB": mb, "h2d_gbs": round(n / th / 1e9, 1), "d2h_gbs": round(n / td / 1e9, 1),
                      "both_ms": round(tb * 1e3, 3), "both_each_gbs": round(n / tb / 1e9, 1),
                      "h2d_ms": round(th * 1e3, 3), "d2h_ms": round(td * 1e3, 3)}), flush=True)
