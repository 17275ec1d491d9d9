"""D2H rate with 1, 2, 3 concurrent streams, 64 MB total per round (diagnostic)."""
import torch

tot = 64 << 20
for ns in (1, 2, 3, 6):
    per = tot // ns
    hs = [torch.empty(per, dtype=torch.uint8).pin_memory() for _ in range(ns)]
    ds = [torch.empty(per, dtype=torch.uint8, device="cuda") for _ in range(ns)]
    sts = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for s in sts:
            s.wait_stream(torch.cuda.current_stream())
        for _ in range(10):
            for h, d, s in zip(hs, ds, sts):
                with torch.cuda.stream(s):
                    h.copy_(d, non_blocking=True)
        for s in sts:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        print(f"d2h streams={ns}: {tot * 10 / (a.elapsed_time(b) / 1e3) / 1e9:.1f} GB/s")
