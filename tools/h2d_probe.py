"""H2D bandwidth from pinned host memory: one stream vs two streams (copy engines)."""
import torch
n = 1 << 28  # 1 GB of int32
h = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(3):
        e0.record()
        part = n // streams
        for i, s in enumerate(ss):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    print(streams, "streams:", round(4 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1), "GB/s")
