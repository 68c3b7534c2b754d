"""Pinned host -> device copy bandwidth (one stream vs two, whole vs chunked)."""
import torch
dev = torch.device("cuda")
n = 280_000_000 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device=dev)
img_h = torch.empty(6_220_800, dtype=torch.float32).pin_memory()
img_d = torch.empty(6_220_800, dtype=torch.float32, device=dev)
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def run(kind, reps=10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        if kind == "one":
            d.copy_(h, non_blocking=True)
        elif kind == "two":
            half = n // 2
            s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
            with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
        elif kind == "chunks":
            c = 8 << 20
            for o in range(0, n, c):
                d[o:o + c].copy_(h[o:o + c], non_blocking=True)
        elif kind == "one+d2h":
            s3.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s3): img_h.copy_(img_d, non_blocking=True)
            d.copy_(h, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s3)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{kind:8s} {ms:7.3f} ms  {n * 4 / ms / 1e6:6.1f} GB/s")
for k in ("one", "two", "chunks", "one+d2h", "one", "two"):
    run(k)
