"""PCIe H2D bandwidth from pinned memory: one stream vs two, whole vs 4 MiB chunks."""
import torch, time
n = 134184960
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(streams, chunk):
    torch.cuda.synchronize(); t = time.perf_counter()
    for i, off in enumerate(range(0, n, chunk)):
        with torch.cuda.stream(streams[i % len(streams)]):
            d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
    torch.cuda.synchronize(); return time.perf_counter() - t
for name, st, ch in [("1 stream whole", [s1], n), ("1 stream 4MiB", [s1], 4 << 20), ("2 streams 4MiB", [s1, s2], 4 << 20)]:
    ts = [run(st, ch) for _ in range(5)]
    print(f"{name:16s} {min(ts)*1e3:6.2f} ms  {n/min(ts)/1e9:6.1f} GB/s")
dd = torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(5): h.copy_(dd, non_blocking=True)
torch.cuda.synchronize(); print(f"D2H {n*5/(time.perf_counter()-t)/1e9:6.1f} GB/s")
