import torch, time
x = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for _ in range(2):
    with torch.cuda.stream(s):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s); d.copy_(x, non_blocking=True); b.record(s)
    torch.cuda.synchronize()
    print("H2D 1 GiB pinned: %.1f GB/s" % ((1 << 30) / (a.elapsed_time(b) * 1e-3) / 1e9))
# concurrent with a compute kernel on another stream
y = torch.randn(8192, 8192, device="cuda")
with torch.cuda.stream(s):
    a.record(s); d.copy_(x, non_blocking=True); b.record(s)
for _ in range(20): y = y @ y * 1e-4
torch.cuda.synchronize()
print("H2D under concurrent GEMMs: %.1f GB/s" % ((1 << 30) / (a.elapsed_time(b) * 1e-3) / 1e9))
