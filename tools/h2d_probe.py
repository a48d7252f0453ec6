import torch, time
x = torch.empty(42*1024*1024, dtype=torch.uint8).pin_memory()
d = torch.empty_like(x, device='cuda')
for _ in range(3): d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): d.copy_(x, non_blocking=True)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b)/10
print(f"H2D 42 MiB: {ms:.3f} ms = {42*1.048576/ms:.1f} GB/s")
