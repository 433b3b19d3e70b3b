import torch, time
x = torch.empty(1<<30, dtype=torch.float64, pin_memory=True)  # 8 GiB
d = torch.empty_like(x, device='cuda')
for _ in range(2): d.copy_(x, non_blocking=True); torch.cuda.synchronize()
t0=time.perf_counter()
for _ in range(3): d.copy_(x, non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t0)/3
print(f"raw pinned H2D 8 GiB: {dt*1e3:.1f} ms = {x.numel()*8/dt/1e9:.1f} GB/s")
