import torch
n = 64 << 20
a = torch.ones(n // 2, dtype=torch.bfloat16, device="cuda:0")
b = torch.empty_like(a, device="cuda:1")
for _ in range(3): b.copy_(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): b.copy_(a)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"torch peer copy 64MB: {ms*1e3:.1f} us {n/ms/1e6:.1f} GB/s, can_access_peer={torch.cuda.can_device_access_peer(0,1)}")
