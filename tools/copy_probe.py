"""torch copy_ / in-place neg_ of 512 MiB, for ncu comparison with the tile kernels."""
import torch

a = torch.empty(1 << 26, dtype=torch.float64, device="cuda").uniform_()
b = torch.empty_like(a)
for _ in range(3):
    b.copy_(a)
    a.neg_()
torch.cuda.synchronize()
print("ok")
