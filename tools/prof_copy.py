import torch, sys
x = torch.rand(3*16384*16384, device="cuda"); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize(); print("done")
