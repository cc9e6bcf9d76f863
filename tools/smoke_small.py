import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1711_09791_b200 import device as dev
from oracle import oracle as orc
w = np.array([1,4,6,4,1], np.float32)/np.float32(16)
x = orc.synthetic(3*64*128, 1, 1).reshape(3,64,128)
out = dev.two_pass(torch.from_numpy(x).cuda(), w)
torch.cuda.synchronize()
print("small ok:", np.array_equal(out.cpu().numpy(), orc.two_pass(x, w)))
