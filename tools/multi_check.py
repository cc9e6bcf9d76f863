"""Multi-rank orchestration check on ONE GPU (dev/CI tool), launched with
    torchrun --nproc-per-node N tools/multi_check.py
Ranks share the GPU and exchange halos over gloo through host memory (no kernel
ever waits on another rank's kernel); every rank checks its band of the banded
fused two-pass bit for bit against the whole-image kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from paper_1711_09791_b200 import device as dev
from paper_1711_09791_b200.multi import BandStepper, band_plan

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
ok = True
for (P, R, C, taps) in ((3, 1000, 2048, [1, 4, 6, 4, 1]), (3, 517, 1920, [-1, -2, 7, -2, -1]), (2, 64, 512, [0.25, 0.5, 0.25])):
    w = np.asarray(taps, np.float32) / (16 if taps[0] == 1 else 1)
    full = dev.synthetic((P, R, C), 7, 2)
    want = dev.two_pass(full, w)
    b = band_plan(R, rank, world, len(w) // 2)
    src = torch.full((P, b.local_rows, C), float("nan"), device="cuda")
    src[:, b.owned] = full[:, b.lo:b.hi]
    out = torch.empty((P, b.hi - b.lo, C), device="cuda")
    st = BandStepper(src, out, b, w)
    for _ in range(3):
        st.step()
    torch.cuda.synchronize()
    ok &= torch.equal(out, want[:, b.lo:b.hi])
flag = torch.tensor([1 if ok else 0])
dist.all_reduce(flag, op=dist.ReduceOp.MIN)
if rank == 0:
    print("multi_check", "OK" if flag.item() == 1 else "MISMATCH", "world", world)
dist.destroy_process_group()
sys.exit(0 if flag.item() == 1 else 1)
