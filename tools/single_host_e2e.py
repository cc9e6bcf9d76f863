"""convolve_image's single-pass variants on numpy planes: the streamed host path
(sc_single_pass_host_f32) next to round 1's stack -> H2D -> kernel -> D2H -> region copies (dev tool)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import Algorithm, ConvVariant, Cuda, Image, Plane, SeparableKernel, convolve_image
from paper_1711_09791_b200 import device as dev
from paper_1711_09791_b200.kernels import outer_product
R = C = int(os.environ.get("SIZE", 4096))
rng = np.random.default_rng(1)
x = rng.random((3, R, C), dtype=np.float32)
k = SeparableKernel(np.array([1, 4, 6, 4, 1], np.float32) / 16)
def old(image, ws, copy_back):
    src = torch.stack([torch.from_numpy(p.data) for p in image.planes]).cuda()
    wsd = torch.stack([torch.from_numpy(p.data) for p in ws.planes]).cuda()
    dev.single_pass(src, outer_product(k).matrix, wsd, copy_back=copy_back)
    src_h, wsd_h = src.cpu().numpy(), wsd.cpu().numpy()
    for p in range(3):
        ws.planes[p].data[2:-2, 2:-2] = wsd_h[p, 2:-2, 2:-2]
        if copy_back: image.planes[p].data[2:-2, 2:-2] = src_h[p, 2:-2, 2:-2]
for copy_back in (False, True):
    image = Image([Plane(p.copy()) for p in x]); ws = Image([Plane(np.zeros_like(p)) for p in x])
    v = ConvVariant(Algorithm.SINGLE_PASS_UNROLLED5, copy_back)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); convolve_image(image, k, v, Cuda(), workspace=ws); ts.append(time.perf_counter() - t0)
    to = []
    for _ in range(3):
        t0 = time.perf_counter(); old(image, ws, copy_back); to.append(time.perf_counter() - t0)
    print(json.dumps({"size": R, "copy_back": copy_back, "streamed_first_ms": round(ts[0] * 1e3, 2),
                      "streamed_ms": round(min(ts[1:]) * 1e3, 2), "round1_path_ms": round(min(to) * 1e3, 2)}), flush=True)
