"""Per-kernel efficiency table at one config (dev tool; evidence for DESIGN section 3).

    python tools/kernel_table.py --cfg cfg5                 # CUDA-event timings -> JSON lines
    python tools/kernel_table.py --cfg cfg5 --ncu-pass      # one launch per op (run under ncu)
    python tools/kernel_table.py --merge launches.csv times.jsonl   # -> markdown table

Every kernel family of the path runs on the same seeded image: fused two-pass
(K1), row pass with zero fill and column pass (the split pair K2/K3), single
pass (and its copy-back), the one-pass split mode, and the PPM u8 payload kernel. For each the
ALGORITHMIC bytes are the minimum one launch must move (a read of every input
sample it needs once, a write of every output sample), so `alg GB/s` is what
the roofline fraction uses; ncu's dram__bytes show the real traffic.
"""
import argparse, csv, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

OPS = ["fused", "split", "hpass_zero", "vpass", "single", "single_general", "single_copyback", "u8"]

# FP32 pipe peak for the FP-bound kernels: 126.7 lane-ops per cycle per SM measured
# for FFMA/FMUL/FADD and their packed forms alike (tools/fp2_rate.cu,
# profiles/r02_fp2_rate.txt) x 148 SMs x the 1965 MHz maximum SM clock
FP32_PEAK_OPS = 126.7 * 148 * 1.965e9


def build_ops(cfg):
    import numpy as np, torch
    from paper_1711_09791_b200 import device as dev
    from paper_1711_09791_b200.configs import CONFIGS
    wl = CONFIGS[cfg]
    w = wl.tap_vector()
    r = len(w) // 2
    shape = (wl.frames, wl.planes, wl.rows, wl.cols) if wl.frames > 1 else (wl.planes, wl.rows, wl.cols)
    x = dev.synthetic(shape, wl.seed, wl.kind)
    y = torch.empty_like(x)
    z = torch.zeros_like(x)
    dense = np.outer(w, w).astype(np.float32)
    from paper_1711_09791_b200.configs import CONFIG_TAPS
    wn = CONFIG_TAPS["normal"]  # asymmetric taps (config 2): a dense matrix with no mirror symmetry
    dense_general = np.outer(wn, wn).astype(np.float32)
    n_px = x.numel()                      # samples of all planes
    R, C = wl.rows, wl.cols
    valid = (R - 2 * r) * (C - 2 * r) * (n_px // (R * C))
    u8 = torch.randint(0, 256, (R, C, 3), dtype=torch.uint8, device=x.device)
    u8o = torch.empty_like(u8)
    ops = {
        # op: (callable, algorithmic bytes per launch, what)
        "fused": (lambda: dev.two_pass(x, w, y), 8 * n_px, "read image + write image"),
        "split": (lambda: dev.two_pass_split(y, z, w), 12 * n_px,
                  "read image + write scratch + write image (the reference's buffer end state)"),
        "hpass_zero": (lambda: dev.hpass(x, w, y, 0, R, zero_fill=True), 8 * n_px,
                       "read image + write scratch (all rows, ring zeroed)"),
        "vpass": (lambda: dev.vpass(y, w, z), 4 * n_px + 4 * valid, "read scratch + write valid region"),
        "single": (lambda: dev.single_pass(x, dense, y), 4 * n_px + 4 * valid, "read image + write valid region"),
        "single_general": (lambda: dev.single_pass(x, dense_general, y), 4 * n_px + 4 * valid,
                           "read image + write valid region (config-2 taps: no mirror symmetry)"),
        "single_copyback": (lambda: dev.single_pass(x, dense, y, copy_back=True), 4 * n_px + 8 * valid,
                            "read image + write valid region to workspace and image"),
        "u8": (lambda: dev.two_pass_u8hwc(u8, w, u8o), 6 * R * C, "read + write 3 B/pixel"),
    }
    return wl, ops


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg5")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ncu-pass", action="store_true")
    ap.add_argument("--merge", nargs=2, metavar=("NCU_CSV", "TIMES_JSONL"))
    a = ap.parse_args()
    if a.merge:
        return merge(*a.merge)
    import numpy as np, torch
    wl, ops = build_ops(a.cfg)
    marker = torch.empty(1, device="cuda")
    for name in OPS:  # warm-up of every op first (plans memoised, modules loaded)
        for _ in range(3):
            ops[name][0]()
    torch.cuda.synchronize()
    for name in OPS:
        fn, alg, what = ops[name]
        if a.ncu_pass:
            marker.fill_(1.0)  # a torch kernel: separates this op's launches in the ncu list
            fn()
            torch.cuda.synchronize()
            continue
        ts = []
        for _ in range(a.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(5):
                fn()
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e) / 5)
        ms = float(np.median(ts))
        W = len(wl.tap_vector())
        R, C = wl.rows, wl.cols
        valid = (R - 2 * (W // 2)) * (C - 2 * (W // 2)) * (wl.frames * wl.planes)
        # the reference algorithm's float32 operations (S/conv.py:86-114, 215-293)
        ops_n = {"single": valid * (2 * W * W - 1), "single_general": valid * (2 * W * W - 1),
                 "single_copyback": valid * (2 * W * W - 1), "fused": valid * 2 * (2 * W - 1),
                 "split": valid * 2 * (2 * W - 1), "u8": (R - 2 * (W // 2)) * (C - 2 * (W // 2)) * 3 * 2 * (2 * W - 1),
                 "hpass_zero": valid * (2 * W - 1), "vpass": valid * (2 * W - 1)}[name]
        print(json.dumps({"cfg": a.cfg, "op": name, "ms": round(ms, 4), "alg_bytes": alg,
                          "alg_GBps": round(alg / ms / 1e6, 1), "fp32_ops": ops_n,
                          "fp32_frac": round(ops_n / (ms / 1e3) / FP32_PEAK_OPS, 3), "what": what}), flush=True)


def merge(ncu_csv, times):
    """ncu --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
    of the --ncu-pass run: each op's launches follow a torch fill kernel (the
    separator); an op's own kernels (namespace sc::) are summed."""
    t = [json.loads(l) for l in open(times) if l.startswith("{")]
    rows = list(csv.DictReader(l for l in open(ncu_csv) if l.startswith('"')))
    by_id = {}
    for r_ in rows:
        d = by_id.setdefault(int(r_["ID"]), {"name": r_["Kernel Name"]})
        v = float(r_["Metric Value"].replace(",", ""))
        d[r_["Metric Name"]] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3,
                                    "ms": 1.0, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}.get(
            r_["Metric Unit"], 1)
    groups, cur = [], None
    for k in sorted(by_id):
        d = by_id[k]
        if "sc::" not in d["name"]:
            cur = []
            groups.append(cur)
        elif cur is not None:
            cur.append(d)
    groups = groups[-len(OPS):]
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    peak = float(peaks.get("hbm_gbs", 6551.4))
    print("| op | kernels | event ms | alg bytes | alg GB/s | frac of measured copy | FP32 ops (ref. algorithm) | "
          "frac of FP32 pipe | ncu ms (sum) | ncu dram bytes | dram / alg |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for d, g in zip(t, groups):
        dram = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in g)
        nms = sum(x.get("gpu__time_duration.sum", 0) for x in g)
        names = ", ".join(sorted({x["name"].split("(")[0].replace("void ", "").replace("sc::", "") for x in g}))
        print(f"| {d['op']} | `{names}` | {d['ms']} | {d['alg_bytes'] / 1e9:.3f} G | {d['alg_GBps']} | "
              f"{d['alg_GBps'] / peak:.3f} | {d.get('fp32_ops', 0) / 1e9:.2f} G | {d.get('fp32_frac', 0):.3f} | "
              f"{nms:.4f} | {dram / 1e9:.3f} G | {dram / d['alg_bytes']:.3f} |")


if __name__ == "__main__":
    main()
