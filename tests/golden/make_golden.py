"""Generate golden fixtures by running the REFERENCE implementation itself.

Run here (not on the GPU box; /root/reference does not exist there):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports sepconv_lab from /root/reference/pkg/src (read-only, no bytecode
written), drives its public entry points on seeded inputs and stores inputs +
outputs as small .npz fixtures next to this script. tests/test_oracle_golden.py
pins the CPU oracle to these fixtures (CPU) and tests/test_parity_gpu.py pins
the CUDA path to them (GPU).

Entry points exercised (S/ = /root/reference/pkg/src/sepconv_lab/):
  conv_two_pass (faithful + extended)          S/conv.py:392-421
  convolve_image TWO_PASS / SINGLE_* x plans   S/executors.py:269-405
  conv_single_pass_generic / _unrolled5        S/conv.py:324-359
  horizontal_pass / vertical_pass              S/conv.py:362-389
  copy_back                                    S/conv.py:424-440
  make_synthetic / splitmix64                  S/image.py:131-162
"""

from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))

import numpy as np  # noqa: E402

import sepconv_lab as ref  # noqa: E402
from paper_1711_09791_b200.configs import CONFIG_TAPS  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

SENTINEL = np.float32(-777.0)


def plane_case(name, planes_data: np.ndarray, taps: np.ndarray):
    """planes_data: (P, R, C) float32. Runs every path entry point of the reference."""
    P, R, C = planes_data.shape
    k = ref.SeparableKernel(taps)
    dense = ref.outer_product(k)
    out = {"input": planes_data.copy(), "taps": k.weights.copy(), "dense": dense.matrix.copy()}

    def image():
        return ref.Image([ref.Plane(planes_data[p].copy()) for p in range(P)])

    # conv_two_pass, faithful and extended (plane + scratch end state)
    for ext in (False, True):
        imgs, scrs = [], []
        for p in range(P):
            pl = ref.Plane(planes_data[p].copy())
            sc = ref.Plane.full(R, C, SENTINEL)  # zeroed by the op (S/conv.py:414)
            ref.conv_two_pass(pl, k, sc, extended=ext)
            imgs.append(pl.data)
            scrs.append(sc.data)
        tag = "ext" if ext else "faithful"
        out[f"two_pass_{tag}_image"] = np.stack(imgs)
        out[f"two_pass_{tag}_scratch"] = np.stack(scrs)

    # convolve_image TWO_PASS under two plans must equal conv_two_pass bitwise
    # (T/test_executors.py:188-231); asserted here so the fixture stores it once.
    for plan in (ref.Sequential(), ref.StaticChunked(3)):
        img = image()
        ws = ref.Image.zeros_like(img)
        variant = ref.ConvVariant(ref.Algorithm.TWO_PASS)
        ref.convolve_image(img, k, variant, plan, workspace=ws)
        res = ref.result_image(img, ws, variant)
        assert np.array_equal(np.stack([p.data for p in res.planes]), out["two_pass_faithful_image"])
        assert np.array_equal(np.stack([p.data for p in ws.planes]), out["two_pass_faithful_scratch"])

    # single pass: generic == unrolled bitwise (T/test_conv.py:64-71), zero and sentinel dst
    zs, ss = [], []
    for p in range(P):
        src = ref.Plane(planes_data[p].copy())
        z = ref.Plane.zeros(R, C)
        ref.conv_single_pass_generic(src, dense, z)
        if k.width == 5:
            z2 = ref.Plane.zeros(R, C)
            ref.conv_single_pass_unrolled5(src, dense, z2)
            assert np.array_equal(z.data, z2.data)
        s = ref.Plane.full(R, C, SENTINEL)
        ref.conv_single_pass_generic(src, dense, s)
        zs.append(z.data)
        ss.append(s.data)
    out["single_zero"] = np.stack(zs)
    out["single_sentinel"] = np.stack(ss)

    # convolve_image single pass, copy-back on/off (image + workspace end states)
    if k.width == 5:
        for copy in (False, True):
            variant = ref.ConvVariant(ref.Algorithm.SINGLE_PASS_UNROLLED5, copy_back=copy)
            img = image()
            ws = ref.Image.zeros_like(img)
            ref.convolve_image(img, k, variant, ref.StaticChunked(2), workspace=ws)
            img_a = np.stack([p.data for p in img.planes])
            ws_a = np.stack([p.data for p in ws.planes])
            assert np.array_equal(ws_a, out["single_zero"])
            if copy:
                out["convolve_single_copy_image"] = img_a
            else:
                assert np.array_equal(img_a, planes_data)
        # copy_back of the single-pass result into the source == the copy-back end state
        res = []
        region = ref.valid_region(R, C, 2)
        for p in range(P):
            a = ref.Plane(planes_data[p].copy())
            b = ref.Plane.zeros(R, C)
            ref.conv_single_pass_unrolled5(a, dense, b)
            ref.copy_back(b, a, region)
            res.append(a.data)
        assert np.array_equal(np.stack(res), out["convolve_single_copy_image"])

    # standalone passes into a sentinel dst (dst outside the valid region untouched)
    for pname, op in (("horizontal", ref.horizontal_pass), ("vertical", ref.vertical_pass)):
        res = []
        for p in range(P):
            d = ref.Plane.full(R, C, SENTINEL)
            op(ref.Plane(planes_data[p].copy()), k, d)
            res.append(d.data)
        out[f"{pname}_sentinel"] = np.stack(res)

    path = os.path.join(OUT, f"{name}.npz")
    np.savez(path, **out)
    return path


def wide_cases():
    """Widths above 9 (the reference takes any odd width, S/kernels.py:17-20)."""
    out = []
    img = ref.make_synthetic(30, 34, 2, 17)
    data = np.stack([p.data for p in img.planes])
    rng = np.random.default_rng(1711)
    for W in (11, 13):
        taps = rng.uniform(-1, 1, size=W).astype(np.float32)
        out.append(plane_case(f"syn_30x34_s17_w{W}", data, taps))
    return out


def subnormal_cases():
    """Products and sums in the float32 subnormal range (|x| < 2^-126 ~ 1.18e-38):
    numpy on x86 keeps subnormals (no FTZ/DAZ), so the reference's bits depend on
    gradual underflow in every multiply and add. Cases: tiny taps x tiny inputs,
    inputs just above and below FLT_MIN with ordinary taps, exact subnormal
    inputs, signed zeros and mixed signs; shapes with C % 4 == 0 (TMA path) and
    odd C (generic path)."""
    out = []
    rng = np.random.default_rng(1126)
    tiny = np.float32(np.finfo(np.float32).tiny)  # 2^-126
    for R, C in ((24, 40), (23, 37)):
        # 1. tiny taps (~1e-20) x tiny inputs (~1e-20): products ~1e-40, subnormal
        a = (rng.uniform(-1, 1, size=(2, R, C)) * 1e-20).astype(np.float32)
        a[0, 3, :] = 0.0
        a[1, :, 5] = -0.0
        out.append(plane_case(f"subnormal_{R}x{C}_tinytaps", a,
                              np.array([1e-20, 3e-20, 5e-20, 3e-20, 1e-20], dtype=np.float32)))
        out.append(plane_case(f"subnormal_{R}x{C}_tinyasym", a,
                              np.array([2e-20, -7e-21, 4e-20, 1.5e-20, -3e-20], dtype=np.float32)))
        # 2. inputs near FLT_MIN (some normal, some subnormal), ordinary taps
        b = (rng.uniform(-4, 4, size=(2, R, C)) * tiny).astype(np.float32)
        b[0, ::3, ::2] = (rng.uniform(-1, 1, size=b[0, ::3, ::2].shape) * 1e-40).astype(np.float32)
        b[1, 7, :] = np.float32(1e-45)  # the smallest subnormal
        for tname in ("gauss5", "sharpen", "normal"):
            out.append(plane_case(f"subnormal_{R}x{C}_fltmin_{tname}", b, CONFIG_TAPS[tname]))
        # 3. ordinary inputs x subnormal taps (width 3)
        c = rng.uniform(0, 256, size=(1, R, C)).astype(np.float32)
        out.append(plane_case(f"subnormal_{R}x{C}_subtaps_w3", c,
                              np.array([3e-41, 1e-40, 3e-41], dtype=np.float32)))
    return out


def subnormal_ppm():
    """u8 payload with subnormal and tiny taps: read_ppm -> two-pass -> write_ppm."""
    res = {}
    rng = np.random.default_rng(77)
    for (R, C), taps in (((32, 48), [1e-40, 2e-40, 5e-40, 2e-40, 1e-40]),
                         ((40, 64), [1e-39, -3e-39, 9e-39, -3e-39, 1e-39])):
        pix = rng.integers(0, 256, size=(R, C, 3), dtype=np.uint8)
        data = f"P6\n{C} {R}\n255\n".encode() + pix.tobytes()
        img = ref.read_ppm_bytes(data)
        k = ref.SeparableKernel(taps)
        ref.convolve_image(img, k, ref.ConvVariant(ref.Algorithm.TWO_PASS), ref.Sequential())
        key = f"{R}x{C}"
        res[f"in_{key}"] = np.frombuffer(data, dtype=np.uint8)
        res[f"out_{key}"] = np.frombuffer(ref.write_ppm_bytes(img), dtype=np.uint8)
        res[f"taps_{key}"] = k.weights
        res[f"planes_out_{key}"] = np.stack([p.data for p in img.planes])
    np.savez(os.path.join(OUT, "subnormal_ppm.npz"), **res)


def main():
    if "--only-wide" in sys.argv:  # add the wide fixtures without rewriting the others
        print(wide_cases())
        return
    if "--only-subnormal" in sys.argv:  # add the subnormal fixtures without rewriting the others
        print(subnormal_cases())
        subnormal_ppm()
        return
    written = []
    # 1. reference-test shapes on make_synthetic inputs (values in [0, 256))
    shapes = [
        ("syn_7x7_s42", 7, 7, 1, 42),      # T/test_conv.py:55-61 golden centre
        ("syn_9x10_s11", 9, 10, 1, 11),    # T/test_conv.py:44-52
        ("syn_12x12_s13", 12, 12, 1, 13),  # T/test_conv.py:194-204
        ("syn_12x13_s3", 12, 13, 3, 3),
        ("syn_16x16_s5", 16, 16, 3, 5),    # faithful rows {2,3,12,13} differ from extended
        ("syn_5x5_s0", 5, 5, 1, 0),        # minimum size
        ("syn_5x9_s1", 5, 9, 2, 1),
        ("syn_37x23_s8", 37, 23, 3, 8),    # SURVEY App. A band probe shape
        ("syn_129x131_s20", 129, 131, 1, 20),  # SPEC.md:491 odd/prime dims
        ("syn_24x64_s21", 24, 64, 3, 21),  # C % 4 == 0: TMA path shape
        ("syn_40x136_s22", 40, 136, 1, 22),
    ]
    for name, R, C, P, seed in shapes:
        img = ref.make_synthetic(R, C, P, seed)
        data = np.stack([p.data for p in img.planes])
        tap_sets = CONFIG_TAPS if R * C * P <= 4000 else {t: CONFIG_TAPS[t] for t in ("gauss5", "sharpen")}
        for tname, taps in tap_sets.items():
            written.append(plane_case(f"{name}_{tname}", data, taps))
    # 2. delta kernel and a non-5 width (generic path only)
    img = ref.make_synthetic(12, 16, 2, 4)
    data = np.stack([p.data for p in img.planes])
    written.append(plane_case("syn_12x16_s4_delta5", data, ref.delta(5).weights))
    written.append(plane_case("syn_12x16_s4_w3", data, np.array([0.1, 0.7, 0.3], dtype=np.float32)))
    written.extend(wide_cases())
    written.extend(subnormal_cases())
    subnormal_ppm()
    # 3. special values: negative, zero rows, large magnitudes (FMA-sensitive)
    rng = np.random.default_rng(1234)
    spec = rng.uniform(-1e4, 1e4, size=(2, 20, 28)).astype(np.float32)
    spec[0, 5, :] = 0.0
    spec[1, :, 7] = -0.0
    for tname, taps in CONFIG_TAPS.items():
        written.append(plane_case(f"special_20x28_{tname}", spec, taps))

    # 4. synthetic generator goldens (S/image.py:144-162) for the oracle's kind 0
    syn = {}
    for (R, C, P, seed) in ((5, 5, 1, 0), (8, 8, 3, 42), (6, 7, 2, 9), (33, 17, 3, 2**63)):
        syn[f"make_synthetic_{R}x{C}x{P}_s{seed}"] = np.stack(
            [p.data for p in ref.make_synthetic(R, C, P, seed).planes]
        )
    syn["splitmix64_s42_64"] = ref.splitmix64(42, 64)
    syn["splitmix64_smax_64"] = ref.splitmix64(2**64 - 1, 64)
    np.savez(os.path.join(OUT, "synthetic.npz"), **syn)

    # 5. PPM either side of the path (S/ppm.py): read -> convolve_image(TWO_PASS) -> write
    ppm = {}
    rng = np.random.default_rng(4242)
    for (R, C, tname) in ((16, 16, "gauss5"), (37, 48, "sharpen"), (64, 80, "gauss5"), (100, 160, "sigma1"),
                          (29, 131, "sharpen"), (24, 1040, "gauss5")):
        pix = rng.integers(0, 256, size=(R, C, 3), dtype=np.uint8)
        pix[0, :4] = 0
        pix[-1, -4:] = 255
        data = f"P6\n{C} {R}\n255\n".encode() + pix.tobytes()
        img = ref.read_ppm_bytes(data)
        k = ref.SeparableKernel(CONFIG_TAPS[tname])
        ref.convolve_image(img, k, ref.ConvVariant(ref.Algorithm.TWO_PASS), ref.Sequential())
        out = ref.write_ppm_bytes(img)
        key = f"{R}x{C}_{tname}"
        ppm[f"in_{key}"] = np.frombuffer(data, dtype=np.uint8)
        ppm[f"out_{key}"] = np.frombuffer(out, dtype=np.uint8)
        ppm[f"taps_{key}"] = k.weights
        ppm[f"planes_{key}"] = np.stack([p.data for p in ref.read_ppm_bytes(data).planes])
    # malformed headers: the reference's error message and byte offset
    bad = [b"P5\n2 2\n255\n" + bytes(12), b"P6x2 2\n255\n" + bytes(12), b"P6\n2 2\n255\n" + bytes(11),
           b"P6\n2 2\n255\n" + bytes(13), b"P6\n2 2\n65535\n" + bytes(24), b"P6\n0 2\n255\n",
           b"P6\n2 # c\n2\n255\n" + bytes(12), b"P6\n2 a\n255\n", b"P6\n2 2\n255", b"P6\n2 2\n255x" + bytes(12),
           b"P6\n2", b"P6 2 2 255\n" + bytes(12)]
    errs = []
    for i, d in enumerate(bad):
        try:
            ref.read_ppm_bytes(d)
            errs.append(("ok", -1))
        except ref.PpmParseError as e:
            errs.append((str(e), e.byte_offset))
        ppm[f"bad_{i}"] = np.frombuffer(d, dtype=np.uint8)
    ppm["bad_messages"] = np.array([m for m, _ in errs])
    ppm["bad_offsets"] = np.array([o for _, o in errs])
    np.savez(os.path.join(OUT, "ppm.npz"), **ppm)

    total = sum(os.path.getsize(p) for p in written)
    print(f"wrote {len(written)} plane fixtures ({total / 1e6:.2f} MB) + synthetic.npz")


if __name__ == "__main__":
    main()
