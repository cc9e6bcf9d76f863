"""bench.py's driver contract on CPU: the reference arm (`--impl reference`,
the reference algorithm timed on host cores) prints ONE JSON line with the keys
the driver reads, and the host-path byte accounting mirrors csrc/stream.cu."""

from __future__ import annotations

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    # cfg1 keeps the CPU suite short; the driver runs the default (cfg5, the full image)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1", "--config", "cfg1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["warmup"] >= 3 and d["value"] > 0
    # the real reference package (baseline/_ref) on the full configured image
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert "sepconv_lab" in d["cpu_baseline"]["sample"] and d["cpu_baseline"]["cpu_model"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("cfg1") and d["config"]["rows"] == 1152


def test_host_chunk_accounting():
    sys.path.insert(0, ROOT)
    import bench

    # one chunk per plane when the plane is small: every byte once each way
    h2d, d2h = bench.host_chunk_bytes(64, 128, 3, 2, 0, 64, 0, 64)
    assert (h2d, d2h) == (3 * 64 * 128 * 4, 3 * 64 * 128 * 4)
    # big planes: 32 MiB chunks, each chunk re-reads the 2r halo rows of its neighbours
    R, C = 16384, 16384
    h2d, d2h = bench.host_chunk_bytes(R, C, 3, 2, 0, R, 0, R)
    ch = (32 << 20) // (C * 4)
    nchunks = -(-R // ch)
    assert d2h == 3 * R * C * 4
    assert h2d == 3 * (R * C * 4 + (nchunks - 1) * 2 * 2 * C * 4)
