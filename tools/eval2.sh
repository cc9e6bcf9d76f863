#!/bin/bash
timeout -s KILL 600 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "not config" 2>&1 | tail -1
echo "== TMA"; python tools/bw_probe.py
for b in 32 128; do SC_BAND_H=$b python tools/bw_probe.py | grep fused_w5 | sed "s/^/band=$b /"; done
for n in 3 6; do SC_NS=$n python tools/bw_probe.py | grep fused_w5 | sed "s/^/ns=$n /"; done
SC_NT=64 python tools/bw_probe.py | grep fused_w5 | sed "s/^/nt=64 /"
echo "== DIRECT"; SC_DIRECT=1 python tools/bw_probe.py
for b in 32 128; do SC_DIRECT=1 SC_BAND_H=$b python tools/bw_probe.py | grep fused_w5 | sed "s/^/band=$b /"; done
echo "== DIRECT du4"; SC_DIRECT=1 SEPCONV_B200_LIB=tools/_variants/lib_du4.so python tools/bw_probe.py | grep -E "pass_w5|fused"
