#!/bin/bash
export SC_DIRECT=1
timeout -s KILL 600 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "not config" 2>&1 | tail -1
python tools/bw_probe.py
for b in 32 128 256; do SC_BAND_H=$b python tools/sweep.py --cfg cfg5 --grid '{}' 2>&1 | grep -v "^\[sc\]" | tail -1 | sed "s/^/band=$b /"; done
for lib in tools/_variants/lib_du4.so tools/_variants/lib_du4m1.so; do echo "== $lib"; SEPCONV_B200_LIB=$lib python tools/bw_probe.py | grep -E "fused|hpass_w5|vpass_w5"; done
