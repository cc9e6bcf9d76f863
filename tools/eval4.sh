#!/bin/bash
for lib in paper_1711_09791_b200/libsepconv_b200.so tools/_variants/lib_srows2.so tools/_variants/lib_srows8.so; do
  echo "=== $lib"
  SEPCONV_B200_LIB=$lib timeout -s KILL 300 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "golden and tma" 2>&1 | tail -1
  SEPCONV_B200_LIB=$lib python tools/bw_probe.py | grep -E "fused_w5|hpass_w5|vpass_w5"
done
for ns in 6 10 12 16; do echo "srows2 ns=$ns"; SC_NS=$ns SEPCONV_B200_LIB=tools/_variants/lib_srows2.so python tools/bw_probe.py | grep -E "fused_w5"; done
for ns in 3 5 6; do echo "srows4 ns=$ns"; SC_NS=$ns python tools/bw_probe.py | grep -E "fused_w5"; done
