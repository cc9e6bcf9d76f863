#!/bin/bash
# Compare kernel build variants (dev tool): parity subset + timing per variant.
for lib in paper_1711_09791_b200/libsepconv_b200.so tools/_variants/lib_*.so; do
  echo "=== $lib"
  SEPCONV_B200_LIB=$lib timeout -s KILL 300 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "golden and (fused or passes)" 2>&1 | tail -1
  SEPCONV_B200_LIB=$lib timeout -s KILL 120 python tools/sweep.py --cfg cfg5 --grid '{};{"SC_NT":64};{"SC_NT":256};{"SC_NS":3};{"SC_NS":6};{"SC_NT":256,"SC_NS":3}' 2>&1 | grep -v "^\[sc\]"
  SEPCONV_B200_LIB=$lib timeout -s KILL 120 python tools/quick_perf.py --cfg cfg5 --ops hpass,single 2>&1 | grep -v "^\[sc\]"
done
