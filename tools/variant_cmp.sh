#!/bin/bash
# Time build variants of the library side by side (dev tool):
#   tools/variant_cmp.sh lib1.so lib2.so ...
# Variants are built beforehand, e.g.
#   python -m paper_1711_09791_b200.build -D SC_STATIC_FIRST=0 --out tools/vlib/x.so
# Per library: CUDA-graph timings of the fused kernel at small sizes, the
# bench's L2-flushed config-1/2 lines, and cfg5/cfg2 fused + single.
for rep in 1 2; do
for lib in "$@"; do
  n=$(basename $lib)
  for s in 1152 1728 2592; do
    SEPCONV_B200_LIB=$lib timeout -s KILL 120 python tools/sweep.py --size $s --op fused --reps 20 --graph --grid '{}' 2>/dev/null | grep -v '^\[sc\]' | tail -1 | sed "s|^|{\"lib\": \"$n\", \"rep\": $rep, \"size\": $s} |"
  done
  for c in cfg1 cfg2; do
    SEPCONV_B200_LIB=$lib timeout -s KILL 120 python bench.py --config $c --steps 200 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib': '$n', 'rep': $rep, 'bench': '$c', 'ms': d['ms_per_step']}))"
  done
  for c in cfg5 cfg2; do
    SEPCONV_B200_LIB=$lib timeout -s KILL 120 python tools/quick_perf.py --cfg $c --ops fused,single --reps 30 2>/dev/null | sed "s|^|{\"lib\": \"$n\", \"rep\": $rep} |"
  done
done
done
