#!/bin/bash
# Small-image comparison of library variants (dev tool): CUDA-graph timings of the
# fused kernel at 3 x S^2 and the bench's L2-flushed config-1 line.
for rep in 1 2; do
for lib in "$@"; do
  n=$(basename $lib)
  for s in 1152 2592; do
    SEPCONV_B200_LIB=$lib timeout -s KILL 120 python tools/sweep.py --size $s --op fused --reps 20 --graph --grid '{}' 2>/dev/null | grep -v '^\[sc\]' | tail -1 | sed "s|^|{\"lib\": \"$n\", \"rep\": $rep, \"size\": $s} |"
  done
  SEPCONV_B200_LIB=$lib timeout -s KILL 120 python bench.py --config cfg1 --steps 200 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib': '$n', 'rep': $rep, 'bench': 'cfg1', 'ms': d['ms_per_step']}))"
done
done
