#!/bin/bash
timeout -s KILL 900 python -m pytest tests -x -q -m gpu -k "not config and not orchestration" 2>&1 | tail -1
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do SC_DEBUG_PLAN=1 python tools/quick_perf.py --cfg $c --ops fused --reps 3 2>&1 | grep "\[sc\]" | head -1; done
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do python tools/sweep.py --cfg $c --reps 30 --grid '{}' 2>&1 | grep -v "^\[sc\]" | tail -1 | sed "s/^/$c /"; done
for c in cfg1 cfg2 cfg3; do python bench.py --config $c --steps 300 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['effective_GBps'], d['roofline']['kernel_ms'])"; done
