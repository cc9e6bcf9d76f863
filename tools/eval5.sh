#!/bin/bash
timeout -s KILL 600 python -m pytest tests -x -q -m gpu -k "not config" 2>&1 | tail -1
SC_DEBUG_PLAN=1 python tools/quick_perf.py --cfg cfg5 --ops fused --reps 3 2>&1 | grep "\[sc\]" | head -1
for cfg in cfg5 cfg4 cfg3; do
python tools/sweep.py --cfg $cfg --grid '{};{"SC_BAND_H":128};{"SC_BAND_H":512};{"SC_BAND_H2":16};{"SC_BAND_H2":64};{"SC_NS":3};{"SC_NS":3,"SC_BAND_H":512};{"SC_BAND_H":64,"SC_BAND_H2":64}' 2>&1 | grep -v "^\[sc\]" | sed "s/^/$cfg /"
done
