#!/bin/bash
timeout -s KILL 900 python -m pytest tests/test_dropin_gpu.py -x -q -m gpu 2>&1 | tail -3
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout -s KILL 300 python tools/sweep.py --cfg cfg5 --grid '{};{"SC_BAND_H":32};{"SC_BAND_H":128};{"SC_BAND_H":256};{"SC_L2_NORMAL":1};{"SC_L2_NORMAL":1,"SC_BAND_H":128};{"SC_NS":3};{"SC_NS":5};{"SC_NS":6};{"SC_NT":96};{"SC_NT":160};{"SC_NT":192}' 2>&1 | grep -v "^\[sc\]"
for c in cfg1 cfg2 cfg3; do timeout -s KILL 120 python tools/sweep.py --cfg $c --grid '{};{"SC_BAND_H":16};{"SC_BAND_H":32};{"SC_L2_NORMAL":1};{"SC_NT":64}' 2>&1 | grep -v "^\[sc\]" | sed "s/^/$c /"; done
