#!/bin/bash
echo "default"; for i in 1 2; do python tools/bw_probe.py | grep -E "fused_w5|hpass_w5"; done
echo "default NS3"; SC_NS=3 python tools/bw_probe.py | grep -E "fused_w5|hpass_w5"
export SEPCONV_B200_LIB=tools/_variants/lib_minb4.so SC_NT=128
SC_FORCE_GENERIC=0 timeout -s KILL 300 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "golden and tma and fused" 2>&1 | tail -1
echo "minb4 NS3"; for i in 1 2; do SC_NS=3 python tools/bw_probe.py | grep -E "fused_w5|hpass_w5"; done
echo "minb4 NS4"; SC_NS=4 python tools/bw_probe.py | grep -E "fused_w5|hpass_w5"
for c in cfg3 cfg4; do SC_NS=3 python tools/sweep.py --cfg $c --reps 20 --grid '{}' 2>&1 | grep -v "^\[sc\]" | tail -1 | sed "s/^/minb4 ns3 $c /"; done
unset SEPCONV_B200_LIB SC_NT
for c in cfg3 cfg4; do python tools/sweep.py --cfg $c --reps 20 --grid '{}' 2>&1 | grep -v "^\[sc\]" | tail -1 | sed "s/^/default $c /"; done
