#!/bin/bash
for cfg in cfg1 cfg2; do
python tools/sweep.py --cfg $cfg --reps 50 --grid '{};{"SC_NT":32};{"SC_NT":64};{"SC_NT":96};{"SC_NT":64,"SC_BAND_H2":16};{"SC_NT":32,"SC_BAND_H2":16};{"SC_NT":64,"SC_BAND_H":64};{"SC_NS":3};{"SC_NT":32,"SC_NS":3}' 2>&1 | grep -v "^\[sc\]" | sed "s/^/$cfg /"
done
CMD="python tools/quick_perf.py --cfg cfg1 --ops fused --reps 5"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:sepconv -s 2 -c 2 $CMD 2>&1 | grep -E "duration|dram|lts" 
CMD="python tools/quick_perf.py --cfg cfg2 --ops fused --reps 5"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sepconv -s 2 -c 2 $CMD 2>&1 | grep -E "duration|dram"
