set -x
for c in cfg5 cfg2; do
python tools/kernel_table.py --cfg $c > gpurun_out/kt_$c.jsonl 2>&1
python tools/kernel_table.py --cfg $c --ncu-pass > gpurun_out/kt_plain_$c.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/kt_ncu_$c.csv python tools/kernel_table.py --cfg $c --ncu-pass > gpurun_out/kt_ncu_$c.log 2>&1
python tools/kernel_table.py --merge gpurun_out/kt_ncu_$c.csv gpurun_out/kt_$c.jsonl > gpurun_out/kt_table_$c.md 2>&1
done
