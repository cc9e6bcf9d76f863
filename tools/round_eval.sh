#!/bin/bash
# Full GPU evaluation: tests, bench, launch list, one full ncu capture, per-config timings.
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout -s KILL 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
timeout -s KILL 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1; cat gpurun_out/bench_ref.json
for c in cfg1 cfg2 cfg3 cfg4; do timeout -s KILL 300 python tools/quick_perf.py --cfg $c --ops fused,split,single,copy 2>&1 | grep -v "^\[sc\]"; done > gpurun_out/configs.jsonl; cat gpurun_out/configs.jsonl
CMD="python bench.py --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
for c in cfg1 cfg2 cfg3 cfg4; do timeout -s KILL 300 python bench.py --config $c --steps 200 --e2e-steps 1 --no-cpu-baseline 2>/dev/null; done > gpurun_out/bench_configs.jsonl; cat gpurun_out/bench_configs.jsonl
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
python tools/prof_one.py --op fused > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sepconv_rows -s 2 -c 1 -f -o gpurun_out/prof_fused_cfg5 python tools/prof_one.py --op fused > gpurun_out/ncu_full.log 2>&1
python tools/prof_one.py --op single > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sepconv_rows -s 2 -c 1 -f -o gpurun_out/prof_single_cfg5 python tools/prof_one.py --op single > gpurun_out/ncu_single.log 2>&1
python tools/misalign_probe.py > gpurun_out/misalign.jsonl 2>&1; cat gpurun_out/misalign.jsonl
python -m paper_1711_09791_b200.ladder --reps 200 --csv gpurun_out/ladder_gpu.csv > /dev/null 2>&1
ls -la gpurun_out
# per-kernel table (every kernel family: event time, DRAM bytes) and full captures of the in-place and u8 kernels
bash tools/kernel_table.sh > gpurun_out/kt.log 2>&1
python tools/kernel_table.py --cfg cfg5 --ncu-pass > gpurun_out/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sepconv_u8 -s 3 -c 1 -f -o gpurun_out/prof_u8_cfg5 python tools/kernel_table.py --cfg cfg5 --ncu-pass > gpurun_out/ncu_u8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sepconv_rows -s 3 -c 1 -f -o gpurun_out/prof_splitf_cfg5 python tools/kernel_table.py --cfg cfg5 --ncu-pass > gpurun_out/ncu_sf.log 2>&1
ls -la gpurun_out
