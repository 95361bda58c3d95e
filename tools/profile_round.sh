#!/bin/bash
# Round evidence on one B200 (run under gpurun): plain bench, launch list, full
# K5 capture, K5 DRAM traffic.  Writes gpurun_out/${TAG}_* (TAG defaults to r02).
set -x
OUT=gpurun_out
T=${TAG:-r02}
python bench.py --steps 300 --warmup 10 --cpu-seconds 10 > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > $OUT/${T}_reference.json 2> $OUT/${T}_reference.err
python bench.py --workload c4 --steps 20 --warmup 3 > $OUT/${T}_bench_c4.json 2> $OUT/${T}_bench_c4.err
python tools/prof_step.py > $OUT/${T}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${T}_launches.csv python tools/prof_step.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_render -s 1 -c 1 -o $OUT/${T}_k_render python tools/prof_step.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $OUT/${T}_kernel_metrics.csv python tools/prof_step.py --frames 1 > /dev/null 2>&1
echo done
