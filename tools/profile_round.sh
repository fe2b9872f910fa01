#!/bin/bash
# ncu evidence for the bench's dominant kernel (run under gpurun, one GPU).
#  1) launch list of the bench command (durations, cold-cache & serialised)
#  2) one --set full capture of a K1 launch of the bench shape
set -x
OUT=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-value-leg > $OUT/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_stencil2d -s 20 -c 1 -o $OUT/k1_full \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-value-leg > $OUT/k1_full.log 2>&1
ls -la $OUT
