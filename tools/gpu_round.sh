#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + one full K1 capture.
# Usage (here): gpurun --timeout 3000 -- 'bash tools/gpu_round.sh [tests|bench|ncu]...'
OUT=gpurun_out
mkdir -p $OUT
steps=${@:-tests bench ncu}
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1; free -g > $OUT/free.txt 2>&1
for s in $steps; do
  case $s in
    tests)
      timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/summary.txt ;;
    bench)
      timeout 1200 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/summary.txt
      tail -1 $OUT/bench.log >> $OUT/summary.txt ;;
    refarm)
      timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $OUT/bench_ref.log 2>&1; echo "ref rc=$?" >> $OUT/summary.txt
      tail -1 $OUT/bench_ref.log >> $OUT/summary.txt ;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-value-leg > $OUT/launches_bench.log 2>&1
      echo "ncu launches rc=$?" >> $OUT/summary.txt
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_stencil2d -s 20 -c 1 -o $OUT/k1_full -f \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-value-leg > $OUT/k1_full.log 2>&1
      echo "ncu full rc=$?" >> $OUT/summary.txt ;;
  esac
done
cat $OUT/summary.txt
