# Same-box A/B of bench chunkings: d / k_on (the B200 planner prefers d=144, k_on=8).
#   gpurun -- 'bash tools/gpu_ab_plan.sh'
OUT=gpurun_out; mkdir -p $OUT; rm -f $OUT/summary.txt
for rep in 1 2; do
  for v in "64 4" "96 4" "144 4" "144 8" "96 8"; do
    set -- $v
    timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-value-leg --d $1 --k-on $2 > $OUT/bench_d$1_k$2_$rep.log 2>&1
    echo "== d=$1 k_on=$2 rc=$?" >> $OUT/summary.txt
    tail -1 $OUT/bench_d$1_k$2_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e', round(d['value'],1), 'frac_e2e', round(d['binding_roofline']['frac_e2e'],3), 'K1 ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3), 'fma', round(d['roofline']['fma']['frac'],3), 'R_pcie', d['binding_roofline']['R_pcie'])" >> $OUT/summary.txt 2>&1
  done
done
cat $OUT/summary.txt
