# Same-box A/B of the bench's chunk count d (k_on=4): d=32 vs d=64, interleaved.
OUT=gpurun_out; mkdir -p $OUT; rm -f $OUT/summary.txt
for rep in 1 2 3; do
  for dd in 64 32; do
    timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --d $dd > $OUT/bench_d${dd}_$rep.log 2>&1
    echo "== d=$dd rc=$?" >> $OUT/summary.txt
    tail -1 $OUT/bench_d${dd}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e', round(d['value'],1), 'frac_e2e', round(d['binding_roofline']['frac_e2e'],3), 'hbm', round(d['hbm_resident']['value'],1), 'K1 ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3), 'pred', round(d['planner']['predicted_for_this_config']['gcell_per_s'],1))" >> $OUT/summary.txt 2>&1
  done
done
cat $OUT/summary.txt
