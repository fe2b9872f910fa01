OUT=gpurun_out; mkdir -p $OUT; rm -f $OUT/summary.txt
free -g > $OUT/free0.txt
for rep in 1 2 3 4 5; do
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$rep.log 2>&1
  tail -1 $OUT/bench_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e', round(d['value'],1), 'K1', round(d['roofline']['avg_launch_ms'],4), 'steps', d['e2e']['rank0_device_ms_per_step'], 'pcie', d['binding_roofline']['pcie_measured']['duplex_combined_GBps'], 'reg_s', round(d['host_register_s'],1))" >> $OUT/summary.txt 2>&1
  free -g | head -2 | tail -1 >> $OUT/summary.txt
done
cat $OUT/summary.txt
