OUT=gpurun_out; mkdir -p $OUT; rm -f $OUT/summary.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_k1_stream.py tests/test_gpu_kernels.py -x -q > $OUT/pytest_k1.log 2>&1; echo "pytest k1 rc=$?" >> $OUT/summary.txt; tail -3 $OUT/pytest_k1.log >> $OUT/summary.txt
SZ=32768 STENCILS=box2d1r,star2d1r,box2d2r KS=1,2,4,8 timeout 600 python tools/k1_bench.py > $OUT/k1_bench.log 2>&1; echo "k1 rc=$?" >> $OUT/summary.txt; cat $OUT/k1_bench.log >> $OUT/summary.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/summary.txt
tail -1 $OUT/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],1), 'hbm', d.get('hbm_resident',{}).get('value'), 'K1 ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3))" >> $OUT/summary.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_k1_variants.py tests/test_gpu_engine.py -x -q > $OUT/pytest_eng.log 2>&1; echo "pytest eng rc=$?" >> $OUT/summary.txt; tail -3 $OUT/pytest_eng.log >> $OUT/summary.txt
cat $OUT/summary.txt
