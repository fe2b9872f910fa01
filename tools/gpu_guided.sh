# A/B of the K1 row segmentation: guided plan (default) vs the r02-mid uniform
# segments (SO2DR_K1_SEGS=uniform: SO2DR_K1_IPW items per warp, r02-mid: 4 below 4096 rows, 6 above).
#   gpurun -- 'bash tools/gpu_guided.sh [tests]'
OUT=gpurun_out; mkdir -p $OUT; rm -f $OUT/summary.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
if [ "$1" = tests ]; then
  timeout 1200 python -m pytest tests/test_gpu_k1_stream.py tests/test_gpu_kernels.py tests/test_gpu_k1_variants.py tests/test_gpu_engine.py tests/test_gpu_3d_f64.py -x -q > $OUT/pytest_k1.log 2>&1
  echo "pytest k1 rc=$?" >> $OUT/summary.txt; tail -3 $OUT/pytest_k1.log >> $OUT/summary.txt
fi
for ipw in guided uniform; do
  if [ $ipw = guided ]; then unset SO2DR_K1_SEGS; else export SO2DR_K1_SEGS=$ipw; fi
  SZ=32768 STENCILS=box2d1r,star2d1r,box2d2r KS=1,2,4,8 timeout 600 python tools/k1_bench.py > $OUT/k1_$ipw.log 2>&1
  SZ3=768 STENCILS=star3d1r,box3d1r KS=1,2,4 timeout 600 python tools/k1_bench.py >> $OUT/k1_$ipw.log 2>&1
  echo "== k1 $ipw rc=$?" >> $OUT/summary.txt
  python -c "
import json,sys
for l in open('$OUT/k1_$ipw.log'):
  try: d=json.loads(l); print(d['stencil'], d['k_on'], d['GCell_s'], d['alg_GBps'], d['fma_frac'])
  except Exception: print(l.strip()[:200])" >> $OUT/summary.txt
done
for ipw in guided uniform guided uniform; do
  if [ $ipw = guided ]; then unset SO2DR_K1_SEGS; else export SO2DR_K1_SEGS=$ipw; fi
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_$ipw.log 2>&1
  echo "== bench $ipw rc=$?" >> $OUT/summary.txt
  tail -1 $OUT/bench_$ipw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e', round(d['value'],1), 'hbm', round(d['hbm_resident']['value'],1), 'K1 ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3))" >> $OUT/summary.txt 2>&1
done
unset SO2DR_K1_SEGS
cat $OUT/summary.txt
