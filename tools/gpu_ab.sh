# A/B of experiment builds: bash tools/gpu_ab.sh "default build/var_x/libso2dr_b200.so ..." [bench]
OUT=gpurun_out; mkdir -p $OUT
for lib in $1; do
  if [ "$lib" = default ]; then unset SO2DR_LIB; tag=default; else export SO2DR_LIB=$PWD/$lib; tag=$(basename $(dirname $lib)); fi
  echo "== $tag" >> $OUT/summary.txt
  SZ=32768 STENCILS=${STENCILS:-box2d1r,star2d1r} KS=${KS:-1,2,4,8} timeout 600 python tools/k1_bench.py > $OUT/k1_$tag.log 2>&1
  cat $OUT/k1_$tag.log | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l); print(d['stencil'], d['k_on'], d['GCell_s'], d['alg_GBps'], d['fma_frac'])
  except Exception: print(l.strip()[:200])" >> $OUT/summary.txt
  if [ -n "$2" ]; then
    timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_$tag.log 2>&1
    tail -1 $OUT/bench_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench value', round(d['value'],1), 'hbm', round(d['hbm_resident']['value'],1), 'K1 ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3))" >> $OUT/summary.txt 2>&1
  fi
done
unset SO2DR_LIB
