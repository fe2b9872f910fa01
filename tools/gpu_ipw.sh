# Guided K1 plan: A/B of the segment-length cap (SO2DR_K1_IPW = uniform items per
# worker that set the cap; r02-guided default was 4 below 4096 rows, 6 above; now 8).
#   gpurun -- 'bash tools/gpu_ipw.sh'
OUT=gpurun_out; mkdir -p $OUT; rm -f $OUT/summary.txt
for ipw in default 6 8; do
  if [ $ipw = default ]; then unset SO2DR_K1_IPW; else export SO2DR_K1_IPW=$ipw; fi
  for rep in 1 2; do
    timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_ipw${ipw}_$rep.log 2>&1
    echo "== bench ipw=$ipw rc=$?" >> $OUT/summary.txt
    tail -1 $OUT/bench_ipw${ipw}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e', round(d['value'],1), 'hbm', round(d['hbm_resident']['value'],1), 'K1 ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3))" >> $OUT/summary.txt 2>&1
  done
done
for ipw in default 8 12; do
  if [ $ipw = default ]; then unset SO2DR_K1_IPW; else export SO2DR_K1_IPW=$ipw; fi
  SZ=32768 STENCILS=box2d1r,star2d1r KS=1,2,4,8 timeout 600 python tools/k1_bench.py > $OUT/k1_ipw$ipw.log 2>&1
  echo "== k1 ipw=$ipw rc=$?" >> $OUT/summary.txt
  python -c "
import json
for l in open('$OUT/k1_ipw$ipw.log'):
  try: d=json.loads(l); print(d['stencil'], d['k_on'], d['GCell_s'], d['alg_GBps'], d['fma_frac'])
  except Exception: print(l.strip()[:200])" >> $OUT/summary.txt
done
unset SO2DR_K1_IPW
cat $OUT/summary.txt
