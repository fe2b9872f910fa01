OUT=gpurun_out; mkdir -p $OUT; rm -f $OUT/summary.txt
for rep in 1 2; do
  for ipw in 8 12 16; do
    SO2DR_K1_IPW=$ipw timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_ipw${ipw}_$rep.log 2>&1
    echo "== bench ipw=$ipw rc=$?" >> $OUT/summary.txt
    tail -1 $OUT/bench_ipw${ipw}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e', round(d['value'],1), 'hbm', round(d['hbm_resident']['value'],1), 'K1 ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3))" >> $OUT/summary.txt 2>&1
  done
done
SO2DR_K1_IPW=16 SZ=32768 STENCILS=box2d1r,star2d1r KS=1,2,4,8 timeout 600 python tools/k1_bench.py > $OUT/k1_ipw16.log 2>&1
python -c "
import json
for l in open('$OUT/k1_ipw16.log'):
  try: d=json.loads(l); print('ipw16', d['stencil'], d['k_on'], d['GCell_s'], d['alg_GBps'], d['fma_frac'])
  except Exception: print(l.strip()[:200])" >> $OUT/summary.txt
cat $OUT/summary.txt
