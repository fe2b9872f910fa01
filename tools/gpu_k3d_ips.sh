# 3D K1: A/B of the uniform z items per SM that cap the guided z segments (SO2DR_K3D_IPS).
OUT=gpurun_out; mkdir -p $OUT; rm -f $OUT/summary.txt
for ips in 8 16 4 32; do
  SO2DR_K3D_IPS=$ips SZ3=768 STENCILS=star3d1r,box3d1r KS=1,2,4 timeout 600 python tools/k1_bench.py > $OUT/k3d_ips$ips.log 2>&1
  echo "== ips=$ips rc=$?" >> $OUT/summary.txt
  python -c "
import json
for l in open('$OUT/k3d_ips$ips.log'):
  try: d=json.loads(l); print(d['stencil'], d['k_on'], d['GCell_s'], d['alg_GBps'])
  except Exception: print(l.strip()[:200])" >> $OUT/summary.txt
done
cat $OUT/summary.txt
