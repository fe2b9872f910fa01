# ncu --set full of one in-core K1 launch per k_on: bash tools/gpu_ncuk1.sh "1 4 8" [tag]
OUT=gpurun_out; mkdir -p $OUT
TAG=${2:-cur}
for k in ${1:-4}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_stencil2d -s 1 -c 1 \
    -o $OUT/k1_${TAG}_k$k -f python tools/k1_one.py $k 32768 ${KIND:-box} > $OUT/k1_${TAG}_k$k.log 2>&1
  echo "ncu k=$k rc=$?" >> $OUT/summary.txt
done
