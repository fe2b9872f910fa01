#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + one full K1 capture.
# Usage (here): gpurun --timeout 3000 -- 'bash tools/gpu_round.sh [tests|bench|ncu]...'
OUT=gpurun_out
mkdir -p $OUT
steps=${@:-tests bench ncu}
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1; free -g > $OUT/free.txt 2>&1
for s in $steps; do
  case $s in
    tests)
      timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/summary.txt ;;
    bench)
      timeout 1200 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/summary.txt
      tail -1 $OUT/bench.log >> $OUT/summary.txt ;;
    refarm)
      timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $OUT/bench_ref.log 2>&1; echo "ref rc=$?" >> $OUT/summary.txt
      tail -1 $OUT/bench_ref.log >> $OUT/summary.txt ;;
    k1)
      SZ=32768 STENCILS=${STENCILS:-box2d1r,star2d1r} KS=${KS:-1,2,4,8} timeout 900 python tools/k1_bench.py > $OUT/k1_bench.log 2>&1
      echo "k1 rc=$?" >> $OUT/summary.txt; cat $OUT/k1_bench.log >> $OUT/summary.txt ;;
    pipe)
      DS=${DS:-16,32,64} NS=${NS:-3} KS=${KS:-4,8} timeout 1200 python tools/pipe_sweep.py > $OUT/pipe_sweep.log 2>&1
      echo "pipe rc=$?" >> $OUT/summary.txt; cat $OUT/pipe_sweep.log >> $OUT/summary.txt ;;
    full)
      timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu --durations=0 > $OUT/pytest_fullsize.log 2>&1
      echo "fullsize rc=$?" >> $OUT/summary.txt; tail -12 $OUT/pytest_fullsize.log >> $OUT/summary.txt ;;
    prof)
      for d in 16 64; do timeout 600 python tools/pipe_profile.py 92160 $d 8 3 > $OUT/pipe_profile_d$d.log 2>&1; done
      echo "prof rc=$?" >> $OUT/summary.txt; head -1 $OUT/pipe_profile_d16.log $OUT/pipe_profile_d64.log >> $OUT/summary.txt ;;
    configs)
      timeout 1500 python tools/config_runs.py $CONFIGS > $OUT/config_runs.log 2>&1
      echo "configs rc=$?" >> $OUT/summary.txt; cat $OUT/config_runs.log >> $OUT/summary.txt ;;
    pcie)
      timeout 300 python tools/pcie_probe.py > $OUT/pcie_probe.log 2>&1; echo "pcie rc=$?" >> $OUT/summary.txt
      cat $OUT/pcie_probe.log >> $OUT/summary.txt ;;
    pcpipe)
      timeout 600 python tools/pcie_pipe.py -v > $OUT/pcie_pipe.log 2>&1; echo "pcpipe rc=$?" >> $OUT/summary.txt
      grep pattern $OUT/pcie_pipe.log >> $OUT/summary.txt ;;
    diag)
      timeout 300 python tools/pipe_profile.py 92160 16 8 3 > $OUT/pp_default.log 2>&1
      SO2DR_DIAG_NO_K1=1 timeout 300 python tools/pipe_profile.py 92160 16 8 3 > $OUT/pp_nok1.log 2>&1
      SO2DR_DIAG_NO_K1=1 SO2DR_DIAG_NO_D2D=1 timeout 300 python tools/pipe_profile.py 92160 16 8 3 > $OUT/pp_nok1_nod2d.log 2>&1
      for f in pp_default pp_nok1 pp_nok1_nod2d; do echo $f >> $OUT/summary.txt; head -1 $OUT/$f.log >> $OUT/summary.txt; done ;;
    fmapeak)
      (cd tools/cu && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_peak fma_peak.cu && ./fma_peak) > $OUT/fma_peak.log 2>&1
      echo "fmapeak rc=$?" >> $OUT/summary.txt; cat $OUT/fma_peak.log >> $OUT/summary.txt ;;
    diag2)
      SO2DR_DIAG_NO_K1=1 timeout 300 python tools/pipe_profile.py 92160 16 8 3 > $OUT/pp_nok1.log 2>&1
      SO2DR_DIAG_NO_K1=1 HOST_ALLOC=torch timeout 300 python tools/pipe_profile.py 92160 16 8 3 > $OUT/pp_nok1_torch.log 2>&1
      SO2DR_DIAG_NO_K1=1 SO2DR_HOST_ALLOC_DEFAULT=1 timeout 300 python tools/pipe_profile.py 92160 16 8 3 > $OUT/pp_nok1_dflt.log 2>&1
      for f in pp_nok1 pp_nok1_torch pp_nok1_dflt; do echo $f >> $OUT/summary.txt; head -1 $OUT/$f.log >> $OUT/summary.txt; grep -E "c 5 (htod|dtoh)" $OUT/$f.log >> $OUT/summary.txt; done ;;
    diag3)
      for sp in 1 2 3; do
        SO2DR_H2D_SPLIT=$sp SO2DR_DIAG_NO_K1=1 timeout 300 python tools/pipe_profile.py 92160 16 8 3 > $OUT/pp_split$sp.log 2>&1
        echo split$sp >> $OUT/summary.txt; head -1 $OUT/pp_split$sp.log >> $OUT/summary.txt; grep -E "c 5 (htod|dtoh)" $OUT/pp_split$sp.log >> $OUT/summary.txt
      done
      for sp in 1 2; do
        SO2DR_H2D_SPLIT=$sp timeout 300 python tools/pipe_profile.py 92160 64 4 3 > $OUT/pp_d64_split$sp.log 2>&1
        echo d64 split$sp >> $OUT/summary.txt; head -1 $OUT/pp_d64_split$sp.log >> $OUT/summary.txt
      done ;;
    pcpipe2)
      timeout 600 python tools/pcie_pipe2.py > $OUT/pcie_pipe2.log 2>&1; echo "pcpipe2 rc=$?" >> $OUT/summary.txt
      cat $OUT/pcie_pipe2.log >> $OUT/summary.txt ;;
    pcpipe3)
      timeout 900 python tools/pcie_pipe3.py > $OUT/pcie_pipe3.log 2>&1; echo "pcpipe3 rc=$?" >> $OUT/summary.txt
      cat $OUT/pcie_pipe3.log >> $OUT/summary.txt ;;
    allocvar)
      timeout 1200 python tools/alloc_var.py > $OUT/alloc_var.log 2>&1; echo "allocvar rc=$?" >> $OUT/summary.txt
      cat $OUT/alloc_var.log >> $OUT/summary.txt ;;
    clockab)
      for cms in 200 1000 200 1000; do
        timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-value-leg --clock-ms $cms > $OUT/bench_c$cms.log 2>&1
        echo "clock_ms=$cms" >> $OUT/summary.txt
        tail -1 $OUT/bench_c$cms.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e']['value'], d['ms_per_step'], d['clocks'])" >> $OUT/summary.txt
      done ;;
    probeab)
      for v in before after before after; do
        flag=""; [ $v = after ] && flag="--pcie-probe-after"
        timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-value-leg $flag > $OUT/bench_p$v.log 2>&1
        echo "probe=$v" >> $OUT/summary.txt
        tail -1 $OUT/bench_p$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e']['value'], d['ms_per_step'], d['binding_roofline']['pcie_measured'])" >> $OUT/summary.txt
      done
      timeout 600 python tools/alloc_var.py > $OUT/alloc_var.log 2>&1; grep alloc $OUT/alloc_var.log >> $OUT/summary.txt ;;
    ipwbench)
      for ipw in 3 4 6 8 12; do
        SO2DR_K1_IPW=$ipw timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > $OUT/bench_ipw$ipw.log 2>&1
        echo "ipw=$ipw" >> $OUT/summary.txt
        tail -1 $OUT/bench_ipw$ipw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'K1 ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3))" >> $OUT/summary.txt
      done ;;
    robust)
      DS=32,64,128 NS=3,4,6 KS=4 timeout 1500 python tools/pipe_sweep.py > $OUT/pipe_sweep_robust.log 2>&1
      echo "robust rc=$?" >> $OUT/summary.txt; cat $OUT/pipe_sweep_robust.log >> $OUT/summary.txt
      timeout 300 python tools/pipe_profile.py 92160 64 4 3 > $OUT/pp_d64.log 2>&1
      head -1 $OUT/pp_d64.log >> $OUT/summary.txt; grep -E "c(20|21|22) (htod|dtoh)" $OUT/pp_d64.log >> $OUT/summary.txt ;;
    robust2)
      DS=64,128,192 NS=3 KS=4,8 timeout 1500 python tools/pipe_sweep.py > $OUT/pipe_sweep_robust2.log 2>&1
      echo "robust2 rc=$?" >> $OUT/summary.txt; cat $OUT/pipe_sweep_robust2.log >> $OUT/summary.txt
      timeout 300 python tools/pipe_profile.py 92160 64 4 3 > $OUT/pp_d64.log 2>&1
      head -1 $OUT/pp_d64.log >> $OUT/summary.txt; grep -E "c(20|21|22) (htod|dtoh)" $OUT/pp_d64.log >> $OUT/summary.txt ;;
    ncuk1)  # one in-core K1 launch per k_on: NCU_KS="1 4 8"
      bash tools/gpu_ncuk1.sh "${NCU_KS:-4}" incore ;;
    k3d)
      SZ3=768 STENCILS=star3d1r,box3d1r KS=1,2,4 timeout 900 python tools/k1_bench.py > $OUT/k3d.log 2>&1
      echo "k3d rc=$?" >> $OUT/summary.txt; cat $OUT/k3d.log >> $OUT/summary.txt
      timeout 900 python -m pytest tests/test_gpu_3d_f64.py tests/test_gpu_fullsize.py -x -q > $OUT/pytest_3d.log 2>&1; echo "pytest 3d rc=$?" >> $OUT/summary.txt ;;
    sanitize)
      # the sanitize workload bare first (must pass), then under each tool
      timeout 300 python tools/sanitize_run.py > $OUT/sanitize_plain.log 2>&1; echo "sanitize plain rc=$?" >> $OUT/summary.txt
      for tool in memcheck racecheck synccheck initcheck; do
        timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_run.py > $OUT/sanitize_$tool.log 2>&1
        echo "sanitize $tool rc=$?" >> $OUT/summary.txt; tail -3 $OUT/sanitize_$tool.log >> $OUT/summary.txt
      done ;;
    ncu3d)
      timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_stencil3d -s 1 -c 1 -o $OUT/k1_3d_star_k4 -f \
        python tools/k1_one3d.py 4 768 star > $OUT/k1_3d.log 2>&1; echo "ncu3d rc=$?" >> $OUT/summary.txt ;;
    multi)
      SO2DR_SHARE_DEVICE=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-value-leg > $OUT/bench_n2_shared.log 2>&1
      echo "multi rc=$?" >> $OUT/summary.txt; tail -1 $OUT/bench_n2_shared.log | cut -c1-1500 >> $OUT/summary.txt
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
        bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > $OUT/bench_ref_n2.log 2>&1
      echo "ref n2 rc=$?" >> $OUT/summary.txt; tail -1 $OUT/bench_ref_n2.log | cut -c1-300 >> $OUT/summary.txt ;;
    ncu)
      # launch list of one bench step (e2e leg): every launch with its device time
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-value-leg > $OUT/launches_bench.log 2>&1
      echo "ncu launches rc=$?" >> $OUT/summary.txt
      # DRAM traffic of chunk 5's 16 K1 launches (steady state)
      timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        -k regex:k1_stencil2d -s 80 -c 16 --csv --log-file $OUT/k1_traffic.csv \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-value-leg > $OUT/k1_traffic.log 2>&1
      echo "ncu traffic rc=$?" >> $OUT/summary.txt
      # one full capture of a steady-state K1 launch
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_stencil2d -s 85 -c 1 -o $OUT/k1_full -f \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-value-leg > $OUT/k1_full.log 2>&1
      echo "ncu full rc=$?" >> $OUT/summary.txt ;;
  esac
done
cat $OUT/summary.txt
