set -x
mkdir -p gpurun_out data_cfg2 /tmp/ncu
./tools/micro/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "block or lu or config1 or singular" > gpurun_out/pytest_lu.log 2>&1
timeout 300 python tools/lu_ab.py > gpurun_out/lu_ab.log 2>&1
oracle/_ref/fsi_ref_harness export cfg2 data_cfg2/cfg2.fsix --no-mult --no-gmres > gpurun_out/export.log 2>&1
export FSI_DATA=data_cfg2/cfg2.fsix
timeout 600 python bench.py --config cfg2full --no-cpu-baseline --no-microbench --steps 5 --warmup 3 > gpurun_out/bench_cfg2full.json 2>gpurun_out/bench_cfg2full.err
FSI_MAXIT=30 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cfg2full_launches.csv python tools/profile_solve.py solve > gpurun_out/ncu_list.log 2>&1
for k in prolong_resid residual restrict fs_smoother; do
  timeout 300 ncu --set full --import-source on --clock-control none --profile-from-start off -c 2 -o /tmp/ncu/cfg2_$k python tools/profile_solve.py kernel:$k:4 > gpurun_out/ncu_$k.log 2>&1
  ncu -i /tmp/ncu/cfg2_$k.ncu-rep --page details --csv > gpurun_out/cfg2_${k}_details.csv 2>&1
  python tools/ncu_lines.py /tmp/ncu/cfg2_$k.ncu-rep 30 > gpurun_out/cfg2_${k}_lines.txt 2>&1
done
timeout 600 python tools/tune_spmv.py data_cfg2/cfg2.fsix 4 3 2 > gpurun_out/tune_cfg2full.txt 2>&1
du -sh gpurun_out
