set -x
mkdir -p gpurun_out data_cfg2
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1
bash tools/ab_multi.sh paper_1909_13201_b200/libfsigpu_base.so paper_1909_13201_b200/libfsigpu.so > gpurun_out/ab_cfg0.txt 2>&1
oracle/_ref/fsi_ref_harness export cfg2 data_cfg2/cfg2.fsix --no-mult --max-iters 30 --block-stride 997 > gpurun_out/export.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k cfg2 > gpurun_out/pytest_cfg2.log 2>&1
timeout 900 python tools/tune_spmv.py data_cfg2/cfg2.fsix 4 3 > gpurun_out/tune_cfg2full_ap.txt 2>&1
timeout 600 python bench.py --config cfg2full --no-cpu-baseline --no-microbench --steps 5 --warmup 3 > gpurun_out/bench_cfg2full.json 2>gpurun_out/bench_cfg2full.err
export FSI_DATA=data_cfg2/cfg2.fsix
FSI_MAXIT=30 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file /tmp/launches.csv python tools/profile_solve.py solve > gpurun_out/ncu_list.log 2>&1
python tools/launch_table.py /tmp/launches.csv > gpurun_out/launch_table_cfg2full.txt 2>&1
du -sh gpurun_out
