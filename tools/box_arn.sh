set -x
mkdir -p gpurun_out/arn data_cfg2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/arn/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/arn/pytest.log
oracle/_ref/fsi_ref_harness export cfg2 data_cfg2/cfg2.fsix --no-mult --max-iters 30 --block-stride 997 > gpurun_out/arn/export.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k cfg2 > gpurun_out/arn/pytest_cfg2.log 2>&1; echo "rc=$?" >> gpurun_out/arn/pytest_cfg2.log
timeout 600 python bench.py --config cfg2full --no-cpu-baseline --no-microbench --steps 5 --warmup 3 > gpurun_out/arn/bench_cfg2full.json 2>gpurun_out/arn/bench_cfg2full.err
export FSI_DATA=data_cfg2/cfg2.fsix
FSI_MAXIT=30 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file /tmp/l.csv python tools/profile_solve.py solve > /dev/null 2>&1
python tools/launch_table.py /tmp/l.csv > gpurun_out/arn/launch_table_cfg2full.txt 2>&1
