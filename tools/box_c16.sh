# CSR16 FS operator: parity, config-0/2 benches, A/B against 32-bit columns, launch table
set -x
mkdir -p gpurun_out/c16 data_cfg2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c16/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c16/pytest.log
timeout 600 python bench.py > gpurun_out/c16/bench_cfg0.json 2> gpurun_out/c16/bench_cfg0.err
FSIGPU_FS_C16=0 timeout 600 python bench.py --no-microbench --no-cpu-baseline > gpurun_out/c16/bench_cfg0_c32.json 2> /dev/null
oracle/_ref/fsi_ref_harness export cfg2 data_cfg2/cfg2.fsix --no-mult --max-iters 30 --block-stride 997 > gpurun_out/c16/export.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k cfg2 > gpurun_out/c16/pytest_cfg2.log 2>&1; echo "rc=$?" >> gpurun_out/c16/pytest_cfg2.log
timeout 600 python bench.py --config cfg2full --no-cpu-baseline --no-microbench --steps 5 --warmup 3 > gpurun_out/c16/bench_cfg2full.json 2>gpurun_out/c16/bench_cfg2full.err
FSIGPU_FS_C16=0 timeout 600 python bench.py --config cfg2full --no-cpu-baseline --no-microbench --steps 5 --warmup 3 > gpurun_out/c16/bench_cfg2full_c32.json 2>/dev/null
export FSI_DATA=data_cfg2/cfg2.fsix
FSI_MAXIT=30 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file /tmp/l.csv python tools/profile_solve.py solve > /dev/null 2>&1
python tools/launch_table.py /tmp/l.csv > gpurun_out/c16/launch_table_cfg2full.txt 2>&1
