set -x
mkdir -p gpurun_out/final data_cfg2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final/pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/final/bench_cfg0.json 2> gpurun_out/final/bench_cfg0.err
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/final/launches_cfg0.csv python tools/profile_solve.py solve > gpurun_out/final/ncu_list_cfg0.log 2>&1
python tools/launch_table.py gpurun_out/final/launches_cfg0.csv > gpurun_out/final/launch_table_cfg0.txt 2>&1
python tools/ncu_class_traffic.py gpurun_out/final/launches_cfg0.csv cfg0 > gpurun_out/final/class_traffic_cfg0.txt 2>&1
timeout 300 ncu --set full --import-source on --clock-control none --profile-from-start off -c 2 -o /tmp/fs2 python tools/profile_solve.py kernel:fs_smoother:2 > gpurun_out/final/ncu_fs2.log 2>&1
ncu -i /tmp/fs2.ncu-rep --page details --csv > gpurun_out/final/ncu_fs2_details.csv 2>&1
python tools/ncu_lines.py /tmp/fs2.ncu-rep 30 > gpurun_out/final/ncu_fs2_lines.txt 2>&1
oracle/_ref/fsi_ref_harness export cfg2 data_cfg2/cfg2.fsix --no-mult --max-iters 30 --block-stride 997 > gpurun_out/final/export.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k cfg2 > gpurun_out/final/pytest_cfg2.log 2>&1
timeout 900 python bench.py --config cfg2full --no-cpu-baseline --no-microbench --steps 5 --warmup 3 > gpurun_out/final/bench_cfg2full.json 2>gpurun_out/final/bench_cfg2full.err
export FSI_DATA=data_cfg2/cfg2.fsix
FSI_MAXIT=30 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/final/launches_cfg2full.csv python tools/profile_solve.py solve > gpurun_out/final/ncu_list_cfg2.log 2>&1
python tools/launch_table.py gpurun_out/final/launches_cfg2full.csv > gpurun_out/final/launch_table_cfg2full.txt 2>&1
python tools/ncu_class_traffic.py gpurun_out/final/launches_cfg2full.csv cfg2full > gpurun_out/final/class_traffic_cfg2.txt 2>&1
cp profiles/ncu_summary.json gpurun_out/final/ncu_summary.json
du -sh gpurun_out
