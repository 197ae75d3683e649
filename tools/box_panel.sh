# shared-memory panel LU (config-4 regime): parity, timing vs the global-memory panel, full GPU tier, bench
set -x
mkdir -p gpurun_out/pn
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pn/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pn/pytest.log
for v in 0 1; do
  FSIGPU_LU_PANEL_GLOBAL=$v timeout 300 python tools/lu_large.py 780 592 > gpurun_out/pn/lu780_global$v.txt 2>&1
  FSIGPU_LU_PANEL_GLOBAL=$v timeout 300 python tools/lu_large.py 500 1184 > gpurun_out/pn/lu500_global$v.txt 2>&1
done
timeout 600 python bench.py > gpurun_out/pn/bench_cfg0.json 2> gpurun_out/pn/bench_cfg0.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pn/lu780_launches.csv python tools/lu_large.py 780 592 > /dev/null 2>&1
