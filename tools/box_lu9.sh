# LU init kernel: single fused pass (copy + row maxima)
set -x
mkdir -p gpurun_out/lu11
timeout 600 python -m pytest tests -m gpu -x -q -k "large_block or lu or singular" > gpurun_out/lu11/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/lu11/pytest.log
for i in 1 2; do
  timeout 300 python tools/lu_large.py 780 592 >> gpurun_out/lu11/lu780.txt 2>&1
  timeout 300 python tools/lu_large.py 500 1184 >> gpurun_out/lu11/lu500.txt 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu11/lu780_launches.csv python tools/lu_large.py 780 592 > /dev/null 2>&1
