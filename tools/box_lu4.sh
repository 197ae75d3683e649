set -x
mkdir -p gpurun_out/lu4
timeout 600 python -m pytest tests -m gpu -x -q -k "large_block" > gpurun_out/lu4/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/lu4/pytest.log
for v in 0 1; do
  FSIGPU_LU_UPDATE_REG=$v timeout 300 python tools/lu_large.py 780 592 > gpurun_out/lu4/lu780_reg$v.txt 2>&1
  FSIGPU_LU_UPDATE_REG=$v timeout 300 python tools/lu_large.py 500 1184 > gpurun_out/lu4/lu500_reg$v.txt 2>&1
done
FSIGPU_LU_UPDATE_REG=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu4/lu780_launches.csv python tools/lu_large.py 780 592 > /dev/null 2>&1
