# A/B of the large-block LU trailing update: 4x8 register tile (default) vs 1x16 strip (FSIGPU_LU_UPDATE_R1=1)
set -x
mkdir -p gpurun_out/lu5
timeout 600 python -m pytest tests -m gpu -x -q -k "large_block or config1" > gpurun_out/lu5/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/lu5/pytest.log
for v in 0 1; do
  FSIGPU_LU_UPDATE_R1=$v timeout 300 python tools/lu_large.py 780 592 > gpurun_out/lu5/lu780_r1$v.txt 2>&1
  FSIGPU_LU_UPDATE_R1=$v timeout 300 python tools/lu_large.py 500 1184 > gpurun_out/lu5/lu500_r1$v.txt 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu5/lu780_launches.csv python tools/lu_large.py 780 592 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:lu_big_update_r4 -c 1 -o gpurun_out/lu5/r4 python tools/lu_large.py 780 592 > gpurun_out/lu5/ncu_full.log 2>&1
