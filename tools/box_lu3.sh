set -x
mkdir -p gpurun_out/lu3
timeout 600 python -m pytest tests -m gpu -x -q -k "large_block or lu" > gpurun_out/lu3/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/lu3/pytest.log
for v in 0 1; do
  FSIGPU_LU_UPDATE_TILES=$v timeout 300 python tools/lu_large.py 780 592 > gpurun_out/lu3/lu780_tiles$v.txt 2>&1
  FSIGPU_LU_UPDATE_TILES=$v timeout 300 python tools/lu_large.py 500 1184 > gpurun_out/lu3/lu500_tiles$v.txt 2>&1
done
timeout 300 python tools/lu_large.py 260 2048 > gpurun_out/lu3/lu260.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu3/lu780_launches.csv python tools/lu_large.py 780 592 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lu_big_panel_smem -s 3 -c 1 -o gpurun_out/lu3/panel python tools/lu_large.py 780 592 > gpurun_out/lu3/ncu_panel.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lu_big_update_strip -s 3 -c 1 -o gpurun_out/lu3/strip python tools/lu_large.py 780 592 > gpurun_out/lu3/ncu_strip.log 2>&1
