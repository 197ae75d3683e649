# LU update 2x8 tile at 3 CTAs/SM (80 registers, small spill) vs the committed 2-CTA build
set -x
mkdir -p gpurun_out/lu8
timeout 600 python -m pytest tests -m gpu -x -q -k "large_block" > gpurun_out/lu8/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/lu8/pytest.log
for i in 1 2; do
  timeout 300 python tools/lu_large.py 780 592 >> gpurun_out/lu8/lu780.txt 2>&1
  timeout 300 python tools/lu_large.py 500 1184 >> gpurun_out/lu8/lu500.txt 2>&1
done
