# A/B of the large-block LU trailing update: 4x8 tile (default, 0) vs 2x8 tile at 256 threads (2)
set -x
mkdir -p gpurun_out/lu7
timeout 600 python -m pytest tests -m gpu -x -q -k "large_block" > gpurun_out/lu7/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/lu7/pytest.log
for i in 1 2; do for v in 0 2; do
  FSIGPU_LU_UPDATE_R1=$v timeout 300 python tools/lu_large.py 780 592 >> gpurun_out/lu7/lu780_$v.txt 2>&1
  FSIGPU_LU_UPDATE_R1=$v timeout 300 python tools/lu_large.py 500 1184 >> gpurun_out/lu7/lu500_$v.txt 2>&1
done; done
