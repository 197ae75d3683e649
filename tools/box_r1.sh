set -x
mkdir -p gpurun_out/r1 data_cfg2
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r1/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1/pytest.log
FSI_WHICH=R timeout 300 python tools/tune_spmv.py data/cfg0.fsix 1 2 > gpurun_out/r1/tune_r_cfg0_cold.txt 2>&1
oracle/_ref/fsi_ref_harness export cfg2 data_cfg2/cfg2.fsix --no-mult --max-iters 30 --block-stride 997 > gpurun_out/r1/export.log 2>&1
FSI_WHICH=R timeout 600 python tools/tune_spmv.py data_cfg2/cfg2.fsix 4 3 2 > gpurun_out/r1/tune_r_cfg2.txt 2>&1
