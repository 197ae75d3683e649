# restriction launch-shape sweep on config 2 (cold) and config 0 (warm)
set -x
mkdir -p gpurun_out/rs data_cfg2
FSI_WHICH=R timeout 300 python tools/tune_spmv.py data/cfg0.fsix 1 2 > gpurun_out/rs/tune_r_cfg0_cold.txt 2>&1
FSI_WARM=1 FSI_WHICH=R timeout 300 python tools/tune_spmv.py data/cfg0.fsix 1 2 > gpurun_out/rs/tune_r_cfg0_warm.txt 2>&1
oracle/_ref/fsi_ref_harness export cfg2 data_cfg2/cfg2.fsix --no-mult --max-iters 30 --block-stride 997 > gpurun_out/rs/export.log 2>&1
FSI_WHICH=R timeout 600 python tools/tune_spmv.py data_cfg2/cfg2.fsix 4 3 2 1 > gpurun_out/rs/tune_r_cfg2.txt 2>&1
