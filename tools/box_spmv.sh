set -x
mkdir -p gpurun_out data_cfg2
FSIGPU_SPMV_PAIR=22 timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_pair22.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_default.log 2>&1
oracle/_ref/fsi_ref_harness export cfg2 data_cfg2/cfg2.fsix --no-mult --no-gmres > gpurun_out/export.log 2>&1
timeout 900 python tools/tune_spmv.py data_cfg2/cfg2.fsix 4 3 2 > gpurun_out/tune_cfg2full_pair.txt 2>&1
for v in 0 22 24; do FSIGPU_SPMV_PAIR=$v timeout 600 python bench.py --config cfg2full --no-cpu-baseline --no-microbench --steps 5 --warmup 3 > gpurun_out/bench_cfg2full_pair$v.json 2>gpurun_out/bench_cfg2full_pair$v.err; done
for v in 0 22; do FSIGPU_SPMV_PAIR=$v timeout 600 python bench.py --no-cpu-baseline --no-microbench > gpurun_out/bench_cfg0_pair$v.json 2>&1; done
du -sh gpurun_out
