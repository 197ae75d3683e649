set -x
mkdir -p gpurun_out/v
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v/pytest.log
timeout 600 python bench.py > gpurun_out/v/bench.json 2> gpurun_out/v/bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/v/smoke.log
