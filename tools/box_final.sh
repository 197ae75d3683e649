# round-end style check: full GPU tier, smoke, bench (ours + reference arm), large-block LU timing
set -x
mkdir -p gpurun_out/fin
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/fin/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fin/smoke.log
timeout 300 python tools/lu_large.py 780 592 > gpurun_out/fin/lu780.txt 2>&1
timeout 300 python tools/lu_large.py 500 1184 > gpurun_out/fin/lu500.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin/lu780_launches.csv python tools/lu_large.py 780 592 > /dev/null 2>&1
timeout 600 python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/fin/bench_ref.json 2> gpurun_out/fin/bench_ref.err
