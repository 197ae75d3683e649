for pad in 0 2 64 300; do
 for lib in paper_1909_13201_b200/libfsigpu_base.so paper_1909_13201_b200/libfsigpu.so; do
  FSI_PAD_MB=$pad FSIGPU_LIB=$PWD/$lib python bench.py --no-cpu-baseline --no-microbench 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pad $pad $lib', round(d['value']), round(d['solve_ms'],3))"
 done
done
