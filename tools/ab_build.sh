# A/B of two in-tree builds on the config-0 bench, alternating:
#   bash tools/ab_build.sh paper_1909_13201_b200/libfsigpu_base.so [rounds]
B=${1:-paper_1909_13201_b200/libfsigpu_base.so}
N=${2:-3}
for i in $(seq $N); do
  for lib in "$B" paper_1909_13201_b200/libfsigpu.so; do
    FSIGPU_LIB=$PWD/$lib python bench.py --no-cpu-baseline --no-microbench 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value']), round(d['solve_ms'],3), d['iterations'])"
  done
done
