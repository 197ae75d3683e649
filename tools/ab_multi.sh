# config-0 bench for several in-tree builds, alternating: bash tools/ab_multi.sh lib1.so lib2.so ...
for i in 1 2; do
  for lib in "$@"; do
    FSIGPU_LIB=$PWD/$lib python bench.py --no-cpu-baseline --no-microbench 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value']), round(d['solve_ms'],3), d['iterations'])"
  done
done
