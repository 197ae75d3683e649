# config-0 bench under FSI_PAD_MB paddings (placement sensitivity):
#   bash tools/ab_pad.sh lib.so pad1 pad2 ...
lib=$1; shift
for pad in "$@"; do
  FSI_PAD_MB=$pad FSIGPU_LIB=$PWD/$lib python bench.py --no-cpu-baseline --no-microbench 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pad $pad $lib', round(d['value']), round(d['solve_ms'],3))"
done
