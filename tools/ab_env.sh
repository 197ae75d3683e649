# config-0 bench of the current build under several environments, alternating:
#   bash tools/ab_env.sh 'A=1' 'B=2' ...   ('-' = none)
for i in 1 2; do
  for e in "$@"; do
    if [ "$e" = "-" ]; then envs=""; else envs="$e"; fi
    env $envs python bench.py --no-cpu-baseline --no-microbench 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['value']), round(d['solve_ms'],3), d['iterations'], round(d['setup_s'],2))"
  done
done
