# bench.py config-2 attention median and step time for alternating library builds.
#   bash tools/ab_bench.sh OUT lib1 lib2 ...
set -u
out=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    NIYAMA_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --steps 200 --warmup 20 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$lib', 'attn median %.1f p10 %.1f p90 %.1f step %.1f us clocks %s' % (d['attention_launch_us']['median'], d['attention_launch_us']['p10'], d['attention_launch_us']['p90'], d['ms_per_step']*1e3, d['clocks']['sm_mhz']))"
  done
done > $out 2>&1
