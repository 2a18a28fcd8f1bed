# Config-4 prefill-CTA count under the bench's own sustained (power-capped) conditions:
# 27-layer steps, alternating settings, two passes.   bash tools/ab_l70b_ctas.sh OUT n1 n2 ...  (0 = planner default; key=val = any tuning field)
set -u
out=$1; shift
for rep in 1 2; do
  for n in "$@"; do
    case "$n" in 0) tun="";; *=*) tun="--tuning $n";; *) tun="--tuning prefill_ctas=$n";; esac
    timeout 600 python bench.py --config l70b --no-cpu-baseline --steps 120 --warmup 10 $tun 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('ctas $n', 'attn median %.1f p10 %.1f p90 %.1f frac %.3f step %.2f ms clocks %s %s' % (d['attention_launch_us']['median'], d['attention_launch_us']['p10'], d['attention_launch_us']['p90'], d['roofline']['frac'], d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons']), flush=True)"
  done
done > $out 2>&1
