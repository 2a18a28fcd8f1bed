# A/B of library builds on the prefill-heavy set (tools/ab_prefill.py), alternating.
#   bash tools/ab_libs.sh OUT lib1 lib2 ...
set -u
out=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib"; NIYAMA_LIB_PATH=$lib timeout 300 python tools/ab_prefill.py 2>&1 | sed -E 's/ +T=.*median= *([0-9.]+)us batched= *([0-9.]+)us.*/ \1 \2/' | grep -v "^lib:"
  done
done > $out 2>&1
