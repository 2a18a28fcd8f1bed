set -u
mkdir -p gpurun_out
for c in dec ragged; do
  echo "== $c path2"; timeout 120 python tools/sanitize_case.py $c path2 2>&1 | tail -3
  echo "== $c memcheck"; timeout 300 compute-sanitizer --tool memcheck python tools/sanitize_case.py $c path2 2>&1 | grep -v "^=========     " | head -30
done > gpurun_out/dbg5.txt 2>&1
