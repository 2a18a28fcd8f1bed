# Final round-2 check on HEAD: parity suite, smoke, bench lines (driver defaults, config 4).
set -u
O=gpurun_out/final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gputests.txt 2>&1; tail -1 $O/gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 600 python bench.py > $O/bench_l8b.json 2> $O/bench_l8b.err
timeout 600 python bench.py --config l70b --steps 60 --warmup 5 --no-cpu-baseline > $O/bench_l70b.json 2> $O/bench_l70b.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
