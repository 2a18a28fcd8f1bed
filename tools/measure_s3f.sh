# Session-3 pass after the early-K/V change: parity suite, smoke, a8 sweeps + iteration sweep
# for the refits, bench lines.
set -u
O=gpurun_out/s3f
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gputests.txt 2>&1; tail -1 $O/gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 1200 python tools/sweep_predictor.py --train-random 1500 --trace-every 0 --raw $O/predictor_sweep_l8b.json > $O/sweep.log 2>&1; tail -1 $O/sweep.log
timeout 1200 python tools/sweep_predictor.py --config l70b --train-random 1000 --trace-every 0 --raw $O/predictor_sweep_l70b.json > $O/sweep70.log 2>&1; tail -1 $O/sweep70.log
timeout 2400 python tools/sweep_iteration.py --out $O/iteration_sweep.json > $O/iteration.log 2>&1; tail -1 $O/iteration.log
timeout 600 python bench.py > $O/bench_l8b.json 2> $O/bench_l8b.err
timeout 900 python bench.py --config l70b --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_l70b.json 2> $O/bench_l70b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 64 --csv --log-file $O/launches_bench_l8b.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
