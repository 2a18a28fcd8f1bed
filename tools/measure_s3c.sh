# Session-3 pass 3 (recalibrated CTA split): predictor + iteration sweeps for the a8 refits,
# bench lines for configs 2 and 4, and a check of config 2's split.
set -u
O=gpurun_out/s3c
mkdir -p $O
timeout 1200 python tools/sweep_predictor.py --train-random 1500 --trace-every 0 --raw $O/predictor_sweep_l8b.json > $O/sweep.log 2>&1; tail -1 $O/sweep.log
timeout 600 python bench.py > $O/bench_l8b.json 2> $O/bench_l8b.err
timeout 600 python bench.py --config l70b --steps 60 --warmup 5 --no-cpu-baseline > $O/bench_l70b.json 2> $O/bench_l70b.err
timeout 600 python tools/cap_sweep_l70b.py 0,80,88 > $O/cap_l70b.txt 2>&1
timeout 2400 python tools/sweep_iteration.py --out $O/iteration_sweep.json > $O/iteration.log 2>&1; tail -2 $O/iteration.log
