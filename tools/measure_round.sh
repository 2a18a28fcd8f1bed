set -x
python bench.py > gpurun_out/bench_l8b.json 2> gpurun_out/bench_l8b.err
python bench.py --config l70b --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_l70b.json 2> gpurun_out/bench_l70b.err
timeout 600 python tools/sweep_predictor.py --out gpurun_out/predictor_fit.json > gpurun_out/sweep.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 60 --csv --log-file gpurun_out/launches_bench_l8b.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hybrid_attn -s 2 -c 1 -o gpurun_out/mixed python tools/prof_case.py mixed 3 > gpurun_out/ncu_mixed.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hybrid_attn -s 2 -c 1 -o gpurun_out/prefill python tools/prof_case.py prefill 3 > gpurun_out/ncu_prefill.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:hybrid_attn -s 2 -c 1 -o gpurun_out/l70b python tools/prof_case.py l70b 3 > gpurun_out/ncu_l70b.log 2>&1
timeout 300 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
