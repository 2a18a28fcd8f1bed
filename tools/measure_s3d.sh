# Session-3 final pass on HEAD: parity suite, smoke, bench lines (driver defaults and config 4),
# launch list, ncu captures of the attention launch, and the single-S-load softmax A/B.
set -u
O=gpurun_out/s3d
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gputests.txt 2>&1; tail -1 $O/gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 600 python bench.py > $O/bench_l8b.json 2> $O/bench_l8b.err
timeout 600 python bench.py --config l70b --steps 60 --warmup 5 --no-cpu-baseline > $O/bench_l70b.json 2> $O/bench_l70b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 60 --csv --log-file $O/launches_bench_l8b.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hybrid_attn -s 2 -c 1 -o $O/mixed python tools/prof_case.py mixed 3 > $O/ncu_mixed.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hybrid_attn -s 2 -c 1 -o $O/l70b python tools/prof_case.py l70b 3 > $O/ncu_l70b.log 2>&1
bash tools/ab_libs.sh $O/ab_onesload.txt paper_2503_22562_b200/libniyama.so paper_2503_22562_b200/_build/variants/libniyama_onesload.so
