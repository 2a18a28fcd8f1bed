set -u
mkdir -p gpurun_out
timeout 300 python tools/bench_gap.py > gpurun_out/gap_l8b.txt 2>&1
export NIYAMA_LIB_PATH=paper_2503_22562_b200/_build/variants/libniyama_tiles.so
for c in l70b l8b l8b-c2048 l8b-mixed l70b-mixed; do timeout 200 python tools/tile_trace.py $c > gpurun_out/tiles_$c.txt 2>&1; done
unset NIYAMA_LIB_PATH
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hybrid_attn -s 2 -c 1 -o gpurun_out/decode_src python tools/prof_case.py decode 3 > gpurun_out/ncu_decode.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hybrid_attn -s 2 -c 1 -o gpurun_out/l70b_src python tools/prof_case.py l70b 3 > gpurun_out/ncu_l70b.log 2>&1
