set -u
mkdir -p gpurun_out
B=paper_2503_22562_b200/_build/variants/libniyama_base.so
N=paper_2503_22562_b200/libniyama.so
for i in 1 2; do
  NIYAMA_LIB_PATH=$B timeout 300 python tools/ab_prefill.py > gpurun_out/ab3_base_$i.txt 2>&1
  NIYAMA_LIB_PATH=$N timeout 300 python tools/ab_prefill.py > gpurun_out/ab3_new_$i.txt 2>&1
done
export NIYAMA_LIB_PATH=paper_2503_22562_b200/_build/variants/libniyama_tiles.so
for c in l70b l8b l8b-mixed l70b-mixed; do timeout 200 python tools/tile_trace.py $c > gpurun_out/tiles3_$c.txt 2>&1; done
unset NIYAMA_LIB_PATH
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests3.txt 2>&1
