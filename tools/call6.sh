set -u
mkdir -p gpurun_out
export NIYAMA_LIB_PATH=paper_2503_22562_b200/_build/variants/libniyama_hang.so
timeout 120 python tools/sanitize_case.py dec path2 > gpurun_out/dbg6.txt 2>&1
