set -u
mkdir -p gpurun_out
NIYAMA_LIB_PATH=paper_2503_22562_b200/_build/variants/libniyama_hang.so timeout 120 python tools/sanitize_case.py dec path2 > gpurun_out/dbg7.txt 2>&1
timeout 120 python tools/sanitize_case.py dec path2 >> gpurun_out/dbg7.txt 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "producer_consumer" > gpurun_out/gputests7.txt 2>&1
tail -3 gpurun_out/gputests7.txt
timeout 600 python tools/ab_tuning.py decode_path 0 2 > gpurun_out/ab7_path2.txt 2>&1
