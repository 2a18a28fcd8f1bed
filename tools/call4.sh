set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "producer_consumer" > gpurun_out/gputests4.txt 2>&1
tail -3 gpurun_out/gputests4.txt
timeout 600 python tools/ab_tuning.py decode_path 0 2 > gpurun_out/ab4_path2.txt 2>&1
