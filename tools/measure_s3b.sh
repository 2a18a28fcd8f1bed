# Session-3 pass 2: parity suite on the final kernel options (decode auto, prefill pairs auto),
# config-4 A/B of pairs, and the config-3 predictor sweep for the a8 refit.
set -u
O=gpurun_out/s3b
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gputests.txt 2>&1; tail -2 $O/gputests.txt
timeout 600 python tools/ab_pairs.py > $O/ab_pairs.txt 2>&1
timeout 3000 python tools/sweep_predictor.py --train-random 1500 --trace-every 0 --raw $O/predictor_sweep_l8b.json > $O/sweep.log 2>&1
tail -2 $O/sweep.log
