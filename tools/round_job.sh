set -u
mkdir -p gpurun_out
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
echo "== sweep big"; timeout 2400 python tools/sweep_predictor.py --train-random 1500 --trace-every 0 --raw gpurun_out/predictor_sweep_l8b_psep_big.json 2>&1 | tail -1
echo "== sweep traced"; timeout 1200 python tools/sweep_predictor.py --raw gpurun_out/predictor_sweep_l8b_psep.json 2>&1 | tail -1
echo "== iteration sweep"; timeout 2400 python tools/sweep_iteration.py --out gpurun_out/iteration_sweep_psep.json 2>&1 | tail -2
echo "== sanitize"; SAN_TIMEOUT=600 bash tools/sanitize.sh 2>&1 | tail -20
