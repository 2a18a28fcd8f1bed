"""CPU test of bench.py's N-rank launch path (a7 plumbing):
`python bench.py --gpus 2` with no WORLD_SIZE re-launches itself under
torch.distributed.run with two ranks; --host-only runs them over gloo with
NIYAMA_DEVICE_NONE pools (no GPU) and prints one line from rank 0."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_self_spawns_two_ranks_host_only():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--host-only", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = lines[0]
    assert out["impl"] == "host-only" and out["n_gpus"] == 2 and out["world_size_seen"] == 2
    assert out["replicated_plans_equal"] is True
    assert out["unique_id_bytes"] == [128, 128]
    assert out["predicted_launch_s"] > 0
