"""bench.py harness logic on CPU: --gpus N self-launches N ranks under torch.distributed.run (the reference
arm needs no GPU), rank 0 alone prints one JSON line, and both arms share one config object."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_n_self_launches_ranks_and_reference_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=600,
                       env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"


def test_both_arms_share_the_config_object():
    sys.path.insert(0, ROOT)
    import bench

    assert bench.workload_config(1) == bench.workload_config(1)
    assert bench.workload_config(4)["global_batch"] == 4 * bench.BATCH
