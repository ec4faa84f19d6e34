"""bench.py --gpus N started without a launcher re-runs itself under
torchrun with N ranks (what the driver's scaling run needs when it calls
`bench.py --gpus N` directly); the plumbing is checked over gloo on CPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_flag_spawns_ranks():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--selftest"], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    line = lines[0]
    assert line["selftest"] == "ok" and line["n_gpus"] == 2
    assert line["rank_sum"] == 3.0 and line["ms_max"] == 2.0
    assert line["nccl_debug"] == "INFO"
