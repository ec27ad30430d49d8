"""bench.py's multi-GPU launcher on CPU: `--gpus 2` without WORLD_SIZE
spawns two ranks itself (torch.distributed.run on 127.0.0.1), the ranks
agree on world size 2, run the broadcast + reduce plumbing of the sharded
C4 step over gloo (--stub: no transform compute), and rank 0 prints one JSON
line with n_gpus = 2."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    return env


def test_bench_spawns_ranks_and_reports_world():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--stub", "--steps", "2",
                        "--warmup", "1", "--L", "1024", "--jmin", "3"],
                       capture_output=True, text=True, timeout=300, env=_env(), cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["stub"] is True and d["scaling"] == "strong"
    loads = d["config"]["rank_loads"]
    assert len(loads) == 2 and max(loads) <= 1.01 * sum(loads) / 2


def test_bench_rejects_world_mismatch():
    env = _env()
    env.update(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--stub", "--steps", "1"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode != 0 and "world size 1 != --gpus 2" in (r.stderr + r.stdout)
