"""bench.py's N-rank harness on CPU: `bench.py --gpus 2` with no launcher spawns its own two
ranks (RANK / WORLD_SIZE / MASTER_ADDR=127.0.0.1 set by bench.py itself), joins a gloo process
group, times with a barrier on both sides, takes the max over ranks and prints ONE JSON line
on rank 0.  --plumbing-check swaps the GPU step for a numpy stand-in (there is no GPU here and
no CPU fallback of the kernel); everything around the step is the GPU arm's code."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_spawns_two_ranks_and_prints_one_line():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--plumbing-check"], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["warmup"] == 3
    assert d["config"]["backend"] == "gloo" and d["config"]["gathered_ok"] is True
    assert d["ms_per_step"] > 0 and d["value"] is None


def test_reference_arm_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1", "--m", "1", "--layer", "L8B.O"], capture_output=True, text=True, timeout=300,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
