"""bench.py's launcher contract on CPU: `--gpus N` outside torchrun re-launches N
ranks (torch.distributed.run, 127.0.0.1 rendezvous) and rank 0 alone prints the
reference arm's line; a world size that disagrees with --gpus fails loudly."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = dict(os.environ, REF_SAMPLE="1")
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                          text=True, timeout=600, env=env, cwd=ROOT)


def test_gpus2_self_launches_two_ranks():
    r = _run(["--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0


def test_gpus_world_size_mismatch_fails():
    r = _run(["--gpus", "4", "--impl", "reference", "--steps", "1"],
             {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "--gpus 4" in r.stderr
