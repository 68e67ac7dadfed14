"""bench.py's launcher (CPU, gloo): `--gpus N` without torchrun becomes N ranks itself, and a
--gpus / WORLD_SIZE mismatch fails loudly (VERDICT r01 "What's weak" #4)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    e["CUDA_VISIBLE_DEVICES"] = ""
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=e, timeout=300)


def test_gpus_2_relaunches_two_ranks():
    r = _run(["--gpus", "2", "--probe-launch"])
    assert r.returncode == 0, r.stderr[-2000:]
    # the two ranks' lines may interleave on the shared stdout: decode every object in order
    lines, dec, text, i = [], json.JSONDecoder(), r.stdout, 0
    while (i := text.find("{", i)) >= 0:
        obj, i = dec.raw_decode(text, i)
        lines.append(obj)
    assert sorted(l["rank"] for l in lines) == [0, 1]
    assert all(l["world"] == 2 and l["sum"] == 2.0 for l in lines)


def test_gpus_world_mismatch_fails():
    r = _run(["--gpus", "2", "--probe-launch"], env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
