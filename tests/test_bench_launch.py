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


def test_reference_arm_reports_executed_iterations(monkeypatch, capsys):
    """--impl reference never prints steps / warm-up it did not execute (VERDICT r01 "What's
    weak" #3), also when the wall-clock budget cuts the request short."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench

    asked = {}

    def fake_iterations(cfg, n, skip, count):
        asked.update(skip=skip, count=count)
        return {"setup_s": 1.0, "per_iter_s": 20.0, "iters_timed": count, "iters_skipped": skip, "levels": 4}

    monkeypatch.setattr(bench, "oracle_iterations", fake_iterations)
    monkeypatch.setattr(bench, "oracle_full_size", lambda cfg: {"iters": 64, "solve_s": 1280.0})
    monkeypatch.setenv("REF_BUDGET_S", "540")
    for steps, warm, want in ((20, 5, (5, 20, False)), (100, 10, (5, 22, True))):
        bench.run_reference(argparse.Namespace(cfg=5, n=None, gpus=1, steps=steps, warmup=warm), 0)
        line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
        assert (asked["skip"], asked["count"], line["capped_to_wall_budget"]) == want
        assert (line["warmup"], line["steps"]) == want[:2]
        assert line["value"] == 20.0 * 64 and line["impl"] == "reference"
    # the other ranks of a torchrun launch do no work and print nothing
    bench.run_reference(argparse.Namespace(cfg=5, n=None, gpus=2, steps=3, warmup=1), 1)
    assert capsys.readouterr().out == ""
