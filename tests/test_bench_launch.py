"""CPU: bench.py's launch plumbing.  `--gpus N` outside torchrun re-launches
the script as N ranks over 127.0.0.1 (one process per GPU); the reference arm
runs the oracle on the whole workload and never maps the product library."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=300):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_gpus_n_spawns_n_ranks():
    d = _run("--gpus", "3", "--dry-run")
    assert d["dry_run"] and d["n_gpus"] == 3
    assert sorted(r["rank"] for r in d["ranks"]) == [0, 1, 2]
    assert len({r["pid"] for r in d["ranks"]}) == 3          # one process per rank
    assert sorted(r["local_rank"] for r in d["ranks"]) == [0, 1, 2]


def test_default_is_one_rank():
    d = _run("--dry-run")
    assert d["n_gpus"] == 1 and len(d["ranks"]) == 1


def test_reference_arm_whole_workload_without_the_product_library():
    d = _run("--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["config"]["same_config"] and d["config"]["registered_bytes_per_rank"] == 64 << 20
    assert d["repo_libs_loaded"] == ["oracle/liboracle.so"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
