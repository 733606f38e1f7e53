"""bench.py's driver contract on CPU: the N = 2 path launches its own ranks (no torchrun
environment), partitions the rows, replicates [K||V] with ONE all-gather (gloo here, NCCL on
GPUs), reduces the timing over ranks and prints one JSON line (--dry-run: no kernel, value null);
and the reference arm (the oracle) prints its line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("config", ["cora", "arxiv"])
def test_bench_two_ranks_dry_run(config):
    j = _run(["--gpus", "2", "--dry-run", "--config", config, "--steps", "3", "--warmup", "3"])
    assert j["n_gpus"] == 2 and j["dry_run"] is True and j["value"] is None
    assert j["checks"] == {"rows_cover": True, "kv_allgather_bitwise": True}
    assert j["all_ranks_ok"] is True
    (b0, e0), (b1, e1) = j["bounds"]
    assert b0 == 0 and e0 == b1 and e1 == j["config"]["n"] and e0 % 16 == 0


def test_bench_batched_dry_run_has_no_collective():
    j = _run(["--gpus", "2", "--dry-run", "--config", "batched", "--steps", "3", "--warmup", "3"])
    assert j["checks"]["kv_allgather_bitwise"] == "batched: no collective" and j["all_ranks_ok"]


def test_reference_arm_line():
    j = _run(["--impl", "reference", "--config", "cora", "--steps", "3", "--warmup", "3"])
    assert j["impl"] == "reference" and j["value"] > 0 and j["cpu_baseline"]["kind"] == "oracle"
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["higher_is_better"] is True
