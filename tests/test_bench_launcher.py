"""bench.py's multi-rank harness on CPU: `--gpus 2` starts two ranks itself
(torch.distributed.run, gloo in --dry-run) and shards config 3's 256
realizations 128 + 128 by global index (homogenize.py:147-171 is what the
sharding replaces)."""

import json
import os
import subprocess
import sys

from conftest import REPO


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True,
                         text=True, timeout=300, env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_two_rank_dry_run_shards_the_config_batch():
    line = _run("--gpus", "2", "--dry-run", "--steps", "1", "--warmup", "0")
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["realizations_per_rank"] == [128, 128]
    assert line["first_seed_index_per_rank"] == [0, 128]
    assert line["config"]["realizations"] == 256
    assert "sharding x2" in line["config"]["parallelism"]


def test_single_rank_dry_run():
    line = _run("--dry-run", "--steps", "1", "--warmup", "0", "--config", "4")
    assert line["n_gpus"] == 1 and line["realizations_per_rank"] == [16]


def test_bench_refuses_debug_flags():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--dry-run"], capture_output=True,
                         text=True, timeout=120, env={**os.environ, "CHK_DEBUG_FLAGS": "1"})
    assert out.returncode != 0 and "CHK_DEBUG_FLAGS" in out.stderr
