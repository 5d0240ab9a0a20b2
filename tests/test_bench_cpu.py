"""bench.py host logic on CPU: the --gpus N launcher (2 ranks over gloo), the
static workload description both arms print, and the reference arm's
application counts (mgrit.py:276-334)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_launcher_spawns_ranks():
    """`bench.py --gpus 2` without torchrun re-launches itself under
    torch.distributed.run with 2 ranks (here: the gloo self-test)."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-check"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["world_size"] == 2 and d["n_gpus"] == 2
    assert sorted(x["rank"] for x in d["ranks"]) == [0, 1]
    assert sorted(x["local_rank"] for x in d["ranks"]) == [0, 1]


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--launch-check"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


@pytest.mark.parametrize("name,levels", [("cfg1", [1024, 128]), ("cfg2", [4096, 1024, 256, 64, 16, 4]),
                                         ("cfg3", [16384, 2048, 256, 32, 4]), ("cfg4", [1024, 256, 64, 16, 4]),
                                         ("cfg5", [2048, 256, 32, 4])])
def test_level_sizes_match_survey(name, levels):
    """SURVEY.md §8a build_hierarchy row: the level sizes of every config."""
    assert bench.level_sizes(bench.CONFIGS[name])[0] == levels
    assert bench.static_config(name)["levels"] == levels


def test_default_workload_is_cfg5():
    assert bench.DEFAULT_CONFIG == "cfg5"
    c = bench.static_config("cfg5")
    assert c["dof"] == 2 ** 31 and c["dim"] == 2 and c["p"] == 5


def test_application_counts():
    """cfg5: fine 2048 (5 - 2/8) = 9728 applications per iteration (three
    F-relaxations, C-relaxation, residual, convergence residual); level 1:
    256 (4 - 2/8) = 960; level 2: 120; coarsest: 4."""
    assert bench.applications("cfg5") == [9728.0, 960.0, 120.0, 4.0]
    est, t_iter = bench.model_estimate("cfg5", 1.0, 2.0, 14)
    assert t_iter == 9728 + 2 * (960 + 120 + 4)
    assert est == 2048 + 14 * t_iter


def test_reference_arm_prints_the_gpu_arm_config():
    """--impl reference prints exactly static_config(name), the dict the GPU
    arm prints, so the driver's same-config check holds."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference"
    assert d["config"] == bench.static_config("cfg1")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
