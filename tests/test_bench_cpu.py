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


def test_phase_bytes_2d_counts_input_rows_and_separable_records():
    """Algorithmic bytes of the fused phases: a 2D
    batched step reads its input row from HBM (8 B) and writes 8 B; per-node
    records add 16 B, separable records nothing; the fine 2D FC phase that
    skips its F-steps is one step per interval.  1D keeps the row on chip."""
    import types

    import bench
    from paper_2203_13382_b200 import _lib

    def level(dim, n, steps, m, kind="fine", separable=False, sig=None):
        grid = types.SimpleNamespace(n_points=n, dim=dim)
        return types.SimpleNamespace(grid=grid, n_steps=steps, cf=m, kind=kind, separable=separable, sig_x=sig)

    n, N, m = 1 << 20, 2048, 8
    nI = N // m
    per_node = bench.phase_bytes(level(2, n, N, m), _lib.PHASE_FC, True)
    sep = bench.phase_bytes(level(2, n, N, m, separable=True), _lib.PHASE_FC, True)
    assert per_node == nI * m * 8 * n * 4            # 2 records + input + output
    assert sep == nI * m * 8 * n * 2                 # input + output
    assert bench.phase_bytes(level(2, n, N, m, separable=True), _lib.PHASE_FC, True, c_only=True) == nI * 16 * n
    # a corrected 2D level is never "separable" for the byte count (per-node records + sigma + G)
    corr = bench.phase_bytes(level(2, n, 256, m, kind="corrected", separable=True, sig=object()), _lib.PHASE_FC, False)
    assert corr == (256 // m) * m * 8 * n * (2 + 1 + 2 + 1 + 1)
    # 1D fine level: left C row once per interval, then record + output per step
    n1 = 4096
    assert bench.phase_bytes(level(1, n1, 4096, 4), _lib.PHASE_FC, True) == (4096 // 4) * (8 * n1 + 4 * 16 * n1)
