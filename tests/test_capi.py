"""The C-ABI library loads and exports every symbol include/mgrit_b200.h
declares; struct layouts agree between the header and the ctypes mirror; the
host-side logic (ERK tableaux, PCG64 jump-ahead, config validation) is right.
CPU only — no compute calls."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "mgrit_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mgrit_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    from paper_2203_13382_b200 import _lib
    lib = _lib.load()
    names = _declared()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_loop_entry_points_reject_bad_arguments():
    """The device-loop entry points validate their arguments before touching
    CUDA (no device needed): the legacy stream cannot be captured, NULL
    handles and buffers are rejected."""
    from paper_2203_13382_b200 import _lib
    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.mgrit_loop_begin(None, ctypes.byref(h)) == _lib.MGRIT_EINVAL
    assert lib.mgrit_loop_check(None, 8, 8, 8, 8, 8, None) == _lib.MGRIT_EINVAL
    assert lib.mgrit_loop_end(None, None) == _lib.MGRIT_EINVAL
    assert lib.mgrit_loop_launch(None, None) == _lib.MGRIT_EINVAL
    assert lib.mgrit_loop_init(None, 8, 8, 8, 1e-10, 1e6, 10, None) == _lib.MGRIT_EINVAL
    assert lib.mgrit_loop_init(8, 8, 8, 8, 1e-10, 1e6, 0, None) == _lib.MGRIT_EINVAL
    lib.mgrit_loop_destroy(None)


def test_launch_policy_names_match_header():
    """Python launch-policy names map onto the header's MGRIT_LAUNCH_* values
    (the C side reads the integer from the level descriptor)."""
    import re as _re
    from paper_2203_13382_b200 import mgrit as M
    src = open(HEADER).read()
    vals = {k: int(v) for k, v in _re.findall(r"MGRIT_LAUNCH_([A-Z0-9_]+)\s*=\s*(\d+)", src)}
    want = {"auto": "AUTO", "cta": "CTA", "cluster": "CLUSTER", "auto_one": "AUTO_ONE",
            "cluster2": "CLUSTER2", "cluster4": "CLUSTER4", "cluster8": "CLUSTER8", "cluster16": "CLUSTER16"}
    assert set(M.LAUNCH_POLICIES) == set(want)
    for name, enum in want.items():
        assert M.LAUNCH_POLICIES[name] == vals[enum], name
    prev = M.set_launch_policy("cluster16")
    assert M.set_launch_policy(prev) == "cluster16"
    with pytest.raises(ValueError):
        M.set_launch_policy("cluster3")


def test_library_is_sm100a():
    from paper_2203_13382_b200 import _lib
    r = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in r.stdout


def test_struct_layout_matches_header(tmp_path):
    from paper_2203_13382_b200 import _lib
    c = tmp_path / "sz.c"
    c.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "%s"\nint main(){printf("%%zu %%zu %%zu %%zu %%zu %%zu\\n",'
                 'sizeof(mgrit_level_desc),sizeof(mgrit_phase_args),sizeof(mgrit_erk_tableau),'
                 'offsetof(mgrit_level_desc,gmres_tol),offsetof(mgrit_phase_args,partial),'
                 'offsetof(mgrit_erk_tableau,c));}' % HEADER)
    exe = tmp_path / "sz"
    subprocess.run(["gcc", str(c), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(_lib.LevelDesc), ctypes.sizeof(_lib.PhaseArgs), ctypes.sizeof(_lib.ErkTableau),
            _lib.LevelDesc.gmres_tol.offset, _lib.PhaseArgs.partial.offset, _lib.ErkTableau.c.offset]
    assert got == want


@pytest.mark.parametrize("order", [1, 3, 5])
def test_erk_tableau_constants(order):
    import oracle as O
    from paper_2203_13382_b200 import _lib
    t = _lib.erk_tableau(order)
    a, b, c = O.erk_tableau(order)
    s = len(b)
    assert t.n_stages == s
    A = np.array(list(t.a)).reshape(6, 6)
    assert np.array_equal(A[:s, :s], a)
    assert np.array_equal(np.array(list(t.b))[:s], b)
    assert np.array_equal(np.array(list(t.c))[:s], c)


def _pcg_emulate(seed, count, start=0):
    """Python model of the device PCG64 kernel (jump-ahead + XSL-RR + 53-bit)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    state, inc = int(st["state"]), int(st["inc"])
    M = (2549297995355413924 << 64) | 4865540595714422341
    mask = (1 << 128) - 1
    # jump ahead `start` steps
    cur_m, cur_p, acc_m, acc_p, d = M, inc, 1, 0, start
    while d:
        if d & 1:
            acc_m = (acc_m * cur_m) & mask
            acc_p = (acc_p * cur_m + cur_p) & mask
        cur_p = ((cur_m + 1) * cur_p) & mask
        cur_m = (cur_m * cur_m) & mask
        d >>= 1
    state = (acc_m * state + acc_p) & mask
    out = []
    for _ in range(count):
        state = (state * M + inc) & mask
        hi, lo = state >> 64, state & ((1 << 64) - 1)
        rot = state >> 122
        x = hi ^ lo
        v = ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)
        out.append((v >> 11) * (1.0 / 9007199254740992.0))
    return np.array(out)


@pytest.mark.parametrize("seed", [0, 1, 4, 123])
def test_pcg64_model_matches_numpy(seed):
    ref = np.random.default_rng(seed).random(300)
    assert np.array_equal(_pcg_emulate(seed, 300), ref)
    assert np.array_equal(_pcg_emulate(seed, 50, start=200), ref[200:250])


def test_solver_config_validation():
    from paper_2203_13382_b200 import SolverConfig
    with pytest.raises(ValueError):
        SolverConfig(n_x=16, n_t=16, p=2)
    with pytest.raises(ValueError):
        SolverConfig(n_x=16, n_t=16, operator_kind="bogus")
    with pytest.raises(ValueError):
        SolverConfig(n_x=16, n_t=16, relaxation="CFC")
    with pytest.raises(ValueError):
        SolverConfig(n_x=16, n_t=16, wave_speed="C4")
    with pytest.raises(ValueError):
        SolverConfig(n_x=16, n_t=16, departure_policy="nope")
    assert SolverConfig(n_x=16, n_t=16, schedule=[16, 4]).schedule_factor(5) == 4


def test_product_fails_loudly_without_cuda():
    import torch
    from paper_2203_13382_b200 import SolverConfig, build_hierarchy
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="CUDA"):
        build_hierarchy(SolverConfig(n_x=16, n_t=16))


def test_cli_parse_and_config(tmp_path):
    """Config file + explicit flags (flags win), per-level schedules, bad input
    -> ValueError / exit status 2 (reference cli.py:93-125 behaviour)."""
    from paper_2203_13382_b200 import cli
    cfgf = tmp_path / "c.json"
    cfgf.write_text('{"n_x": 64, "n_t": 128, "p": 3, "wave_speed": "C3"}')
    cfg = cli.make_config({"p": 5}, str(cfgf))
    assert (cfg.n_x, cfg.n_t, cfg.p, cfg.wave_speed) == (64, 128, 5, "C3")
    assert cli.make_config({"n_x": 8, "n_t": 64, "schedule": "16,4"}, None).schedule == [16, 4]
    assert cli.make_config({"n_x": 8, "n_t": 64, "schedule": "8"}, None).schedule == 8
    bad = tmp_path / "b.json"
    bad.write_text('{"n_x": 64, "n_t": 128, "bogus": 1}')
    with pytest.raises(ValueError):
        cli.make_config({}, str(bad))
    with pytest.raises(ValueError):
        cli.make_config({"n_x": 64}, None)
    assert cli.main(["run", "--config", str(bad)]) == 2
    assert cli.main(["run", "--nx", "64"]) == 2
