"""The `raysurf` command line on the B200 engine (paper_2209_02878_b200.io_cli),
following the reference's CLI tests (tests/test_io_cli.py): binary readers
and writers, the positional / long-flag grammar, exit codes 1/2/3, and
end-to-end runs whose result files hold exactly the reference's results."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from golden_io import MODES, expected, load
from paper_2209_02878_b200 import io_cli

REPO = Path(__file__).resolve().parents[1]


def run_cli(args, cwd):
    env = dict(os.environ, PYTHONPATH=str(REPO))
    return subprocess.run([sys.executable, "-m", "paper_2209_02878_b200", *map(str, args)],
                          cwd=cwd, env=env, capture_output=True, text=True, timeout=300)


def write_scene(tmp_path, name="scene_s19"):
    fx = load(name)
    paths = io_cli.write_input_files(tmp_path / "input", fx["vertices"], fx["triangles"],
                                     fx["starts"], fx["ends"])
    return fx, [paths[n] for n in io_cli.DEFAULT_FILE_NAMES]


# ---------------------------------------------------------- CPU-only paths --

def test_readers_roundtrip(tmp_path):
    fx, files = write_scene(tmp_path)
    assert np.array_equal(io_cli.read_vertices(files[0]), fx["vertices"])
    assert np.array_equal(io_cli.read_triangles(files[1], fx["vertices"].shape[0]), fx["triangles"])
    seg = io_cli.read_segments(files[2], files[3])
    assert np.array_equal(seg.starts, fx["starts"]) and np.array_equal(seg.ends, fx["ends"])


@pytest.mark.parametrize("argv", [["a", "b"], ["a", "b", "c", "d", "loud"],
                                  ["a", "b", "c", "d", "silent", "fast"], ["--mode", "nope"],
                                  ["a", "b", "c", "d", "e", "f", "g"]])
def test_usage_errors_exit_1(tmp_path, argv):
    r = run_cli(argv, tmp_path)
    assert r.returncode == 1, r.stderr
    assert "raysurf: error" in r.stderr


def test_input_errors_exit_2(tmp_path):
    _, files = write_scene(tmp_path)
    bad = tmp_path / "bad_f32"
    bad.write_bytes(b"\0" * 13)  # not a multiple of 12 (test_io_cli.py)
    assert run_cli([bad, files[1], files[2], files[3]], tmp_path).returncode == 2
    assert run_cli([tmp_path / "missing", files[1], files[2], files[3]], tmp_path).returncode == 2
    short = tmp_path / "short_f32"
    np.zeros((3, 3), np.float32).tofile(short)  # 3 ends vs the batch's starts
    assert run_cli([files[0], files[1], files[2], short], tmp_path).returncode == 2
    assert run_cli([], tmp_path / "input").returncode == 2  # no ./input/input defaults


def test_validation_errors_exit_3(tmp_path):
    fx, files = write_scene(tmp_path)
    t = fx["triangles"].copy()
    t[5, 1] = fx["vertices"].shape[0]  # out of range (io_cli.py:86-96)
    badt = tmp_path / "tris_i32"
    t.astype("<i4").tofile(badt)
    r = run_cli([files[0], badt, files[2], files[3]], tmp_path)
    assert r.returncode == 3 and "triangle 5" in r.stderr


# ------------------------------------------------------------- end to end --

@pytest.mark.gpu
@pytest.mark.parametrize("mode", MODES)
def test_cli_results_match_reference(tmp_path, mode):
    fx, files = write_scene(tmp_path)
    out = tmp_path / "out"
    argv = files + ["silent"] + (["barycentric"] if mode == "barycentric" else
                                 ["intercept_count"] if mode == "count" else [])
    if mode == "boolean":
        argv = files + ["silent"]
    r = run_cli(argv + ["--out-dir", out], tmp_path)
    assert r.returncode == 0, r.stderr
    assert r.stdout == ""
    want = expected(fx, "batch", mode)
    if mode == "boolean":
        assert np.array_equal(io_cli.read_boolean_results(out), want["crossing"])
    elif mode == "count":
        assert np.array_equal(io_cli.read_count_results(out), want["counts"])
    else:
        rays, dist, tris, pts = io_cli.read_barycentric_results(out)
        assert np.array_equal(rays, want["ray_index"])
        assert np.array_equal(dist, want["distance"])
        assert np.array_equal(tris, want["triangle_id"])
        assert np.array_equal(pts, want["point"])


@pytest.mark.gpu
def test_cli_defaults_flags_and_report(tmp_path):
    fx, _ = write_scene(tmp_path)
    r = run_cli(["--mode", "count", "--sort-rays", "--workers", "2"], tmp_path)
    assert r.returncode == 0, r.stderr
    assert f"rays     : {fx['starts'].shape[0]}" in r.stdout
    assert "phase timings (ms):" in r.stdout
    # the reference's phase report (io_cli.py:52-61,254-263), every phase timed on device
    for phase in ("ray sort", "ray boxes", "quantization", "encoding", "sorting", "reset",
                  "construct", "query"):
        assert f"  {phase:<12} " in r.stdout, (phase, r.stdout)
    assert np.array_equal(io_cli.read_count_results(tmp_path), expected(fx, "batch", "count")["counts"])
    # byte-determinism across repeats (test_io_cli.py)
    first = (tmp_path / io_cli.RESULT_FILE_COUNT).read_bytes()
    assert run_cli(["--mode", "count"], tmp_path).returncode == 0
    assert (tmp_path / io_cli.RESULT_FILE_COUNT).read_bytes() == first
