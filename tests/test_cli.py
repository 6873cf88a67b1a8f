"""The `silt-gpu` command line (paper_1307_0491_b200/cli/silt_main.cpp) against
the reference's CLI flow (the same source built with -DSILT_CLI_REFERENCE:
silt::run_parallel + silt::write_snapshot on the CPU, tests/cpp/_build/silt-ref-cli;
proj/tools/src/main.cpp:100-203, 261-317).

GPU STRICT runs write byte-identical snapshots, final.csv and config.txt; the
stdout report matches line for line except the wall time; timing.csv has one
row per worker strip with the reference's columns and a compute/exchange split.
"""
from __future__ import annotations

import os
import subprocess

import pytest

from conftest import ROOT

GPU_CLI = os.path.join(ROOT, "paper_1307_0491_b200", "lib", "silt-gpu")
REF_CLI = os.path.join(ROOT, "tests", "cpp", "_build", "silt-ref-cli")


def _run(exe, args, cwd):
    r = subprocess.run([exe] + args, capture_output=True, text=True, cwd=cwd, timeout=600)
    return r.returncode, r.stdout, r.stderr


def _need(exe):
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make -C paper_1307_0491_b200/cli)")


def test_cli_binaries_exist_and_reject_bad_flags(tmp_path):
    """CPU: the CLI is built; unknown flags and malformed dims fail like the
    reference's parser (exit 1, "error: ..."), no GPU needed."""
    for exe in (GPU_CLI, REF_CLI):
        _need(exe)
        rc, out, err = _run(exe, ["simulate", "--bogus", "1"], tmp_path)
        assert rc == 1 and "unknown option --bogus" in err
        rc, out, err = _run(exe, ["simulate", "--cells", "12y4"], tmp_path)
        assert rc == 1 and "--cells: expected positive integers" in err
        rc, out, err = _run(exe, ["regime", "1.0", "0.5"], tmp_path)
        assert rc == 0 and "regime     dune" in out
    rc_a, a, _ = _run(GPU_CLI, ["flux-table", "--points", "5"], tmp_path)
    rc_b, b, _ = _run(REF_CLI, ["flux-table", "--points", "5"], tmp_path)
    assert rc_a == rc_b == 0 and a == b


def _strip_wall(text):
    return [ln for ln in text.splitlines() if not ln.startswith(("wall time", "output"))]


@pytest.mark.gpu
@pytest.mark.parametrize("case", [
    ["--scenario", "bump2d", "--cells", "64x48", "--t-end", "6", "--snap-every", "2",
     "--workers", "1x3", "--ag", "1.0"],
    ["--scenario", "dune1d", "--cells", "500", "--t-end", "40", "--snap-at", "10,25"],
    ["--scenario", "antidune1d", "--cells", "300", "--t-end", "3", "--snap-every", "1"],
    ["--scenario", "bump2d", "--cells", "40x30", "--max-steps", "25", "--workers", "2x2",
     "--snap-at", "0,1.5", "--law", "mpm", "--friction", "darcy-weisbach"],
])
def test_simulate_matches_reference_cli(tmp_path, case):
    _need(GPU_CLI)
    _need(REF_CLI)
    d_gpu, d_ref = tmp_path / "gpu", tmp_path / "ref"
    rc, out_gpu, err = _run(GPU_CLI, ["simulate"] + case + ["--out", str(d_gpu), "--variant",
                                                            "strict"], tmp_path)
    assert rc == 0, err
    rc, out_ref, err = _run(REF_CLI, ["simulate"] + case + ["--out", str(d_ref)], tmp_path)
    assert rc == 0, err
    assert _strip_wall(out_gpu) == _strip_wall(out_ref)
    files = sorted(os.listdir(d_ref))
    assert sorted(os.listdir(d_gpu)) == files
    for f in files:
        if f in ("timing.csv", "config.txt"):
            continue
        assert (d_gpu / f).read_bytes() == (d_ref / f).read_bytes(), f
    # config.txt: the same keys; out_dir differs by design (two directories)
    cg = [ln for ln in (d_gpu / "config.txt").read_text().splitlines() if not ln.startswith("out_dir")]
    cr = [ln for ln in (d_ref / "config.txt").read_text().splitlines() if not ln.startswith("out_dir")]
    assert cg == cr
    rows = (d_gpu / "timing.csv").read_text().splitlines()
    assert rows[0] == "rank,steps,compute_seconds,exchange_seconds"
    body = [r.split(",") for r in rows[1:]]
    steps = {r[1] for r in body}
    assert len(steps) == 1
    assert all(float(r[2]) > 0 and float(r[3]) >= 0 for r in body)


@pytest.mark.gpu
def test_simulate_fast_variant_and_bench_speedup(tmp_path):
    """The default (FAST) variant runs the same flow; bench-speedup writes the
    reference's speedup CSV over the GPU strip layouts."""
    _need(GPU_CLI)
    rc, out, err = _run(GPU_CLI, ["simulate", "--scenario", "bump2d", "--cells", "128x96",
                                  "--t-end", "20", "--workers", "1x2", "--out",
                                  str(tmp_path / "f")], tmp_path)
    assert rc == 0, err
    assert "workers    1x2" in out and (tmp_path / "f" / "final.csv").exists()
    rc, out, err = _run(GPU_CLI, ["bench-speedup", "--cells", "128x96", "--t-end", "5",
                                  "--layouts", "1x1,1x2,1x4", "--out", str(tmp_path / "s.csv")],
                        tmp_path)
    assert rc == 0, err
    csv = (tmp_path / "s.csv").read_text().splitlines()
    assert csv[0] == "workers,seconds,speedup,efficiency"
    assert [r.split(",")[0] for r in csv[1:]] == ["1", "2", "4"]
    assert "layout 1x4:" in out
