"""The reference CLI (``fcasep.cli``) with its estimator routed through the device.

The reference package is the caller here: its installed copy (``baseline/_ref``, the reference
arm's install) drives scene synthesis, WAV I/O, SDR and the CSV report, while
``paper_1805_09498_b200.cli.install`` rebinds ``cli._run_estimator`` / ``cli._images_from_run``
(cli.py:202-214) to the B200 path.  The reproducibility test is the reference's own
``test_bench_reproducible_and_counted`` (test_cli.py:109-135) run through that path, plus a
comparison of the device CSV against the stock CPU CLI on the same scenes.
"""

import csv
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "baseline", "_ref"))

SMALL = ["--sources", "2", "--channels", "2", "--duration", "1.0", "--frame-length", "256",
         "--frame-shift", "128"]


@pytest.fixture(scope="module")
def ref_cli():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    cli = pytest.importorskip("fcasep.cli", reason="reference package not installed in baseline/_ref")
    return cli


def read_csv(path):
    with open(path, newline="") as fh:
        return list(csv.DictReader(fh))


def _device(monkeypatch, ref_cli):
    from paper_1805_09498_b200 import cli as dev_cli

    calls = []

    def run_estimator(*a, **k):
        calls.append(1)
        return dev_cli.run_estimator(*a, **k)

    monkeypatch.setattr(ref_cli, "_run_estimator", run_estimator)
    monkeypatch.setattr(ref_cli, "_images_from_run", dev_cli.images_from_run)
    return calls


def test_bench_through_device_reproducible_and_counted(tmp_path, monkeypatch, ref_cli):
    from fcasep.evalkit import TIMING_COLUMNS

    args = ["bench", "--trials", "2", "--iterations", "2", "--seed", "3", *SMALL]
    cpu_out = tmp_path / "cpu"
    assert ref_cli.main(args + ["--out", str(cpu_out)]) == 0  # stock CLI, CPU estimator
    calls = _device(monkeypatch, ref_cli)
    out_a, out_b = tmp_path / "a", tmp_path / "b"
    assert ref_cli.main(args + ["--out", str(out_a)]) == 0
    assert ref_cli.main(args + ["--out", str(out_b)]) == 0
    assert len(calls) == 8  # 2 runs x 2 trials x 2 algorithms went through the device
    rows_a, rows_b, rows_c = read_csv(out_a / "bench.csv"), read_csv(out_b / "bench.csv"), read_csv(
        cpu_out / "bench.csv")
    assert len(rows_a) == 4  # two trials x two algorithms
    for ra, rb in zip(rows_a, rows_b):  # bit-identical apart from the timing columns (test_cli.py:109-135)
        for key, value in ra.items():
            if key in TIMING_COLUMNS:
                continue
            assert value == rb[key], key
    for row in rows_a:  # counter columns reproduce the formulas exactly
        N, F = int(row["N"]), int(row["F"])
        if row["algorithm"] == "fca":
            assert int(row["inversions"]) == 2 * (2 + N) * F
            assert int(row["matmuls"]) == 2 * 2 * 2 * N * F
        else:
            assert int(row["inversions"]) == 2 * (2 + 1) * F
            assert int(row["matmuls"]) == 0
    for ra, rc in zip(rows_a, rows_c):  # the device CSV against the stock CPU CLI
        assert ra["algorithm"] == rc["algorithm"] and ra["inversions"] == rc["inversions"]
        for key in ra:
            if key.startswith("sdr"):
                assert abs(float(ra[key]) - float(rc[key])) <= 1e-6, key


@pytest.mark.parametrize("algorithm", ["fca", "fastfca"])
def test_separate_through_device_matches_cpu(tmp_path, monkeypatch, ref_cli, algorithm):
    from fcasep.stft import read_wav

    scene_dir = tmp_path / "scene"
    assert ref_cli.main(["synth", "--seed", "4", "--out", str(scene_dir), *SMALL]) == 0
    sep = ["separate", "--scene-dir", str(scene_dir), "--algorithm", algorithm, "--iterations", "5", "--seed", "4",
           *SMALL]
    assert ref_cli.main(sep + ["--out", str(tmp_path / "cpu")]) == 0
    calls = _device(monkeypatch, ref_cli)
    assert ref_cli.main(sep + ["--out", str(tmp_path / "dev")]) == 0
    assert len(calls) == 1
    for j in (1, 2):
        a, _ = read_wav(tmp_path / "dev" / f"source_{j}.wav")
        b, _ = read_wav(tmp_path / "cpu" / f"source_{j}.wav")
        assert np.abs(a - b).max() <= 1e-6 * max(np.abs(b).max(), 1e-30) + 1e-9
    dev = read_csv(tmp_path / "dev" / "report.csv")[0]
    cpu = read_csv(tmp_path / "cpu" / "report.csv")[0]
    assert dev["inversions"] == cpu["inversions"] and dev["matmuls"] == cpu["matmuls"]


def test_main_device_option(tmp_path, ref_cli):
    from paper_1805_09498_b200 import cli as dev_cli

    saved = ref_cli._run_estimator, ref_cli._images_from_run
    try:
        out = tmp_path / "b"
        assert dev_cli.main(["bench", "--trials", "1", "--iterations", "1", "--seed", "5", "--device", "cuda",
                             "--out", str(out), *SMALL], cli_module=ref_cli) == 0
        assert len(read_csv(out / "bench.csv")) == 2
        assert ref_cli._run_estimator is dev_cli.run_estimator
    finally:
        ref_cli._run_estimator, ref_cli._images_from_run = saved
