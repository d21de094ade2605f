"""MPS ingest and the command-line runner.

* include/batchlp/mps.hpp is exercised by the reference's own test_mps.cpp
  and acceptance criterion 10 (tests/test_cpp.py) and by our round trip in
  tests/cpp/test_dropin.cpp.
* tools/batchlp_run end to end on the B200: a set-cover instance written as
  MPS goes through `fsb` (root relaxation + strong branching on every
  fractional integer column, all on the device) and `bench` (the reference
  CLI's CSV row); the branch results match the compiled reference's run_fsb
  (oracle/_ref) on the same candidates: statuses identical, objectives
  within 1e-6 relative, iterations within 10 %.
"""
import csv
import io
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUN = os.path.join(ROOT, "tools", "_build", "batchlp_run")
DROPIN = os.path.join(ROOT, "tests", "cpp", "_build", "dropin_tests")
STATUS = {"optimal": 0, "primal_infeasible": 1, "dual_infeasible": 2, "iteration_limit": 3}


def _require(path):
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run __graft_entry__.build()")


def test_runner_rejects_bad_usage_and_missing_files(tmp_path):
    _require(RUN)
    r = subprocess.run([RUN], capture_output=True, text=True)
    assert r.returncode == 1 and "usage" in r.stderr
    r = subprocess.run([RUN, "solve", str(tmp_path / "nope.mps")], capture_output=True,
                       text=True)
    assert r.returncode == 2 and "cannot open" in r.stderr
    bad = tmp_path / "bad.mps"
    bad.write_text("NAME X\nROWS\n N obj\n N obj\nENDATA\n")
    r = subprocess.run([RUN, "solve", str(bad)], capture_output=True, text=True)
    assert r.returncode == 2 and "mps:4: duplicate row" in r.stderr


@pytest.mark.gpu
def test_mps_fsb_and_bench_match_reference(tmp_path, ref):
    _require(RUN)
    _require(DROPIN)
    import paper_2601_21990_b200 as bl
    from paper_2601_21990_b200 import instances as I
    rows, cols, dens, seed = 250, 500, 0.02, 3  # 10 fractional root columns
    mps = tmp_path / "setcover.mps"
    subprocess.run([DROPIN, "--write-mps", str(rows), str(cols), str(dens), str(seed),
                    str(mps)], check=True)
    out = tmp_path / "fsb.json"
    subprocess.run([RUN, "fsb", str(mps), "--json", str(out)], check=True, timeout=600)
    rep = json.loads(out.read_text())
    assert rep["format_version"] == "1" and rep["command"] == "fsb"
    assert (rep["m"], rep["n"]) == (rows, cols)
    # the same instance and the device root point (MPS round trip is exact)
    p = I.set_cover(rows, cols, dens, seed)
    root = bl.solve(p)
    assert abs(rep["root"]["objective"] - root.objective) <= 1e-12 * (1 + abs(root.objective))
    x = np.asarray(root.x)
    frac = [c for c in range(cols) if abs(x[c] - np.round(x[c])) > 1e-6]
    assert frac and len(rep["fsb"]["branches"]) == len(frac)
    want = ref.run_fsb(p, x, frac)
    for k, b in enumerate(rep["fsb"]["branches"]):
        assert b["variable"] == frac[k]
        for side in ("up", "down"):
            g = b[side]
            assert STATUS[g["status"]] == int(want[f"{side}_status"][k]), (k, side)
            wi = int(want[f"{side}_iterations"][k])
            assert abs(g["iterations"] - wi) <= 0.1 * max(wi, 1), (k, side)
            wo = float(want[f"{side}_objective"][k])
            if np.isfinite(wo) and g["status"] == "optimal":
                assert abs(g["objective"] - wo) <= 1e-6 * (1 + abs(wo)), (k, side)
    # the bench CSV row of the same flow
    r = subprocess.run([RUN, "bench", str(mps)], capture_output=True, text=True, check=True,
                       timeout=600)
    rows_ = list(csv.DictReader(io.StringIO(r.stdout)))
    assert list(rows_[0].keys()) == ["family", "instance", "m", "n", "nnz", "S", "runtime_s",
                                     "iters"]
    row = rows_[0]
    assert (row["family"], row["instance"]) == ("mps", "setcover")
    assert (int(row["m"]), int(row["n"]), int(row["nnz"])) == (rows, cols, p.A.nnz())
    assert int(row["S"]) == 2 * len(frac)
    assert int(row["iters"]) == root.iterations + rep["fsb"]["iterations"]
    assert float(row["runtime_s"]) > 0.0
