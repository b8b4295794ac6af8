"""Host-side pieces of the recall loop and the CLI (no GPU): the CSV
schema (reference cli.py:59-63, 111-147), the keyed generator contract
(simdata.py), the SERIAL cost columns (cost.py:77-110) and the exit codes
of validation failures raised before any device work.  Pinned to
tests/golden/recall_cli.json (oracle/make_golden.py --recall, generated
from the reference)."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2412_04358_b200 import cli, simdata

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "recall_cli.json")))


def test_columns_match_reference_header():
    # the header line of a reference-produced CSV
    header = GOLD["corr"][0]["stdout"].splitlines()[1].split(",")
    assert cli.COLUMNS == header


def test_reference_csv_round_trips_byte_identical():
    text = GOLD["corr"][0]["stdout"]
    assert cli.render_csv(*cli.read_csv(text)) == text


def test_write_csv_rejects_non_canonical_columns():
    import io
    with pytest.raises(ValueError):
        cli.write_csv(io.StringIO(), [{"n": 1, "gpu": 3}])


def test_derive_seed_known_answers():
    for seed, step, want in GOLD["derive_seed"]:
        assert simdata.derive_seed(seed, step) == want


def test_ar1_and_permute_match_reference():
    a = GOLD["ar1"]
    x = simdata.ar1_batch(a["trials"], a["n"], a["rho"], seed=a["seed"])
    assert hashlib.sha256(x.tobytes()).hexdigest() == a["sha"]
    p = GOLD["permute"]
    assert simdata.permute(np.arange(p["n"]), seed=p["seed"], row=p["row"]).tolist() == p["out"]


def test_iid_normal_rows_are_blocking_invariant():
    full = simdata.iid_normal(5, 33, seed=12)
    part = simdata.normal_rows(12, 2, 3, 33)
    assert np.array_equal(full[2:], part)


def test_serial_cost_matches_reference():
    for c in GOLD["cost"]:
        assert cli._serial_cost(float(c["n"]), float(c["k"]), float(c["m"])) == c["exact"]
        assert cli._approx_serial_cost(c["n"], c["k"], c["m"], c["b"], c["kb"]) == c["approx"]


def test_run_validation_failure_exits_two(tmp_path, capsys):
    path = tmp_path / "row.csv"
    path.write_text("11,3,10,6,1,4,8,5,2,9,7\n")
    code = cli.main(["run", "--k", "4", "--b", "2", "--kb", "1", "--input", str(path)])
    assert code == 2
    assert "b*kb < k" in capsys.readouterr().err


def test_bench_missing_scheme_exits_two(capsys):
    assert cli.main(["bench", "--n", "64", "--k", "4", "--ops", "approx_per_bucket"]) == 2


def test_ragged_input_exits_two(tmp_path):
    path = tmp_path / "rows.csv"
    path.write_text("1,2,3\n4,5\n")
    assert cli.main(["run", "--k", "1", "--exact", "--input", str(path)]) == 2
