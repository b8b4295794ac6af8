"""GPU recall loop and CLI against the reference's own outputs
(tests/golden/recall_cli.json, from oracle/make_golden.py --recall):

* monte_carlo_recall — identical mean and standard error (reference
  recall.py:231-268): same keyed inputs, exact float64 selections on the
  GPU, membership counts in btk_recall_hits;
* empirical_recall_rows — identical per-row recalls (recall.py:218-228);
* `run` — the reference's JSON payload byte for byte (cli.py:232-278);
* `correlation` — the reference's CSV byte for byte (cli.py:347-392);
* `bench` — schema, protocol flags, bytes and cost columns (cli.py:395-443).
"""

import contextlib
import io
import json
import os

import numpy as np
import pytest
import torch

import paper_2412_04358_b200 as btk
from paper_2412_04358_b200 import cli, recall

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "recall_cli.json")))


def _run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = cli.main(list(argv))
    return code, buf.getvalue()


@pytest.mark.parametrize("case", GOLD["mc"], ids=lambda c: f"n{c['n']}-k{c['k']}-b{c['b']}-kb{c['kb']}")
def test_monte_carlo_recall_equals_reference(case):
    asg = btk.Assignment.from_string(case["asg"])
    mc = recall.monte_carlo_recall(btk.ProblemShape(m=1, n=case["n"], k=case["k"]),
                                   btk.BucketScheme(case["b"], case["kb"], asg),
                                   trials=case["trials"], seed=case["seed"], block_rows=64)
    assert mc.mean_recall == case["mean_recall"]
    assert mc.stderr == case["stderr"]
    assert mc.trials == case["trials"]


def test_monte_carlo_recall_blocking_invariant():
    shape, scheme = btk.ProblemShape(m=1, n=512, k=32), btk.BucketScheme(32, 1)
    a = recall.monte_carlo_recall(shape, scheme, trials=200, seed=9)
    b = recall.monte_carlo_recall(shape, scheme, trials=200, seed=9, block_rows=17)
    assert a == b


def test_empirical_recall_rows_equals_reference():
    g = GOLD["rows"]
    x = np.random.default_rng(g["seed"]).standard_normal((g["m"], g["n"]))
    got = btk.approx_topk(x, g["k"], btk.BucketScheme(g["b"], g["kb"]))
    want = btk.exact_topk_oracle(x, g["k"])
    assert recall.empirical_recall_rows(got, want).tolist() == g["recall"]
    for r in range(g["m"]):
        assert recall.empirical_recall(got.row(r), want.row(r), g["k"]) == g["recall"][r]


def test_recall_hits_arbitrary_index_rows():
    """Membership counts on arbitrary (non-selection) rows: disjoint,
    identical, repeated approx entries, a truth duplicate across hash
    chunks, the sentinel value -1, and k larger than one pass."""
    a = torch.tensor([[0, 1, 2], [3, 4, 5], [7, 7, 9], [-1, 2, 3]], device="cuda")
    t = torch.tensor([[3, 4, 5], [5, 4, 3], [7, 8, 9], [3, -1, 8]], device="cuda")
    assert recall.recall_hits(a, t).tolist() == [0, 3, 3, 2]
    rng = np.random.default_rng(0)
    k = 20000
    tr = rng.permutation(10 ** 6)[:k]
    tr[-1] = tr[0]  # a duplicate in a later hash chunk
    ap = np.concatenate([tr[: k // 2], rng.integers(10 ** 6, 2 * 10 ** 6, size=k - k // 2)])
    want = int(np.isin(ap, tr).sum())
    assert int(recall.recall_hits(torch.from_numpy(ap[None]).cuda(), torch.from_numpy(tr[None]).cuda())[0]) == want


@pytest.mark.parametrize("case", GOLD["cli"], ids=lambda c: " ".join(c["argv"][:6]))
def test_cli_run_equals_reference(case):
    code, out = _run(case["argv"])
    assert code == case["code"]
    assert out == case["stdout"]


def test_cli_worked_example(tmp_path):
    path = tmp_path / "row.csv"
    path.write_text("11,3,10,6,1,4,8,5,2,9,7\n")
    code, out = _run(["run", "--k", "4", "--b", "3", "--kb", "2", "--input", str(path)])
    assert code == 0
    row = json.loads(out)["rows"][0]
    assert row["values"] == [11.0, 10.0, 9.0, 7.0] and row["indices"] == [0, 2, 9, 10]
    code, out = _run(["run", "--k", "4", "--exact", "--input", str(path)])
    assert json.loads(out)["rows"][0]["values"] == [11.0, 10.0, 9.0, 8.0]


@pytest.mark.parametrize("case", GOLD["corr"], ids=lambda c: "correlation")
def test_cli_correlation_equals_reference(case):
    code, out = _run(case["argv"])
    assert code == case["code"]
    assert out == case["stdout"]


def test_cli_bench_schema_and_columns(monkeypatch):
    monkeypatch.setenv("BUCKETED_TOPK_WORKERS", "1")
    code, out = _run(["bench", "--n", "256", "--k", "16", "--m", "2", "--b", "16", "--kb", "1",
                      "--ops", "priority_queue,approx_per_bucket", "--warmup", "2", "--iters", "4"])
    assert code == 0
    comments, header, rows = cli.read_csv(out)
    assert header == cli.COLUMNS and comments == ["# seed=0"]
    rows = [dict(zip(header, r)) for r in rows]
    assert [r["mode"] for r in rows] == ["priority_queue", "approx_per_bucket"]
    c = GOLD["cost"][0]
    for r in rows:
        assert float(r["mean_ns"]) > 0
        assert "warmup=2" in r["flags"] and "iters=4" in r["flags"] and "dtype=float64" in r["flags"]
        assert ("stable" in r["flags"]) or ("unstable" in r["flags"])
        assert int(r["bytes_moved"]) == 2 * (256 * 8 + 16 * 16)
    assert float(rows[0]["cost"]) == c["exact"] and float(rows[1]["cost"]) == c["approx"]
    # bf16 on the device: same schema, 2-byte values accounted by --value-bytes
    code, out = _run(["bench", "--n", "65536", "--k", "64", "--m", "8", "--b", "64", "--kb", "1",
                      "--ops", "approx_per_bucket", "--warmup", "2", "--iters", "3", "--dtype", "bfloat16",
                      "--value-bytes", "2"])
    assert code == 0 and "dtype=bfloat16" in out
