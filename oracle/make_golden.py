"""Generate golden fixtures from the REAL reference implementation.

TEST INFRASTRUCTURE.  Run in the build container, where the read-only
reference is mounted:

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py

It imports `bucketed_topk` from /root/reference/pkg/src (pure NumPy; the
reference cannot travel to the GPU box) and writes `tests/golden/*.npz`.
The fixtures pin both the NumPy oracle (`oracle/bucketed_oracle.py`) and
the CUDA product path to the reference's own outputs.

Large inputs are not stored: they are regenerated from a seed with
`numpy.random.default_rng` (same image on the GPU box) and checked
against a stored SHA-256 of the input bytes before use.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(REPO, "tests", "golden")
REF_SRC = "/root/reference/pkg/src"


def _ref():
    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import bucketed_topk.approx as approx
    import bucketed_topk.core as core
    import bucketed_topk.exact as exact
    return approx, core, exact


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16, returned as float32 values."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return (u.astype(np.uint32) << 16).view(np.float32)


def gen_input(kind: str, m: int, n: int, seed: int) -> np.ndarray:
    """Deterministic generator shared by this script and the tests."""
    rng = np.random.default_rng(seed)
    if kind == "normal_f32":
        return rng.standard_normal((m, n), dtype=np.float32)
    if kind == "normal_bf16":
        return bf16_round(rng.standard_normal((m, n), dtype=np.float32))
    if kind == "normal_f16":
        return rng.standard_normal((m, n), dtype=np.float32).astype(np.float16).astype(np.float32)
    if kind == "ties":
        return rng.integers(0, 4, size=(m, n)).astype(np.float32)
    if kind == "signed_zero":
        x = rng.integers(-1, 2, size=(m, n)).astype(np.float32) * 0.0
        x[rng.random((m, n)) < 0.3] = -1.0
        return x  # mix of +0.0, -0.0 and -1.0
    raise ValueError(kind)


def sha(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float32).tobytes()).hexdigest()


def main() -> None:
    approx, core, exact = _ref()
    I, C = core.Assignment.INTERLEAVED, core.Assignment.CONTIGUOUS
    os.makedirs(OUT, exist_ok=True)

    # ---- 1. small explicit cases with stored inputs --------------------------------
    small = []  # (name, x(m,n) f32, k, b, kb, assignment)
    fig = np.array([[11.0, 3.0, 10.0, 6.0, 1.0, 4.0, 8.0, 5.0, 2.0, 9.0, 7.0]], np.float32)
    small.append(("worked_example", fig, 4, 3, 2, "interleaved"))
    small.append(("worked_example_contig", fig, 4, 3, 2, "contiguous"))
    small.append(("short_bucket_kb4", fig, 10, 3, 4, "interleaved"))
    small.append(("all_equal", np.full((1, 9), 3.0, np.float32), 2, 9, 1, "interleaved"))
    small.append(("five_five_five", np.array([[5.0, 5.0, 5.0, 1.0]], np.float32), 2, 1, 2, "interleaved"))
    small.append(("pos_neg_zero", np.array([[0.0, -0.0, -1.0]], np.float32), 2, 3, 1, "interleaved"))
    small.append(("neg_zero_sign_kept", np.array([[-0.0, 0.0, -1.0, -0.0]], np.float32), 3, 4, 1, "interleaved"))
    sub = np.array([[1.4e-45, 2.8e-45, 0.0, -1.4e-45]], np.float32)
    small.append(("subnormals", sub, 4, 1, 4, "interleaved"))
    small.append(("subnormals_b2", sub, 2, 2, 1, "interleaved"))
    rng = np.random.default_rng(1234)
    cnt = 0
    for assignment in ("interleaved", "contiguous"):
        for kind in ("normal_f32", "ties", "signed_zero", "normal_bf16"):
            for _ in range(12):
                n = int(rng.integers(1, 700))
                b = int(rng.integers(1, n + 1))
                cap = -(-n // b)
                kb = int(rng.integers(1, min(cap, 40) + 1))
                kmax = min(n, b * kb)
                k = int(rng.integers(kb, kmax + 1)) if kmax >= kb else kmax
                x = gen_input(kind, 3, n, int(rng.integers(1 << 30)))
                small.append((f"rand{cnt:03d}_{assignment[:3]}_{kind}", x, k, b, kb, assignment))
                cnt += 1
    # degenerate exact schemes (reference test_approx.py:107-115)
    for n in (2, 17, 64, 150):
        x = gen_input("ties", 2, n, n)
        small.append((f"degen_b1_n{n}", x, min(n, 9), 1, min(n, 9), "interleaved"))
        small.append((f"degen_bn_n{n}", x, min(n, 9), n, 1, "interleaved"))

    rec = {}
    for name, x, k, b, kb, asg in small:
        scheme = core.BucketScheme(b=b, k_b=kb, assignment=I if asg == "interleaved" else C)
        r = approx.approx_topk(x, k, scheme)
        s1 = approx.stage1(x, scheme)
        ex = exact.exact_topk_oracle(x, k)
        rec[name] = dict(x=x, k=k, b=b, kb=kb, asg=asg, values=r.values, indices=r.indices,
                         s1_values=s1.values, s1_indices=s1.indices, s1_per_bucket=s1.per_bucket,
                         ex_values=ex.values, ex_indices=ex.indices)
    flat = {}
    for name, d in rec.items():
        for key, v in d.items():
            flat[f"{name}/{key}"] = np.asarray(v)
    np.savez_compressed(os.path.join(OUT, "small_cases.npz"), names=np.array(list(rec)), **flat)

    # ---- 2. carried-label stage 2 (reference test_exact.py:141-147) -------------------
    v = np.array([[1.0, 9.0, 5.0, 9.0]])
    lab = np.array([[40, 30, 20, 10]])
    t = exact.topk_with_indices(v, lab, 3)
    rng = np.random.default_rng(99)
    v2 = rng.integers(0, 5, size=(4, 300)).astype(np.float32)
    lab2 = np.stack([rng.permutation(100000)[:300] for _ in range(4)]).astype(np.int64)
    t2 = exact.topk_with_indices(v2, lab2, 57)
    np.savez_compressed(os.path.join(OUT, "carried_labels.npz"),
                        v=v, lab=lab, k=3, values=t.values, indices=t.indices,
                        v2=v2, lab2=lab2, k2=57, values2=t2.values, indices2=t2.indices)

    # ---- 3. validation codes --------------------------------------------------------
    grid = []
    rng = np.random.default_rng(5)
    for _ in range(400):
        m, n, k, b, kb = (int(v) for v in rng.integers(-1, 40, size=5))
        try:
            core.check_parameters(m, n, k, b, kb)
            code = ""
        except core.ConfigError as e:
            code = e.code
        grid.append((m, n, k, b, kb, code))
    extra = [(1, 8, 4, 2, 1), (1, 8, 9, 1, 8), (1, 8, 4, 9, 1), (1, 11, 8, 3, 5), (1, 64, 2, 4, 3),
             (1, 11, 8, 3, 4), (0, 8, 2, 4, 1), (1, 65536, 64, 64, 1)]
    for m, n, k, b, kb in extra:
        try:
            core.check_parameters(m, n, k, b, kb)
            code = ""
        except core.ConfigError as e:
            code = e.code
        grid.append((m, n, k, b, kb, code))
    np.savez_compressed(os.path.join(OUT, "validation.npz"),
                        params=np.array([g[:5] for g in grid], np.int64),
                        codes=np.array([g[5] for g in grid]))

    # ---- 4. BASELINE-shaped cases (inputs regenerated from seed, hash-checked) ---------
    big = [  # name, kind, m, n, k, b, kb, seed
        ("cfg1", "normal_f32", 4, 65536, 64, 64, 1, 101),
        ("cfg2_kb2", "normal_f32", 2, 65536, 16384, 8192, 2, 102),
        ("cfg2_kb4", "normal_f32", 2, 65536, 16384, 4096, 4, 103),
        ("cfg2_kb8", "normal_f32", 2, 65536, 16384, 2048, 8, 104),
        ("cfg3_r1", "normal_bf16", 1, 1 << 20, 256, 256, 1, 105),
        ("cfg3_r8", "normal_bf16", 1, 1 << 20, 256, 2048, 1, 106),
        ("cfg3_kb2", "normal_bf16", 1, 1 << 20, 256, 256, 2, 107),
        ("cfg4", "normal_bf16", 8, 32768, 512, 512, 1, 108),
        ("cfg5_kb2", "normal_bf16", 1, 1 << 20, 65536, 65536, 2, 109),
        ("cfg1_ties", "ties", 2, 65536, 64, 64, 1, 110),
        ("cfg4_f16", "normal_f16", 4, 32768, 512, 512, 1, 111),
    ]
    out = {}
    for name, kind, m, n, k, b, kb, seed in big:
        x = gen_input(kind, m, n, seed)
        scheme = core.BucketScheme(b=b, k_b=kb, assignment=I)
        r = approx.approx_topk(x, k, scheme, workers=os.cpu_count() or 1)
        out[f"{name}/meta"] = np.array([m, n, k, b, kb, seed], np.int64)
        out[f"{name}/kind"] = np.array(kind)
        out[f"{name}/sha"] = np.array(sha(x))
        out[f"{name}/indices"] = r.indices.astype(np.int32)
        out[f"{name}/values"] = r.values.astype(np.float32)
        print(name, "done", flush=True)
    np.savez_compressed(os.path.join(OUT, "baseline_shapes.npz"),
                        names=np.array([b[0] for b in big]), **out)
    print("golden fixtures written to", OUT)


def cfg5_rows() -> None:
    """cfg5 at m = 8 rows (b = 65536, k_b = 2, k = 65536 of n = 2^20, bf16
    values): outputs stored as SHA-256 of the int64 indices and of the
    float32 value bits (8 x 65536 pairs would be MBs of fixture), plus
    row 0 in full for diagnosis."""
    approx, core, _ = _ref()
    m, n, k, b, kb, seed = 8, 1 << 20, 65536, 65536, 2, 112
    x = gen_input("normal_bf16", m, n, seed)
    r = approx.approx_topk(x, k, core.BucketScheme(b=b, k_b=kb, assignment=core.Assignment.INTERLEAVED),
                           workers=os.cpu_count() or 1)
    idx = np.ascontiguousarray(r.indices, dtype=np.int64)
    val = np.ascontiguousarray(r.values, dtype=np.float32)
    np.savez_compressed(os.path.join(OUT, "cfg5_rows.npz"), meta=np.array([m, n, k, b, kb, seed], np.int64),
                        kind=np.array("normal_bf16"), sha=np.array(sha(x)),
                        sha_indices=np.array(hashlib.sha256(idx.tobytes()).hexdigest()),
                        sha_values=np.array(hashlib.sha256(val.tobytes()).hexdigest()),
                        row0_indices=idx[0].astype(np.int32), row0_values=val[0])
    print("cfg5_rows done", flush=True)


def philox_normal_rows(seed: int, first_row: int, rows: int, n: int) -> np.ndarray:
    """Restatement of the reference's keyed generator (simdata.py:38-66):
    row r is standard_normal(n) from Philox keyed (seed << 64) | (0 << 56) | r."""
    out = np.empty((rows, n), dtype=np.float64)
    for r in range(rows):
        out[r] = np.random.Generator(np.random.Philox(key=(seed << 64) | (first_row + r))).standard_normal(n)
    return out


# float64 cases on the reference's own inputs (simdata.iid_normal): name,
# m, n, k, b, kb, assignment, seed
F64_CASES = [
    ("f64_cfg1like", 16, 4096, 64, 64, 1, "interleaved", 201),
    ("f64_kb2", 8, 65536, 512, 512, 2, "interleaved", 202),
    ("f64_contig_kb4", 8, 10000, 100, 50, 4, "contiguous", 203),
    ("f64_kb30", 4, 20000, 300, 10, 30, "interleaved", 204),
    ("f64_ragged", 6, 10007, 333, 97, 5, "interleaved", 205),
    ("f64_bigpool", 2, 131072, 12000, 8192, 2, "interleaved", 206),
    ("f64_exact_b1", 4, 20000, 500, 1, 500, "interleaved", 207),
    ("f64_exact_long", 2, 50000, 9000, 1, 9000, "contiguous", 208),
]


def f64_cases() -> None:
    """Reference outputs on its own float64 generator (simdata.iid_normal):
    approx_topk, stage1 and exact_topk_oracle, stored in full."""
    approx, core, exact = _ref()
    import bucketed_topk.simdata as simdata
    out = {}
    for name, m, n, k, b, kb, asg, seed in F64_CASES:
        x = simdata.iid_normal(m, n, seed=seed)
        assert np.array_equal(x, philox_normal_rows(seed, 0, m, n))
        A = core.Assignment.INTERLEAVED if asg == "interleaved" else core.Assignment.CONTIGUOUS
        scheme = core.BucketScheme(b=b, k_b=kb, assignment=A)
        r = approx.approx_topk(x, k, scheme)
        s1 = approx.stage1(x, scheme)
        ex = exact.exact_topk_oracle(x, k)
        out[f"{name}/meta"] = np.array([m, n, k, b, kb, seed], np.int64)
        out[f"{name}/asg"] = np.array(asg)
        out[f"{name}/sha"] = np.array(hashlib.sha256(x.tobytes()).hexdigest())
        out[f"{name}/values"] = r.values
        out[f"{name}/indices"] = r.indices
        out[f"{name}/s1_values"] = s1.values
        out[f"{name}/s1_indices"] = s1.indices
        out[f"{name}/ex_values"] = ex.values
        out[f"{name}/ex_indices"] = ex.indices
        print(name, "done", flush=True)
    # carried labels in float64 with repeated labels and signed zeros
    rng = np.random.default_rng(301)
    v = rng.integers(-2, 3, size=(3, 5000)).astype(np.float64) * rng.choice([1.0, 0.5e-310], size=(3, 5000))
    v[:, ::7] = -0.0
    lab = rng.integers(0, 600, size=(3, 5000)).astype(np.int64)
    t = exact.topk_with_indices(v, lab, 777)
    out["labels/v"], out["labels/lab"], out["labels/k"] = v, lab, np.array(777)
    out["labels/values"], out["labels/indices"] = t.values, t.indices
    np.savez_compressed(os.path.join(OUT, "f64_iid.npz"), names=np.array([c[0] for c in F64_CASES]), **out)
    print("f64 cases done", flush=True)


# Monte-Carlo recall configs: (n, k, b, kb, assignment, trials, seed)
MC_CASES = [
    (512, 32, 32, 1, "interleaved", 200, 9),
    (2048, 64, 32, 2, "interleaved", 300, 3),
    (1000, 50, 50, 2, "contiguous", 150, 4),
    (4096, 256, 128, 4, "interleaved", 100, 5),
    (64, 8, 1, 8, "interleaved", 50, 0),
]
# CLI argument sets whose stdout / CSV the GPU CLI must reproduce
CLI_RUNS = [
    ["run", "--n", "128", "--k", "8", "--b", "16", "--kb", "1", "--seed", "3"],
    ["run", "--n", "1000", "--m", "3", "--k", "20", "--b", "10", "--kb", "3", "--seed", "7",
     "--assignment", "contiguous"],
    ["run", "--n", "4096", "--m", "2", "--k", "64", "--exact", "--seed", "11"],
    ["run", "--n", "300", "--m", "2", "--k", "30", "--b", "7", "--kb", "5", "--seed", "1", "--mode", "auto"],
]
CLI_CORR = [
    ["correlation", "--n", "512", "--k", "64", "--rho-list", "0.0,0.99", "--kb-list", "1,2,3",
     "--trials", "200", "--shuffle", "--seed", "2"],
]


def recall_cli() -> None:
    """Reference outputs for the recall loop and the CLI commands (run,
    correlation) — the GPU versions must reproduce them exactly."""
    import contextlib
    import io
    import json

    approx, core, exact = _ref()
    import bucketed_topk.cli as cli
    import bucketed_topk.recall as recall

    out = {"mc": [], "rows": None, "cli": [], "corr": []}
    for n, k, b, kb, asg, trials, seed in MC_CASES:
        A = core.Assignment.INTERLEAVED if asg == "interleaved" else core.Assignment.CONTIGUOUS
        mc = recall.monte_carlo_recall(core.ProblemShape(m=1, n=n, k=k), core.BucketScheme(b=b, k_b=kb, assignment=A),
                                       trials=trials, seed=seed, block_rows=64)
        out["mc"].append({"n": n, "k": k, "b": b, "kb": kb, "asg": asg, "trials": trials, "seed": seed,
                          "mean_recall": mc.mean_recall, "stderr": mc.stderr})
        print("mc", n, k, b, kb, flush=True)
    rng = np.random.default_rng(77)
    x = rng.standard_normal((6, 2000))
    got = approx.approx_topk(x, 40, core.BucketScheme(b=20, k_b=2))
    want = exact.exact_topk_oracle(x, 40)
    out["rows"] = {"seed": 77, "m": 6, "n": 2000, "k": 40, "b": 20, "kb": 2,
                   "recall": recall.empirical_recall_rows(got, want).tolist()}
    for argv in CLI_RUNS + CLI_CORR:
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            code = cli.main(list(argv))
        (out["corr"] if argv[0] == "correlation" else out["cli"]).append(
            {"argv": argv, "code": code, "stdout": buf.getvalue()})
        print("cli", argv[0], flush=True)
    import bucketed_topk.cost as cost
    import bucketed_topk.simdata as simdata
    out["derive_seed"] = [[sd, st, simdata.derive_seed(sd, st)] for sd, st in ((0, 0), (7, 3), (2**63 + 5, 1000))]
    ar = simdata.ar1_batch(3, 257, 0.9, seed=4)
    out["ar1"] = {"trials": 3, "n": 257, "rho": 0.9, "seed": 4, "sha": hashlib.sha256(ar.tobytes()).hexdigest()}
    perm = simdata.permute(np.arange(50), seed=3, row=2)
    out["permute"] = {"n": 50, "seed": 3, "row": 2, "out": perm.tolist()}
    S = cost.CostModelKind.SERIAL
    out["cost"] = [{"n": n, "k": k, "m": m, "b": b, "kb": kb, "exact": cost.exact_cost(S, n, k, m),
                    "approx": cost.approx_cost(S, n, k, m, b, kb)}
                   for n, k, m, b, kb in ((256, 16, 2, 16, 1), (65536, 64, 128, 64, 1), (4096, 64, 3, 16, 8))]
    with open(os.path.join(OUT, "recall_cli.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("recall/cli done", flush=True)


if __name__ == "__main__":
    if "--recall" in sys.argv:
        recall_cli()
    elif "--cfg5" in sys.argv:
        cfg5_rows()
    elif "--f64" in sys.argv:
        f64_cases()
    else:
        main()
        cfg5_rows()
        f64_cases()
