"""Command-line front end on the GPU, drop-in for the reference CLI's
selection commands (reference cli.py).

    python -m paper_2412_04358_b200.cli run   --k 4 --b 3 --kb 2 --input row.csv
    python -m paper_2412_04358_b200.cli bench --n 65536 --k 64 --m 128 --b 64 --kb 1
    python -m paper_2412_04358_b200.cli correlation --n 512 --k 64 --rho-list 0.99 --shuffle

* ``run``          one selection, JSON on stdout — the reference payload
                   exactly (cli.py:232-278); float64 inputs take the exact
                   float64 GPU path, so the numbers are the reference's.
* ``bench``        timing + bandwidth CSV (cli.py:395-443) under the
                   reference protocol (bench.py:76-135: refill outside the
                   timed span, warmup, stderr/mean <= 5% stability flag);
                   the selection is timed with CUDA events.  GPU facts
                   (device, dtype, kernel family) go into the flags column.
* ``correlation``  AR(1) assignment experiment (cli.py:347-392): recall of
                   interleaved vs contiguous buckets on correlated rows,
                   selections and recall counts on the GPU.

The CSV schema is the reference's COLUMNS (cli.py:59-63), byte for byte;
auxiliary facts go into ``flags`` as ``;``-separated tokens and the seed
is echoed as ``# seed=N``.  Exit codes: 0 success, 2 validation / usage
error, 1 internal error.  BUCKETED_TOPK_WORKERS (or --workers) picks how
many GPUs the rows are sharded over (the reference's worker threads).
The analytic-model commands (``tradeoff``, ``recall``) are outside this
package's scope.
"""

from __future__ import annotations

import argparse
import json
import logging
import math
import os
import sys
from typing import List, Optional, Sequence, TextIO

import numpy as np
import torch

from . import simdata
from .approx import ChunkedMerge, ExecutionMode, PerBucket, approx_topk, select_mode
from .core import Assignment, BucketScheme, ConfigError, NonFiniteInputError, ProblemShape, validate
from .exact import exact_topk_oracle, priority_queue_topk
from .recall import recall_hits

log = logging.getLogger(__name__)

WORKERS_ENV = "BUCKETED_TOPK_WORKERS"

COLUMNS = [
    "model", "n", "k", "m", "b", "k_b", "ratio", "assignment", "mode",
    "analytic_error", "mc_error", "mc_stderr", "cost", "relative_cost",
    "mean_ns", "stderr_ns", "bytes_moved", "gbytes_per_s", "flags",
]

SELECTION_OPS = ("exact_oracle", "priority_queue", "approx_per_bucket", "approx_chunked_merge")
STABILITY_LIMIT = 0.05
_DTYPES = {"float64": torch.float64, "float32": torch.float32, "bfloat16": torch.bfloat16,
           "float16": torch.float16}


# ---------------------------------------------------------------------------- CSV
def _fmt(value) -> str:
    if value is None or value == "":
        return ""
    if isinstance(value, float):
        return repr(value)
    return str(value)


def write_csv(stream: TextIO, rows: Sequence[dict], seed: Optional[int] = None) -> None:
    if seed is not None:
        stream.write(f"# seed={seed}\n")
    stream.write(",".join(COLUMNS) + "\n")
    for row in rows:
        extra = set(row) - set(COLUMNS)
        if extra:
            raise ValueError(f"row has non-canonical columns: {sorted(extra)}")
        stream.write(",".join(_fmt(row.get(c)) for c in COLUMNS) + "\n")


def read_csv(text: str):
    """(comments, header, rows of strings)."""
    comments, header, rows = [], None, []
    for line in text.splitlines():
        if line.startswith("#"):
            comments.append(line)
        elif header is None:
            header = line.split(",")
        elif line:
            rows.append(line.split(","))
    return comments, header, rows


def render_csv(comments: List[str], header: List[str], rows: List[List[str]]) -> str:
    return "\n".join(list(comments) + [",".join(header)] + [",".join(r) for r in rows]) + "\n"


def _flags(*tokens) -> str:
    return ";".join(t for t in tokens if t)


def _emit(rows, seed, out) -> None:
    if out in (None, "-"):
        write_csv(sys.stdout, rows, seed=seed)
        return
    with open(out, "w", encoding="utf-8") as fh:
        write_csv(fh, rows, seed=seed)


# ---------------------------------------------------------------------------- helpers
def _int_list(text: str) -> List[int]:
    return [int(t) for t in text.split(",") if t]


def _float_list(text: str) -> List[float]:
    return [float(t) for t in text.split(",") if t]


def _parse_mode(text: str, shape: ProblemShape, scheme: BucketScheme) -> ExecutionMode:
    t = text.lower()
    if t in ("per-bucket", "perbucket"):
        return PerBucket()
    if t == "auto":
        return select_mode(shape, scheme, lanes=os.cpu_count() or 1)
    if t.startswith("chunked"):
        _, _, arg = t.partition(":")
        return ChunkedMerge(int(arg) if arg else 64)
    raise ConfigError("mode", f"unknown mode {text!r} (expected per-bucket, chunked[:c], or auto)")


def _mode_label(mode: ExecutionMode) -> str:
    return f"chunked:{mode.chunks_per_bucket}" if isinstance(mode, ChunkedMerge) else "per-bucket"


def _workers(args) -> int:
    if getattr(args, "workers", None):
        return args.workers
    env = os.environ.get(WORKERS_ENV)
    if env:
        try:
            return max(1, int(env))
        except ValueError:
            log.warning("ignoring non-integer %s=%r", WORKERS_ENV, env)
    return 1


def _devices(workers: int):
    """Worker count -> the GPUs rows are sharded over (None: current device)."""
    n = min(workers, torch.cuda.device_count())
    return [torch.device("cuda", i) for i in range(n)] if n > 1 else None


def _read_input_matrix(path: str) -> np.ndarray:
    rows = []
    with open(path, "r", encoding="utf-8") as fh:
        for line in fh:
            line = line.strip()
            if line:
                rows.append([float(t) for t in line.split(",")])
    if not rows:
        raise ConfigError("empty_input", f"input file {path} holds no rows")
    widths = {len(r) for r in rows}
    if len(widths) != 1:
        raise ConfigError("ragged_input", f"input rows differ in length: {sorted(widths)}")
    return np.asarray(rows, dtype=np.float64)


def _serial_cost(n: float, k: float, m: float) -> float:
    """SERIAL operation-count model (reference cost.py:77-85): the cheaper of
    an insertion-sorted queue scan and a radix select."""
    return min(m * n * (3.0 * k - 1.0), m * n * (4.0 * math.log2(n) + 4.0))


def _approx_serial_cost(n: int, k: int, m: int, b: int, kb: int) -> float:
    """Stage 1 over (m*b, n/b) plus stage 2 when b*k_b > k (cost.py:98-110)."""
    total = _serial_cost(n / b, float(kb), float(m * b))
    if b * kb > k:
        total += _serial_cost(float(b * kb), float(k), float(m))
    return total


# ---------------------------------------------------------------------------- commands
def cmd_run(args) -> int:
    if args.input:
        scores = _read_input_matrix(args.input)
    else:
        if not args.n:
            raise ConfigError("missing", "--n is required without --input")
        scores = simdata.iid_normal(args.m, args.n, seed=args.seed)
    m, n = scores.shape
    shape = ProblemShape(m=m, n=n, k=args.k)
    devices = _devices(_workers(args))
    if args.exact:
        fn = priority_queue_topk if args.priority_queue else exact_topk_oracle
        result = fn(scores, args.k)
        params = {"exact": True, "priority_queue": bool(args.priority_queue)}
    else:
        if not args.b or not args.kb:
            raise ConfigError("missing", "--b and --kb are required unless --exact")
        scheme = BucketScheme(b=args.b, k_b=args.kb, assignment=Assignment.from_string(args.assignment))
        validate(shape, scheme)
        mode = _parse_mode(args.mode, shape, scheme)
        result = approx_topk(scores, args.k, scheme, mode, devices=devices)
        params = {"b": args.b, "kb": args.kb, "assignment": scheme.assignment.value,
                  "mode": _mode_label(mode)}
    vals = result.values.double().cpu().numpy()
    idx = result.indices.cpu().numpy()
    payload = {
        "command": "run", "m": m, "n": n, "k": args.k, "seed": args.seed, "params": params,
        "rows": [{"values": [float(v) for v in vals[r]], "indices": [int(i) for i in idx[r]]}
                 for r in range(vals.shape[0])],
    }
    print(json.dumps(payload, sort_keys=True))
    return 0


def time_selection(op: str, shape: ProblemShape, scheme: Optional[BucketScheme], mode,
                   warmup: int, iters: int, seed: int, dtype=torch.float64, devices=None):
    """Reference bench.py:101-135 protocol on the GPU: a fresh seeded batch
    per iteration (generated and uploaded outside the timed span), CUDA
    events around the selection call.  Returns (mean_ns, stderr_ns)."""
    if op not in SELECTION_OPS:
        raise ConfigError("op", f"op must be one of {SELECTION_OPS}, got {op!r}")
    if iters < 1 or warmup < 0:
        raise ValueError(f"need iters >= 1 and warmup >= 0, got {iters}, {warmup}")
    if op.startswith("approx"):
        if scheme is None:
            raise ConfigError("missing", f"{op} requires --b and --kb")
        validate(shape, scheme)
        mode = PerBucket() if op == "approx_per_bucket" else (
            mode if isinstance(mode, ChunkedMerge) else ChunkedMerge(64))
        run = lambda x: approx_topk(x, shape.k, scheme, mode, devices=devices)
    elif op == "exact_oracle":
        run = lambda x: exact_topk_oracle(x, shape.k)
    else:
        run = lambda x: priority_queue_topk(x, shape.k)
    dev = torch.device("cuda", torch.cuda.current_device())

    def refill(step):
        x = simdata.iid_normal(shape.m, shape.n, seed=simdata.derive_seed(seed, step))
        return torch.from_numpy(x).to(dev).to(dtype)

    for step in range(warmup):
        run(refill(step))
    samples = np.empty(iters)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(iters):
        x = refill(warmup + i)
        torch.cuda.synchronize(dev)
        e0.record()
        run(x)
        e1.record()
        e1.synchronize()
        samples[i] = e0.elapsed_time(e1) * 1e6
    mean = float(samples.mean())
    stderr = float(samples.std(ddof=1) / np.sqrt(iters)) if iters > 1 else 0.0
    return mean, stderr


def cmd_bench(args) -> int:
    shape = ProblemShape(m=args.m, n=args.n, k=args.k)
    scheme = None
    if args.b and args.kb:
        scheme = BucketScheme(b=args.b, k_b=args.kb, assignment=Assignment.from_string(args.assignment))
        validate(shape, scheme)
    workers = _workers(args)
    devices = _devices(workers)
    dtype = _DTYPES[args.dtype]
    rows = []
    exact_c = _serial_cost(float(args.n), float(args.k), float(args.m))
    for op in args.ops:
        if op.startswith("approx") and scheme is None:
            raise ConfigError("missing", f"{op} requires --b and --kb")
        mode = ChunkedMerge(args.chunks) if op == "approx_chunked_merge" else None
        mean_ns, stderr_ns = time_selection(op, shape, scheme, mode, args.warmup, args.iters,
                                            args.seed, dtype=dtype, devices=devices)
        moved = args.m * (args.n * args.value_bytes + args.k * (args.value_bytes + args.index_bytes))
        stable = args.iters >= 2 and mean_ns > 0 and stderr_ns / mean_ns <= STABILITY_LIMIT
        approx = op.startswith("approx")
        cost = _approx_serial_cost(args.n, args.k, args.m, scheme.b, scheme.k_b) if approx else exact_c
        rows.append({
            "model": "serial", "n": args.n, "k": args.k, "m": args.m,
            "b": scheme.b if approx else "", "k_b": scheme.k_b if approx else "",
            "ratio": (scheme.b * scheme.k_b / args.k) if approx else "",
            "assignment": scheme.assignment.value if approx else "",
            "mode": op, "cost": cost, "relative_cost": cost / exact_c,
            "mean_ns": mean_ns, "stderr_ns": stderr_ns, "bytes_moved": moved,
            "gbytes_per_s": moved / mean_ns,
            "flags": _flags(f"warmup={args.warmup}", f"iters={args.iters}",
                            "stable" if stable else "unstable", f"workers={workers}",
                            f"device=cuda:{torch.cuda.current_device()}", f"dtype={args.dtype}",
                            f"gpus={len(devices) if devices else 1}"),
        })
    _emit(rows, args.seed, args.out)
    return 0


def _correlation_runs(shuffle: bool):
    for assignment in (Assignment.INTERLEAVED, Assignment.CONTIGUOUS):
        for shuf in ([False, True] if shuffle else [False]):
            if shuf and assignment is not Assignment.CONTIGUOUS:
                continue  # shuffling only matters where assignment is order-sensitive
            yield assignment, shuf


def cmd_correlation(args) -> int:
    rows = []
    k, n = args.k, args.n
    dev = torch.device("cuda", torch.cuda.current_device())
    for rho in args.rho_list:
        for kb in args.kb_list:
            if k % kb:
                log.info("skipping k_b=%s: does not divide k=%s", kb, k)
                continue
            b = k // kb
            data = simdata.ar1_batch(args.trials, n, rho, seed=args.seed)
            xd = torch.from_numpy(data).to(dev)
            truth = exact_topk_oracle(xd, k)
            for assignment, shuf in _correlation_runs(args.shuffle):
                scheme = BucketScheme(b=b, k_b=kb, assignment=assignment)
                validate(ProblemShape(m=args.trials, n=n, k=k), scheme)
                if shuf:
                    xs = np.stack([simdata.permute(data[t], seed=args.seed, row=t) for t in range(args.trials)])
                    xs_d = torch.from_numpy(xs).to(dev)
                    got, want = approx_topk(xs_d, k, scheme), exact_topk_oracle(xs_d, k)
                else:
                    got, want = approx_topk(xd, k, scheme), truth
                recalls = recall_hits(got.indices, want.indices).cpu().numpy().astype(np.float64) / k
                mean = float(recalls.mean())
                stderr = float(recalls.std(ddof=1) / math.sqrt(args.trials))
                rows.append({
                    "model": "", "n": n, "k": k, "m": args.trials, "b": b, "k_b": kb,
                    "ratio": b * kb / k, "assignment": assignment.value,
                    "mc_error": 1.0 - mean, "mc_stderr": stderr,
                    "flags": _flags(f"rho={rho}", "shuffled" if shuf else ""),
                })
    _emit(rows, args.seed, args.out)
    return 0


# ---------------------------------------------------------------------------- parser
def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="bucketed-topk-b200",
                                     description="Bucketed approximate top-k on the B200.")
    parser.add_argument("-v", "--verbose", action="store_true", help="log skipped points")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("run", help="run one selection, JSON on stdout")
    p.add_argument("--n", type=int, help="row length (ignored with --input)")
    p.add_argument("--m", type=int, default=1, help="batch rows to generate")
    p.add_argument("--k", type=int, required=True)
    p.add_argument("--b", type=int)
    p.add_argument("--kb", type=int)
    p.add_argument("--assignment", default="interleaved")
    p.add_argument("--mode", default="per-bucket", help="per-bucket | chunked[:c] | auto")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--input", help="CSV of score rows (no header)")
    p.add_argument("--exact", action="store_true", help="exact selection instead")
    p.add_argument("--priority-queue", action="store_true", help="with --exact: same contract")
    p.add_argument("--workers", type=int, help="GPUs to shard rows over")
    p.set_defaults(func=cmd_run)

    p = sub.add_parser("bench", help="timing and bandwidth, CSV")
    p.add_argument("--ops", type=lambda s: s.split(","), default=list(SELECTION_OPS),
                   help=f"comma list from {SELECTION_OPS}")
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--k", type=int, required=True)
    p.add_argument("--m", type=int, default=1)
    p.add_argument("--b", type=int)
    p.add_argument("--kb", type=int)
    p.add_argument("--assignment", default="interleaved")
    p.add_argument("--chunks", type=int, default=64)
    p.add_argument("--warmup", type=int, default=16)
    p.add_argument("--iters", type=int, default=512)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--value-bytes", type=int, default=8)
    p.add_argument("--index-bytes", type=int, default=8)
    p.add_argument("--dtype", default="float64", choices=sorted(_DTYPES),
                   help="device dtype of the scores (float64 = the reference's)")
    p.add_argument("--workers", type=int, help="GPUs to shard rows over")
    p.add_argument("--out")
    p.set_defaults(func=cmd_bench)

    p = sub.add_parser("correlation", help="assignment experiment on AR(1) data, CSV")
    p.add_argument("--n", type=int, default=2048)
    p.add_argument("--k", type=int, default=256)
    p.add_argument("--rho-list", type=_float_list, default=[0.0, 0.9, 0.99])
    p.add_argument("--kb-list", type=_int_list, default=[1, 2, 4])
    p.add_argument("--trials", type=int, default=1000)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--shuffle", action="store_true",
                   help="also run contiguous assignment on shuffled rows")
    p.add_argument("--out")
    p.set_defaults(func=cmd_correlation)
    return parser


def main(argv: Optional[Sequence[str]] = None) -> int:
    args = build_parser().parse_args(argv)
    logging.basicConfig(level=logging.INFO if args.verbose else logging.WARNING,
                        format="%(levelname)s %(message)s")
    try:
        return args.func(args)
    except (ConfigError, NonFiniteInputError) as err:
        print(f"error: {err}", file=sys.stderr)
        return 2
    except BrokenPipeError:
        return 0
    except Exception as err:  # internal failure
        log.exception("internal error")
        print(f"internal error: {err}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
