"""Long randomised parity sweep of approx_topk against the oracle over every
dtype, both layouts and random shapes (development tool; run under gpurun).
Prints mismatching cases; exits non-zero if any."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_2412_04358_b200 as btk
from paper_2412_04358_b200 import _lib
from oracle import bucketed_oracle as O
from special_inputs import special, to_dtype, TORCH

budget = float(os.environ.get("SWEEP_SECONDS", "600"))
rng = np.random.default_rng(int(os.environ.get("SWEEP_SEED", "2024")))
lib = _lib.load()
DTC = {"f32": _lib.BTK_F32, "bf16": _lib.BTK_BF16, "f16": _lib.BTK_F16}
t0 = time.time()
n_cases = fails = 0
fams = {}
while time.time() - t0 < budget:
    dn = str(rng.choice(["f32", "bf16", "f16"]))
    asg = btk.Assignment.INTERLEAVED if rng.random() < 0.75 else btk.Assignment.CONTIGUOUS
    m = int(rng.choice([1, 2, 3, 5, 17, 300, 1300]))
    if rng.random() < 0.5:  # power-of-two-ish large shapes (fused / exchange families)
        b = int(2 ** rng.integers(3, 17))
        s = int(rng.choice([1, 2, 3, 4, 7, 8, 16, 33]))
        n = b * s
    else:
        n = int(rng.integers(8, 200000))
        b = int(rng.integers(1, min(n, 70000) + 1))
    n = min(n, 1 << 21)
    if m * n > (1 << 23):
        m = max(1, (1 << 23) // n)
    s = -(-n // b)
    kb = int(min(rng.choice([1, 1, 2, 3, 4, 8, 17]), s))
    P = b * kb
    k = int(rng.integers(1, min(P, n) + 1)) if rng.random() < 0.8 else int(min(P, n))
    try:
        btk.check_parameters(m, n, k, b, kb)
    except btk.ConfigError:
        continue
    kind = str(rng.choice(["normal", "ties", "pm0", "subnormal"]))
    if kind == "normal":
        x32 = rng.standard_normal((m, n), dtype=np.float32)
    elif kind == "ties":
        x32 = np.round(rng.standard_normal((m, n), dtype=np.float32) * 4) / 4
    else:
        x32 = special(rng, kind, m, n, dn)
    x = torch.from_numpy(np.ascontiguousarray(x32)).to(TORCH[dn])
    x32 = x.float().numpy()
    fam = lib.btk_kernel_family(m, n, k, b, kb, DTC[dn], 0 if asg == btk.Assignment.INTERLEAVED else 1, n)
    fams[fam] = fams.get(fam, 0) + 1
    xd = x.cuda()
    if rng.random() < 0.35:  # prepared op, BTK_INPUT_READY, launched right behind another launch
        op = btk.ApproxTopK(m, n, k, btk.BucketScheme(b, kb, asg), dtype=xd.dtype, device=xd.device,
                            inputs_ready=True)
        other = torch.randn_like(xd, dtype=torch.float32).to(xd.dtype)
        op.launch(other)
        op.launch(xd)
        r = btk.TopKResult(values=op.values.clone(), indices=op.indices.clone())
    else:
        r = btk.approx_topk(xd, k, btk.BucketScheme(b, kb, asg))
    wv, wi = O.approx_topk(x32, k, b, kb, assignment=O.INTERLEAVED if asg == btk.Assignment.INTERLEAVED else O.CONTIGUOUS)
    gi = r.indices.cpu().numpy()
    gv = r.values.float().cpu().numpy()
    ok = np.array_equal(gi, wi) and np.array_equal(gv.view(np.int32), np.asarray(wv, np.float32).view(np.int32))
    n_cases += 1
    if not ok:
        fails += 1
        print("MISMATCH", dn, asg, m, n, k, b, kb, kind, "family", fam, flush=True)
print("cases", n_cases, "fails", fails, "families", dict(sorted(fams.items())), flush=True)
sys.exit(1 if fails else 0)
