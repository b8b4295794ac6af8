"""Quick GPU parity sweep of the exchange family against the oracle, every
dtype / k_b / input kind (development tool): the batched pipeline by
default, the cluster kernel with BTK_XB=0, fp32 through it with BTK_XC=1."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import paper_2412_04358_b200 as btk
from paper_2412_04358_b200 import _lib
from oracle import bucketed_oracle as O
from special_inputs import special, to_dtype, TORCH

DTC = {"f32": _lib.BTK_F32, "bf16": _lib.BTK_BF16, "f16": _lib.BTK_F16}
lib = _lib.load()
rng = np.random.default_rng(1)
fails = 0
cases = [
    ("bf16", 3, 1 << 20, 65536, 65536, 2),
    ("f16", 2, 1 << 20, 65536, 65536, 2),
    ("bf16", 3, 131072, 16384, 16384, 2),
    ("bf16", 2, 262144, 20000, 16384, 2),
    ("f16", 2, 262144, 30000, 8192, 4),
    ("bf16", 2, 262144, 30000, 8192, 4),
    ("bf16", 2, 262144, 9000, 16384, 1),
    ("f32", 3, 65536, 16384, 8192, 2),
    ("f32", 2, 65536, 16384, 4096, 4),
    ("f32", 2, 65536, 16384, 2048, 8),
    ("f32", 3, 65536, 10000, 8192, 2),
    ("f32", 2, 131072, 30000, 16384, 2),
]
for (dn, m, n, k, b, kb) in cases:
    fam = lib.btk_kernel_family(m, n, k, b, kb, DTC[dn], _lib.BTK_INTERLEAVED, n)
    for kind in ("normal", "ties", "pm0", "subnormal", "subnormal_ties", "mixed"):
        if kind == "normal":
            x32 = rng.standard_normal((m, n), dtype=np.float32)
        elif kind == "ties":
            x32 = np.round(rng.standard_normal((m, n), dtype=np.float32) * 4) / 4
        elif kind == "mixed":
            x32 = special(rng, "pm0", m, n, dn)
            x32[0] = rng.standard_normal(n, dtype=np.float32)
        else:
            x32 = special(rng, kind, m, n, dn)
        x = torch.from_numpy(x32).to(TORCH[dn])
        x32 = x.float().numpy()
        t0 = time.time()
        r = btk.approx_topk(x.cuda(), k, btk.BucketScheme(b, kb))
        torch.cuda.synchronize()
        wv, wi = O.approx_topk(x32, k, b, kb)
        gi = r.indices.cpu().numpy()
        gv = r.values.float().cpu().numpy()
        ok_i = np.array_equal(gi, wi)
        ok_v = np.array_equal(gv.view(np.int32), wv.astype(np.float32).view(np.int32))
        bad_rows = [int(q) for q in np.nonzero((gi != wi).any(1))[0]] if not ok_i else []
        if not (ok_i and ok_v):
            fails += 1
        print(f"{dn} m={m} n={n} k={k} b={b} kb={kb} fam={fam} {kind}: idx {ok_i} val {ok_v} bad_rows={bad_rows[:8]}"
              f" ({time.time()-t0:.1f}s)", flush=True)
print("FAILS", fails)
