"""Fallback-row census of the cluster kernel fused_xchg (run with BTK_XB=0;
rowmask reasons; development tool).  tools/xb_why.py is the batched
pipeline's counterpart."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2412_04358_b200 as btk
from bench import CONFIGS
for cfg in sys.argv[1:] or ["cfg5", "cfg2_kb2"]:
    dt, m, n, k, b, kb, _, _ = CONFIGS[cfg]
    m = min(m, 64)
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[dt]
    x = torch.randn(m, n, device="cuda").to(tdt)
    op = btk.ApproxTopK(m, n, k, btk.BucketScheme(b, kb), dtype=tdt, device="cuda")
    op.launch(x); torch.cuda.synchronize()
    cnt = int(op.ws[:4].view(torch.int32).item())
    print(cfg, "fallback rows:", cnt, op.ws[256:256 + 4 * m].view(torch.int32)[:cnt].cpu().tolist())
