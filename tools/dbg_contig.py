import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2412_04358_b200 as btk
from oracle import bucketed_oracle as O
from golden_io import small_cases
c = [c for c in small_cases() if c["name"] == "rand086_con_normal_bf16"][0]
x32 = np.ascontiguousarray(c["x"], np.float32)
k, b, kb = c["k"], c["b"], c["kb"]
for dt in (torch.float32, torch.bfloat16):
    x = torch.from_numpy(x32).to(dt).cuda()
    s = btk.stage1(x, btk.BucketScheme(b, kb, btk.Assignment.CONTIGUOUS))
    sv, si, _ = O.stage1(O.as_matrix(x.float().cpu().numpy()), b, kb, "contiguous")
    gi = s.indices.cpu().numpy()
    bad = np.argwhere(gi != si)
    print(dt, "stage1 mismatches", len(bad), bad[:5].tolist())
    for (r, p) in bad[:4]:
        print("  row", r, "pos", p, "got", gi[r, p], "want", si[r, p], "vals", x32[r, gi[r, p]], x32[r, si[r, p]])
