import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2412_04358_b200 as btk
from tests.golden_io import f64_cases
for c in f64_cases()[:3]:
    x = c["gen"]()
    sch = btk.BucketScheme(c["b"], c["kb"], btk.Assignment.INTERLEAVED if c["asg"]=="interleaved" else btk.Assignment.CONTIGUOUS)
    r = btk.approx_topk(x, c["k"], sch)
    print(c["name"], "approx", np.array_equal(r.indices.cpu().numpy(), c["indices"]), r.indices[0,:4].tolist())
    s1 = btk.stage1(x, sch)
    print(c["name"], "s1", np.array_equal(s1.indices.cpu().numpy(), c["s1_indices"]))
    e = btk.exact_topk_oracle(x, c["k"])
    print(c["name"], "exact", np.array_equal(e.indices.cpu().numpy(), c["ex_indices"]), e.indices[0,:4].tolist())
    r = btk.approx_topk(x, c["k"], sch)
    print(c["name"], "approx again", np.array_equal(r.indices.cpu().numpy(), c["indices"]), r.indices[0,:4].tolist())
