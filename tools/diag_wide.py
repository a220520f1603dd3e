"""Run the wide tcgen05 filter once in debug-dump mode (compute-sanitizer target)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_17573_b200 as H  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dt = sys.argv[2] if len(sys.argv) > 2 else "f32"
dim = int(sys.argv[3]) if len(sys.argv) > 3 else 64
mode = sys.argv[4] if len(sys.argv) > 4 else "dump"
n = 2000
col = H.Collection(dim, capacity=n, dtype=dt)
col.generate(H.EXACT, 5, n)
q = H.gen_queries(H.EXACT, 6, 5, n, 0, B, dim)
if mode == "dump":
    out = col.debug_sim_scores(q, variant=1)
else:
    out = col.search_topk_exact(q, 8)[1]
torch.cuda.synchronize()
print("ok", B, dt, dim, mode, out.shape)
