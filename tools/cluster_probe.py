"""Print the max co-resident clusters of the wide kernel per cluster size (diagnostic)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import paper_2603_17573_b200 as H  # noqa: E402
import torch  # noqa: E402

col = H.Collection(4096, capacity=200000)
col.generate(H.REAL, 1, 200000)
for B in (256, 512, 700, 1024):
    q = H.gen_queries(H.REAL, 2, 1, 200000, 0, B, 4096)
    col.search_topk_exact(q, 8)
torch.cuda.synchronize()
print("ok")
