"""Small invocation of every device entry point, for compute-sanitizer
(memcheck / racecheck / synccheck).  python tools/sanitize_smoke.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_17573_b200 as H  # noqa: E402
from paper_2603_17573_b200 import synth  # noqa: E402

torch.cuda.set_device(0)
n, dim = 3000, 128
for dtype in ("f32", "bf16"):
    col = H.Collection(dim, capacity=n, dtype=dtype)
    col.generate(H.REAL, 3, n)
    for path in (["tc", "rows", "tile", "tc1", "tc3"] if dtype == "f32" else ["tc"]):
        H.set_sim_path(path)
        for B in (1, 5, 64, 300):
            if path in ("tc1", "tc3", "rows", "tile") and B > 64:
                continue
            q = H.gen_queries(H.REAL, 4, 3, n, 0, B, dim)
            sc, ids = col.search_topk_exact(q, 8)
    H.set_sim_path("auto")
    if dtype == "f32":
        col.set_filter("bf16_copy")
        q = H.gen_queries(H.REAL, 4, 3, n, 0, 700, dim)
        col.search_topk_exact(q, 8)
    rows = H.query_rows(4, H.REAL, n, 0, 64)
    lg = H.gen_logits(col, 3, rows, 7)
    fn, fp = H.gen_features(5, 64, 64)
    q = H.gen_queries(H.REAL, 4, 3, n, 0, 64, dim)
    sc, ids = col.search_topk_exact(q, 8)
    col.verify_round(ids, lg, [H.VerifyParams.make(skip_enabled=True), H.VerifyParams.make(relaxed=False)],
                     feat_now=fn, feat_prev=fp)
xyz = torch.as_tensor(synth.trajectory_windows(64, 15, seed=3)[0], device="cuda")
H.window_features(xyz, derivatives=True)
col = H.Collection(64, capacity=64 * 40, dtype="bf16")
col.generate(H.REAL, 7, 64 * 40, payload=H.PAYLOAD_TRAJ, traj_T=64)
loop = H.HybridLoop(col, H.hybrid_params(40, traj_T=64, d_f=64, seed=5, db_seed=7), max_rounds=20)
loop.step(20)
loop.reports()
f = torch.randn(60, 64, device="cuda")
f = f / f.norm(dim=1, keepdim=True)
try:
    H.calibrate_skip(f, [0, 30, 60], 0.0)
except H.CalibrationError:
    pass
torch.cuda.synchronize()
print("sanitize smoke ok")
