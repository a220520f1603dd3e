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
    for path in ("auto", "filter", "scan", "tc_single"):
        H.set_sim_path(path)
        for B in (1, 5, 64, 200, 300):
            q = H.gen_queries(H.REAL, 4, 3, n, 0, B, dim)
            sc, ids = col.search_topk_exact(q, 8)
    H.set_sim_path("auto")
    if dtype == "f32":
        col.set_filter("bf16_copy")
        q = H.gen_queries(H.REAL, 4, 3, n, 0, 700, dim)
        col.search_topk_exact(q, 8)
    # the approximate index: build (exact assignment, counting sort, centroids) and search
    idx = H.Index(col, nlist=24, n_iter=2)
    for B in (1, 70, 1100):
        q = H.gen_queries(H.REAL, 6, 3, n, 0, B, dim)
        idx.search_topk(q, 8, nprobe=3, return_probes=True)
    idx.close()
    rows = H.query_rows(4, H.REAL, n, 0, 64)
    lg = H.gen_logits(col, 3, rows, 7)
    fn, fp = H.gen_features(5, 64, 64)
    q = H.gen_queries(H.REAL, 4, 3, n, 0, 64, dim)
    sc, ids = col.search_topk_exact(q, 8)
    col.verify_round(ids, lg, [H.VerifyParams.make(skip_enabled=True), H.VerifyParams.make(relaxed=False)],
                     feat_now=fn, feat_prev=fp)
# the range fallback: runs of near-duplicate rows
cl = H.Collection(dim, capacity=4096)
cl.generate(H.CLUSTER, 9, 4096)
for B in (1, 64):
    cl.search_topk_exact(H.gen_queries(H.CLUSTER, 4, 9, 4096, 0, B, dim), 8)
# per-chain verification and percentile bounds
ids8 = ids[:16].contiguous()
nch, ab, ctoks = H.enumerate_chains(ids8, 7, col=col)
H.verify_round_chains(ids8, H.VerifyParams.make(), torch.zeros(16, dtype=torch.int32, device="cuda"),
                      chain_greedy=ctoks, col=col)
H.percentile_bounds(torch.rand(1000, dtype=torch.float64, device="cuda"))
xyz = torch.as_tensor(synth.trajectory_windows(64, 15, seed=3)[0], device="cuda")
H.window_features(xyz, derivatives=True)
# engine step: K5 + the skip similarity on the side stream, K1 / K2 / K4 on the main stream
col = H.Collection(dim, capacity=n)
col.generate(H.REAL, 3, n)
eng = H.Engine(col, 64, 8, 7, 64, 15)
rows = H.query_rows(4, H.REAL, n, 0, 64)
fn, fp = H.gen_features(5, 64, 64)
dev = "cuda"
buf = H.StepBuffers(queries=H.gen_queries(H.REAL, 4, 3, n, 0, 64, dim), logits=H.gen_logits(col, 3, rows, 7),
                    feat_now=fn, feat_prev=fp, xyz=xyz, history=torch.full((64,), 100, dtype=torch.int32, device=dev),
                    scores=torch.empty((64, 8), dtype=torch.float64, device=dev),
                    ids=torch.empty((64, 8), dtype=torch.int32, device=dev),
                    out=torch.empty((64, 20), dtype=torch.uint8, device=dev),
                    tokens=torch.empty((64, 7), dtype=torch.uint8, device=dev),
                    R=torch.empty(64, dtype=torch.float64, device=dev), D=torch.empty(64, dtype=torch.float64, device=dev),
                    F=torch.empty(64, dtype=torch.float64, device=dev),
                    decision=torch.empty(64, dtype=torch.int32, device=dev))
eng.step(64, buf, H.VerifyParams.make(skip_enabled=True, min_S=0.95, O_dist=5), gap_d=1)
torch.cuda.synchronize()
# batch 1 on the exact scan: K4 launched early (PDL) under K1x, its own skip similarity
eng1 = H.Engine(col, 1, 8, 7, 64, 15)
b1 = H.StepBuffers(**{kk: (v[:1] if hasattr(v, "shape") else v) for kk, v in buf.__dict__.items()})
for _ in range(3):
    eng1.step(1, b1, H.VerifyParams.make(skip_enabled=True, min_S=0.95, O_dist=5), gap_d=1)
torch.cuda.synchronize()
# k > 32: every row's chain + radix sort; index search with k > 32
q = H.gen_queries(H.REAL, 4, 3, n, 0, 5, dim)
col.search_topk_exact(q, 100)
col.search_topk_exact(q, n + 3, row_range=(10, 400))
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
