"""Approximate index (IVF-flat) at a configuration-2 shape: build time, search
time per batch (CUDA events, median of iters) and recall@k against the exact
search.  One JSON line per (B, nprobe) on stdout.

  python tools/bench_index.py --n 1000000 --dim 4096 --nlist 1024 --iters 5
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_17573_b200 as H  # noqa: E402


def similar_recall(ids, ref, ref_sc, floor=0.5):
    """Recall over the exact top-k neighbours with cosine >= floor (the steps of a
    query's own run; pure-noise neighbours at cosine ~0.05 carry no signal)."""
    hit = tot = 0
    for a, b, s in zip(ids, ref, ref_sc):
        want = set(b[(b >= 0) & (s >= floor)].tolist())
        hit += len(want & set(a.tolist()))
        tot += len(want)
    return (hit / tot if tot else None), tot


def recall(ids, ref):
    hit = sum(len(set(a[a >= 0].tolist()) & set(b[b >= 0].tolist())) for a, b in zip(ids, ref))
    return hit / max(1, int((ref >= 0).sum()))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=1_000_000)
    p.add_argument("--dim", type=int, default=4096)
    p.add_argument("--nlist", type=int, default=1024)
    p.add_argument("--n-iter", type=int, default=5)
    p.add_argument("--k", type=int, default=8)
    p.add_argument("--batches", default="1,8,64")
    p.add_argument("--nprobes", default="4,8,16,32")
    p.add_argument("--iters", type=int, default=5)
    p.add_argument("--kind", type=int, default=H.CLUSTER)
    p.add_argument("--filter", default="bf16_copy", choices=["native", "bf16_copy"])
    a = p.parse_args()
    torch.cuda.set_device(0)
    col = H.Collection(a.dim, capacity=a.n)
    col.generate(a.kind, 7, a.n)
    col.set_filter(a.filter)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    idx = H.Index(col, nlist=a.nlist, n_iter=a.n_iter)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    inf = idx.info()
    print(json.dumps({"family": {0: "EXACT", 1: "REAL", 2: "CLUSTER"}[a.kind], "build_s": build_s, **inf, "n": a.n, "dim": a.dim, "n_iter": a.n_iter,
                      "filter": a.filter}), flush=True)
    for B in [int(x) for x in a.batches.split(",")]:
        q = H.gen_queries(a.kind, 8, 7, a.n, 0, B, a.dim)
        nd = np.array([b for b, r in enumerate(H.query_rows(8, a.kind, a.n, 0, B)) if r >= 0], np.int64)
        es, ei = col.search_topk_exact(q, a.k)
        ei, es = ei.cpu().numpy(), es.cpu().numpy()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tex = []
        for _ in range(a.iters):
            ev0.record()
            col.search_topk_exact(q, a.k)
            ev1.record()
            torch.cuda.synchronize()
            tex.append(ev0.elapsed_time(ev1))
        for npb in [int(x) for x in a.nprobes.split(",")]:
            ts = []
            for it in range(a.iters + 1):
                ev0.record()
                s, i = idx.search_topk(q, a.k, nprobe=npb)
                ev1.record()
                torch.cuda.synchronize()
                if it:
                    ts.append(ev0.elapsed_time(ev1))
            ii = i.cpu().numpy()
            r = recall(ii, ei)
            r_nd = recall(ii[nd], ei[nd]) if len(nd) else None
            r_sim, n_sim = similar_recall(ii, ei, es)
            top1 = float(np.mean(ii[:, 0] == ei[:, 0]))
            ms = float(np.median(ts))
            frac_rows = npb / inf["nlist"]
            print(json.dumps({"B": B, "nprobe": npb, "recall_at_k": r, "recall_at_k_near_dup": r_nd,
                              "recall_similar_neighbours": r_sim, "similar_neighbours": n_sim, "top1_match": top1, "ms": ms, "queries_per_s": B / ms * 1e3,
                              "exact_ms": float(np.median(tex)), "speedup_vs_exact": float(np.median(tex)) / ms,
                              "est_list_GBps": B * frac_rows * a.n * a.dim * 2 / (ms * 1e-3) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
