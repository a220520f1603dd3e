"""Diagnostics for the tcgen05 similarity kernel: which split-precision terms
reach the accumulator (compares the dumped filter scores with the Kh*Qh,
Kh*Ql, Kl*Qh decomposition computed on the host), plus a one-launch driver for
ncu (`--profile`)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2603_17573_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402


def trunc(x):
    return (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def terms():
    import torch

    n, dim, B = 1024, 4096, 64
    col = H.Collection(dim, capacity=n)
    col.generate(O.REAL, 5, n)
    q = H.gen_queries(O.REAL, 6, 5, n, 0, B, dim)
    approx = col.debug_sim_scores(q).cpu().numpy().astype(np.float64)
    K = O.gen_keys(O.REAL, 5, 0, n, dim)
    Q = q.cpu().numpy()
    Kh, Qh = trunc(K), trunc(Q)
    Kl, Ql = (K - Kh), (Q - Qh)
    f = lambda a, b: a.astype(np.float64) @ b.astype(np.float64).T
    hh, hl, lh = f(Qh, Kh), f(Ql, Kh), f(Qh, Kl)
    exact = f(Q, K)
    for name, v in [("hh+hl+lh", hh + hl + lh), ("hh+hl", hh + hl), ("hh+lh", hh + lh), ("hh", hh),
                    ("exact", exact), ("hh+2hl", hh + 2 * hl), ("hh+hl+2lh", hh + hl + 2 * lh)]:
        print(f"{name:12s} max|approx - model| = {np.abs(approx - v).max():.3e}")
    # per-query / per-row structure of the residual
    r = approx - exact
    print("worst rows (mod 128):", np.bincount(np.argsort(-np.abs(r).max(0))[:64] % 128, minlength=128).nonzero()[0][:20])
    print("worst queries:", np.argsort(-np.abs(r).max(1))[:10])


def profile(n):
    import torch

    dim, B = 4096, 64
    col = H.Collection(dim, capacity=n)
    col.generate(O.REAL, 2026, n)
    q = H.gen_queries(O.REAL, 7, 2026, n, 0, B, dim)
    for _ in range(3):
        col.search_topk_exact(q, 8)
    torch.cuda.synchronize()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--n", type=int, default=1_000_000)
    a = ap.parse_args()
    if a.profile:
        profile(a.n)
    else:
        terms()
