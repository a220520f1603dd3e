"""Micro-benchmark of the batched exact search (K1 similarity + K2 select) per
path / key dtype / batch, device-timed with CUDA events on the launching
stream.  Prints one JSON line per configuration.

  python tools/bench_search.py --n 1000000 --dim 4096 --batches 64,128,256 --dtypes f32,bf16
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=4096)
    ap.add_argument("--batches", default="64,128,256")
    ap.add_argument("--dtypes", default="f32,bf16")
    ap.add_argument("--paths", default="tc")
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    import torch

    import paper_2603_17573_b200 as H

    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    for dt in a.dtypes.split(","):
        col = H.Collection(a.dim, capacity=a.n, dtype=dt)
        col.generate(H.REAL, 2026, a.n)
        esz = 2 if dt == "bf16" else 4
        for path in a.paths.split(","):
            if dt == "bf16" and path != "tc":
                continue
            H.set_sim_path(path)
            for B in [int(x) for x in a.batches.split(",")]:
                q = H.gen_queries(H.REAL, 7, 2026, a.n, 0, B, a.dim)
                for _ in range(3):
                    col.search_topk_exact(q, a.k)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(s)
                for _ in range(a.iters):
                    col.search_topk_exact(q, a.k)
                e1.record(s)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.iters
                gbs = a.n * a.dim * esz * ((B + 1023) // 1024 if path == "tc" else (B + 63) // 64) / (ms / 1e3) / 1e9
                print(json.dumps({"dtype": dt, "path": path, "B": B, "n": a.n, "dim": a.dim, "ms": ms,
                                  "queries_per_s": B / (ms / 1e3), "key_stream_GBps": gbs,
                                  "overflow": col.overflow_count()}), flush=True)
            H.set_sim_path("auto")
        col.close()
        del col
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
