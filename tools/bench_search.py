"""Micro-benchmark of the batched exact search per search path / key dtype /
batch, device-timed with CUDA events on the launching stream (L2 flushed
before every timed search with --flush).  Prints one JSON line per
configuration.

  python tools/bench_search.py --n 10000 --dim 4096 --batches 1,2,4 --paths filter,scan --flush
  python tools/bench_search.py --n 1000000 --dim 4096 --batches 64,256 --dtypes f32,bf16
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
    ap.add_argument("--paths", default="auto", help="comma list of auto | filter | scan | tc_single")
    ap.add_argument("--shadow", action="store_true", help="fp32 collections keep the bf16 filter copy")
    ap.add_argument("--flush", action="store_true", help="write 512 MB between timed searches (cold L2)")
    ap.add_argument("--flush-read", action="store_true",
                    help="with --flush: then read 256 MB, so the write's dirty lines drain outside the timing")
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import torch

    import paper_2603_17573_b200 as H

    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if a.flush else None
    rd = torch.zeros(64 << 20, dtype=torch.int32, device="cuda") if a.flush and a.flush_read else None
    for dt in a.dtypes.split(","):
        col = H.Collection(a.dim, capacity=a.n, dtype=dt)
        col.generate(H.REAL, 2026, a.n)
        if a.shadow and dt == "f32":
            col.set_filter("bf16_copy")
        for path in a.paths.split(","):
            H.set_sim_path(path)
            for B in [int(x) for x in a.batches.split(",")]:
                q = H.gen_queries(H.REAL, 7, 2026, a.n, 0, B, a.dim)
                for _ in range(3):
                    col.search_topk_exact(q, a.k)
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in range(a.iters)]
                torch.cuda.synchronize()
                for e0, e1 in ev:
                    if flush is not None:
                        flush.fill_(1)
                        if rd is not None:
                            rd.sum()
                    e0.record(s)
                    col.search_topk_exact(q, a.k)
                    e1.record(s)
                torch.cuda.synchronize()
                t = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
                ms = sum(t) / len(t)
                print(json.dumps({"dtype": dt, "path": path, "shadow": bool(a.shadow), "B": B, "n": a.n,
                                  "dim": a.dim, "ms": ms, "ms_min": t[0], "ms_median": t[len(t) // 2],
                                  "queries_per_s": B / (ms / 1e3), "l2_flushed": bool(a.flush),
                                  "stats": col.search_stats(reset=True)}), flush=True)
            H.set_sim_path("auto")
        col.close()
        del col
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
