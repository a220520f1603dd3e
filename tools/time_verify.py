"""K4 latency / throughput at several episode counts (CUDA events around
back-to-back hsd_verify_round calls on one stream; device-resident inputs).

  python tools/time_verify.py
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_17573_b200 as H  # noqa: E402


def main():
    torch.cuda.set_device(0)
    n, dim, k, L, d_f = 4096, 64, 8, 7, 4096
    col = H.Collection(dim, capacity=n)
    col.generate(H.REAL, 7, n)
    skip = (H.VerifyParams * 1)(H.VerifyParams.make(skip_enabled=True, min_S=0.95, O_dist=5))
    noskip = (H.VerifyParams * 1)(H.VerifyParams.make(skip_enabled=False))
    for E in (1, 8, 64, 512, 4096):
        q = H.gen_queries(H.REAL, 8, 7, n, 0, E, dim)
        _, ids = col.search_topk_exact(q, k)
        rows = H.query_rows(8, H.REAL, n, 0, E)
        lg = H.gen_logits(col, 3, rows, L)
        now, prev = H.gen_features(5, E, d_f)
        out = torch.empty((1, E, C.sizeof(H.Outcome)), dtype=torch.uint8, device="cuda")
        toks = torch.empty((1, E, L), dtype=torch.uint8, device="cuda")
        s = torch.cuda.current_stream()
        for feats in (False, True):
            fn, fp = (now, prev) if feats else (None, None)
            arr = skip if feats else noskip

            def call():
                H.check(H.lib().hsd_verify_round(col.handle, H._ptr(ids), E, k, L, H._ptr(lg), H._ptr(fn),
                                                 H._ptr(fp), d_f if feats else 0, None, 1,
                                                 C.cast(arr, C.c_void_p), 1, H._ptr(out), H._ptr(toks),
                                                 C.c_void_p(s.cuda_stream)))
            for _ in range(5):
                call()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            it = 50
            e0.record()
            for _ in range(it):
                call()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / it
            print(json.dumps({"E": E, "features_in_kernel": feats, "us_per_call": round(us, 2)}), flush=True)


if __name__ == "__main__":
    main()
