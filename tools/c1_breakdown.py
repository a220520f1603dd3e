"""Config-1 step breakdown on one B200 (L2 flushed before every timed call,
CUDA events on the launching stream): the search alone (K1x), the step
without K5 / verify-skip, and the full step; eager and early-K4 variants are
selected by HSD_NO_EARLY_VERIFY in the environment.

    python tools/c1_breakdown.py [--n 10000] [--dim 4096] [--iters 100]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_17573_b200 as H  # noqa: E402
from paper_2603_17573_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000)
    ap.add_argument("--dim", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=100)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    B, k, L, d_f = 1, 8, 7, 4096
    col = H.Collection(a.dim, capacity=a.n)
    col.generate(H.REAL, 2026, a.n)
    q = H.gen_queries(H.REAL, 7, 2026, a.n, 0, B, a.dim)
    rows = synth.query_rows(7, H.REAL, a.n, 0, B)
    lg = H.gen_logits(col, 3, rows, L)
    now, prev = H.gen_features(5, B, d_f)
    xyz = torch.as_tensor(synth.trajectory_windows(B, 15, seed=4)[0], device=dev)
    hist = torch.full((B,), 100, dtype=torch.int32, device=dev)
    outs = dict(scores=torch.empty((B, k), dtype=torch.float64, device=dev),
                ids=torch.empty((B, k), dtype=torch.int32, device=dev),
                out=torch.empty((B, 20), dtype=torch.uint8, device=dev),
                tokens=torch.empty((B, L), dtype=torch.uint8, device=dev),
                R=torch.empty(B, dtype=torch.float64, device=dev), D=torch.empty(B, dtype=torch.float64, device=dev),
                F=torch.empty(B, dtype=torch.float64, device=dev),
                decision=torch.empty(B, dtype=torch.int32, device=dev))
    full = H.StepBuffers(queries=q, logits=lg, feat_now=now, feat_prev=prev, xyz=xyz, history=hist, **outs)
    bare = H.StepBuffers(queries=q, logits=lg, history=hist, **outs)
    skipb = H.StepBuffers(queries=q, logits=lg, feat_now=now, feat_prev=prev, history=hist, **outs)
    eng = H.Engine(col, B, k, L, d_f, 15)
    vp_skip = H.VerifyParams.make(relaxed=True, skip_enabled=True, min_S=0.95, O_dist=5)
    vp_plain = H.VerifyParams.make(relaxed=True, skip_enabled=False)
    l2 = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    l2rd = torch.zeros(64 << 20, dtype=torch.int32, device=dev)
    small = torch.empty(16, dtype=torch.float64, device=dev)
    host = torch.zeros(16, dtype=torch.float64)
    stream = torch.cuda.current_stream()

    def timed(fn):
        ts = []
        for i in range(a.iters + 3):
            l2.fill_(i & 0xFF)
            l2rd.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
        return float(np.median(ts)), float(np.min(ts)), float(np.mean(ts)), float(np.percentile(ts, 90))

    res = {
        "empty bracket": timed(lambda: None),
        "H2D 128 B pageable": timed(lambda: small.copy_(host, non_blocking=True)),
        "search (K1x)": timed(lambda: col.search_topk_exact(q, k)),
        "step: K1x + K4, no K5 / skip": timed(lambda: eng.step(B, bare, vp_plain, gap_d=1)),
        "step: K1x + K4 + skip (K4 or side cos)": timed(lambda: eng.step(B, skipb, vp_skip, gap_d=1)),
        "step: full (K5 side + skip)": timed(lambda: eng.step(B, full, vp_skip, gap_d=1)),
    }
    # bench-like: 200 steps enqueued without a host sync, 4 rotating input batches
    qs = [H.gen_queries(H.REAL, 7, 2026, a.n, s * B, B, a.dim) for s in range(4)]
    bl = [H.StepBuffers(queries=qs[s], logits=lg, feat_now=now, feat_prev=prev, xyz=xyz, history=hist, **outs)
          for s in range(4)]
    for poll in (False, True):
        stop = [False]
        th = None
        if poll:  # an NVML clock poller, as bench.py's ClockSampler
            import threading

            import pynvml as N

            N.nvmlInit()
            hd = N.nvmlDeviceGetHandleByIndex(0)

            def run():
                import time
                while not stop[0]:
                    N.nvmlDeviceGetClockInfo(hd, N.NVML_CLOCK_SM)
                    N.nvmlDeviceGetCurrentClocksEventReasons(hd)
                    time.sleep(0.001)
            th = threading.Thread(target=run, daemon=True)
            th.start()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
        torch.cuda.synchronize()
        for i in range(200):
            l2.fill_(i & 0xFF)
            l2rd.sum()
            evs[i][0].record(stream)
            eng.step(B, bl[i % 4], vp_skip, gap_d=1)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        stop[0] = True
        ts = np.array([x.elapsed_time(y) * 1e3 for x, y in evs])
        res[f"bench-like 200 steps{' + NVML poller' if poll else ''}"] = (
            float(np.median(ts)), float(ts.min()), float(ts.mean()), float(np.percentile(ts, 90)))
    # host cost per call (wall clock of the enqueue loop, then the total with the sync)
    import time
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    hin = dict(queries=pin(q), logits=pin(lg), feat_now=pin(now), feat_prev=pin(prev), xyz=pin(xyz),
               history=pin(hist))
    hout = {kk: torch.empty_like(v, device="cpu").pin_memory() for kk, v in outs.items()}
    hb = H.StepBuffers(**hin, **hout)
    host = {}
    for name, fn in (("eng.step (device buffers)", lambda: eng.step(B, full, vp_skip, gap_d=1)),
                     ("eng.step_host_async (pinned host buffers)", lambda: eng.step_host_async(B, hb, vp_skip, gap_d=1))):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            fn()
        t1 = time.perf_counter()
        eng.sync()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        host[name] = ((t1 - t0) / 200 * 1e6, (t2 - t0) / 200 * 1e6)
    for name, (enq, tot) in host.items():
        print(f"host   {name:42s} enqueue {enq:7.2f} us/call   with sync {tot:7.2f} us/call")
    tag = "base" if os.environ.get("HSD_NO_EARLY_VERIFY") else "early"
    for name, (med, mn, mean, p90) in res.items():
        print(f"{tag:5s}  {name:42s} median {med:7.2f}  min {mn:7.2f}  mean {mean:7.2f}  p90 {p90:7.2f} us")


if __name__ == "__main__":
    main()
