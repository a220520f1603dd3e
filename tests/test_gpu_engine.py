"""The fused decode-round engine (hsd_step / hsd_step_host / hsd_step_host_async):
host-buffer steps equal device-buffer steps, and the double-buffered async path
keeps every in-flight step's inputs and outputs separate."""
import numpy as np
import pytest

import paper_2603_17573_b200 as H
from paper_2603_17573_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


def make_inputs(torch, col, n, dim, B, L, d_f, s):
    q = H.gen_queries(H.REAL, 7 + s, 5, n, 0, B, dim)
    rows = H.query_rows(7 + s, H.REAL, n, 0, B)
    lg = H.gen_logits(col, 3 + s, rows, L)
    fn, fp = H.gen_features(5 + s, B, d_f)
    xyz = torch.as_tensor(synth.trajectory_windows(B, 15, seed=4 + s)[0], device="cuda")
    hist = torch.full((B,), 100, dtype=torch.int32, device="cuda")
    return dict(queries=q, logits=lg, feat_now=fn, feat_prev=fp, xyz=xyz, history=hist)


def outputs(torch, B, k, L, device):
    pin = device == "cpu"
    mk = lambda shape, dt: (torch.empty(shape, dtype=dt, device=device).pin_memory() if pin  # noqa: E731
                            else torch.empty(shape, dtype=dt, device=device))
    return dict(scores=mk((B, k), torch.float64), ids=mk((B, k), torch.int32), out=mk((B, 20), torch.uint8),
                tokens=mk((B, L), torch.uint8), R=mk((B,), torch.float64), D=mk((B,), torch.float64),
                F=mk((B,), torch.float64), decision=mk((B,), torch.int32))


def test_host_and_async_steps_match_device_steps(torch):
    n, dim, B, k, L, d_f = 20000, 256, 48, 8, 7, 256
    col = H.Collection(dim, capacity=n)
    col.generate(H.REAL, 5, n)
    eng = H.Engine(col, B, k, L, d_f, 15)
    vp = H.VerifyParams.make(skip_enabled=True, min_S=0.95, O_dist=5)
    S = 5
    ins = [make_inputs(torch, col, n, dim, B, L, d_f, s) for s in range(S)]
    ref = []
    for s in range(S):
        o = outputs(torch, B, k, L, "cuda")
        eng.step(B, H.StepBuffers(**ins[s], **o), vp)
        torch.cuda.synchronize()
        ref.append({kk: v.cpu() for kk, v in o.items()})
    h_in = [{kk: v.cpu().pin_memory() for kk, v in d.items()} for d in ins]
    # synchronous host-buffer step
    o = outputs(torch, B, k, L, "cpu")
    eng.step_host(B, H.StepBuffers(**h_in[2], **o), vp)
    for kk in o:
        assert torch.equal(o[kk], ref[2][kk]), kk
    # async: all S steps in flight through the two staging slots, distinct host outputs
    outs = [outputs(torch, B, k, L, "cpu") for _ in range(S)]
    for rep in range(2):
        for s in range(S):
            eng.step_host_async(B, H.StepBuffers(**h_in[s], **outs[s]), vp)
        eng.sync()
        for s in range(S):
            for kk in outs[s]:
                assert torch.equal(outs[s][kk], ref[s][kk]), (rep, s, kk)


def test_graph_replay_matches_eager(torch):
    """hsd_step_graph: the captured round replays to the eager results (B = 1, config-1 shape)."""
    n, dim, B, k, L, d_f = 10000, 4096, 1, 8, 7, 4096
    col = H.Collection(dim, capacity=n)
    col.generate(H.REAL, 5, n)
    col.set_filter("bf16_copy")
    eng = H.Engine(col, B, k, L, d_f, 15)
    vp = H.VerifyParams.make(skip_enabled=True, min_S=0.95, O_dist=5)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ins = [make_inputs(torch, col, n, dim, B, L, d_f, s) for s in range(3)]
        ref, got = [], []
        for s in range(3):
            o = outputs(torch, B, k, L, "cuda")
            eng.step(B, H.StepBuffers(**ins[s], **o), vp, stream=st)
            st.synchronize()
            ref.append({kk: v.clone() for kk, v in o.items()})
        bufs = [(outputs(torch, B, k, L, "cuda")) for _ in range(3)]
        for rep in range(3):  # miss (eager + capture), then replays
            for s in range(3):
                for v in bufs[s].values():
                    v.zero_()
                eng.step(B, H.StepBuffers(**ins[s], **bufs[s]), vp, stream=st, graph=True)
            st.synchronize()
            for s in range(3):
                for kk in bufs[s]:
                    assert torch.equal(bufs[s][kk], ref[s][kk]), (rep, s, kk)


@pytest.mark.parametrize("B", [1, 3, 48, 200])
def test_cohorts_on_two_streams_match_serial_steps(torch, B):
    """Two engines over one collection, each on its own stream, their steps
    interleaved with no synchronisation between them (the bench's cohort
    pipelining; B = 200 runs the CTA-pair filter, B <= 4 the exact scan with
    K4 launched under it): every step's outputs equal the same step run alone."""
    n, dim, k, L, d_f = 20000, 256, 8, 7, 256
    col = H.Collection(dim, capacity=n)
    col.generate(H.REAL, 5, n)
    vp = H.VerifyParams.make(skip_enabled=True, min_S=0.95, O_dist=5)
    S = 6
    ins = [make_inputs(torch, col, n, dim, B, L, d_f, s) for s in range(S)]
    solo = H.Engine(col, B, k, L, d_f, 15)
    ref = []
    for s in range(S):
        o = outputs(torch, B, k, L, "cuda")
        solo.step(B, H.StepBuffers(**ins[s], **o), vp)
        torch.cuda.synchronize()
        ref.append({kk: v.cpu() for kk, v in o.items()})
    engs = [H.Engine(col, B, k, L, d_f, 15) for _ in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [outputs(torch, B, k, L, "cuda") for _ in range(S)]
    for rep in range(3):  # repeat: the interleaving differs run to run
        for s in range(S):
            engs[s % 2].step(B, H.StepBuffers(**ins[s], **outs[s]), vp, stream=streams[s % 2])
        torch.cuda.synchronize()
        for s in range(S):
            for kk in outs[s]:
                assert torch.equal(outs[s][kk].cpu(), ref[s][kk]), (rep, s, kk)


def test_graphs_alternating_batch_and_params(torch):
    """Cached graphs keep their own parameters and the engine's fixed scratch:
    graphs captured for (B = 8, strict), (B = 160, relaxed + skip) and
    (B = 40, tight caps) replayed in alternation equal the eager steps (a
    larger B used to reallocate the scratch an older graph still pointed at,
    and every graph read the last parameters copied)."""
    n, dim, k, L, d_f = 30000, 256, 8, 7, 256
    col = H.Collection(dim, capacity=n)
    col.generate(H.REAL, 5, n)
    col.set_filter("bf16_copy")
    eng = H.Engine(col, 160, k, L, d_f, 15)
    cases = [(8, H.VerifyParams.make(relaxed=False)),
             (160, H.VerifyParams.make(skip_enabled=True, min_S=0.9, O_dist=5)),
             (40, H.VerifyParams.make(bias_seq_max=4, bias_token_max=2))]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ins = [make_inputs(torch, col, n, dim, B, L, d_f, i) for i, (B, _) in enumerate(cases)]
        ref = []
        for i, (B, vp) in enumerate(cases):
            o = outputs(torch, B, k, L, "cuda")
            eng.step(B, H.StepBuffers(**ins[i], **o), vp, stream=st)
            st.synchronize()
            ref.append({kk: v.clone() for kk, v in o.items()})
        bufs = [outputs(torch, B, k, L, "cuda") for B, _ in cases]
        for rep in range(4):
            order = [0, 1, 2] if rep % 2 == 0 else [2, 0, 1]
            for i in order:
                B, vp = cases[i]
                for v in bufs[i].values():
                    v.zero_()
                eng.step(B, H.StepBuffers(**ins[i], **bufs[i]), vp, stream=st, graph=True)
                # an eager step in between with other parameters must not leak into the graphs
                eng.step(B, H.StepBuffers(**ins[i], **outputs(torch, B, k, L, "cuda")),
                         H.VerifyParams.make(relaxed=True, bias_seq_max=0, bias_token_max=0), stream=st)
            st.synchronize()
            for i in range(3):
                for kk in bufs[i]:
                    assert torch.equal(bufs[i][kk], ref[i][kk]), (rep, i, kk)


def test_multi_pass_batch_scratch(torch):
    """B = 1280 over 24k rows: two passes with different filter-list counts
    (1024-query clusters, then a 256-query pair pass) share one scratch."""
    from oracle import oracle as O
    n, dim = 24_000, 64
    col = H.Collection(dim, capacity=n)
    col.generate(O.REAL, 3, n)
    for B in (1280, 1100, 2100):
        q = H.gen_queries(O.REAL, 4, 3, n, 0, B, dim)
        sc, ids = col.search_topk_exact(q, 8)
        osc, oid = O.search_synth(O.REAL, 3, n, q.cpu().numpy(), 8, threads=0)
        np.testing.assert_array_equal(ids.cpu().numpy(), oid)
        np.testing.assert_array_equal(sc.cpu().numpy(), osc)
