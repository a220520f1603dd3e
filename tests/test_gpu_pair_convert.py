"""CTA-pair filter over fp32 keys with on-chip bf16 conversion (k_sim_wide.cu,
sim_pair_kernel<false, G, true>; passes of 129..1024 queries over an fp32
collection without the bf16 filter copy; above 256 queries clusters of G
pairs share multicast raw key tiles).

The converter warps round every fp32 key to bf16 RN-even — the rounding the
bf16 filter copy stores — and the queries go through the same bf16 slab, so
the kind::f16 MMAs see the copy path's operands in the same order: the filter
scores, hence the rescored candidate sets, equal the copy path's.  That is
what ties this kernel to the copy path's bound (sim_wide_gamma with the copy
flag, tested on rounding-adversarial inputs in test_gpu_tc.py).  Results are
checked bit-exact against the oracle (ids and fp64 score bits)."""
import numpy as np
import pytest

import paper_2603_17573_b200 as H
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


def _run(col, q, k):
    col.search_stats(reset=True)
    sc, ids = col.search_topk_exact(q, k)
    return sc, ids, col.search_stats(reset=True)


@pytest.mark.parametrize("kind", [O.EXACT, O.REAL, O.CLUSTER])
@pytest.mark.parametrize("dim,n,B", [(64, 6000, 256), (4096, 2500, 200), (100, 3000, 129), (4352, 1500, 160),
                                     (136, 4000, 250), (256, 5000, 300), (4096, 1200, 513), (64, 9000, 700),
                                     (512, 3000, 1024)])
def test_converted_pair_matches_oracle_and_copy_path(torch, kind, dim, n, B):
    col = H.Collection(dim, capacity=n)
    col.generate(kind, 11, n)
    q = H.gen_queries(kind, 12, 11, n, 0, B, dim)
    osc, oid = O.search_synth(kind, 11, n, q.cpu().numpy(), 8)
    sc, ids, st_conv = _run(col, q, 8)  # native fp32 collection: on-chip conversion
    np.testing.assert_array_equal(ids.cpu().numpy(), oid)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    if dim % 8:  # no bf16 slab / copy for these rows (16-B TMA stride): the TF32 pair kernel ran
        return
    col.set_filter("bf16_copy")
    sc2, ids2, st_copy = _run(col, q, 8)
    assert torch.equal(ids, ids2) and torch.equal(sc, sc2)
    assert st_conv == st_copy, (st_conv, st_copy)  # identical filter scores -> identical candidate sets


def test_converted_pair_midpoint_adversarial(torch):
    """Keys and queries at bf16 rounding midpoints (every product rounded the
    same way, ~2^-7 relative): exact results, and the same candidates as the
    bf16 copy whose scores test_gpu_tc.py bounds on these inputs."""
    rng = np.random.default_rng(3)
    n, dim, B = 2000, 512, 200
    mant = np.float32(1.0 + 2.0**-8 - 2.0**-20)
    keys = (mant * np.float32(2.0) ** (-5 - rng.integers(0, 3, size=(n, dim))).astype(np.float32)
            * np.where(rng.random((n, dim)) < 0.5, -1, 1)).astype(np.float32)
    q = (mant * np.float32(2.0) ** (-5 - rng.integers(0, 3, size=(B, dim))).astype(np.float32)
         * np.where(rng.random((B, dim)) < 0.5, -1, 1)).astype(np.float32)
    q[: B // 2] = np.abs(q[: B // 2]) * np.sign(keys[: B // 2])  # half the queries: all products > 0 with row b
    col = H.Collection(dim, capacity=n)
    col.insert(keys, np.zeros((n, 3, 7)))
    qd = torch.as_tensor(q, device="cuda")
    sc, ids, st_conv = _run(col, qd, 8)
    osc, oid = O.search_topk(keys, q, 8)
    np.testing.assert_array_equal(ids.cpu().numpy(), oid)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    col.set_filter("bf16_copy")
    _, _, st_copy = _run(col, qd, 8)
    assert st_conv == st_copy, (st_conv, st_copy)


def test_converted_pair_ragged_ranges(torch):
    """Range searches whose ends split key blocks and block pairs."""
    n, dim, B = 5000, 256, 180
    col = H.Collection(dim, capacity=n)
    col.generate(O.REAL, 21, n)
    q = H.gen_queries(O.REAL, 22, 21, n, 0, B, dim)
    keys = O.gen_keys(O.REAL, 21, 0, n, dim)
    for rb, re in ((0, 1), (3, 130), (127, 385), (1000, 4999), (0, n)):
        sc, ids = col.search_topk_exact(q, 8, row_range=(rb, re))
        osc, oid = O.search_topk(keys[rb:re], q.cpu().numpy(), 8)
        kk = oid.shape[1]
        np.testing.assert_array_equal(ids[:, :kk].cpu().numpy(), oid + rb, err_msg=f"{rb}:{re}")
        np.testing.assert_array_equal(sc[:, :kk].cpu().numpy(), osc, err_msg=f"{rb}:{re}")


def test_search_plan_reports_the_conversion(torch):
    col = H.Collection(256, capacity=5000)
    col.generate(O.REAL, 1, 5000)
    assert col.search_plan(200, 8) == "filter_bf16_onchip"
    assert col.search_plan(100, 8) == "filter"  # one CTA per key range: TF32
    assert col.search_plan(700, 8) == "filter_bf16_onchip"  # clusters of 3 pairs
    col.set_filter("bf16_copy")
    assert col.search_plan(200, 8) == "filter"  # the copy is streamed instead
    odd = H.Collection(100, capacity=3000)
    odd.generate(O.REAL, 1, 3000)
    assert odd.search_plan(200, 8) == "filter"  # dim % 8: no bf16 slab, TF32 pair kernel
