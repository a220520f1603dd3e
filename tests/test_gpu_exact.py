"""Exactness is unconditional (k_select.cu): whatever the DB holds, the top-k
equals the reference's search_topk_exact (store.cpp:59-73) bit for bit.

* CLUSTER family (hsd_synth.h): runs of 64-512 consecutive near-duplicate or
  identical rows, the layout of a demonstration DB.
  A query near a run has hundreds of rows inside the filter's error window, so
  a filter list cannot bound its rows and the exact range fallback rescans it.
* Forced pool overflow: more than 256 candidates spread over every list.
* Every kernel variant: 1-CTA (B <= 128), CTA pairs (129..1024 queries,
  stride-2 lists), multicast clusters, the single-CTA ablation, range searches.
"""
import numpy as np
import pytest

import paper_2603_17573_b200 as H
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


@pytest.fixture(autouse=True)
def filter_path():
    """This module covers the filter + rescoring path's exactness machinery (the
    candidate margin and the range fallback): small batches would otherwise take
    the exact scan (tests/test_gpu_scan.py covers that path on these families)."""
    H.set_sim_path("filter")
    yield
    H.set_sim_path("auto")


def check(col, kind, seed, n, q, k, row_range=None):
    sc, ids = col.search_topk_exact(q, k, row_range=row_range)
    if row_range is None:
        osc, oid = O.search_synth(kind, seed, n, q.cpu().numpy(), k, threads=0)
    else:
        keys = O.gen_keys(kind, seed, row_range[0], row_range[1] - row_range[0], col.dim())
        osc, oid = O.search_topk(keys, q.cpu().numpy(), k)
        oid = oid + row_range[0]
    kk = oid.shape[1]
    np.testing.assert_array_equal(ids.cpu().numpy()[:, :kk], oid)
    np.testing.assert_array_equal(sc.cpu().numpy()[:, :kk], osc)
    assert np.all(ids.cpu().numpy()[:, kk:] == -1)


def test_cluster_generator_matches_host(torch):
    n, dim = 3000, 64
    for dtype, kk in (("f32", O.CLUSTER), ("bf16", O.CLUSTER | O.KEYS_BF16)):
        col = H.Collection(dim, capacity=n, dtype=dtype)
        col.generate(O.CLUSTER, 13, n)
        keys, _ = col.keys_view()
        np.testing.assert_array_equal(keys.float().cpu().numpy(), O.gen_keys(kk, 13, 0, n, dim))
    q = H.gen_queries(O.CLUSTER, 14, 13, n, 0, 50, dim)
    np.testing.assert_array_equal(q.cpu().numpy(), O.gen_queries(O.CLUSTER, 14, 13, n, 0, 50, dim))
    k64 = O.gen_keys(O.CLUSTER, 13, 0, 1024, dim).astype(np.float64)
    cos = k64[1:] @ k64[:-1].T
    assert np.diag(cos).max() > 0.9999  # runs: consecutive rows nearly (or exactly) parallel


@pytest.mark.parametrize("filt", ["native", "bf16_copy", "bf16"])
@pytest.mark.parametrize("B", [1, 64, 256, 1024])
def test_cluster_family_bit_exact(torch, B, filt):
    n, dim = (40_000, 256) if B < 1024 else (20_000, 128)
    dtype = "bf16" if filt == "bf16" else "f32"
    col = H.Collection(dim, capacity=n, dtype=dtype)
    col.generate(O.CLUSTER, 51, n)
    if filt == "bf16_copy":
        col.set_filter("bf16_copy")
    kind = O.CLUSTER | (O.KEYS_BF16 if dtype == "bf16" else 0)
    q = H.gen_queries(O.CLUSTER, 52, 51, n, 0, B, dim)
    col.search_stats(reset=True)
    check(col, kind, 51, n, q, 8)
    st = col.search_stats()
    if B >= 64:  # near-duplicate queries of run rows exercise the range fallback
        assert st["fallback_queries"] >= 1, st


@pytest.mark.parametrize("B", [3, 64, 200])
def test_cluster_dim4096_and_ranges(torch, B):
    n, dim = 6000, 4096
    col = H.Collection(dim, capacity=n)
    col.generate(O.CLUSTER, 61, n)
    col.set_filter("bf16_copy")
    q = H.gen_queries(O.CLUSTER, 62, 61, n, 0, B, dim)
    col.search_stats(reset=True)
    check(col, O.CLUSTER, 61, n, q, 8)
    check(col, O.CLUSTER, 61, n, q, 32)
    assert col.search_stats()["fallback_queries"] >= 1
    for rg in ((100, 1900), (513, 515), (4000, 6000)):
        check(col, O.CLUSTER, 61, n, q, 5, row_range=rg)


@pytest.mark.parametrize("path", ["auto", "tc_single"])
def test_cluster_all_pass_widths(torch, path):
    H.set_sim_path("filter" if path == "auto" else path)
    try:
        n, dim = 12_000, 64
        col = H.Collection(dim, capacity=n)
        col.generate(O.CLUSTER, 71, n)
        for B in (129, 300, 513, 1100):
            q = H.gen_queries(O.CLUSTER, 72, 71, n, 0, B, dim)
            check(col, O.CLUSTER, 71, n, q, 8)
    finally:
        H.set_sim_path("auto")


def test_forced_pool_overflow_all_lists(torch):
    """20 copies of the best row in every filter list: > 256 candidates, none
    of the lists exhausted -> every list with a candidate is rescanned."""
    rng = np.random.default_rng(5)
    dim, nsm_rows = 64, 148 * 128 * 2
    emb = rng.standard_normal((nsm_rows, dim)).astype(np.float32) * 0.1
    q = rng.standard_normal((4, dim)).astype(np.float32)
    best = q[0] / np.linalg.norm(q[0])
    per = nsm_rows // 148
    for lst in range(148):
        for j in range(20):
            emb[lst * per + 7 * j] = best
    col = H.Collection(dim, capacity=nsm_rows)
    col.insert(emb, np.zeros((nsm_rows, 3, 7)))
    qd = torch.as_tensor(q, device="cuda")
    col.search_stats(reset=True)
    for k in (1, 8, 32):
        sc, ids = col.search_topk_exact(qd, k)
        osc, oid = O.search_topk(emb, q, k)
        np.testing.assert_array_equal(ids.cpu().numpy(), oid)
        np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    st = col.search_stats()
    assert st["fallback_queries"] >= 3 and st["fallback_lists"] >= 3 * 100, st


def test_identical_rows_everywhere(torch):
    """A DB of one repeated row: every list is exhausted; the answer is ids 0..k-1."""
    dim, n = 128, 50_000
    row = np.random.default_rng(1).standard_normal(dim).astype(np.float32)
    col = H.Collection(dim, capacity=n)
    col.insert(np.tile(row, (n, 1)), np.zeros((n, 3, 7)))
    q = torch.as_tensor(np.stack([row, -row, row * 0.5]), device="cuda")
    sc, ids = col.search_topk_exact(q, 16)
    np.testing.assert_array_equal(ids.cpu().numpy(), np.tile(np.arange(16), (3, 1)))
    osc, _ = O.search_topk(np.tile(row, (16, 1)), q.cpu().numpy(), 16)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)
