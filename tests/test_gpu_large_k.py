"""k > HSD_K_MAX (32): the large-k exact path (every row's fp64 chain from the
K1x scan, then a stable radix sort of (order key, row id) per query) against
the oracle restatement of store.cpp:59-73 — ids and fp64 score bits, ties by
id (EXACT has duplicate rows, CLUSTER runs of near-duplicates), k up to and
past the collection size."""
import numpy as np
import pytest

import paper_2603_17573_b200 as H
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


def _keys(col, torch):
    keys, _ = col.keys_view()
    return keys.to(torch.float32).cpu().numpy()


@pytest.mark.parametrize("kind", [O.EXACT, O.REAL, O.CLUSTER])
@pytest.mark.parametrize("B", [1, 3, 6])
def test_large_k_parity(torch, kind, B):
    n, dim = 3000, 64
    col = H.Collection(dim, capacity=n)
    col.generate(kind, 40 + B, n)
    q = H.gen_queries(kind, 50 + B, 40 + B, n, 0, B, dim)
    for k in (33, 257, n - 1, n, n + 5):
        sc, ids = col.search_topk_exact(q, k)
        osc, oid = O.search_synth(kind, 40 + B, n, q.cpu().numpy(), k)
        kk = min(k, n)
        np.testing.assert_array_equal(ids[:, :kk].cpu().numpy(), oid)
        np.testing.assert_array_equal(sc[:, :kk].cpu().numpy(), osc)
        assert (ids[:, kk:] == -1).all() and torch.isinf(sc[:, kk:]).all()


def test_large_k_prefix_equals_small_k(torch):
    """the first 32 of a k = 100 search are the k = 32 search (the filter path)."""
    n, dim = 20_000, 4096
    col = H.Collection(dim, capacity=n)
    col.generate(O.REAL, 5, n)
    q = H.gen_queries(O.REAL, 6, 5, n, 0, 8, dim)
    s32, i32 = col.search_topk_exact(q, 32)
    s100, i100 = col.search_topk_exact(q, 100)
    assert torch.equal(i100[:, :32], i32) and torch.equal(s100[:, :32], s32)
    osc, oid = O.search_synth(O.REAL, 5, n, q[:2].cpu().numpy(), 100, threads=0)
    np.testing.assert_array_equal(i100[:2].cpu().numpy(), oid)
    np.testing.assert_array_equal(s100[:2].cpu().numpy(), osc)


def test_large_k_bf16_and_range(torch):
    n, dim = 4000, 128
    col = H.Collection(dim, capacity=n, dtype="bf16")
    col.generate(O.CLUSTER, 8, n)
    q = H.gen_queries(O.CLUSTER, 9, 8, n, 0, 5, dim)
    keys = _keys(col, torch)
    sc, ids = col.search_topk_exact(q, 300)
    osc, oid = O.search_topk(keys, q.cpu().numpy(), 300)
    np.testing.assert_array_equal(ids.cpu().numpy(), oid)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    sc, ids = col.search_topk_exact(q, 1200, row_range=(700, 1500))  # 800 rows: 400 trailing -1
    osc, oid = O.search_topk(keys[700:1500], q.cpu().numpy(), 1200)
    np.testing.assert_array_equal(ids[:, :800].cpu().numpy(), oid + 700)
    np.testing.assert_array_equal(sc[:, :800].cpu().numpy(), osc)
    assert (ids[:, 800:] == -1).all()


def test_large_k_index_answers_exact(torch):
    n, dim = 5000, 64
    col = H.Collection(dim, capacity=n)
    col.generate(O.CLUSTER, 3, n)
    col.build_hnsw(nlist=64, n_iter=4, nprobe=2)
    q = H.gen_queries(O.CLUSTER, 4, 3, n, 0, 4, dim)
    sc, ids = col.search_topk(q, 64)
    esc, eid = col.search_topk_exact(q, 64)
    assert torch.equal(ids, eid) and torch.equal(sc, esc)


def test_large_k_empty_and_errors(torch):
    col = H.Collection(64, capacity=16)
    q = H.gen_queries(O.REAL, 1, 1, 10, 0, 2, 64)
    sc, ids = col.search_topk_exact(q, 1000)
    assert (ids == -1).all() and torch.isinf(sc).all()
    col.generate(O.REAL, 1, 10)
    with pytest.raises(H.InvalidInputError):
        col.search_topk_exact(q, 0)


def test_large_k_wide_rows_and_limit(torch):
    """Wide rows: the fp64 query slab of the scan bounds the dim (one query per pass near the
    limit); beyond it k > 32 is rejected with InvalidInput, k <= 32 still searches."""
    n, dim = 400, 16384
    col = H.Collection(dim, capacity=n)
    col.generate(O.REAL, 12, n)
    q = H.gen_queries(O.REAL, 13, 12, n, 0, 3, dim)
    sc, ids = col.search_topk_exact(q, 50)
    osc, oid = O.search_synth(O.REAL, 12, n, q.cpu().numpy(), 50)
    np.testing.assert_array_equal(ids.cpu().numpy(), oid)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    big = H.Collection(20480, capacity=64)
    big.generate(O.REAL, 14, 64)
    qb = H.gen_queries(O.REAL, 15, 14, 64, 0, 1, 20480)
    with pytest.raises(H.InvalidInputError):
        big.search_topk_exact(qb, 40)
    sc, ids = big.search_topk_exact(qb, 8)
    osc, oid = O.search_synth(O.REAL, 14, 64, qb.cpu().numpy(), 8)
    np.testing.assert_array_equal(ids.cpu().numpy(), oid)
