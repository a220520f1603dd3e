"""Approximate device index (IVF-flat), the stand-in for
the reference's HNSW behind Collection::build_hnsw / search_topk
(store.cpp:75-92).

What is pinned bit for bit against the oracle:
  * the build: every record sits in the list of its best centroid by the
    reference's exact search (score desc, id asc), lists in ascending id
    order (perm / offs), centroids = normalized list means;
  * the search: the probed lists are the best nprobe centroids (up to fp32
    near-ties), and the result is the exact top-k over the probed lists' rows
    (ids and fp64 score bits) — returned scores are always the reference's
    cosine_similarity of the returned ids (store.cpp:86-90);
  * a stale index (rows inserted after the build) searches exactly, as the
    reference drops the index on insert.
Recall against search_topk_exact is measured, with floors.
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


def make_db(kind, seed, n, dim, dtype="f32"):
    col = H.Collection(dim, capacity=n, dtype=dtype)
    col.generate(kind, seed, n)
    return col


def recall(ids, ref_ids):
    hit = 0
    for a, b in zip(ids, ref_ids):
        hit += len(set(int(x) for x in a if x >= 0) & set(int(x) for x in b if x >= 0))
    return hit / max(1, sum(int((b >= 0).sum()) for b in ref_ids))


@pytest.mark.parametrize("kind,n,dim,nlist,n_iter", [(O.REAL, 6000, 128, 48, 4), (O.CLUSTER, 5000, 64, 40, 3),
                                                     (O.EXACT, 3000, 100, 17, 2), (O.REAL, 700, 64, 1, 1)])
def test_build_matches_oracle_definition(torch, kind, n, dim, nlist, n_iter):
    col = make_db(kind, 5, n, dim)
    idx = H.Index(col, nlist=nlist, n_iter=n_iter)
    inf = idx.info()
    assert inf["nlist"] == min(nlist, n) and inf["n_rows"] == n and not inf["stale"]
    offs, perm, cent = idx.lists()
    keys = O.gen_keys(kind, 5, 0, n, dim)
    # every record in the list of its exact best centroid; stable list order
    ref_assign = O.ivf_assign(keys, cent)
    roffs, rperm = O.ivf_lists(ref_assign, inf["nlist"])
    np.testing.assert_array_equal(offs, roffs)
    np.testing.assert_array_equal(perm, rperm)
    assert inf["max_list"] == int(np.diff(offs).max())
    # unit-norm centroids
    nr = np.linalg.norm(cent.astype(np.float64), axis=1)
    assert np.all(np.abs(nr[nr > 0] - 1.0) < 1e-5)


def test_build_seeds_and_one_iteration_match_oracle(torch):
    n, dim, nlist = 4000, 64, 32
    col = make_db(O.REAL, 9, n, dim)
    keys = O.gen_keys(O.REAL, 9, 0, n, dim)
    for n_iter in (0, 1, 3):
        cent_o, offs_o, perm_o = O.ivf_build(keys, nlist, n_iter)
        offs, perm, cent = H.Index(col, nlist=nlist, n_iter=n_iter).lists()
        np.testing.assert_allclose(cent, cent_o, rtol=0, atol=2e-7)
        np.testing.assert_array_equal(offs, offs_o)
        np.testing.assert_array_equal(perm, perm_o)


def test_build_is_deterministic(torch):
    col = make_db(O.CLUSTER, 3, 8000, 128)
    a = H.Index(col, nlist=64, n_iter=5).lists()
    b = H.Index(col, nlist=64, n_iter=5).lists()
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("B,nprobe", [(1, 4), (16, 8), (64, 3), (1100, 2)])
def test_search_is_exact_over_probed_lists(torch, dtype, B, nprobe):
    n, dim, nlist, k = 12000, 128, 64, 8
    col = make_db(O.REAL, 21, n, dim, dtype)
    idx = H.Index(col, nlist=nlist, n_iter=4)
    offs, perm, cent = idx.lists()
    q = H.gen_queries(O.REAL, 4, 21, n, 0, B, dim)
    sc, ids, probes = idx.search_topk(q, k, nprobe=nprobe, return_probes=True)
    sc, ids, probes = sc.cpu().numpy(), ids.cpu().numpy(), probes.cpu().numpy()
    keys = O.gen_keys(O.REAL | (O.KEYS_BF16 if dtype == "bf16" else 0), 21, 0, n, dim) if dtype == "bf16" \
        else O.gen_keys(O.REAL, 21, 0, n, dim)
    qn = q.cpu().numpy()
    # probes: the nprobe best centroids by the exact score, up to fp32 near-ties at the boundary
    cs = qn.astype(np.float64) @ cent.astype(np.float64).T
    for b in range(B):
        got = set(int(x) for x in probes[b])
        assert len(got) == nprobe
        order = np.argsort(-cs[b], kind="stable")
        want = set(int(x) for x in order[:nprobe])
        if got != want:
            edge = cs[b, order[nprobe - 1]]
            for l in got ^ want:
                assert abs(cs[b, l] - edge) < 1e-4, (b, l, cs[b, l], edge)
    # results: the exact top-k over the probed lists' rows
    rs, ri = O.ivf_search_lists(keys, offs, perm, probes, qn, k)
    np.testing.assert_array_equal(ids, ri)
    np.testing.assert_array_equal(sc, rs)


@pytest.mark.parametrize("nlist,nprobe,B", [(1, 1, 1100), (2, 2, 300), (3, 1, 1)])
def test_few_long_lists(torch, nlist, nprobe, B):
    # a handful of huge lists: units span many 32/128-row chunks (the per-pass unit cap)
    n, dim, k = 20000, 64, 8
    col = make_db(O.REAL, 31, n, dim)
    idx = H.Index(col, nlist=nlist, n_iter=1)
    offs, perm, cent = idx.lists()
    q = H.gen_queries(O.REAL, 2, 31, n, 0, B, dim)
    sc, ids, probes = idx.search_topk(q, k, nprobe=nprobe, return_probes=True)
    rs, ri = O.ivf_search_lists(O.gen_keys(O.REAL, 31, 0, n, dim), offs, perm, probes.cpu().numpy(),
                                q.cpu().numpy(), k)
    np.testing.assert_array_equal(ids.cpu().numpy(), ri)
    np.testing.assert_array_equal(sc.cpu().numpy(), rs)
    if nprobe == nlist:  # every list probed: the exact search
        es, ei = col.search_topk_exact(q, k)
        np.testing.assert_array_equal(ids.cpu().numpy(), ei.cpu().numpy())


def test_recall_and_full_probe(torch):
    n, dim, k = 20000, 256, 8
    col = make_db(O.REAL, 2, n, dim)
    idx = H.Index(col, nlist=32, n_iter=6)
    q = H.gen_queries(O.REAL, 7, 2, n, 0, 128, dim)
    es, ei = col.search_topk_exact(q, k)
    es, ei = es.cpu().numpy(), ei.cpu().numpy()
    r = {}
    for nprobe in (1, 4, 16, 32):
        s, i = idx.search_topk(q, k, nprobe=nprobe)
        r[nprobe] = recall(i.cpu().numpy(), ei)
    # more lists never hurt; every list probed = exhaustive over the bf16 candidates
    assert r[1] <= r[4] + 1e-9 <= r[16] + 2e-9 <= r[32] + 3e-9
    assert r[32] >= 0.999, r
    s, i = idx.search_topk(q, k, nprobe=32)
    same = (i.cpu().numpy() == ei).all(axis=1)
    np.testing.assert_array_equal(s.cpu().numpy()[same], es[same])


def similar_recall(ids, ref_ids, ref_scores, floor=0.5):
    """Recall over the exact top-k neighbours that are genuinely similar (score >= floor)."""
    hit = tot = 0
    for a, b, s in zip(ids, ref_ids, ref_scores):
        want = set(int(x) for x, v in zip(b, s) if x >= 0 and v >= floor)
        hit += len(want & set(int(x) for x in a))
        tot += len(want)
    return hit / max(1, tot), tot


@pytest.mark.parametrize("filt", ["native", "bf16_copy"])
def test_recall_on_trajectory_runs(torch, filt):
    # CLUSTER rows: runs of near-duplicate consecutive steps.
    # A query's similar neighbours (cosine >= 0.5: the steps of its run) share its
    # list; neighbours of pure-noise rows sit at cosine ~0.1 and are not retrievable
    # by any partition, so recall is measured over the similar ones.
    n, dim, k = 40000, 256, 8
    col = make_db(O.CLUSTER, 8, n, dim)
    if filt == "bf16_copy":
        col.set_filter("bf16_copy")
    idx = H.Index(col, nlist=64, n_iter=6)
    q = H.gen_queries(O.CLUSTER, 3, 8, n, 0, 256, dim)
    es, ei = col.search_topk_exact(q, k)
    s, i = idx.search_topk(q, k, nprobe=4)
    r, tot = similar_recall(i.cpu().numpy(), ei.cpu().numpy(), es.cpu().numpy())
    assert tot >= 300 and r >= 0.95, (r, tot)


def test_near_duplicate_queries_find_their_row(torch):
    # REAL queries q < B/2 are near-duplicates of a DB row (top-1 cosine ~0.95)
    n, dim = 30000, 256
    col = make_db(O.REAL, 12, n, dim)
    idx = H.Index(col, nlist=128, n_iter=5)
    B = 256
    q = H.gen_queries(O.REAL, 13, 12, n, 0, B, dim)
    rows = H.query_rows(13, O.REAL, n, 0, B)
    s, i = idx.search_topk(q, 8, nprobe=8)
    i = i.cpu().numpy()
    nd = [b for b in range(B) if rows[b] >= 0]
    found = np.mean([rows[b] in set(i[b]) for b in nd])
    assert found >= 0.95, found


def test_stale_index_searches_exactly(torch):
    n, dim = 3000, 64
    col = make_db(O.REAL, 4, n, dim)
    col.build_hnsw(nlist=16, n_iter=2, nprobe=1)
    assert col.has_hnsw()
    q = H.gen_queries(O.REAL, 5, 4, n, 0, 32, dim)
    s1, i1 = col.search_topk(q, 8)
    col.generate(O.REAL, 4, 500)  # insert after the build: the index is dropped (store.cpp:44-57)
    assert not col.has_hnsw()
    assert col._index.info()["stale"]
    s2, i2 = col.search_topk(q, 8)
    es, ei = col.search_topk_exact(q, 8)
    np.testing.assert_array_equal(i2.cpu().numpy(), ei.cpu().numpy())
    np.testing.assert_array_equal(s2.cpu().numpy(), es.cpu().numpy())
    # the index object itself also falls back once stale
    s3, i3 = col._index.search_topk(q, 8, nprobe=1)
    np.testing.assert_array_equal(i3.cpu().numpy(), ei.cpu().numpy())


def test_small_lists_pad_and_errors(torch):
    col = make_db(O.REAL, 6, 40, 64)
    idx = H.Index(col, nlist=100, n_iter=1)  # clamped to the row count: one record per list
    assert idx.info()["nlist"] == 40
    q = H.gen_queries(O.REAL, 1, 6, 40, 0, 3, 64)
    s, i = idx.search_topk(q, 8, nprobe=2)  # <= 2 records probed: the rest -1 / -inf
    i = i.cpu().numpy()
    s = s.cpu().numpy()
    assert ((i >= 0).sum(axis=1) <= 2).all() and ((i >= 0).sum(axis=1) >= 1).all()
    assert np.isneginf(s[i < 0]).all()
    with pytest.raises(H.InvalidInputError):
        idx.search_topk(q, 0, nprobe=2)
    with pytest.raises(H.InvalidInputError):
        idx.search_topk(q, 8, nprobe=0)
    with pytest.raises(H.InvalidInputError):
        idx.search_topk(q, 8, nprobe=33)
    empty = H.Collection(64, capacity=4)
    with pytest.raises(H.InvalidInputError, match="empty collection"):
        H.Index(empty, nlist=4)
    with pytest.raises(H.ConfigError):
        H.Index(col, nlist=0)


def test_destroy_order_leaves_no_error(torch):
    # a reference cycle (Collection <-> its build_hnsw index) is finalized in any
    # order by Python's GC: an index outliving its collection must destroy cleanly
    import ctypes as C
    col = make_db(O.REAL, 8, 500, 64)
    idx = H.Index(col, nlist=8, n_iter=1)
    L = H.lib()
    L.hsd_debug_last_cuda_error()
    assert L.hsd_collection_destroy(col.handle) == 0
    col._h = C.c_void_p()  # closed
    with pytest.raises(H.InvalidInputError, match="closed"):
        idx.search_topk(H.gen_queries(O.REAL, 1, 8, 500, 0, 2, 64), 4)
    idx.close()
    assert L.hsd_debug_last_cuda_error() == 0

