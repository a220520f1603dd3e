"""GPU parity of the retrieval path (K0 synth, K1 similarity, K2 select)
against the CPU oracle and the reference fixtures: ids AND fp64 scores
bit-exact (ties broken by id as in store.cpp:67-70)."""
import os

import numpy as np
import pytest

import paper_2603_17573_b200 as H
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


def make_db(kind, seed, n, dim):
    col = H.Collection(dim, capacity=n)
    col.generate(kind, seed, n)
    return col


def test_device_generator_matches_host(torch):
    for kind in (O.EXACT, O.REAL):
        col = make_db(kind, 7, 3000, 64)
        keys, toks = col.keys_view()
        np.testing.assert_array_equal(keys.cpu().numpy(), O.gen_keys(kind, 7, 0, 3000, 64))
        np.testing.assert_array_equal(toks[:, :21].cpu().numpy(), O.synth_tokens(7, np.arange(3000)))
        assert (toks[:, 21:] == 0).all()
        q = H.gen_queries(kind, 9, 7, 3000, 5, 40, 64)
        np.testing.assert_array_equal(q.cpu().numpy(), O.gen_queries(kind, 9, 7, 3000, 5, 40, 64))
    now, prev = H.gen_features(5, 16, 4096)
    hn, hp = O.gen_features(5, 0, 16, 4096)
    np.testing.assert_array_equal(now.cpu().numpy(), hn)
    np.testing.assert_array_equal(prev.cpu().numpy(), hp)
    col = make_db(O.REAL, 11, 500, 64)
    rows = np.array([5, -1, 499, 0, 17])
    lg = H.gen_logits(col, 3, rows, 21)
    np.testing.assert_array_equal(lg.cpu().numpy(), O.gen_logits(11, 3, rows, 0, 21))


@pytest.mark.parametrize("name", ["search_exact_64", "search_real_64", "search_exact_4096", "search_real_4096"])
def test_search_matches_reference_fixture(torch, name):
    z = np.load(os.path.join(GOLD, name + ".npz"))
    kind, n, dim, B, k = int(z["kind"]), int(z["n"]), int(z["dim"]), int(z["B"]), int(z["k"])
    col = make_db(kind, int(z["db_seed"]), n, dim)
    q = H.gen_queries(kind, int(z["q_seed"]), int(z["db_seed"]), n, 0, B, dim)
    sc, ids = col.search_topk_exact(q, k)
    np.testing.assert_array_equal(ids.cpu().numpy(), z["ids"])
    np.testing.assert_array_equal(sc.cpu().numpy(), z["scores"])
    assert col.overflow_count() == 0


@pytest.mark.parametrize("path", ["auto", "filter"])
@pytest.mark.parametrize("kind", [O.EXACT, O.REAL])
@pytest.mark.parametrize("B", [1, 2, 3, 5, 8, 9, 24, 64, 100])
@pytest.mark.parametrize("dim", [64, 4096])
def test_search_parity_vs_oracle(torch, kind, B, dim, path):
    """auto: the exact scan for small rows x batch (B <= 4), else the filter; filter: K1 + K2 always."""
    if path == "filter" and B > 4:
        pytest.skip("auto already takes the filter path")
    n = 20_000 if dim == 64 else 6000
    col = make_db(kind, 100 + B, n, dim)
    q = H.gen_queries(kind, 200 + B, 100 + B, n, 0, B, dim)
    H.set_sim_path(path)
    try:
        for k in (1, 8, 32):
            sc, ids = col.search_topk_exact(q, k)
            osc, oid = O.search_synth(kind, 100 + B, n, q.cpu().numpy(), k, threads=0)
            np.testing.assert_array_equal(ids.cpu().numpy(), oid)
            np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    finally:
        H.set_sim_path("auto")
    assert col.overflow_count() == 0


def test_search_edge_cases(torch):
    col = H.Collection(64, capacity=16)
    q = H.gen_queries(O.REAL, 1, 1, 10, 0, 3, 64)
    sc, ids = col.search_topk_exact(q, 5)  # empty collection -> empty result, no error
    assert (ids == -1).all() and torch.isinf(sc).all()
    col.generate(O.REAL, 1, 10)
    sc, ids = col.search_topk_exact(q, 32)  # k > N -> N hits (store.cpp:71)
    osc, oid = O.search_synth(O.REAL, 1, 10, q.cpu().numpy(), 32)
    np.testing.assert_array_equal(ids[:, :10].cpu().numpy(), oid)
    assert (ids[:, 10:] == -1).all()
    with pytest.raises(H.InvalidInputError):
        col.search_topk_exact(q, 0)  # store.cpp:60
    sc, ids = col.search_topk_exact(q, 33)  # k > HSD_K_MAX: the large-k path, same contract
    np.testing.assert_array_equal(ids[:, :10].cpu().numpy(), oid)
    np.testing.assert_array_equal(sc[:, :10].cpu().numpy(), osc)
    assert (ids[:, 10:] == -1).all() and torch.isinf(sc[:, 10:]).all()
    with pytest.raises(H.InvalidInputError):
        col.search_topk_exact(torch.zeros((2, 32), device="cuda"), 3)  # dim mismatch (store.cpp:30)
    misaligned = torch.zeros(3 * 64 + 1, device="cuda")[1:].view(3, 64)  # 4-byte offset view
    with pytest.raises(H.InvalidInputError):
        col.search_topk_exact(misaligned, 3)


def test_range_search_is_a_task_shard(torch):
    col = make_db(O.EXACT, 3, 9000, 64)
    q = H.gen_queries(O.EXACT, 4, 3, 9000, 0, 16, 64)
    sc, ids = col.search_topk_exact(q, 8, row_range=(3000, 6500))
    keys = O.gen_keys(O.EXACT, 3, 3000, 3500, 64)
    osc, oid = O.search_topk(keys, q.cpu().numpy(), 8)
    np.testing.assert_array_equal(ids.cpu().numpy(), oid + 3000)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)


def test_insert_path_quantizes_like_reference(torch):
    rng = np.random.default_rng(0)
    n, dim = 2000, 64
    emb = rng.standard_normal((n, dim)).astype(np.float32)
    acts = rng.uniform(-1.3, 1.3, (n, 21))
    col = H.Collection(dim, capacity=8)  # forces growth
    assert col.insert(emb[:700], acts[:700]) == 0
    assert col.insert(emb[700:], acts[700:]) == 700
    assert col.size() == n
    _, toks = col.keys_view()
    want = np.array([[O.quantize(a[s * 7:(s + 1) * 7])[1] for s in range(3)] for a in acts]).reshape(n, 21)
    np.testing.assert_array_equal(toks[:, :21].cpu().numpy(), want)
    q = torch.as_tensor(emb[[5, 77, 1999]], device="cuda")
    sc, ids = col.search_topk_exact(q, 4)
    osc, oid = O.search_topk(emb, emb[[5, 77, 1999]], 4)
    np.testing.assert_array_equal(ids.cpu().numpy(), oid)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    with pytest.raises(H.SchemaError):
        col.insert(emb[:1], acts[:1], episode_idx=[-1])  # store.cpp:50-52
    bad = acts[:1].copy()
    bad[0, 3] = np.nan
    with pytest.raises(H.InvalidInputError):
        col.insert(emb[:1], bad)  # actions.cpp:38-40
    assert col.size() == n


def test_device_quantize_bit_exact(torch):
    z = np.load(os.path.join(GOLD, "quantize.npz"))
    a = torch.as_tensor(z["acts"], device="cuda")
    np.testing.assert_array_equal(H.quantize(a).cpu().numpy(), z["bins"])
    np.testing.assert_array_equal(H.quantize(a, z["lo2"], z["hi2"]).cpu().numpy(), z["bins2"])
    with pytest.raises(H.ConfigError):
        H.quantize(a, 1.0, 1.0)


@pytest.mark.slow
def test_full_size_c2_sampled(torch):
    """BASELINE config 2 size (1M x 4096, B = 64): the oracle streams the
    counter-generated DB and checks a sample of 8 queries bit-exactly."""
    n, dim, B = 1_000_000, 4096, 64
    col = make_db(O.REAL, 2026, n, dim)
    q = H.gen_queries(O.REAL, 7, 2026, n, 0, B, dim)
    sc, ids = col.search_topk_exact(q, 8)
    assert col.overflow_count() == 0
    sel = [0, 1, 2, 3, 17, 31, 48, 63]
    osc, oid = O.search_synth(O.REAL, 2026, n, q.cpu().numpy()[sel], 8, threads=0)
    np.testing.assert_array_equal(ids.cpu().numpy()[sel], oid)
    np.testing.assert_array_equal(sc.cpu().numpy()[sel], osc)
    # size-independent properties on all 64: sorted (score desc, id asc), near-dup queries find their source row
    s = sc.cpu().numpy()
    i = ids.cpu().numpy()
    assert np.all((s[:, :-1] > s[:, 1:]) | ((s[:, :-1] == s[:, 1:]) & (i[:, :-1] < i[:, 1:])))
    rows = H.query_rows(7, O.REAL, n, 0, B)
    hit = rows >= 0
    assert np.all(i[hit, 0] == rows[hit])
