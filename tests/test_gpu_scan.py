"""K1x exact scan (k_exact.cu): every row's fp64 chain in the reference's order
(store.cpp:29-34) + the (score desc, id asc) top-k (store.cpp:59-73), for
small rows x batch.  Bit-exact ids and scores vs the oracle on every family
(EXACT: heavy exact ties and duplicate rows; CLUSTER: runs of near-duplicate
and identical rows), fp32 and bf16 keys, B = 1..4, k = 1..32, ragged dims,
one-tile and multi-tile (persistent) grids, row ranges, fewer rows than k,
and the auto path choice; the forced filter path returns the same bits."""
import numpy as np
import pytest

import paper_2603_17573_b200 as H
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture
def scan_path():
    H.set_sim_path("scan")
    yield
    H.set_sim_path("auto")


def check(col, kind, seed, n, q, k, row_range=None):
    sc, ids = col.search_topk_exact(q, k, row_range=row_range)
    if row_range is None:
        osc, oid = O.search_synth(kind, seed, n, q.cpu().numpy(), k, threads=0)
    else:
        keys = O.gen_keys(kind, seed, row_range[0], row_range[1] - row_range[0], col.dim())
        osc, oid = O.search_topk(keys, q.cpu().numpy(), k)
        oid = np.where(oid >= 0, oid + row_range[0], -1)
    kk = oid.shape[1]
    np.testing.assert_array_equal(ids.cpu().numpy()[:, :kk], oid)
    np.testing.assert_array_equal(sc.cpu().numpy()[:, :kk], osc)
    assert np.all(ids.cpu().numpy()[:, kk:] == -1)
    return sc, ids


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("kind", [O.REAL, O.EXACT, O.CLUSTER])
@pytest.mark.parametrize("B", [1, 2, 3, 4])
def test_scan_bit_exact(scan_path, dtype, kind, B):
    n, dim = 5000, 256
    col = H.Collection(dim, capacity=n, dtype=dtype)
    col.generate(kind, 71, n)
    q = H.gen_queries(kind, 72 + B, 71, n, 0, B, dim)
    okind = kind | (O.KEYS_BF16 if dtype == "bf16" else 0)
    for k in (1, 8, 32):
        check(col, okind, 71, n, q, k)


@pytest.mark.parametrize("n, dim", [(10_000, 4096), (40_000, 512), (3, 64), (147, 96), (1, 4), (20_000, 100)])
def test_scan_shapes(scan_path, n, dim):
    """C1's shape; multi-tile persistent grids (40k rows > 148 x 128); fewer rows than k; dim not a multiple
    of the 32-column chunk (zero-padded query tail)."""
    col = H.Collection(dim, capacity=n)
    col.generate(O.REAL, 81, n)
    for B in (1, 4):
        q = H.gen_queries(O.REAL, 82 + B, 81, n, 0, B, dim)
        check(col, O.REAL, 81, n, q, 8)


def test_scan_ranges_and_insert_growth(scan_path):
    n, dim = 9000, 128
    col = H.Collection(dim, capacity=1000)  # grows through the inserts
    col.generate(O.EXACT, 91, n)
    q = H.gen_queries(O.EXACT, 92, 91, n, 0, 3, dim)
    for rr in [(0, n), (17, 4099), (8990, 9000), (5000, 5001)]:
        check(col, O.EXACT, 91, n, q, 8, row_range=rr)


def test_auto_choice_equals_filter_path():
    """Auto picks the exact scan at config 1's shape; the filter + rescoring path gives the same bits."""
    n, dim = 10_000, 4096
    col = H.Collection(dim, capacity=n)
    col.generate(O.REAL, 7, n)
    col.set_filter("bf16_copy")
    q = H.gen_queries(O.REAL, 8, 7, n, 0, 1, dim)
    col.search_stats(reset=True)
    s1, i1 = check(col, O.REAL, 7, n, q, 8)
    st = col.search_stats()
    assert st["candidates"] == 0, st  # no filter candidates: the scan ran
    H.set_sim_path("filter")
    try:
        s2, i2 = col.search_topk_exact(q, 8)
        assert col.search_stats()["candidates"] > 0
    finally:
        H.set_sim_path("auto")
    np.testing.assert_array_equal(i1.cpu().numpy(), i2.cpu().numpy())
    np.testing.assert_array_equal(s1.cpu().numpy(), s2.cpu().numpy())


def test_scan_repeated_launches_and_streams(scan_path):
    """The last-CTA ticket resets itself: many launches, two streams with their own scratch."""
    import torch

    n, dim = 7000, 256
    col = H.Collection(dim, capacity=n)
    col.generate(O.REAL, 101, n)
    qs = [H.gen_queries(O.REAL, 200 + i, 101, n, 0, 1 + i % 4, dim) for i in range(12)]
    ref = [O.search_synth(O.REAL, 101, n, q.cpu().numpy(), 8, threads=0) for q in qs]
    s2 = torch.cuda.Stream()
    for rep in range(3):
        for i, q in enumerate(qs):
            st = s2 if i % 2 else torch.cuda.current_stream()
            with torch.cuda.stream(st):
                sc, ids = col.search_topk_exact(q, 8)
            st.synchronize()
            np.testing.assert_array_equal(ids.cpu().numpy(), ref[i][1])
            np.testing.assert_array_equal(sc.cpu().numpy(), ref[i][0])


def _edge_keys(rng, n, dim):
    keys = rng.standard_normal((n, dim)).astype(np.float32)
    keys[1, :] = 0.0
    keys[2, :] = -0.0
    keys[3, ::3] = np.float32(1e-40)  # fp32 subnormals
    keys[4, ::5] = np.float32(-3e-45)
    keys[5, :7] = np.float32(3.0e38)  # near FLT_MAX
    keys[6, :] = keys[9, :]  # exact duplicate rows: the id decides
    keys[10:20, :] *= np.float32(1e-30)
    return keys


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_scan_widening_edge_values(scan_path, dtype):
    """Zeros, fp32 subnormals, values near FLT_MAX in keys and queries: the same bits as the reference's
    (double)a * (double)b chain."""
    rng = np.random.default_rng(5)
    n, dim = 300, 64
    keys = _edge_keys(rng, n, dim)
    col = H.Collection(dim, capacity=n, dtype=dtype)
    col.insert(keys, np.zeros((n, 21)))
    stored = col.keys_view()[0].float().cpu().numpy()
    q = rng.standard_normal((4, dim)).astype(np.float32)
    q[1, ::2] = np.float32(1e-42)
    q[2, :3] = np.float32(-2.5e38)
    q[3, :] = 0.0
    import torch

    qt = torch.as_tensor(q, device="cuda")
    for B in (1, 2, 3, 4):
        sc, ids = col.search_topk_exact(qt[:B], 16)
        osc, oid = O.search_topk(stored, q[:B], 16)
        np.testing.assert_array_equal(ids.cpu().numpy(), oid)
        np.testing.assert_array_equal(sc.cpu().numpy(), osc)


def test_scan_nonfinite_keys(scan_path):
    """A key holding +-inf: scores are +-inf as in the reference."""
    rng = np.random.default_rng(6)
    n, dim = 200, 32
    keys = rng.standard_normal((n, dim)).astype(np.float32)
    keys[5, 0] = np.inf
    keys[7, 0] = -np.inf
    col = H.Collection(dim, capacity=n)
    col.insert(keys, np.zeros((n, 21)))
    q = np.abs(rng.standard_normal((2, dim))).astype(np.float32) + 0.1
    import torch

    sc, ids = col.search_topk_exact(torch.as_tensor(q, device="cuda"), 8)
    osc, oid = O.search_topk(keys, q, 8)
    np.testing.assert_array_equal(ids.cpu().numpy(), oid)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    assert ids[0, 0].item() == 5 and sc[0, 0].item() == np.inf
