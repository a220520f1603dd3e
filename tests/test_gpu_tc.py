"""tcgen05 3xTF32 similarity kernel (K1'): its approximate filter scores stay
inside the error bound the exact rescoring relies on (k_sim_tc.cu,
sim_tc_gamma), and every similarity path gives bit-identical top-k results."""
import numpy as np
import pytest

import paper_2603_17573_b200 as H
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


def gamma_tc(dim, variant):
    if variant == 3:  # 3xTF32 (k_sim_tc.cu sim_tc_gamma)
        return 3.0 / 2**20 + (3.0 * dim + 16.0) / 2**23
    return (2.0 + 1.0 / 1024) / 1024 * 1.0001 + (dim + 16.0) / 2**23  # TF32 (k_sim_tc1.cu)


@pytest.mark.parametrize("variant", [1, 2, 3])
@pytest.mark.parametrize("kind", [O.EXACT, O.REAL])
@pytest.mark.parametrize("dim,n,B", [(64, 3000, 64), (4096, 3000, 64), (4096, 1000, 13), (256, 777, 1)])
def test_tc_scores_within_bound(torch, kind, dim, n, B, variant):
    col = H.Collection(dim, capacity=n)
    col.generate(kind, 5, n)
    q = H.gen_queries(kind, 6, 5, n, 0, B, dim)
    approx = col.debug_sim_scores(q, variant=variant).cpu().numpy().astype(np.float64)
    keys = O.gen_keys(kind, 5, 0, n, dim).astype(np.float64)
    qq = q.cpu().numpy().astype(np.float64)
    exact = qq @ keys.T
    bound = gamma_tc(dim, variant) * (np.abs(qq) @ np.abs(keys).T)
    err = np.abs(approx - exact)
    assert np.all(err <= bound), float((err / np.maximum(bound, 1e-300)).max())
    scale = np.linalg.norm(qq, axis=1, keepdims=True) * np.linalg.norm(keys, axis=1)[None, :]
    rel = float((err / scale).max())
    if variant == 3:
        # all three split terms reach the accumulator: the residual is the
        # tensor core's (truncating) fp32 accumulation, far inside the bound
        assert rel < 1e-4
    else:
        assert rel < 2e-3
    if kind == O.EXACT:  # k/16 values are exact in TF32 -> exact scores
        assert np.array_equal(approx, exact)


@pytest.mark.parametrize("path", ["rows", "tile", "tc", "tc1", "tc3"])
@pytest.mark.parametrize("kind", [O.EXACT, O.REAL])
def test_paths_bit_identical(torch, path, kind):
    try:
        H.set_sim_path(path)
        for dim, n in ((64, 5000), (4096, 2500), (4352, 1200)):
            col = H.Collection(dim, capacity=n)
            col.generate(kind, 17, n)
            for B in (1, 4, 8, 13, 64, 70):
                q = H.gen_queries(kind, 18, 17, n, 3, B, dim)
                sc, ids = col.search_topk_exact(q, 8)
                osc, oid = O.search_synth(kind, 17, n, q.cpu().numpy(), 8)
                np.testing.assert_array_equal(ids.cpu().numpy(), oid, err_msg=f"{path} dim={dim} B={B}")
                np.testing.assert_array_equal(sc.cpu().numpy(), osc)
            assert col.overflow_count() == 0
    finally:
        H.set_sim_path("auto")


@pytest.mark.parametrize("path", ["tc", "tc1", "tc3"])
def test_tc_ragged_tail_and_range(torch, path):
    """Row counts that are not multiples of the 128-key block, and sub-ranges."""
    H.set_sim_path(path)
    try:
        n, dim = 1000 * 3 + 77, 128
        col = H.Collection(dim, capacity=n)
        col.generate(O.REAL, 9, n)
        q = H.gen_queries(O.REAL, 10, 9, n, 0, 32, dim)
        for rng in ((0, n), (5, 133), (1000, 2999), (n - 1, n)):
            sc, ids = col.search_topk_exact(q, 5, row_range=rng)
            keys = O.gen_keys(O.REAL, 9, rng[0], rng[1] - rng[0], dim)
            osc, oid = O.search_topk(keys, q.cpu().numpy(), 5)
            kk = oid.shape[1]
            np.testing.assert_array_equal(ids.cpu().numpy()[:, :kk], oid + rng[0])
            np.testing.assert_array_equal(sc.cpu().numpy()[:, :kk], osc)
    finally:
        H.set_sim_path("auto")


# ----------------------------------------------------------------------------- wide kernel (k_sim_wide.cu)
def gamma_wide(dim, bf16):
    acc = (dim + 16.0) / 2**23
    return (1.0 / 512 * 1.0001 + acc) if bf16 else ((2.0 + 1.0 / 1024) / 1024 * 1.0001 + acc)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("kind", [O.EXACT, O.REAL])
@pytest.mark.parametrize("dim,n,B", [(64, 2000, 256), (4096, 1500, 200), (4096, 900, 128), (256, 777, 65),
                                     (4352, 600, 7)])
def test_wide_scores_within_bound(torch, kind, dim, n, B, dtype):
    """The wide filter (N = 64/128/256 queries per UMMA) stays inside gamma * sum|k q|."""
    bf16 = dtype == "bf16"
    col = H.Collection(dim, capacity=n, dtype=dtype)
    col.generate(kind, 5, n)
    q = H.gen_queries(kind, 6, 5, n, 0, B, dim)
    approx = col.debug_sim_scores(q, variant=1).cpu().numpy().astype(np.float64)
    keys = O.gen_keys(kind | (O.KEYS_BF16 if bf16 else 0), 5, 0, n, dim).astype(np.float64)
    qq = q.cpu().numpy().astype(np.float64)
    exact = qq @ keys.T
    bound = gamma_wide(dim, bf16) * (np.abs(qq) @ np.abs(keys).T)
    err = np.abs(approx - exact)
    assert np.all(err <= bound), float((err / np.maximum(bound, 1e-300)).max())
    if kind == O.EXACT:  # k/16 values are exact in TF32 and bf16 -> exact scores
        assert np.array_equal(approx, exact)


@pytest.mark.parametrize("path", ["auto", "tc_single"])
@pytest.mark.parametrize("kind", [O.EXACT, O.REAL])
def test_wide_batches_bit_identical(torch, kind, path):
    """One pass serves up to 1024 queries (CTA pairs above 128, clusters of
    query groups above 256); tc_single = the single-CTA kernels (ablation)."""
    H.set_sim_path(path)
    try:
        for dim, n in ((64, 4000), (4096, 1800)):
            col = H.Collection(dim, capacity=n)
            col.generate(kind, 21, n)
            for B in (5, 65, 127, 128, 129, 200, 256, 300, 513, 700, 1024, 1100):
                q = H.gen_queries(kind, 22, 21, n, 1, B, dim)
                sc, ids = col.search_topk_exact(q, 8)
                osc, oid = O.search_synth(kind, 21, n, q.cpu().numpy(), 8)
                np.testing.assert_array_equal(ids.cpu().numpy(), oid, err_msg=f"dim={dim} B={B}")
                np.testing.assert_array_equal(sc.cpu().numpy(), osc)
            assert col.overflow_count() == 0
    finally:
        H.set_sim_path("auto")


@pytest.mark.parametrize("kind", [O.EXACT, O.REAL])
def test_bf16_collection_exact_over_stored_keys(torch, kind):
    """bf16 collections: ids and fp64 scores bit-identical to the reference's
    search over the bf16-rounded keys (store.cpp:59-73 on the stored DB)."""
    for dim, n in ((64, 3000), (4096, 1500), (4352, 700)):
        col = H.Collection(dim, capacity=n, dtype="bf16")
        col.generate(kind, 31, n)
        keys, _ = col.keys_view()
        assert keys.dtype == torch.bfloat16
        ok = O.gen_keys(kind | O.KEYS_BF16, 31, 0, n, dim)
        np.testing.assert_array_equal(keys.float().cpu().numpy(), ok)
        for B, k in ((1, 8), (3, 1), (64, 8), (100, 32), (256, 8), (683, 3), (1024, 8)):
            q = H.gen_queries(kind, 32, 31, n, 0, B, dim)
            sc, ids = col.search_topk_exact(q, k)
            osc, oid = O.search_synth(kind | O.KEYS_BF16, 31, n, q.cpu().numpy(), k)
            np.testing.assert_array_equal(ids.cpu().numpy(), oid, err_msg=f"dim={dim} B={B}")
            np.testing.assert_array_equal(sc.cpu().numpy(), osc)
        assert col.overflow_count() == 0


def test_bf16_insert_and_range(torch):
    rng = np.random.default_rng(3)
    n, dim = 1300, 128
    emb = rng.standard_normal((n, dim)).astype(np.float32)
    acts = rng.uniform(-1, 1, (n, 3, 7))
    col = H.Collection(dim, capacity=16, dtype="bf16")
    col.insert(emb, acts)
    stored = torch.as_tensor(emb).to(torch.bfloat16).float().numpy()  # RN-even, as hsd_bf16_bits
    keys, _ = col.keys_view()
    np.testing.assert_array_equal(keys.float().cpu().numpy(), stored)
    q = torch.as_tensor(rng.standard_normal((40, dim)).astype(np.float32), device="cuda")
    for rg in ((0, n), (17, 900), (n - 3, n)):
        sc, ids = col.search_topk_exact(q, 6, row_range=rg)
        osc, oid = O.search_topk(stored[rg[0]:rg[1]], q.cpu().numpy(), 6)
        kk = oid.shape[1]
        np.testing.assert_array_equal(ids.cpu().numpy()[:, :kk], oid + rg[0])
        np.testing.assert_array_equal(sc.cpu().numpy()[:, :kk], osc)


def test_bf16_config_errors(torch):
    with pytest.raises(H.ConfigError):
        H.Collection(36, capacity=4, dtype="bf16")  # dim % 8
    with pytest.raises(H.ConfigError):
        H.Collection(64, capacity=4, dtype="fp8")


# ----------------------------------------------------------------------------- bf16 filter copy of fp32 keys
GAMMA_COPY = lambda dim: (1.0 / 256 + 1.0 / 262144) * 1.0001 + (dim + 16.0) / 2**23  # noqa: E731


@pytest.mark.parametrize("kind", [O.EXACT, O.REAL])
@pytest.mark.parametrize("dim,n,B", [(64, 2000, 256), (4096, 1200, 100), (4352, 600, 7)])
def test_filter_copy_scores_within_bound(torch, kind, dim, n, B):
    col = H.Collection(dim, capacity=n)
    col.generate(kind, 5, n)
    col.set_filter("bf16_copy")
    q = H.gen_queries(kind, 6, 5, n, 0, B, dim)
    approx = col.debug_sim_scores(q, variant=4).cpu().numpy().astype(np.float64)
    keys = O.gen_keys(kind, 5, 0, n, dim).astype(np.float64)
    qq = q.cpu().numpy().astype(np.float64)
    err = np.abs(approx - qq @ keys.T)
    bound = GAMMA_COPY(dim) * (np.abs(qq) @ np.abs(keys).T)
    assert np.all(err <= bound), float((err / np.maximum(bound, 1e-300)).max())


@pytest.mark.parametrize("kind", [O.EXACT, O.REAL])
def test_filter_copy_results_bit_identical(torch, kind):
    """With the bf16 filter copy the ids and fp64 scores are still the reference's over the fp32 keys."""
    for dim, n in ((64, 5000), (4096, 1500)):
        col = H.Collection(dim, capacity=n // 2)
        col.generate(kind, 41, n // 2)
        col.set_filter("bf16_copy")
        assert col.filter() == "bf16_copy"
        col.generate(kind, 41, n - n // 2)  # appended rows refresh the copy (and grow it)
        for B, k in ((1, 8), (4, 3), (5, 8), (64, 8), (300, 8), (1024, 32)):
            q = H.gen_queries(kind, 42, 41, n, 2, B, dim)
            sc, ids = col.search_topk_exact(q, k)
            osc, oid = O.search_synth(kind, 41, n, q.cpu().numpy(), k)
            np.testing.assert_array_equal(ids.cpu().numpy(), oid, err_msg=f"dim={dim} B={B}")
            np.testing.assert_array_equal(sc.cpu().numpy(), osc)
        assert col.overflow_count() == 0
        col.set_filter("native")
        assert col.filter() == "native"


def test_filter_copy_insert_and_range(torch):
    rng = np.random.default_rng(9)
    n, dim = 900, 128
    emb = rng.standard_normal((n, dim)).astype(np.float32)
    col = H.Collection(dim, capacity=8)
    col.set_filter("bf16_copy")
    col.insert(emb[:300], rng.uniform(-1, 1, (300, 3, 7)))
    col.insert(emb[300:], rng.uniform(-1, 1, (n - 300, 3, 7)))
    q = torch.as_tensor(rng.standard_normal((50, dim)).astype(np.float32), device="cuda")
    for rg in ((0, n), (10, 777)):
        sc, ids = col.search_topk_exact(q, 5, row_range=rg)
        osc, oid = O.search_topk(emb[rg[0]:rg[1]], q.cpu().numpy(), 5)
        np.testing.assert_array_equal(ids.cpu().numpy(), oid + rg[0])
        np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    with pytest.raises(H.ConfigError):
        H.Collection(64, capacity=4, dtype="bf16").set_filter("bf16_copy")


@pytest.mark.parametrize("dtype,filt", [("f32", "native"), ("f32", "bf16_copy"), ("bf16", "native")])
def test_edge_shapes_all_kernels(torch, dtype, filt):
    """Dims that are not a multiple of the 128-B k-chunk (TMA zero fill), tiny
    and partial key blocks, k > n, sub-ranges, and every pass width (one
    CTA, 2-4 query groups per cluster, several passes)."""
    rng = np.random.default_rng(77)
    for dim in (8, 40, 72, 136):
        if dtype == "bf16" and dim % 8:
            continue
        for n in (1, 5, 127, 129, 700):
            emb = rng.standard_normal((n, dim)).astype(np.float32)
            col = H.Collection(dim, capacity=n, dtype=dtype)
            col.insert(emb, rng.uniform(-1, 1, (n, 3, 7)))
            if filt == "bf16_copy":
                col.set_filter("bf16_copy")
            stored = emb if dtype == "f32" else torch.as_tensor(emb).bfloat16().float().numpy()
            for B in (1, 3, 70, 200, 300, 1030):
                q = torch.as_tensor(rng.standard_normal((B, dim)).astype(np.float32), device="cuda")
                for k, rg in ((1, (0, n)), (9, (0, n)), (4, (n // 3, n))):
                    if rg[0] >= rg[1]:
                        continue
                    sc, ids = col.search_topk_exact(q, k, row_range=rg)
                    osc, oid = O.search_topk(stored[rg[0]:rg[1]], q.cpu().numpy(), k)
                    kk = oid.shape[1]
                    np.testing.assert_array_equal(ids.cpu().numpy()[:, :kk], oid + rg[0],
                                                  err_msg=f"dim={dim} n={n} B={B} k={k} rg={rg}")
                    np.testing.assert_array_equal(sc.cpu().numpy()[:, :kk], osc)
                    assert np.all(ids.cpu().numpy()[:, kk:] == -1)
            assert col.overflow_count() == 0
