"""tcgen05 filter kernels (K1, k_sim_wide.cu): the approximate filter scores
stay inside the forward error bound the exact selection relies on
(sim_wide_gamma), including on rounding-adversarial inputs, and every kernel
variant gives bit-identical top-k results."""
import numpy as np
import pytest

import paper_2603_17573_b200 as H
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


# ----------------------------------------------------------------------------- wide kernel (k_sim_wide.cu)
def acc_term(dim):
    return (dim + 16.0) * 2.0**-22 * 1.02  # fp32 tensor-core accumulation (sim_wide_gamma)


def gamma_wide(dim, bf16):
    """bf16 keys: query rounded to bf16, u = 2^-8; fp32 keys: TF32 truncation 2^-10 per operand."""
    return (2.0**-8 * 1.0001 + acc_term(dim)) if bf16 else ((2.0**-9 + 2.0**-20) * 1.0001 + acc_term(dim))


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
def GAMMA_COPY(dim):
    """bf16 copy of fp32 keys: both operands RN-even to bf16 (u = 2^-8 each)."""
    return (2.0**-7 + 2.0**-16) * 1.0001 + acc_term(dim)


# round-1 constants (unit roundoff taken as 2^-9): the adversarial inputs below must violate them
OLD_GAMMA_COPY = lambda dim: (1.0 / 256 + 1.0 / 262144) * 1.0001 + (dim + 16.0) / 2**23  # noqa: E731
OLD_GAMMA_BF16 = lambda dim: 1.0 / 512 * 1.0001 + (dim + 16.0) / 2**23  # noqa: E731


def midpoint_vectors(rows, dim, seed):
    """fp32 vectors whose every component sits just below a bf16 rounding
    midpoint (1 + 2^-8 - 2^-20 times a power of two, random sign), so RN-even
    rounds every one DOWN in magnitude by ~2^-8 relative."""
    rng = np.random.default_rng(seed)
    mant = np.float32(1.0 + 2.0**-8 - 2.0**-20)
    scale = np.float32(2.0) ** (-5 - rng.integers(0, 3, size=(rows, dim))).astype(np.float32)
    sign = np.where(rng.random((rows, dim)) < 0.5, -1, 1).astype(np.float32)
    return (mant * scale * sign).astype(np.float32), sign


@pytest.mark.parametrize("dim", [64, 4096])
def test_filter_bound_midpoint_adversarial(torch, dim):
    """Every product rounded the same way: the bf16 filter copy errs by ~2^-7
    relative (both operands) and bf16 keys by ~2^-8 (query only).  The errors
    exceed the round-1 constants and stay inside sim_wide_gamma."""
    n, B = 300, 8
    keys, sign = midpoint_vectors(n, dim, 1)
    q = (np.abs(midpoint_vectors(B, dim, 2)[0]) * sign[:B]).astype(np.float32)  # same signs: products all > 0
    qd = torch.as_tensor(q, device="cuda")
    acts = np.zeros((n, 3, 7))
    exact = q.astype(np.float64) @ keys.astype(np.float64).T
    absum = np.abs(q.astype(np.float64)) @ np.abs(keys.astype(np.float64)).T
    # bf16 filter copy of fp32 keys
    col = H.Collection(dim, capacity=n)
    col.insert(keys, acts)
    col.set_filter("bf16_copy")
    approx = col.debug_sim_scores(qd, variant=4).cpu().numpy().astype(np.float64)
    rel = np.abs(approx - exact) / absum
    assert rel[np.arange(B), np.arange(B)].min() > OLD_GAMMA_COPY(dim), rel.max()
    assert np.all(rel <= GAMMA_COPY(dim)), rel.max()
    sc, ids = col.search_topk_exact(qd, 8)
    osc, oid = O.search_topk(keys, q, 8)
    np.testing.assert_array_equal(ids.cpu().numpy(), oid)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    # bf16 collection: the stored keys are exact, the query is rounded
    colb = H.Collection(dim, capacity=n, dtype="bf16")
    stored = torch.as_tensor(keys).bfloat16().float().numpy().astype(np.float64)
    colb.insert(keys, acts)
    approx = colb.debug_sim_scores(qd, variant=1).cpu().numpy().astype(np.float64)
    ex_b = q.astype(np.float64) @ stored.T
    ab_b = np.abs(q.astype(np.float64)) @ np.abs(stored).T
    rel = np.abs(approx - ex_b) / ab_b
    assert rel.max() > OLD_GAMMA_BF16(dim), rel.max()
    assert np.all(rel <= gamma_wide(dim, True)), rel.max()
    # TF32 over the fp32 keys (truncation), inside its own bound
    col.set_filter("native")
    approx = col.debug_sim_scores(qd, variant=1).cpu().numpy().astype(np.float64)
    rel = np.abs(approx - exact) / absum
    assert np.all(rel <= gamma_wide(dim, False)), rel.max()


@pytest.mark.parametrize("path", ["auto", "tc_single"])
def test_ragged_tail_and_range(torch, path):
    """Row counts that are not multiples of the 128-key block, and sub-ranges."""
    H.set_sim_path(path)
    try:
        n, dim = 1000 * 3 + 77, 128
        col = H.Collection(dim, capacity=n)
        col.generate(O.REAL, 9, n)
        for B in (32, 200):
            q = H.gen_queries(O.REAL, 10, 9, n, 0, B, dim)
            for rng in ((0, n), (5, 133), (1000, 2999), (n - 1, n)):
                sc, ids = col.search_topk_exact(q, 5, row_range=rng)
                keys = O.gen_keys(O.REAL, 9, rng[0], rng[1] - rng[0], dim)
                osc, oid = O.search_topk(keys, q.cpu().numpy(), 5)
                kk = oid.shape[1]
                np.testing.assert_array_equal(ids.cpu().numpy()[:, :kk], oid + rng[0])
                np.testing.assert_array_equal(sc.cpu().numpy()[:, :kk], osc)
    finally:
        H.set_sim_path("auto")


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
