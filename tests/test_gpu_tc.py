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


@pytest.mark.parametrize("variant", [1, 3])
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


@pytest.mark.parametrize("path", ["rows", "tile", "tc", "tc3"])
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


@pytest.mark.parametrize("path", ["tc", "tc3"])
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
