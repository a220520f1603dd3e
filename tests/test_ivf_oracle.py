"""CPU checks of the oracle's IVF restatement (oracle/oracle.py ivf_*), the
checker behind tests/test_gpu_index.py: assignment = the reference's exact
best centroid (score desc, id asc), stable lists, unit centroids, and the
probed-lists search = the reference's exact search over those rows."""
import numpy as np

from oracle import oracle as O


def test_ivf_build_is_consistent():
    keys = O.gen_keys(O.CLUSTER, 3, 0, 1500, 32)
    cent, offs, perm = O.ivf_build(keys, 12, 3)
    assert offs[0] == 0 and offs[-1] == 1500 and np.all(np.diff(offs) >= 0)
    assert sorted(perm.tolist()) == list(range(1500))
    for l in range(12):
        rows = perm[offs[l]:offs[l + 1]]
        assert np.all(np.diff(rows) > 0)  # ascending record ids within a list
    s = keys.astype(np.float64) @ cent.astype(np.float64).T
    assign = np.empty(1500, np.int64)
    for l in range(12):
        assign[perm[offs[l]:offs[l + 1]]] = l
    best = s.max(axis=1)
    assert np.all(s[np.arange(1500), assign] >= best - 1e-12)
    nr = np.linalg.norm(cent.astype(np.float64), axis=1)
    assert np.allclose(nr, 1.0, atol=1e-6)


def test_ivf_seeds_and_clamp():
    np.testing.assert_array_equal(O.ivf_seed_rows(10, 4), [1, 3, 6, 8])
    keys = O.gen_keys(O.REAL, 1, 0, 5, 16)
    cent, offs, perm = O.ivf_build(keys, 9, 0)  # nlist clamped to the row count: one row per list
    assert cent.shape[0] == 5 and np.all(np.diff(offs) == 1)


def test_ivf_search_lists_matches_exact_when_every_list_is_probed():
    keys = O.gen_keys(O.REAL, 4, 0, 800, 64)
    cent, offs, perm = O.ivf_build(keys, 8, 2)
    q = O.gen_queries(O.REAL, 5, 4, 800, 0, 6, 64)
    probes = np.tile(np.arange(8), (6, 1))
    s, i = O.ivf_search_lists(keys, offs, perm, probes, q, 5)
    es, ei = O.search_topk(keys, q, 5)
    np.testing.assert_array_equal(i, ei)
    np.testing.assert_array_equal(s, es)
