"""Pin the CPU oracle before trusting it.

(1) Against fixtures produced by the reference itself (tests/golden/*.npz,
    made by tests/golden/make_golden.py from the unmodified store.cpp /
    actions.cpp): search ids/scores bit-exact, quantize bit-exact.
(2) Against every known-answer vector the reference's spec holds for the path
    (SPEC.md line numbers cited per test).
"""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ reference fixtures
@pytest.mark.parametrize("name", ["search_exact_64", "search_real_64", "search_exact_4096", "search_real_4096"])
def test_oracle_search_matches_reference_fixture(name):
    z = np.load(os.path.join(GOLD, name + ".npz"))
    kind, n, dim, B, k = int(z["kind"]), int(z["n"]), int(z["dim"]), int(z["B"]), int(z["k"])
    q = O.gen_queries(kind, int(z["q_seed"]), int(z["db_seed"]), n, 0, B, dim)
    keys = O.gen_keys(kind, int(z["db_seed"]), 0, n, dim)
    sc, ids = O.search_topk(keys, q, k)
    np.testing.assert_array_equal(ids, z["ids"])
    np.testing.assert_array_equal(sc, z["scores"])  # bit-exact fp64
    sc2, ids2 = O.search_synth(kind, int(z["db_seed"]), n, q, k, threads=3)
    np.testing.assert_array_equal(ids2, z["ids"])
    np.testing.assert_array_equal(sc2, z["scores"])
    # retrieve_drafts tokens = quantize(next_actions) of each hit
    np.testing.assert_array_equal(O.synth_tokens(int(z["db_seed"]), z["ids"].ravel()).reshape(z["tokens"].shape),
                                  z["tokens"])


def test_oracle_quantize_matches_reference_fixture():
    z = np.load(os.path.join(GOLD, "quantize.npz"))
    for a, b, b2 in zip(z["acts"], z["bins"], z["bins2"]):
        rc, out = O.quantize(a)
        assert rc == 0
        np.testing.assert_array_equal(out, b)
        rc, out = O.quantize(a, z["lo2"], z["hi2"])
        np.testing.assert_array_equal(out, b2)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_oracle_search_matches_live_reference_ties():
    """EXACT family has heavy exact ties + duplicate rows: (score desc, id asc)."""
    R = O.ref()
    dim, n = 16, 4000
    col = R.hsdref_collection_new(dim)
    assert R.hsdref_insert_synth(col, O.EXACT, 5, 0, n, dim) == 0
    q = O.gen_queries(O.EXACT, 6, 5, n, 0, 40, dim)
    sc_r, ids_r, _ = O.ref_search(col, q, 25, threads=4)
    R.hsdref_collection_free(col)
    sc, ids = O.search_synth(O.EXACT, 5, n, q, 25, threads=2)
    np.testing.assert_array_equal(ids, ids_r)
    np.testing.assert_array_equal(sc, sc_r)
    # ties really are exercised
    assert (np.diff(sc_r, axis=1) == 0).sum() > 50


# ------------------------------------------------------------------ actions (AC1 :733)
def test_quantize_known_answers():
    assert O.quantize([-1.0] * 7)[1].tolist() == [0] * 7
    assert O.quantize([1.0] * 7)[1].tolist() == [255] * 7
    assert O.quantize([0.0] * 7)[1].tolist() == [127] * 7
    assert O.quantize([float("nan")] + [0.0] * 6)[0] == -1  # InvalidInput
    assert O.quantize([0.0] * 7, lo=1.0, hi=1.0)[0] == -2  # ConfigError
    assert O.quantize([0.0] * 7, k_bins=1)[0] == -2


def test_quantize_roundtrip_monotone():
    rng = np.random.default_rng(0)
    a = rng.uniform(-1, 1, size=(20000, 7))
    q = np.array([O.quantize(x)[1] for x in a])
    deq = -1.0 + q / 255.0 * 2.0
    assert np.all(np.abs(deq - a) <= 2.0 / 255.0 + 1e-12)
    order = np.argsort(a[:, 0])
    assert np.all(np.diff(q[order, 0]) >= 0)
    # SPEC.md:67 claims quantize(dequantize(b)) == b for every bin, but the
    # reference's own floor formula (actions.cpp:43-44 after :63) breaks it for
    # 20 of 256 bins (e.g. b=1 -> 0.99999.. -> 0).  The oracle follows the
    # reference, not the spec prose: exactly those 20 bins drop by one.
    bad = [b for b in range(256) if O.quantize([-1.0 + b / 255.0 * 2.0] * 7)[1][0] != b]
    assert len(bad) == 20 and bad[:4] == [1, 2, 5, 9]
    assert all(O.quantize([-1.0 + b / 255.0 * 2.0] * 7)[1][0] == b - 1 for b in bad)


# ------------------------------------------------------------------ search (AC5 :737)
def test_search_known_answers():
    rng = np.random.default_rng(1)
    keys = rng.standard_normal((1000, 64)).astype(np.float32)
    keys /= np.linalg.norm(keys, axis=1, keepdims=True)
    sc, ids = O.search_topk(keys, keys[17], 1)
    assert ids[0, 0] == 17 and abs(sc[0, 0] - 1.0) < 1e-6
    one = np.zeros((1, 64), np.float32)
    one[0, 0] = 1
    orth = np.zeros(64, np.float32)
    orth[1] = 1
    sc, ids = O.search_topk(one, orth, 3)
    assert ids.shape == (1, 1) and sc[0, 0] == 0.0
    with pytest.raises(ValueError):
        O.search_topk(keys, keys[0], 0)
    sc, ids = O.search_topk(keys[:0], keys[0], 3)  # empty collection -> empty result
    assert ids.shape == (1, 0)
    q = rng.standard_normal((100, 64)).astype(np.float32)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    full = q.astype(np.float64) @ keys.astype(np.float64).T
    for k in (1, 3, 5, 10):
        sc, ids = O.search_topk(keys, q, k)
        for b in range(100):
            want = np.lexsort((np.arange(1000), -full[b]))[:k]
            assert set(want.tolist()) == set(ids[b].tolist())


# ------------------------------------------------------------------ verification
def test_token_bias():
    L = O.lib()
    assert L.hsdo_token_bias(100, 100) == 0
    assert L.hsdo_token_bias(100, 115) == 15
    assert L.hsdo_token_bias(0, 255) == 255


def test_accept_sequence_known_answers():
    v = [100, 100, 100]
    assert O.accept_sequence([115, 85, 100], v)  # biases (15,15,0)
    assert not O.accept_sequence([116, 100, 100], v)  # (16,0,0)
    assert not O.accept_sequence([111, 110, 110], v)  # (11,10,10) sum 31
    assert not O.accept_sequence([101], [100], gripper=True)
    assert O.accept_sequence([100], [100], gripper=True)
    assert not O.accept_sequence([101, 100, 100], v, enabled=False)


def test_accept_sequence_monotone():
    rng = np.random.default_rng(3)
    for _ in range(10000):
        b = rng.integers(0, 25, size=3)
        smaller = b - rng.integers(0, 3, size=3).clip(0, b)
        v = np.full(3, 128)
        if O.accept_sequence(v + b, v):
            assert O.accept_sequence(v + smaller, v)


def test_argmax_ties_lowest_index():
    x = np.zeros(256, np.float32)
    x[[7, 200]] = 3.0
    assert O.argmax(x) == 7


def test_verify_tree_known_answers():
    rng = np.random.default_rng(4)
    g = rng.integers(0, 256, size=21).astype(np.int32)
    out = O.verify_round(g[None, :], g, enabled=False)  # perfect draft, strict
    assert out.accept_len == 21 and not out.fallback and out.calls == 1
    bad = g.copy()
    bad[0] = (g[0] + 100) % 256
    out = O.verify_round(np.stack([bad, bad]), g)
    assert out.accept_len == 0 and out.fallback and out.n_emit == 1 and out.tokens[0] == g[0]
    # chain 2 (2 groups) beats chain 1 (1 group)
    c1 = g.copy()
    c1[3] = (g[3] + 100) % 256  # rot0 rejected -> 1 group
    c2 = g.copy()
    c2[6] = (g[6] + 1) % 256  # grip0 rejected -> 2 groups
    out = O.verify_round(np.stack([c1, c2]), g)
    assert out.accept_len == 6 and (out.win_a, out.win_b) == (0, 1)


def test_chain_enumeration():
    rng = np.random.default_rng(5)
    d = rng.integers(0, 256, size=(2, 21)).astype(np.int32)
    chains, a, b = O.enumerate_chains(d, cap=64)
    assert len(chains) == 4 and (a[0], b[0]) == (0, 0)
    np.testing.assert_array_equal(chains[0], d[0])  # first chain is all-rank-0
    chains, a, b = O.enumerate_chains(d, cap=1)
    assert len(chains) == 1
    d[1, :3] = d[0, :3]  # identical pos0 groups -> dedup
    chains, a, b = O.enumerate_chains(d, cap=64)
    assert len(chains) == 2
    # gripper isolation: every chain's gripper tokens come from one rank
    d8 = rng.integers(0, 256, size=(8, 21)).astype(np.int32)
    chains, a, b = O.enumerate_chains(d8, cap=64)
    assert len(chains) == 64
    for c, bb in zip(chains, b):
        assert all(c[6 + 7 * s] == d8[bb, 6 + 7 * s] for s in range(3))


def test_should_skip_known_answers():
    st = O.SkipState(0.9, 0.95, 5, 0.1, 0)
    f = np.zeros(64, np.float32)
    f[0] = 1
    g = np.zeros(64, np.float32)
    g[1] = 1
    assert O.should_skip(O.feature_cos(f, f), st, 1, 10)
    assert not O.should_skip(O.feature_cos(f, g), st, 1, 10)
    assert not O.should_skip(0.96, st, 6, 10)
    assert not O.should_skip(0.99, st, 3, 2)  # insufficient history


def test_feature_cos_exact():
    rng = np.random.default_rng(6)
    a = rng.standard_normal(4096).astype(np.float32)
    b = rng.standard_normal(4096).astype(np.float32)
    from fractions import Fraction

    exact = sum(Fraction(float(x)) * Fraction(float(y)) for x, y in zip(a, b))
    assert O.feature_cos(a, b) == float(exact)


def test_alg1_offline_and_online():
    n = 40
    S = np.array([[1.0 - 0.01 * abs(j - i) for j in range(n)] for i in range(n)])
    m, o = O.calibrate([S], 0.9)
    assert o == 9 and abs(m - 0.91) < 1e-12
    m, o = O.calibrate([np.ones((12, 12))], 0.9)
    assert m == 1.0 and o == 1  # constant: first pair in (i, d) order
    assert O.calibrate([S], 1.0) is None
    st = O.update_skip_state(O.SkipState(0.5, 0.90, 5, 0.1, 0), True, 0.95, 0.90)
    assert abs(st.min_S - 0.905) < 1e-12 and st.O_dist == 6
    st = O.update_skip_state(O.SkipState(0.5, 0.90, 5, 0.1, 0), False, 0.95, 0.90)
    assert abs(st.min_S - 0.895) < 1e-12 and st.O_dist == 4
    st = O.update_skip_state(O.SkipState(0.5, 1.0, 5, 0.1, 0), True, 0.95, 0.90)
    assert st.min_S == 1.0
    st = O.update_skip_state(O.SkipState(0.5, 0.9, 1, 0.1, 0), False, 0.95, 0.90)
    assert st.O_dist == 1


# ------------------------------------------------------------------ kinematics (AC2/AC3)
def circle_pts(r, cx, cy, w=15, arc=2 * math.pi, phase=0.0):
    t = phase + np.arange(w) * (arc / (w if arc >= 2 * math.pi - 1e-12 else w - 1))
    return np.stack([cx + r * np.cos(t), cy + r * np.sin(t)], axis=1)


def test_circle_center_fixture():
    uv = circle_pts(0.05, 0.2, -0.1)
    (cu, cv), deg, it = O.fit_circle_center(uv)
    assert not deg and abs(cu - 0.2) < 1e-6 and abs(cv + 0.1) < 1e-6
    (cu, cv), deg, it = O.fit_circle_center(np.tile([[0.3, 0.4]], (15, 1)))
    assert deg and abs(cu - 0.3) < 1e-15 and abs(cv - 0.4) < 1e-15  # centroid, kinematics.cpp:116-127


def test_curvature_radius_fixtures():
    xy = circle_pts(0.05, 0.0, 0.0)
    xyz = np.concatenate([xy, np.zeros((15, 1))], axis=1)
    assert abs(O.curvature_radius(xyz) - 0.05) < 1e-6
    assert O.curvature_radius(np.tile([[0.1, 0.2, 0.3]], (15, 1))) == 0.0
    line = np.stack([np.arange(15) * 0.01, np.zeros(15), np.zeros(15)], axis=1)
    assert O.curvature_radius(line, r_cap=1.0) == 1.0


def test_circle_ac2_random():
    rng = np.random.default_rng(8)
    for _ in range(200):
        r = rng.uniform(0.01, 0.5)
        c = rng.uniform(-1, 1, size=3)
        arc = rng.uniform(0.5, 2 * math.pi)
        xy = circle_pts(r, 0, 0, arc=arc, phase=rng.uniform(0, 6.28))
        # random rotation into 3-D
        Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        xyz = np.concatenate([xy, np.zeros((15, 1))], axis=1) @ Q.T + c
        R = O.curvature_radius(xyz, r_cap=10.0)
        assert abs(R - r) / r < 1e-5


def test_displacement_fixtures():
    line = np.stack([np.arange(15) * 0.01, np.zeros(15), np.zeros(15)], axis=1)
    assert abs(O.cumulative_displacement(line) - 0.14) < 1e-12
    assert O.cumulative_displacement(np.zeros((15, 3))) == 0.0
    aba = np.array([[0, 0, 0], [0.03, 0, 0], [0, 0, 0]], float)
    assert abs(O.cumulative_displacement(aba) - 0.06) < 1e-15
    with pytest.raises(ValueError):
        O.cumulative_displacement(np.zeros((1, 3)))


def test_normalize_percentile_fused():
    assert O.normalize(0.123381, 0.000009, 0.123381) == 1.0
    assert O.normalize(0.000009, 0.000009, 0.123381) == 0.0
    assert O.normalize(1.0, 0.0, 2.0) == 0.5
    assert O.normalize(-5.0, 0.0, 2.0) == 0.0
    assert O.normalize(3.0, 2.0, 2.0) == 0.0
    assert O.percentile_bounds(np.arange(1, 101)) == (1.0, 95.0)
    assert O.percentile_bounds([7.0]) == (7.0, 7.0)
    assert O.percentile_bounds([5.0, 5.0, 5.0]) == (5.0, 5.0)
    p = O.MetricParams(0.5, 15, 0.5, 1.0)
    b = O.NormBounds(0.0, 1.0, 0.0, 1.0)
    assert O.fused_metric(0.2, 0.8, p, b) == 0.5
    assert O.lib().hsdo_classify(0.5, 0.5) == 0  # F == theta -> drafter
    assert O.lib().hsdo_classify(0.9, 0.5) == 1


def test_decide_sd_fixtures():
    p = O.MetricParams(0.5, 15, 0.5, 1.0)
    b = O.NormBounds(0.000009, 0.123381, 0.000001, 0.014989)  # LIBERO-Goal
    with pytest.raises(ValueError):  # 14 points with w = 15
        O.window_features(np.zeros((14, 3)), p, b)
    R, D, F, dec = O.window_features(np.tile([[0.2, 0.1, 0.3]], (15, 1)), p, b)
    assert (R, D, F, dec) == (0.0, 0.0, 0.0, 0)
    fast = np.stack([np.arange(15) * 0.02, np.arange(15) * 0.01, np.zeros(15)], axis=1)
    R, D, F, dec = O.window_features(fast, p, b)
    assert dec == 1 and F == 1.0


def test_bf16_key_rounding_matches_torch_rn_even():
    """hsd_bf16_bits (bf16 collections, oracle KEYS_BF16) is IEEE RN-even."""
    import torch

    for kind in (O.EXACT, O.REAL):
        k32 = O.gen_keys(kind, 11, 0, 64, 4096)
        kb = O.gen_keys(kind | O.KEYS_BF16, 11, 0, 64, 4096)
        ref = torch.as_tensor(k32).to(torch.bfloat16).float().numpy()
        np.testing.assert_array_equal(kb, ref)
        if kind == O.EXACT:  # k/16 values are exact in bf16
            np.testing.assert_array_equal(kb, k32)
