"""verify_tree with a real verifier (teacher-forced greedy tokens per chain,
models.hpp:34-37), the greedy rule on non-finite logits (std::max_element),
and compute_percentile_bounds (kinematics.cpp:238-247) — GPU vs the oracle."""
import numpy as np
import pytest

import paper_2603_17573_b200 as H
from oracle import oracle as O
from paper_2603_17573_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


def t(torch, a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def make_drafts(rng, E, k, L):
    """Pre-gathered draft records [E][k][32] with duplicated pos0 groups, duplicated later parts and whole
    duplicate candidates (dedup), plus truncated candidate lists."""
    base = rng.integers(0, 256, size=(E, k, L)).astype(np.uint8)
    for e in range(E):
        if k > 1 and e % 3 == 0:
            base[e, 1, :3] = base[e, 0, :3]  # same pos0
        if k > 2 and e % 4 == 1:
            base[e, 2, 3:] = base[e, 0, 3:]  # same later part
        if k > 3 and e % 5 == 2:
            base[e, 3] = base[e, 1]  # identical candidate
    drafts = np.zeros((E, k, 32), np.uint8)
    drafts[:, :, :L] = base
    ids = np.tile(np.arange(k, dtype=np.int32), (E, 1))
    ids[7::9, k // 2:] = -1
    ids[11::17] = -1  # empty shard
    return ids, drafts


def perturb(rng, tok, L):
    """Greedy tokens near the draft: exact, inside the relaxed caps, or outside; gripper mostly exact."""
    d = np.where(rng.random(tok.shape) < 0.6, 0,
                 np.where(rng.random(tok.shape) < 0.75, rng.integers(-12, 13, tok.shape),
                          rng.integers(-60, 61, tok.shape)))
    grip = (np.arange(L) % 7) == 6
    d[..., grip] = np.where(rng.random(d[..., grip].shape) < 0.8, 0, 1)
    return np.clip(tok.astype(np.int64) + d, 0, 255).astype(np.uint8)


def oracle_chains(drafts_e, ids_e, L, cap, chain_greedy_e, g_ctx, skip, p):
    valid = ids_e >= 0
    dr = drafts_e[valid][:, :L].astype(np.int32)
    return O.verify_round_chains(dr if len(dr) else np.zeros((0, L), np.int32), chain_greedy_e, g_ctx, skip=skip,
                                 cap=cap, enabled=bool(p.relaxed), seq_max=p.bias_seq_max, tok_max=p.bias_token_max)


@pytest.mark.parametrize("L", [7, 21])
@pytest.mark.parametrize("k", [3, 8])
@pytest.mark.parametrize("cap", [64, 7, 1])
def test_enumerate_chains_matches_brute_force(torch, L, k, cap):
    rng = np.random.default_rng(L * 10 + k + cap)
    E = 200
    ids, drafts = make_drafts(rng, E, k, L)
    n, ab, tok = H.enumerate_chains(t(torch, ids), L, cap=cap, drafts=t(torch, drafts))
    n, ab, tok = n.cpu().numpy(), ab.cpu().numpy(), tok.cpu().numpy()
    for e in range(E):
        valid = ids[e] >= 0
        ch, a, b = O.enumerate_chains(drafts[e][valid][:, :L].astype(np.int32), cap=cap) if valid.any() else (
            np.zeros((0, L)), np.zeros(0), np.zeros(0))
        assert n[e] == len(ch), e
        np.testing.assert_array_equal(ab[e, :n[e], 0], a)
        np.testing.assert_array_equal(ab[e, :n[e], 1], b)
        np.testing.assert_array_equal(tok[e, :n[e]], ch)


@pytest.mark.parametrize("L", [7, 21])
@pytest.mark.parametrize("k", [3, 8])
@pytest.mark.parametrize("variant", ["greedy", "logits"])
@pytest.mark.parametrize("pset", ["relaxed", "strict", "cap7", "skip"])
def test_verify_round_chains_parity(torch, L, k, variant, pset):
    rng = np.random.default_rng(1000 + L * 10 + k)
    E, d_f = 300, 128
    cap = 7 if pset == "cap7" else 64
    p = {"relaxed": H.VerifyParams.make(relaxed=True),
         "strict": H.VerifyParams.make(relaxed=False),
         "cap7": H.VerifyParams.make(relaxed=True, bias_seq_max=20, bias_token_max=10, chain_cap=7),
         "skip": H.VerifyParams.make(relaxed=True, skip_enabled=True, min_S=0.97, O_dist=3)}[pset]
    ids, drafts = make_drafts(rng, E, k, L)
    n, _, chain_tok = H.enumerate_chains(t(torch, ids), L, cap=cap, drafts=t(torch, drafts))
    chain_tok = chain_tok.cpu().numpy()
    greedy = perturb(rng, chain_tok, L)  # [E][cap][L] (rows >= n_chains unused)
    # every 3rd episode: the verifier departs from every chain after pos0 (partial prefixes)
    g2 = greedy.astype(np.int64)
    g2[::3, :, 3:6] = (g2[::3, :, 3:6] + 40 + rng.integers(0, 40, g2[::3, :, 3:6].shape)) % 256
    greedy = g2.astype(np.uint8)
    g_ctx = rng.integers(0, 256, size=E).astype(np.int32)
    now, prev = O.gen_features(7, 0, E, d_f)
    hist = rng.integers(0, 6, size=E).astype(np.int32)
    kw = dict(drafts=t(torch, drafts), feat_now=t(torch, now), feat_prev=t(torch, prev), history=t(torch, hist),
              gap_d=2)
    if variant == "greedy":
        out, toks = H.verify_round_chains(t(torch, ids), p, t(torch, g_ctx), chain_greedy=t(torch, greedy), **kw)
    else:  # logits whose argmax (lowest bin on exact ties) is the greedy token
        lg = rng.standard_normal((E, cap, L, 256)).astype(np.float32)
        e_i, c_i, p_i = np.indices((E, cap, L))
        lg[e_i, c_i, p_i, greedy.astype(np.int64)] = 9.0
        tie = rng.random((E, cap, L)) < 0.05
        hi_bin = np.minimum(greedy.astype(np.int64) + 1 + rng.integers(0, 40, greedy.shape), 255)
        lg[e_i[tie], c_i[tie], p_i[tie], hi_bin[tie]] = 9.0  # tie at a higher bin: the lower one wins
        out, toks = H.verify_round_chains(t(torch, ids), p, t(torch, g_ctx), chain_logits=t(torch, lg), **kw)
    toks = toks.cpu().numpy()
    n = n.cpu().numpy()
    seen = {"fallback": 0, "partial": 0, "full": 0, "skipped": 0}
    for e in range(E):
        skip = False
        if p.skip_enabled and (ids[e] >= 0).any():
            skip = O.should_skip(O.feature_cos(now[e], prev[e]), O.SkipState(0.0, p.min_S, p.O_dist, 0.0, 0), 2,
                                 int(hist[e]))
        o = oracle_chains(drafts[e], ids[e], L, cap, greedy[e, :max(n[e], 1)], int(g_ctx[e]), skip, p)
        g = out[e]
        got = (g["accept_len"], g["fallback"], g["skipped"], g["calls"], g["n_emit"])
        want = (o.accept_len, o.fallback, o.skipped, o.calls, o.n_emit)
        assert got == want, (e, got, want)
        if not o.skipped and not o.fallback:
            assert (g["win_a"], g["win_b"]) == (o.win_a, o.win_b), e
        np.testing.assert_array_equal(toks[e, :o.n_emit], np.array(o.tokens[:o.n_emit]))
        seen["fallback"] += o.fallback
        seen["skipped"] += o.skipped
        seen["partial"] += 0 < o.accept_len < L
        seen["full"] += o.accept_len == L and not o.skipped
    assert seen["fallback"] > 0 and seen["partial"] > 0, seen
    if pset == "skip":
        assert seen["skipped"] > 0


def test_chain_teacher_forcing_differs_from_context_free(torch):
    """The per-chain path is not the context-free one: make chain 0's greedy tokens reject everything while a later
    chain's accept all groups — the later chain must win."""
    E, k, L = 4, 3, 7
    rng = np.random.default_rng(3)
    ids = np.tile(np.arange(k, dtype=np.int32), (E, 1))
    drafts = np.zeros((E, k, 32), np.uint8)
    drafts[:, :, :L] = rng.integers(0, 200, size=(E, k, L))
    n, ab, chain_tok = H.enumerate_chains(t(torch, ids), L, cap=64, drafts=t(torch, drafts))
    greedy = chain_tok.cpu().numpy().copy()
    greedy[:, 0, 0] = (greedy[:, 0, 0].astype(int) + 100) % 256  # chain 0 rejected at pos0
    greedy[:, 1:, :] = (greedy[:, 1:, :].astype(int) + 50) % 256  # every other chain rejected ...
    greedy[:, 4, :] = chain_tok.cpu().numpy()[:, 4, :]  # ... except chain 4: fully accepted
    out, toks = H.verify_round_chains(t(torch, ids), H.VerifyParams.make(relaxed=False), t(torch, np.zeros(E, np.int32)),
                                      chain_greedy=t(torch, greedy), drafts=t(torch, drafts))
    ab = ab.cpu().numpy()
    for e in range(E):
        assert out[e]["accept_len"] == L and (out[e]["win_a"], out[e]["win_b"]) == tuple(ab[e, 4])
        np.testing.assert_array_equal(toks.cpu().numpy()[e], chain_tok.cpu().numpy()[e, 4])


def test_chains_validation(torch):
    ids = t(torch, np.zeros((2, 3), np.int32))
    dr = t(torch, np.zeros((2, 3, 32), np.uint8))
    g = t(torch, np.zeros((2, 64, 7), np.uint8))
    ctx = t(torch, np.zeros(2, np.int32))
    with pytest.raises(H.ConfigError):  # cap mismatch with the parameters
        H.verify_round_chains(ids, H.VerifyParams.make(chain_cap=5), ctx, chain_greedy=g, drafts=dr)
    with pytest.raises(H.InvalidInputError):
        H.enumerate_chains(ids, 9, drafts=dr)  # L must be 7 or 21


# ----------------------------------------------------------------------------- greedy rule on non-finite logits
def test_nonfinite_logits_follow_max_element(torch):
    """K4's argmax reproduces std::max_element / the oracle's `if (v[b] > v[best])` scan: a NaN in bin 0 is
    never replaced, a later NaN is never selected, +-inf compare normally, equal maxima -> lowest bin."""
    rng = np.random.default_rng(8)
    E, L, k, n = 256, 7, 4, 300
    col = H.Collection(64, capacity=n)
    col.generate(O.REAL, 21, n)
    ids = rng.integers(0, n, size=(E, k)).astype(np.int32)
    tok = O.synth_tokens(21, np.arange(n))[:, :L].astype(np.int64)
    lg = rng.standard_normal((E, L, 256)).astype(np.float32)
    e_i, p_i = np.indices((E, L))
    lg[e_i, p_i, tok[ids[:, 0]]] = 5.0  # greedy == rank-0 draft unless disturbed below
    kinds = rng.integers(0, 8, size=(E, L))
    for e in range(E):
        for p in range(L):
            kd = kinds[e, p]
            if kd == 1:
                lg[e, p, 0] = np.nan
            elif kd == 2:
                lg[e, p, rng.integers(0, 256, 5)] = np.nan
            elif kd == 3:
                lg[e, p, :] = np.nan
            elif kd == 4:
                lg[e, p, rng.integers(1, 256)] = np.inf
            elif kd == 5:
                lg[e, p, :] = -np.inf
            elif kd == 6:
                lg[e, p, rng.integers(0, 256, 3)] = np.inf
                lg[e, p, 0] = np.nan
    out, toks = col.verify_round(t(torch, ids), t(torch, lg), H.VerifyParams.make(relaxed=False))
    toks = toks.cpu().numpy()
    for e in range(E):
        greedy = np.array([O.argmax(lg[e, p]) for p in range(L)], np.int32)
        o = O.verify_round(tok[ids[e]].astype(np.int32), greedy, enabled=False)
        g = out[0, e]
        assert (g["accept_len"], g["fallback"], g["calls"], g["n_emit"], g["greedy0"]) == (
            o.accept_len, o.fallback, o.calls, o.n_emit, greedy[0]), e
        np.testing.assert_array_equal(toks[0, e, :o.n_emit], np.array(o.tokens[:o.n_emit]))


# ----------------------------------------------------------------------------- percentile bounds (A29)
def test_percentile_bounds_spec_examples(torch):
    f64 = lambda a: torch.as_tensor(np.asarray(a, np.float64), device="cuda")  # noqa: E731
    assert H.percentile_bounds(f64(np.arange(1, 101))) == (1.0, 95.0)  # SPEC.md:163, AC3 (:735)
    assert H.percentile_bounds(f64([7.0])) == (7.0, 7.0)
    assert H.percentile_bounds(f64([5.0, 5.0, 5.0])) == (5.0, 5.0)
    rng = np.random.default_rng(2)
    for n in (1, 2, 19, 20, 21, 39, 40, 41, 1000, 100_003):
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, n)
        assert H.percentile_bounds(f64(x)) == O.percentile_bounds(x), n
    with pytest.raises(H.InvalidInputError):
        H.percentile_bounds(f64([1.0, np.nan, 2.0]))
    with pytest.raises(H.InvalidInputError):
        H.percentile_bounds(f64([1.0, np.inf]))
    with pytest.raises(H.InvalidInputError):
        H.percentile_bounds(f64(np.zeros(0)))


def test_norm_bounds_from_windows(torch):
    xyz, _ = synth.trajectory_windows(500, 15, seed=12)
    nb = H.norm_bounds_from_windows(torch.as_tensor(xyz, device="cuda"))
    mp = O.MetricParams(0.5, 15, 0.5, 1.0)
    unit = O.NormBounds(0.0, 1.0, 0.0, 1.0)
    R, D = zip(*[O.window_features(xyz[i], mp, unit)[:2] for i in range(len(xyz))])
    r_lo, r_hi = O.percentile_bounds(np.array(R))
    d_lo, d_hi = O.percentile_bounds(np.array(D))
    for got, want in ((nb.r_min, r_lo), (nb.r_max95, r_hi), (nb.d_min, d_lo), (nb.d_max95, d_hi)):
        assert abs(got - want) <= 1e-5 * max(abs(want), 1e-12), (got, want)
