"""GPU parity of K4 (gather + verify-skip + relaxed acceptance + accepted
length) against the oracle's restatement of SPEC.md:398-506: every outcome
field and every emitted token bit-exact, over a tolerance / skip-threshold
sweep read from one pass (BASELINE config 3 shape at reduced E)."""
import numpy as np
import pytest

import paper_2603_17573_b200 as H
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


SWEEP = [
    H.VerifyParams.make(relaxed=True, bias_seq_max=30, bias_token_max=15),
    H.VerifyParams.make(relaxed=False),
    H.VerifyParams.make(relaxed=True, bias_seq_max=10, bias_token_max=5),
    H.VerifyParams.make(relaxed=True, skip_enabled=True, min_S=0.95, O_dist=5),
    H.VerifyParams.make(relaxed=True, skip_enabled=True, min_S=0.99, O_dist=1),
    H.VerifyParams.make(relaxed=True, bias_seq_max=60, bias_token_max=30, chain_cap=7),
    H.VerifyParams.make(relaxed=True, chain_cap=1),
]


def oracle_round(drafts, greedy, cosv, hist, gap_d, p):
    st = O.SkipState(0.0, p.min_S, p.O_dist, 0.0, 0)
    skip = bool(p.skip_enabled) and len(drafts) > 0 and O.should_skip(cosv, st, gap_d, hist)
    return O.verify_round(np.asarray(drafts, np.int32).reshape(len(drafts), -1) if len(drafts) else
                          np.zeros((0, len(greedy)), np.int32), greedy, skip=skip, cap=p.chain_cap,
                          enabled=bool(p.relaxed), seq_max=p.bias_seq_max, tok_max=p.bias_token_max)


@pytest.mark.parametrize("L", [7, 21])
@pytest.mark.parametrize("k", [1, 3, 8, 12])
def test_verify_parity(torch, L, k):
    _parity(torch, L, k, 512)


@pytest.mark.parametrize("L", [7, 21])
def test_verify_parity_large_round(torch, L):
    """A round of 1100 episodes (more CTAs than one wave of the 2-episode K4
    CTAs on some SM counts); the reported skip similarity matches too."""
    _parity(torch, L, 8, 1100)


def test_verify_skip_threshold_at_the_exact_similarity(torch):
    """min_S equal to an episode's exactly rounded similarity (R >= min_S holds
    with equality) and one ulp above it: only an exactly rounded dot decides
    these like the oracle."""
    E, d_f = 64, 256
    now, prev = O.gen_features(9, 0, E, d_f)
    cos = [O.feature_cos(now[e], prev[e]) for e in range(4)]
    sweep = [H.VerifyParams.make(relaxed=True, skip_enabled=True, min_S=c, O_dist=8) for c in cos]
    sweep += [H.VerifyParams.make(relaxed=True, skip_enabled=True, min_S=float(np.nextafter(c, 2.0)), O_dist=8)
              for c in cos]
    stats = _parity(torch, 7, 8, E, sweep=sweep, feats=(now, prev))
    assert stats["skipped"] > 0


def _parity(torch, L, k, E, sweep=None, feats=None):
    sweep = SWEEP if sweep is None else sweep
    n, d_f = 400, 256
    db_seed, lseed, fseed = 21, 5, 9
    col = H.Collection(64, capacity=n)
    col.generate(O.REAL, db_seed, n)
    rng = np.random.default_rng(L * 100 + k)
    ids = rng.integers(0, n, size=(E, k)).astype(np.int32)
    # duplicate candidates (dedup), truncated lists (k > N shards) and duplicated tokens
    ids[::7, 1:] = ids[::7, :1]
    ids[3::11, k // 2:] = -1
    ids[5::13] = -1
    src = np.where(rng.random(E) < 0.7, ids[:, 0], -1).astype(np.int64)
    src[ids[:, 0] < 0] = -1
    logits = O.gen_logits(db_seed, lseed, src, 0, L)
    now, prev = O.gen_features(fseed, 0, E, d_f) if feats is None else feats
    hist = rng.integers(0, 8, size=E).astype(np.int32)
    gap_d = 2
    t = lambda a: torch.as_tensor(a, device="cuda")
    out, toks = col.verify_round(t(ids), t(logits), sweep, feat_now=t(now), feat_prev=t(prev), history=t(hist),
                                 gap_d=gap_d)
    toks = toks.cpu().numpy()
    tok_db = O.synth_tokens(db_seed, np.arange(n))[:, :L].astype(np.int32)
    stats = {"skipped": 0, "fallback": 0, "partial": 0}
    for e in range(E):
        valid = ids[e][ids[e] >= 0]
        drafts = tok_db[valid]
        greedy = np.array([O.argmax(logits[e, p]) for p in range(L)], np.int32)
        cosv = O.feature_cos(now[e], prev[e])
        for pi, p in enumerate(sweep):
            o = oracle_round(drafts, greedy, cosv, int(hist[e]), gap_d, p)
            g = out[pi, e]
            got = (g["accept_len"], g["fallback"], g["skipped"], g["calls"], g["n_emit"])
            want = (o.accept_len, o.fallback, o.skipped, o.calls, o.n_emit)
            assert got == want, (e, pi, got, want)
            if not o.skipped and not o.fallback:
                assert (g["win_a"], g["win_b"]) == (o.win_a, o.win_b), (e, pi)
            np.testing.assert_array_equal(toks[pi, e, :o.n_emit], np.array(o.tokens[:o.n_emit]))
            assert g["greedy0"] == greedy[0]
            if p.skip_enabled:
                assert g["cos_sim"] == np.float32(cosv), (e, pi)
            stats["skipped"] += o.skipped
            stats["fallback"] += o.fallback
            stats["partial"] += 0 < o.accept_len < L
    # every branch is exercised
    if sweep is SWEEP:
        assert all(v > 0 for v in stats.values()), stats
    return stats


def test_verify_validation(torch):
    col = H.Collection(64, capacity=10)
    col.generate(O.REAL, 1, 10)
    ids = torch.zeros((4, 8), dtype=torch.int32, device="cuda")
    lg = torch.zeros((4, 7, 256), device="cuda")
    with pytest.raises(H.ConfigError):
        col.verify_round(ids, lg, H.VerifyParams.make(bias_seq_max=10, bias_token_max=15))
    with pytest.raises(H.InvalidInputError):
        col.verify_round(ids, torch.zeros((4, 5, 256), device="cuda"), H.VerifyParams.make())
    with pytest.raises(H.InvalidInputError):  # skip needs features
        col.verify_round(ids, lg, H.VerifyParams.make(skip_enabled=True))
