"""Verify-skip lifecycle (Alg. 1):
update_skip_state through the C ABI (host arithmetic) against the SPEC
fixtures and the oracle; offline calibration on the GPU (k_calib.cu) against
the oracle's exhaustive pair scan."""
import numpy as np
import pytest

import paper_2603_17573_b200 as H
from oracle import oracle as O


@pytest.mark.parametrize("success,min_S,O_dist,exp_S,exp_O", [
    (True, 0.90, 5, 0.905, 6), (False, 0.90, 5, 0.895, 4), (True, 1.0, 5, 1.0, 6), (False, 0.9, 1, 0.895, 1)])
def test_update_skip_state_spec_fixtures(success, min_S, O_dist, exp_S, exp_O):
    """SPEC.md:473-475 (Δ = 0.1, |S_c − min_S_h| = 0.05)."""
    st = H.update_skip_state(H.SkipState(0.5, min_S, O_dist, 0.1, 0), success, 0.95, 0.90)
    assert abs(st.min_S - exp_S) < 1e-12 and st.O_dist == exp_O


def test_update_skip_state_matches_oracle():
    rng = np.random.default_rng(0)
    for _ in range(500):
        T, ms, od, dl, inv = rng.uniform(0.3, 0.95), rng.uniform(0.2, 1.0), int(rng.integers(1, 9)), \
            rng.uniform(0, 0.5), int(rng.integers(0, 2))
        succ, sc, mh = bool(rng.integers(0, 2)), rng.uniform(0, 1), rng.uniform(0, 1)
        a = H.update_skip_state(H.SkipState(T, ms, od, dl, inv), succ, sc, mh)
        b = O.update_skip_state(O.SkipState(T, ms, od, dl, inv), succ, sc, mh)
        assert a.min_S == b.min_S and a.O_dist == b.O_dist
        assert T <= a.min_S <= 1.0 and a.O_dist >= 1


def trajectories(rng, lengths, d_f, dup_every=0):
    """Per-episode features whose similarity decays with the step gap (the
    Fig. 3(a) premise): f_i = normalize(base + drift * i + noise), fp32."""
    feats = []
    for n in lengths:
        base = rng.standard_normal(d_f)
        drift = rng.standard_normal(d_f) * 0.08
        for i in range(n):
            v = base + drift * i + rng.standard_normal(d_f) * 0.02
            if dup_every and i % dup_every == 1:
                v = prev  # noqa: F821 — exact duplicate of the previous point (ties)
            prev = v
            feats.append((v / np.linalg.norm(v)).astype(np.float32))
    off = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    return np.array(feats, np.float32).reshape(-1, d_f), off


def oracle_calibrate(feats, off, T):
    sims = []
    for t in range(off.size - 1):
        f = feats[off[t]:off[t + 1]]
        n = f.shape[0]
        s = np.zeros((n, n))
        for i in range(n):
            for j in range(i + 1, n):
                s[i, j] = O.feature_cos(f[i], f[j])
        sims.append(s)
    return O.calibrate(sims, T)


@pytest.mark.gpu
@pytest.mark.parametrize("d_f,lengths,T,dup", [
    (64, [40, 1, 2, 33, 70], 0.9, 0), (64, [50, 50], 0.95, 3), (512, [97, 12, 31], 0.8, 0),
    (4096, [20, 45], 0.9, 4)])
def test_gpu_calibration_matches_oracle(d_f, lengths, T, dup):
    import torch

    rng = np.random.default_rng(d_f + len(lengths))
    feats, off = trajectories(rng, lengths, d_f, dup_every=dup)
    exp = oracle_calibrate(feats, off, T)
    assert exp is not None
    got = H.calibrate_skip(torch.as_tensor(feats, device="cuda"), off, T)
    assert got[0] == exp[0] and got[1] == exp[1], (got, exp)


@pytest.mark.gpu
def test_gpu_calibration_constant_and_failure():
    import torch

    f = np.zeros((12, 64), np.float32)
    f[:, 3] = 1.0  # identical unit features: every S is exactly 1.0
    ft = torch.as_tensor(f, device="cuda")
    assert H.calibrate_skip(ft, [0, 12], 0.9) == (1.0, 1)  # first pair in (i, d) order (oracle reading)
    with pytest.raises(H.CalibrationError):
        H.calibrate_skip(ft, [0, 12], 1.0)  # T = 1 -> no pair strictly exceeds
    with pytest.raises(H.InvalidInputError):
        H.calibrate_skip(ft, [0, 13, 12], 0.9)
