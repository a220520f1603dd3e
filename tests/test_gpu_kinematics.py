"""GPU parity of K5 (kinematic fused metric + hybrid-boundary decision)
against the oracle's Eigen-free restatement of kinematics.cpp: R, D, F within
1e-5 relative (north_star tolerance), decisions identical away from theta,
plus the SPEC fixtures evaluated on the device."""
import math

import numpy as np
import pytest

import paper_2603_17573_b200 as H
from paper_2603_17573_b200 import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-12)


@pytest.mark.parametrize("bounds", ["libero", "unit"])
def test_kinematics_parity(torch, bounds):
    nb = H.LIBERO_GOAL if bounds == "libero" else H.NormBounds(0.0, 0.5, 0.0, 0.5)
    onb = O.NormBounds(nb.d_min, nb.d_max95, nb.r_min, nb.r_max95)
    mp = H.MetricParams(0.5, 15, 0.5, 1.0)
    omp = O.MetricParams(0.5, 15, 0.5, 1.0)
    xyz, kind = synth.trajectory_windows(1200, 15, seed=11)
    hist = np.where(np.arange(1200) % 10 == 0, 9, 40).astype(np.int32)
    R, D, F, dec = H.window_features(torch.as_tensor(xyz, device="cuda"), mp, nb,
                                     history=torch.as_tensor(hist, device="cuda"))
    R, D, F, dec = (x.cpu().numpy() for x in (R, D, F, dec))
    worst = {}
    near = 0
    for i in range(len(xyz)):
        r, d, f, od = O.window_features(xyz[i], omp, onb)
        if hist[i] < 15:
            od = 0  # cold start
        k = synth.KINDS[kind[i]]
        e = max(rel(R[i], r) if r > 1e-12 else abs(R[i] - r), rel(D[i], d) if d > 0 else abs(D[i]), abs(F[i] - f))
        worst[k] = max(worst.get(k, 0.0), e)
        if abs(f - mp.threshold) < 1e-9:
            near += 1
            continue
        assert dec[i] == od, (i, k, f, F[i])
    for k, e in worst.items():
        assert e < 1e-5, (k, e)


def test_kinematics_fixtures_on_device(torch):
    mp = H.MetricParams(0.5, 15, 0.5, 1.0)
    th = np.arange(15) * 2 * math.pi / 15
    circle = np.stack([0.05 * np.cos(th), 0.05 * np.sin(th), np.zeros(15)], 1)
    line = np.stack([np.arange(15) * 0.01, np.zeros(15), np.zeros(15)], 1)
    stationary = np.tile([[0.1, 0.2, 0.3]], (15, 1))
    fast = np.stack([np.arange(15) * 0.02, np.arange(15) * 0.01, np.zeros(15)], 1)
    bad = line.copy()
    bad[4, 1] = np.nan
    x = torch.as_tensor(np.stack([circle, line, stationary, fast, bad]), device="cuda")
    R, D, F, dec = (t.cpu().numpy() for t in H.window_features(x, mp, H.LIBERO_GOAL))
    assert abs(R[0] - 0.05) < 1e-6
    assert R[1] == 1.0 and abs(D[1] - 0.14) < 1e-12  # :138, :145
    assert R[2] == 0.0 and D[2] == 0.0 and F[2] == 0.0 and dec[2] == 0  # :137, :535
    assert dec[3] == 1 and F[3] == 1.0  # straight fast window -> retrieval (:534)
    assert dec[4] == -1  # non-finite -> InvalidInputError
    cold = torch.as_tensor(np.array([14, 15, 14, 15, 15], np.int32), device="cuda")
    dec2 = H.window_features(x, mp, H.LIBERO_GOAL, history=cold)[3].cpu().numpy()
    assert dec2[3] == 1 and dec2[0] == 0  # 14 points of history -> drafter (:533)
    with pytest.raises(H.InvalidInputError):
        H.window_features(x[:, :14].contiguous(), mp, H.LIBERO_GOAL)


def test_velocity_acceleration_jerk_diagnostics(torch):
    """K5's windowed finite-difference kinematics (north-star diagnostics) match
    the oracle's sequential restatement; R/D/F/decisions are unchanged."""
    from paper_2603_17573_b200 import synth

    xyz, _ = synth.trajectory_windows(300, 15, seed=11)
    x = torch.as_tensor(xyz, device="cuda")
    R0, D0, F0, d0 = H.window_features(x)
    R, D, F, dec, vaj = H.window_features(x, derivatives=True)
    assert torch.equal(R, R0) and torch.equal(D, D0) and torch.equal(F, F0) and torch.equal(dec, d0)
    got = vaj.cpu().numpy()
    for i in range(xyz.shape[0]):
        exp = O.window_derivatives(xyz[i])
        np.testing.assert_allclose(got[i], exp, rtol=1e-12, atol=1e-300)
    # a straight constant-speed window: |a| = |j| = 0 up to rounding, |v| = the step
    line = np.stack([np.linspace(0, 0.14, 15), np.zeros(15), np.zeros(15)], 1)[None]
    _, _, _, _, v = H.window_features(torch.as_tensor(line, device="cuda"), derivatives=True)
    assert abs(v[0, 0].item() - 0.01) < 1e-12 and v[0, 1].item() < 1e-12 and v[0, 2].item() < 1e-12
