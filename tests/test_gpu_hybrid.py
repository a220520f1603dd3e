"""GPU parity of the config-5 hybrid decoding loop (hsd_hybrid_*, k_hybrid.cu)
against the oracle loop (hsdo_hybrid_run): per-round StepRecords, ToyEnv
positions and EpisodeReports bit-identical (F within 1e-5 relative)."""
import numpy as np
import pytest

import paper_2603_17573_b200 as H
from oracle import oracle as O

pytestmark = pytest.mark.gpu

T, N_EPI, DIM = 64, 40, 64


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


def make_db(dtype, kind=H.REAL, n=T * N_EPI, dim=DIM):
    col = H.Collection(dim, capacity=n, dtype=dtype)
    col.generate(kind, 7, n, payload=H.PAYLOAD_TRAJ, traj_T=T)
    return col


def oracle_params(hp, kind_flags):
    v = hp.verify
    return O.HybridParams(robots=hp.robots, k=hp.k, mode=hp.mode, traj_T=hp.traj_T, drafter_p_pct=hp.drafter_p_pct,
                          drafter_L=hp.drafter_L, gap_d=hp.gap_d, d_f=hp.d_f, seed=hp.seed, db_seed=hp.db_seed,
                          key_kind=kind_flags, relaxed=v.relaxed, bias_seq_max=v.bias_seq_max,
                          bias_token_max=v.bias_token_max, skip_enabled=v.skip_enabled, O_dist=v.O_dist,
                          chain_cap=v.chain_cap, min_S=v.min_S,
                          metric=O.MetricParams(hp.metric.alpha, hp.metric.w, hp.metric.threshold, hp.metric.r_cap),
                          bounds=O.NormBounds(hp.bounds.d_min, hp.bounds.d_max95, hp.bounds.r_min, hp.bounds.r_max95),
                          cost_verifier=hp.cost_verifier, cost_drafter_token=hp.cost_drafter_token,
                          cost_retrieval=hp.cost_retrieval)


def compare(loop, hp, kind_flags, rounds, n_rows=T * N_EPI, dim=DIM):
    tr = loop.trace()
    otr, opos, orep = O.hybrid_run(oracle_params(hp, kind_flags), n_rows, dim, rounds)
    for f in ("mode", "accept_len", "verifier_calls", "n_emit", "skipped"):
        np.testing.assert_array_equal(tr[f], otr[f], err_msg=f)
    np.testing.assert_allclose(tr["F"], otr["F"], rtol=1e-5, atol=1e-6)
    np.testing.assert_array_equal(tr["cost"], otr["cost"])
    np.testing.assert_array_equal(loop.positions(), opos)
    rep = loop.reports()
    for f in O.EPISODE_REPORT_DTYPE.names:
        np.testing.assert_array_equal(rep[f], orep[f], err_msg=f)
    return tr, rep


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("skip", [True, False])
def test_hybrid_loop_matches_oracle(torch, dtype, skip):
    col = make_db(dtype)
    hp = H.hybrid_params(48, k=3, traj_T=T, d_f=64 if skip else 0, seed=5, db_seed=7)
    rounds = 45
    loop = H.HybridLoop(col, hp, max_rounds=rounds)
    loop.step(rounds)
    tr, rep = compare(loop, hp, H.REAL | (O.KEYS_BF16 if dtype == "bf16" else 0), rounds)
    assert set(np.unique(tr["mode"])) == {0, 1}
    nr, nd = loop.counts()
    assert nr == int((tr["mode"] == 1).sum()) and nd == int((tr["mode"] == 0).sum())


@pytest.mark.parametrize("mode", [H.MODE_PURE_RETRIEVAL, H.MODE_PURE_DRAFTER, H.MODE_AUTOREGRESSIVE])
def test_hybrid_pure_modes(torch, mode):
    col = make_db("f32")
    hp = H.hybrid_params(40, k=4, mode=mode, traj_T=T, d_f=64, seed=9, db_seed=7)
    loop = H.HybridLoop(col, hp, max_rounds=25)
    loop.step(25)
    compare(loop, hp, H.REAL, 25)
    if mode == H.MODE_AUTOREGRESSIVE:
        rep = loop.reports()
        np.testing.assert_array_equal(rep["tokens"].astype(np.float64), rep["cost"])


def test_hybrid_relaxed_off_exact_family_and_k8(torch):
    col = make_db("f32", kind=H.EXACT)
    v = H.VerifyParams.make(relaxed=False, skip_enabled=True, min_S=0.9, O_dist=3)
    hp = H.hybrid_params(33, k=8, traj_T=T, d_f=128, seed=3, db_seed=7, key_kind=H.EXACT, verify=v)
    loop = H.HybridLoop(col, hp, max_rounds=40)
    loop.step(40)
    compare(loop, hp, H.EXACT, 40)


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
def test_hybrid_sharded_world1_equals_single(torch, exchange):
    """The sharded retrieval path (NCCL all-gather or peer-memory publish + merge, world 1) gives the same loop."""
    col = make_db("bf16")
    hp = H.hybrid_params(32, k=3, traj_T=T, d_f=64, seed=4, db_seed=7)
    single = H.HybridLoop(col, hp, max_rounds=30)
    single.step(30)
    if exchange == "nccl":
        comm = H.Comm(H.Comm.unique_id(), 1, 0, 0)
    else:
        comm = H.Comm(None, 1, 0, 0)
        comm.p2p_import([comm.p2p_export(1024, 32)])
    sharded = H.HybridLoop(col, hp, max_rounds=30, comm=comm, n_total_rows=col.size())
    sharded.step(30)
    np.testing.assert_array_equal(single.positions(), sharded.positions())
    a, b = single.trace(), sharded.trace()
    for f in STEP_FIELDS:
        np.testing.assert_array_equal(a[f], b[f])
    sharded.close()
    comm.close()


STEP_FIELDS = ("mode", "accept_len", "verifier_calls", "n_emit", "skipped", "cost", "F")


def test_hybrid_config_errors(torch):
    col = make_db("f32")
    with pytest.raises(H.ConfigError):
        H.HybridLoop(col, H.hybrid_params(8, k=0, traj_T=T))
    with pytest.raises(H.ConfigError):
        H.HybridLoop(col, H.hybrid_params(8, traj_T=T, drafter_L=5))
    with pytest.raises(H.ConfigError):
        H.HybridLoop(col, H.hybrid_params(8, traj_T=T, cost_retrieval=-1.0))
