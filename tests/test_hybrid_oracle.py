"""CPU oracle of the config-5 hybrid decoding loop (oracle/hsd_oracle.c
hsdo_hybrid_run): SPEC scheduler invariants."""
import numpy as np
import pytest

from oracle import oracle as O


def params(mode=0, relaxed=1, skip=1, R=24, d_f=64, k=3, p_pct=85, traj_T=64, kind=O.REAL):
    return O.HybridParams(robots=R, k=k, mode=mode, traj_T=traj_T, drafter_p_pct=p_pct, drafter_L=7, gap_d=1,
                          d_f=d_f if skip else 0, seed=5, db_seed=7, key_kind=kind, relaxed=relaxed, bias_seq_max=30,
                          bias_token_max=15, skip_enabled=skip, O_dist=5, chain_cap=64, min_S=0.95,
                          metric=O.MetricParams(0.5, 15, 0.5, 1.0),
                          bounds=O.NormBounds(0.000009, 0.123381, 0.000001, 0.014989), cost_verifier=1.0,
                          cost_drafter_token=0.1, cost_retrieval=0.37)


N_ROWS, DIM = 40 * 64, 64


def test_autoregressive_speedup_is_one():
    """speedup proxy of autoregressive mode = 1 identically; 7 calls / slice."""
    tr, pos, rep = O.hybrid_run(params(mode=3), N_ROWS, DIM, 30)
    assert np.all(tr["mode"] == 2) and np.all(tr["n_emit"] == 7) and np.all(tr["verifier_calls"] == 7)
    np.testing.assert_array_equal(rep["tokens"].astype(np.float64), rep["cost"])


def test_strict_hybrid_equals_autoregressive_trajectory():
    """strict mode (relaxation off, skip off) emits the AR trajectory step for step."""
    p = params(mode=0, relaxed=0, skip=0)
    tr, pos, rep = O.hybrid_run(p, N_ROWS, DIM, 40)
    n_demo = N_ROWS // p.traj_T
    assert set(np.unique(tr["mode"])) == {0, 1}  # both SD kinds occur
    for r in range(p.robots):
        n_act = int(rep["tokens"][r]) // 7
        np.testing.assert_array_equal(pos[r], O.ar_position(p.db_seed, p.seed, r, n_demo, n_act))


def test_trace_is_self_consistent():
    """per-episode cost = sum of step costs; AL recomputes from the trace; decision mix sums."""
    tr, pos, rep = O.hybrid_run(params(), N_ROWS, DIM, 50)
    assert np.all(rep["rounds"] == 50)
    np.testing.assert_array_equal(tr["n_emit"].sum(0), rep["tokens"])
    np.testing.assert_array_equal(tr["accept_len"].sum(0), rep["accepted"])
    np.testing.assert_array_equal(tr["verifier_calls"].sum(0), rep["verifier_calls"])
    np.testing.assert_allclose(tr["cost"].astype(np.float64).sum(0), rep["cost"], rtol=1e-5)
    assert np.all(rep["n_retrieval"] + rep["n_drafter"] == 50)
    assert np.all(tr["n_emit"] % 7 == 0) and np.all(tr["n_emit"] >= 7)
    # cold start: the first w-1 rounds have < w trajectory points -> drafter
    assert np.all(tr["mode"][:14] == 0)
    # skips fire only in retrieval mode and emit the whole 21-token draft at retrieval cost only
    sk = tr["skipped"] == 1
    assert np.all(tr["mode"][sk] == 1) and np.all(tr["n_emit"][sk] == 21) and np.all(tr["verifier_calls"][sk] == 0)
    np.testing.assert_allclose(tr["cost"][sk], 0.37, rtol=1e-6)


def test_skip_on_retrieval_replay_beats_drafter():
    """Pure retrieval on recorded demonstrations with skip on -> speedup proxy > 2 (SPEC.md:643-645 analogue)."""
    tr, pos, rep = O.hybrid_run(params(mode=1), N_ROWS, DIM, 30)
    seen = rep["n_fallback"] == 0
    assert rep["tokens"][seen].sum() / rep["cost"][seen].sum() > 2.0
