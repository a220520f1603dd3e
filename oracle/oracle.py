"""CPU ORACLE bindings (test infrastructure only).

ctypes access to
  * oracle/_build/libhsd_oracle.so — the C restatement (hsd_oracle.c), and
  * oracle/_ref/libhsdref.so      — the reference's own store/actions/hnsw
                                   sources compiled in place (oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module.  The product package (paper_2603_17573_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libhsd_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libhsdref.so")

_lib = None
_ref = None

_f = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_d = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_l = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build() -> None:
    """Build the oracle (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class AcceptParams(C.Structure):
    _fields_ = [("enabled", C.c_int), ("bias_seq_max", C.c_int), ("bias_token_max", C.c_int)]


class SkipState(C.Structure):
    _fields_ = [("T", C.c_double), ("min_S", C.c_double), ("O_dist", C.c_int), ("delta", C.c_double),
                ("inverted", C.c_int)]


class Outcome(C.Structure):
    _fields_ = [("accept_len", C.c_int), ("win_a", C.c_int), ("win_b", C.c_int), ("fallback", C.c_int),
                ("calls", C.c_int), ("skipped", C.c_int), ("n_emit", C.c_int), ("tokens", C.c_int * 64)]


class Calib(C.Structure):
    _fields_ = [("min_S", C.c_double), ("O_dist", C.c_int), ("found", C.c_int)]


class MetricParams(C.Structure):
    _fields_ = [("alpha", C.c_double), ("w", C.c_int), ("threshold", C.c_double), ("r_cap", C.c_double)]


class NormBounds(C.Structure):
    _fields_ = [("d_min", C.c_double), ("d_max95", C.c_double), ("r_min", C.c_double), ("r_max95", C.c_double)]


class HybridParams(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("robots", "k", "mode", "traj_T", "drafter_p_pct", "drafter_L", "gap_d", "d_f")] + [
        ("seed", C.c_uint64), ("db_seed", C.c_uint64), ("key_kind", C.c_int)] + [
        (n, C.c_int) for n in ("relaxed", "bias_seq_max", "bias_token_max", "skip_enabled", "O_dist", "chain_cap")] + [
        ("min_S", C.c_double), ("metric", MetricParams), ("bounds", NormBounds), ("cost_verifier", C.c_double),
        ("cost_drafter_token", C.c_double), ("cost_retrieval", C.c_double)]


STEP_RECORD_DTYPE = np.dtype([("F", np.float32), ("accept_len", np.int16), ("verifier_calls", np.int16),
                              ("n_emit", np.int16), ("mode", np.int8), ("skipped", np.int8), ("cost", np.float32)])
EPISODE_REPORT_DTYPE = np.dtype([("rounds", np.int64), ("tokens", np.int64), ("accepted", np.int64),
                                 ("verifier_calls", np.int64), ("cost", np.float64), ("n_retrieval", np.int32),
                                 ("n_drafter", np.int32), ("n_skipped", np.int32), ("n_fallback", np.int32)])


def hybrid_run(params: HybridParams, n_rows: int, dim: int, rounds: int):
    """Oracle hybrid loop (hsdo_hybrid_run) -> (trace [rounds, R], pos [R, 3], reports [R])."""
    R = params.robots
    trace = np.zeros(rounds * R, STEP_RECORD_DTYPE)
    pos = np.zeros((R, 3), np.float64)
    rep = np.zeros(R, EPISODE_REPORT_DTYPE)
    rc = lib().hsdo_hybrid_run(C.byref(params), n_rows, dim, rounds, trace.ctypes.data, pos.ctypes.data,
                               rep.ctypes.data)
    assert rc == 0, rc
    return trace.reshape(rounds, R), pos, rep


def policy_token(db_seed: int, e: int, j: int, d: int) -> int:
    return lib().hsdo_policy_token(db_seed, e, j, d)


def robot_greedy(db_seed, seed, r, n_demo, j, d) -> int:
    return lib().hsdo_robot_greedy(db_seed, seed, r, n_demo, j, d)


def robot_start(seed, r, d) -> float:
    return lib().hsdo_robot_start(seed, r, d)


def dequantize_bin(b, lo=-1.0, hi=1.0, k_bins=256) -> float:
    return lib().hsdo_dequantize_bin(b, lo, hi, k_bins)


ENV_SCALE = 0.01  # HSD_ENV_SCALE


def ar_position(db_seed, seed, r, n_demo, n_actions):
    """ToyEnv position after the robot's first n_actions greedy (verifier) actions: the autoregressive trajectory."""
    p = [robot_start(seed, r, d) for d in range(3)]
    for j in range(n_actions):
        for d in range(3):
            p[d] = p[d] + ENV_SCALE * dequantize_bin(robot_greedy(db_seed, seed, r, n_demo, j, d))
    return np.array(p)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.hsdo_dot_f32.restype = C.c_double
        L.hsdo_dot_f32.argtypes = [_f, _f, C.c_int]
        L.hsdo_search_topk_exact.argtypes = [_f, C.c_int64, C.c_int, _f, C.c_int, _d, _l]
        L.hsdo_search_synth.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int, _f, C.c_int, C.c_int, _d, _l, C.c_int]
        L.hsdo_gen_keys.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_int, _f]
        L.hsdo_gen_queries.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_int, C.c_int, _f]
        L.hsdo_gen_features.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_int, _f, _f]
        L.hsdo_gen_logits.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p, C.c_int64, C.c_int, C.c_int, _f]
        L.hsdo_quantize.argtypes = [_d, _d, _d, C.c_int, _i]
        L.hsdo_synth_tokens.argtypes = [C.c_uint64, C.c_int64, _u8]
        L.hsdo_token_bias.argtypes = [C.c_int, C.c_int]
        L.hsdo_accept_sequence.argtypes = [_i, _i, C.c_int, C.c_int, C.POINTER(AcceptParams)]
        L.hsdo_argmax.argtypes = [_f, C.c_int]
        L.hsdo_feature_cos.restype = C.c_double
        L.hsdo_feature_cos.argtypes = [_f, _f, C.c_int]
        L.hsdo_should_skip.argtypes = [C.c_double, C.POINTER(SkipState), C.c_int, C.c_int]
        L.hsdo_verify_round.argtypes = [_i, C.c_int, C.c_int, _i, C.c_int, C.c_int, C.POINTER(AcceptParams),
                                        C.POINTER(Outcome)]
        L.hsdo_enumerate_chains.argtypes = [_i, C.c_int, C.c_int, C.c_int, _i, _i, _i]
        L.hsdo_verify_round_chains.argtypes = [_i, C.c_int, C.c_int, _i, C.c_int, C.c_int, C.c_int,
                                               C.POINTER(AcceptParams), C.POINTER(Outcome)]
        L.hsdo_calibrate_init.argtypes = [C.POINTER(Calib)]
        L.hsdo_calibrate_accumulate.argtypes = [C.POINTER(Calib), _d, C.c_int, C.c_double]
        L.hsdo_calibrate_finish.argtypes = [C.POINTER(Calib), C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.hsdo_update_skip_state.argtypes = [C.POINTER(SkipState), C.c_int, C.c_double, C.c_double]
        L.hsdo_project_window.argtypes = [_d, C.c_int, _d]
        L.hsdo_fit_circle_center.argtypes = [_d, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                             C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.hsdo_curvature_radius.argtypes = [_d, C.c_int, C.c_double, C.POINTER(C.c_double)]
        L.hsdo_cumulative_displacement.argtypes = [_d, C.c_int, C.POINTER(C.c_double)]
        L.hsdo_normalize.restype = C.c_double
        L.hsdo_normalize.argtypes = [C.c_double, C.c_double, C.c_double]
        L.hsdo_percentile_bounds.argtypes = [_d, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.hsdo_fused_metric.restype = C.c_double
        L.hsdo_fused_metric.argtypes = [C.c_double, C.c_double, C.POINTER(MetricParams), C.POINTER(NormBounds)]
        L.hsdo_classify.argtypes = [C.c_double, C.c_double]
        L.hsdo_window_features.argtypes = [_d, C.c_int, C.POINTER(MetricParams), C.POINTER(NormBounds),
                                           C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                           C.POINTER(C.c_int)]
        L.hsdo_hybrid_run.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.hsdo_hybrid_run.restype = C.c_int
        L.hsdo_policy_token.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int]
        L.hsdo_policy_token.restype = C.c_int
        L.hsdo_robot_greedy.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_int]
        L.hsdo_robot_greedy.restype = C.c_int
        L.hsdo_robot_start.argtypes = [C.c_uint64, C.c_int64, C.c_int]
        L.hsdo_robot_start.restype = C.c_double
        L.hsdo_dequantize_bin.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int]
        L.hsdo_dequantize_bin.restype = C.c_double
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        R = C.CDLL(REF_PATH)
        R.hsdref_collection_new.restype = C.c_void_p
        R.hsdref_collection_new.argtypes = [C.c_int]
        R.hsdref_collection_free.argtypes = [C.c_void_p]
        R.hsdref_collection_size.restype = C.c_long
        R.hsdref_collection_size.argtypes = [C.c_void_p]
        R.hsdref_insert.argtypes = [C.c_void_p, _f, _d, C.c_int64, C.c_int, C.c_int]
        R.hsdref_insert_synth.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_int]
        R.hsdref_insert_synth_mt.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_int, C.c_int]
        R.hsdref_search.argtypes = [C.c_void_p, _d, C.c_int, C.c_int, _d, _i, C.c_void_p]
        R.hsdref_search_batch.argtypes = [C.c_void_p, _f, C.c_int, C.c_int, C.c_int, C.c_int, _d, _i, C.c_void_p]
        R.hsdref_quantize.argtypes = [_d, _d, _d, C.c_int, _i]
        R.hsdref_dequantize.argtypes = [_i, _d, _d, C.c_int, _d]
        R.hsdref_l2_normalize.argtypes = [_d, C.c_int, _d]
        R.hsdref_cosine.restype = C.c_double
        R.hsdref_cosine.argtypes = [_d, _d, C.c_int]
        R.hsdref_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_long)]
        R.hsdref_save.argtypes = [C.c_void_p, C.c_char_p]
        R.hsdref_dim.argtypes = [C.c_void_p]
        R.hsdref_record.argtypes = [C.c_void_p, C.c_long, _d, _d, C.POINTER(C.c_int), C.POINTER(C.c_int), _d, C.c_int]
        _ref = R
    return _ref


def ref_load(path: str):
    """The reference's own load_collection (store.cpp:152-191): (status, line, dict | None).
    status: 0 ok, -5 ParseError, -6 VersionError, -2 ConfigError, -4 IoError, -99 a non-hsd exception."""
    R = ref()
    h, line = C.c_void_p(), C.c_long()
    st = R.hsdref_load(os.fsencode(path), C.byref(h), C.byref(line))
    if st != 0:
        return st, line.value, None
    n, dim = R.hsdref_collection_size(h), R.hsdref_dim(h)
    out = {"n": n, "dim": dim, "embedding": np.zeros((n, dim)), "next_actions": np.zeros((n, 3, 7)),
           "episode_idx": np.zeros(n, np.int32), "step_idx": np.zeros(n, np.int32), "features": []}
    e, nx, fb = np.zeros(max(dim, 1)), np.zeros(21), np.zeros(1 << 16)
    ep, stp = C.c_int(), C.c_int()
    for r in range(n):
        nf = R.hsdref_record(h, r, e, nx, C.byref(ep), C.byref(stp), fb, fb.size)
        out["embedding"][r] = e[:dim]
        out["next_actions"][r] = nx.reshape(3, 7)
        out["episode_idx"][r], out["step_idx"][r] = ep.value, stp.value
        out["features"].append(None if nf < 0 else fb[:nf].copy())
    out["_handle"] = h
    return 0, 0, out


def ref_save(loaded: dict, path: str) -> int:
    return ref().hsdref_save(loaded["_handle"], os.fsencode(path))


# ---------------------------------------------------------------- helpers
EXACT, REAL, CLUSTER = 0, 1, 2
KEYS_BF16 = 0x100  # OR into `kind`: the DB stores bf16-rounded keys (hsd_oracle.h HSDO_KEYS_BF16)


def gen_keys(kind: int, db_seed: int, row0: int, n: int, dim: int) -> np.ndarray:
    out = np.empty((n, dim), np.float32)
    lib().hsdo_gen_keys(kind, db_seed, row0, n, dim, out)
    return out


def gen_queries(kind: int, q_seed: int, db_seed: int, n_rows: int, q0: int, B: int, dim: int) -> np.ndarray:
    out = np.empty((B, dim), np.float32)
    lib().hsdo_gen_queries(kind, q_seed, db_seed, n_rows, q0, B, dim, out)
    return out


def gen_features(seed: int, e0: int, E: int, d_f: int):
    now = np.empty((E, d_f), np.float32)
    prev = np.empty((E, d_f), np.float32)
    lib().hsdo_gen_features(seed, e0, E, d_f, now, prev)
    return now, prev


def gen_logits(db_seed: int, seed: int, rows, e0: int, L: int) -> np.ndarray:
    rows = np.ascontiguousarray(rows, np.int64)
    E = rows.size
    out = np.empty((E, L, 256), np.float32)
    lib().hsdo_gen_logits(db_seed, seed, rows.ctypes.data, e0, E, L, out)
    return out


def synth_tokens(db_seed: int, rows) -> np.ndarray:
    rows = np.asarray(rows, np.int64).ravel()
    out = np.empty((rows.size, 21), np.uint8)
    t = np.empty(21, np.uint8)
    for i, r in enumerate(rows):
        lib().hsdo_synth_tokens(db_seed, int(r), t)
        out[i] = t
    return out


def search_topk(keys: np.ndarray, queries: np.ndarray, k: int):
    """Reference search semantics on materialised fp32 keys -> (scores f64, ids i64)."""
    keys = np.ascontiguousarray(keys, np.float32)
    queries = np.ascontiguousarray(np.atleast_2d(queries), np.float32)
    n, dim = keys.shape
    B = queries.shape[0]
    kk = min(k, n) if n else 0
    sc = np.zeros((B, max(k, 1)), np.float64)
    ids = np.full((B, max(k, 1)), -1, np.int64)
    for b in range(B):
        s = np.zeros(max(k, 1), np.float64)
        i = np.zeros(max(k, 1), np.int64)
        rc = lib().hsdo_search_topk_exact(keys, n, dim, queries[b], k, s, i)
        if rc < 0:
            raise ValueError("k must be >= 1")
        sc[b], ids[b] = s, i
    return sc[:, :kk], ids[:, :kk]


def search_synth(kind: int, db_seed: int, n: int, queries: np.ndarray, k: int, threads: int = 0):
    queries = np.ascontiguousarray(np.atleast_2d(queries), np.float32)
    B, dim = queries.shape
    sc = np.zeros((B, k), np.float64)
    ids = np.full((B, k), -1, np.int64)
    rc = lib().hsdo_search_synth(kind, db_seed, n, dim, queries, B, k, sc, ids, threads)
    if rc < 0:
        raise ValueError("k must be >= 1")
    kk = min(k, n)
    return sc[:, :kk], ids[:, :kk]


def quantize(a7, lo=-1.0, hi=1.0, k_bins=256):
    a = np.ascontiguousarray(a7, np.float64)
    lo7 = np.full(7, lo, np.float64) if np.isscalar(lo) else np.ascontiguousarray(lo, np.float64)
    hi7 = np.full(7, hi, np.float64) if np.isscalar(hi) else np.ascontiguousarray(hi, np.float64)
    out = np.zeros(7, np.int32)
    rc = lib().hsdo_quantize(a, lo7, hi7, k_bins, out)
    return rc, out


def argmax(logits) -> int:
    return lib().hsdo_argmax(np.ascontiguousarray(logits, np.float32), len(logits))


def feature_cos(a, b) -> float:
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return lib().hsdo_feature_cos(a, b, a.size)


def should_skip(cos: float, state: SkipState, gap_d: int, history: int) -> bool:
    return bool(lib().hsdo_should_skip(cos, C.byref(state), gap_d, history))


def accept_sequence(draft, verify, gripper=False, enabled=True, seq_max=30, tok_max=15) -> bool:
    d = np.ascontiguousarray(draft, np.int32)
    v = np.ascontiguousarray(verify, np.int32)
    p = AcceptParams(int(enabled), seq_max, tok_max)
    return bool(lib().hsdo_accept_sequence(d, v, d.size, int(gripper), C.byref(p)))


def verify_round(drafts, greedy, skip=False, cap=64, enabled=True, seq_max=30, tok_max=15) -> Outcome:
    drafts = np.ascontiguousarray(np.atleast_2d(drafts), np.int32)
    greedy = np.ascontiguousarray(greedy, np.int32)
    n_cand, L = drafts.shape
    out = Outcome()
    p = AcceptParams(int(enabled), seq_max, tok_max)
    lib().hsdo_verify_round(drafts, n_cand, L, greedy, int(skip), cap, C.byref(p), C.byref(out))
    return out


def verify_round_chains(drafts, chain_greedy, greedy_ctx, skip=False, cap=64, enabled=True, seq_max=30,
                        tok_max=15) -> Outcome:
    """verify_tree with per-chain (teacher-forced) greedy tokens chain_greedy [cap][L] (hsdo_verify_round_chains)."""
    drafts = np.ascontiguousarray(np.atleast_2d(drafts), np.int32)
    n_cand, L = drafts.shape if drafts.size else (0, np.asarray(chain_greedy).shape[-1])
    cg = np.ascontiguousarray(np.asarray(chain_greedy).reshape(-1, L), np.int32)
    out = Outcome()
    p = AcceptParams(int(enabled), seq_max, tok_max)
    lib().hsdo_verify_round_chains(drafts, n_cand, L, cg, int(greedy_ctx), int(skip), cap, C.byref(p), C.byref(out))
    return out


def enumerate_chains(drafts, cap=64):
    drafts = np.ascontiguousarray(np.atleast_2d(drafts), np.int32)
    n_cand, L = drafts.shape
    chains = np.zeros((cap, L), np.int32)
    a = np.zeros(cap, np.int32)
    b = np.zeros(cap, np.int32)
    n = lib().hsdo_enumerate_chains(drafts, n_cand, L, cap, chains, a, b)
    return chains[:n], a[:n], b[:n]


def calibrate(sims_list, T):
    c = Calib()
    lib().hsdo_calibrate_init(C.byref(c))
    for s in sims_list:
        s = np.ascontiguousarray(s, np.float64)
        lib().hsdo_calibrate_accumulate(C.byref(c), s, s.shape[0], T)
    m = C.c_double()
    o = C.c_int()
    rc = lib().hsdo_calibrate_finish(C.byref(c), C.byref(m), C.byref(o))
    if rc < 0:
        return None
    return m.value, o.value


def update_skip_state(state: SkipState, success: bool, S_c: float, min_S_h: float) -> SkipState:
    lib().hsdo_update_skip_state(C.byref(state), int(success), S_c, min_S_h)
    return state


def project_window(xyz):
    xyz = np.ascontiguousarray(xyz, np.float64)
    uv = np.zeros((xyz.shape[0], 2), np.float64)
    rc = lib().hsdo_project_window(xyz, xyz.shape[0], uv)
    if rc < 0:
        raise ValueError(rc)
    return uv


def fit_circle_center(uv):
    uv = np.ascontiguousarray(uv, np.float64)
    cu, cv = C.c_double(), C.c_double()
    deg, it = C.c_int(), C.c_int()
    rc = lib().hsdo_fit_circle_center(uv, uv.shape[0], C.byref(cu), C.byref(cv), C.byref(deg), C.byref(it))
    if rc < 0:
        raise ValueError(rc)
    return (cu.value, cv.value), bool(deg.value), it.value


def curvature_radius(xyz, r_cap=1.0) -> float:
    xyz = np.ascontiguousarray(xyz, np.float64)
    R = C.c_double()
    rc = lib().hsdo_curvature_radius(xyz, xyz.shape[0], r_cap, C.byref(R))
    if rc < 0:
        raise ValueError(rc)
    return R.value


def cumulative_displacement(xyz) -> float:
    xyz = np.ascontiguousarray(xyz, np.float64)
    D = C.c_double()
    rc = lib().hsdo_cumulative_displacement(xyz, xyz.shape[0], C.byref(D))
    if rc < 0:
        raise ValueError(rc)
    return D.value


def normalize(x, lo, hi95) -> float:
    return lib().hsdo_normalize(x, lo, hi95)


def percentile_bounds(samples):
    s = np.ascontiguousarray(samples, np.float64)
    lo, hi = C.c_double(), C.c_double()
    rc = lib().hsdo_percentile_bounds(s, s.size, C.byref(lo), C.byref(hi))
    if rc < 0:
        raise ValueError(rc)
    return lo.value, hi.value


def fused_metric(R, D, params: MetricParams, bounds: NormBounds) -> float:
    return lib().hsdo_fused_metric(R, D, C.byref(params), C.byref(bounds))


def window_features(xyz, params: MetricParams, bounds: NormBounds):
    xyz = np.ascontiguousarray(xyz, np.float64)
    R, D, F = C.c_double(), C.c_double(), C.c_double()
    dec = C.c_int()
    rc = lib().hsdo_window_features(xyz, xyz.shape[0], C.byref(params), C.byref(bounds), C.byref(R), C.byref(D),
                                    C.byref(F), C.byref(dec))
    if rc < 0:
        raise ValueError(rc)
    return R.value, D.value, F.value, dec.value


def ref_search(col, queries: np.ndarray, k: int, threads: int = 1):
    """Reference Collection::search_topk_exact over fp32 queries widened to fp64."""
    q = np.ascontiguousarray(np.atleast_2d(queries), np.float32)
    B, dim = q.shape
    sc = np.zeros((B, k), np.float64)
    ids = np.full((B, k), -1, np.int32)
    tok = np.zeros((B, k, 21), np.uint8)
    rc = ref().hsdref_search_batch(col, q, B, dim, k, threads, sc, ids, tok.ctypes.data)
    if rc < 0:
        raise RuntimeError(f"reference search failed: {rc}")
    n = ref().hsdref_collection_size(col)
    kk = min(k, n)
    return sc[:, :kk], ids[:, :kk], tok[:, :kk]


def window_derivatives(xyz) -> np.ndarray:
    """Mean |velocity|, |acceleration|, |jerk| per step of one window (hsdo_window_derivatives)."""
    x = np.ascontiguousarray(xyz, np.float64)
    out = np.zeros(3, np.float64)
    lib().hsdo_window_derivatives(x.ctypes.data_as(C.c_void_p), x.shape[0], out.ctypes.data_as(C.c_void_p))
    return out


# ---- approximate index (IVF-flat) restatement ----------------------------------
# The product's device index (paper_2603_17573_b200/csrc/k_ivf.cu) stands in for
# the reference's HNSW behind Collection::build_hnsw / search_topk
# (store.cpp:75-92).  HNSW's graph has no bit-level counterpart, so the oracle
# pins the index's own definition: exact assignment of every record to its best
# centroid (the reference's score and (score desc, id asc) order, store.cpp:59-73),
# the stable list order, normalized list means, and search_topk's contract that
# returned scores are the reference's cosine_similarity of the returned ids
# (store.cpp:86-90).

def ivf_seed_rows(n: int, nlist: int) -> np.ndarray:
    """Row floor((2l + 1) n / (2 nlist)) of each of nlist strata (k_ivf.cu ivf_seed_kernel)."""
    l = np.arange(nlist, dtype=np.float64)
    return ((2.0 * l + 1.0) * float(n) / (2.0 * nlist)).astype(np.int64)


def ivf_assign(keys: np.ndarray, cent: np.ndarray) -> np.ndarray:
    """Best centroid of every row by the reference's exact search (row = query)."""
    _, ids = search_topk(cent, keys, 1)
    return ids[:, 0].astype(np.int32)


def ivf_lists(assign: np.ndarray, nlist: int):
    """Stable counting sort: offs [nlist + 1], perm (record ids, ascending within a list)."""
    counts = np.bincount(assign, minlength=nlist)
    offs = np.zeros(nlist + 1, np.int32)
    offs[1:] = np.cumsum(counts)
    perm = np.argsort(assign, kind="stable").astype(np.int32)
    return offs, perm


def ivf_centroids(keys: np.ndarray, offs: np.ndarray, perm: np.ndarray, old: np.ndarray) -> np.ndarray:
    """List means normalized to unit length (fp64 sums, fp32 result); empty lists keep the old centroid."""
    out = old.astype(np.float32).copy()
    for l in range(len(offs) - 1):
        rows = perm[offs[l]:offs[l + 1]]
        if len(rows) == 0:
            continue
        s = keys[rows].astype(np.float64).sum(axis=0)
        nrm = np.sqrt((s * s).sum())
        if nrm > 0 and np.isfinite(nrm):
            out[l] = (s / nrm).astype(np.float32)
    return out


def ivf_build(keys: np.ndarray, nlist: int, n_iter: int):
    """The whole build on the CPU (small cases): (centroids, offs, perm)."""
    keys = np.ascontiguousarray(keys, np.float32)
    n = keys.shape[0]
    nlist = min(nlist, n)
    seeds = keys[ivf_seed_rows(n, nlist)].astype(np.float64)
    nrm = np.sqrt((seeds * seeds).sum(axis=1, keepdims=True))
    cent = np.where(nrm > 0, seeds / np.where(nrm > 0, nrm, 1.0), 0.0).astype(np.float32)
    for it in range(n_iter + 1):
        offs, perm = ivf_lists(ivf_assign(keys, cent), nlist)
        if it == n_iter:
            break
        cent = ivf_centroids(keys, offs, perm, cent)
    return cent, offs, perm


def ivf_search_lists(keys: np.ndarray, offs: np.ndarray, perm: np.ndarray, probes: np.ndarray,
                     queries: np.ndarray, k: int):
    """Exact top-k of each query over the rows of its probed lists: ids are
    record ids, scores the reference's sequential fp64 sum (store.cpp:29-34)."""
    queries = np.ascontiguousarray(np.atleast_2d(queries), np.float32)
    B = queries.shape[0]
    sc = np.full((B, k), -np.inf, np.float64)
    ids = np.full((B, k), -1, np.int64)
    for b in range(B):
        rows = np.sort(np.concatenate([perm[offs[l]:offs[l + 1]] for l in set(int(p) for p in probes[b])]))
        if len(rows) == 0:
            continue
        s, i = search_topk(keys[rows], queries[b:b + 1], k)
        m = s.shape[1]
        sc[b, :m] = s[0]
        ids[b, :m] = rows[i[0]]
    return sc, ids
