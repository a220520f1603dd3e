"""paper_2603_17573_b200 — B200-native HeiSD retrieval-side speculative-decoding hot path.

Python mirror of the C ABI in include/hsd/hsd_gpu.h (the drop-in boundary for
the reference's C++ API in proj/include/hsd).  The compute
lives in libhsd_gpu.so (hand-written sm_100a CUDA, built in-tree by
``__graft_entry__.build()``); this module only marshals pointers.  There is no
CPU fallback: if the shared library is missing the import fails, and every
compute call without an sm_100 device raises NoDeviceError.

Names follow the reference: Collection.insert / search_topk_exact
(store.hpp:59-96), quantize (actions.hpp:55), window_features /
classify_segment (kinematics.hpp:88-93), and the SPEC names for the spec-only
verification ops (verify_round ~ retrieve_drafts + should_skip + verify_tree).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhsd_gpu.so")

HSD_K_MAX = 32
TOKENS_STRIDE = 32
EXACT, REAL, CLUSTER = 0, 1, 2
F32, BF16 = 0, 1  # hsd_dtype (key storage)
_DTYPES = {"f32": F32, "fp32": F32, "float32": F32, F32: F32, "bf16": BF16, "bfloat16": BF16, BF16: BF16}


# --------------------------------------------------------------------------- errors
class HsdError(RuntimeError):
    """hsd::Error (errors.hpp:10)."""


class InvalidInputError(HsdError, ValueError):
    pass


class ConfigError(HsdError, ValueError):
    pass


class SchemaError(HsdError, ValueError):
    pass


class IoError(HsdError):
    pass


class ParseError(HsdError):
    pass


class VersionError(HsdError):
    pass


class CalibrationError(HsdError):
    pass


class CudaError(HsdError):
    pass


class NcclError(HsdError):
    pass


class OutOfMemoryError(HsdError, MemoryError):
    pass


class NoDeviceError(HsdError):
    pass


_STATUS = {1: InvalidInputError, 2: ConfigError, 3: SchemaError, 4: IoError, 5: ParseError, 6: VersionError,
           7: CalibrationError, 100: CudaError, 101: NcclError, 102: OutOfMemoryError, 103: NoDeviceError}


# --------------------------------------------------------------------------- ABI structs
class VerifyParams(C.Structure):
    _fields_ = [("relaxed", C.c_int32), ("bias_seq_max", C.c_int32), ("bias_token_max", C.c_int32),
                ("skip_enabled", C.c_int32), ("min_S", C.c_double), ("O_dist", C.c_int32), ("chain_cap", C.c_int32)]

    @classmethod
    def make(cls, relaxed=True, bias_seq_max=30, bias_token_max=15, skip_enabled=False, min_S=0.95, O_dist=5,
             chain_cap=64):
        return cls(int(relaxed), bias_seq_max, bias_token_max, int(skip_enabled), float(min_S), O_dist, chain_cap)


class Outcome(C.Structure):
    _fields_ = [("accept_len", C.c_int32), ("win_a", C.c_int16), ("win_b", C.c_int16), ("calls", C.c_int16),
                ("fallback", C.c_int8), ("skipped", C.c_int8), ("n_emit", C.c_int16), ("greedy0", C.c_int16),
                ("cos_sim", C.c_float)]


OUTCOME_DTYPE = np.dtype([("accept_len", np.int32), ("win_a", np.int16), ("win_b", np.int16), ("calls", np.int16),
                          ("fallback", np.int8), ("skipped", np.int8), ("n_emit", np.int16), ("greedy0", np.int16),
                          ("cos_sim", np.float32)])
assert OUTCOME_DTYPE.itemsize == C.sizeof(Outcome) == 20


class MetricParams(C.Structure):
    _fields_ = [("alpha", C.c_double), ("w", C.c_int32), ("threshold", C.c_double), ("r_cap", C.c_double)]


class NormBounds(C.Structure):
    _fields_ = [("d_min", C.c_double), ("d_max95", C.c_double), ("r_min", C.c_double), ("r_max95", C.c_double)]


class HybridParams(C.Structure):
    """hsd_hybrid_params (include/hsd/hsd_gpu.h): HybridConfig + CostModel of the SPEC scheduler."""
    _fields_ = [(n, C.c_int32) for n in ("robots", "k", "mode", "traj_T", "drafter_p_pct", "drafter_L", "gap_d",
                                         "d_f")] + [
        ("seed", C.c_uint64), ("db_seed", C.c_uint64), ("key_kind", C.c_int32), ("record_trace", C.c_int32),
        ("verify", VerifyParams), ("metric", MetricParams), ("bounds", NormBounds), ("cost_verifier", C.c_double),
        ("cost_drafter_token", C.c_double), ("cost_retrieval", C.c_double)]


STEP_RECORD_DTYPE = np.dtype([("F", np.float32), ("accept_len", np.int16), ("verifier_calls", np.int16),
                              ("n_emit", np.int16), ("mode", np.int8), ("skipped", np.int8), ("cost", np.float32)])
EPISODE_REPORT_DTYPE = np.dtype([("rounds", np.int64), ("tokens", np.int64), ("accepted", np.int64),
                                 ("verifier_calls", np.int64), ("cost", np.float64), ("n_retrieval", np.int32),
                                 ("n_drafter", np.int32), ("n_skipped", np.int32), ("n_fallback", np.int32)])
MODE_HYBRID, MODE_PURE_RETRIEVAL, MODE_PURE_DRAFTER, MODE_AUTOREGRESSIVE = 0, 1, 2, 3
PAYLOAD_RANDOM, PAYLOAD_TRAJ = 0, 1


class IvfParams(C.Structure):
    _fields_ = [("nlist", C.c_int), ("n_iter", C.c_int)]


class SkipState(C.Structure):
    """hsd_skip_state: VerifySkipState."""
    _fields_ = [("T", C.c_double), ("min_S", C.c_double), ("O_dist", C.c_int32), ("delta", C.c_double),
                ("inverted", C.c_int32)]


class StepIO(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("queries", "logits", "feat_now", "feat_prev", "xyz", "history", "scores",
                                          "ids", "out", "tokens", "R", "D", "F", "decision")]


# LIBERO-Goal bounds and FusedMetricParams defaults (kinematics.hpp:38-45)
LIBERO_GOAL = NormBounds(0.000009, 0.123381, 0.000001, 0.014989)
DEFAULT_METRIC = MetricParams(0.5, 15, 0.5, 1.0)


# --------------------------------------------------------------------------- loader
_lib = None
_vp = C.c_void_p


def lib():
    """Load libhsd_gpu.so (fails loudly; there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing — build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the HeiSD hot path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.hsd_last_error.restype = C.c_char_p
    L.hsd_last_error_line.restype = C.c_long
    L.hsd_abi_version.restype = C.c_int
    sig = {
        "hsd_device_count": [C.POINTER(C.c_int)],
        "hsd_collection_create": [C.c_int, C.c_int, C.c_int64, C.POINTER(_vp)],
        "hsd_collection_create_ex": [C.c_int, C.c_int, C.c_int64, C.c_int, C.POINTER(_vp)],
        "hsd_collection_dtype": [_vp, C.POINTER(C.c_int)],
        "hsd_collection_set_filter": [_vp, C.c_int],
        "hsd_collection_get_filter": [_vp, C.POINTER(C.c_int)],
        "hsd_collection_data": [_vp, C.POINTER(_vp), C.POINTER(_vp)],
        "hsd_collection_destroy": [_vp],
        "hsd_collection_size": [_vp, C.POINTER(C.c_int64)],
        "hsd_collection_dim": [_vp, C.POINTER(C.c_int)],
        "hsd_collection_device": [_vp, C.POINTER(C.c_int)],
        "hsd_collection_keys": [_vp, C.POINTER(_vp), C.POINTER(_vp)],
        "hsd_collection_insert": [_vp, _vp, _vp, _vp, _vp, C.c_int64, C.POINTER(C.c_int64)],
        "hsd_collection_generate": [_vp, C.c_int, C.c_uint64, C.c_int64],
        "hsd_search_topk_exact": [_vp, _vp, C.c_int, C.c_int, _vp, _vp, _vp],
        "hsd_search_topk_range": [_vp, _vp, C.c_int, C.c_int, C.c_int64, C.c_int64, _vp, _vp, _vp],
        "hsd_search_overflow_count": [_vp, _vp, C.POINTER(C.c_int)],
        "hsd_search_stats": [_vp, _vp, C.c_int, C.POINTER(C.c_int * 3)],
        "hsd_engine_stats": [_vp, C.c_int, C.POINTER(C.c_int * 3)],
        "hsd_engine_stage_marks": [_vp, _vp, C.c_int, _vp, C.POINTER(C.c_int)],
        "hsd_collection_set_features": [_vp, C.c_int64, C.c_int64, C.c_int, _vp, _vp],
        "hsd_collection_features": [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(C.c_int)],
        "hsd_enumerate_chains": [_vp, C.c_int, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp],
        "hsd_verify_round_chains": [_vp, C.c_int, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp,
                                    _vp, C.c_int, _vp, C.c_int, C.POINTER(VerifyParams), _vp, _vp, _vp],
        "hsd_percentile_bounds": [C.c_int, _vp, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double), _vp],
        "hsd_norm_bounds_from_windows": [C.c_int, _vp, C.c_int, C.POINTER(MetricParams), C.POINTER(NormBounds), _vp],
        "hsd_verify_round": [_vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int, _vp, C.c_int, _vp, C.c_int,
                             _vp, _vp, _vp],
        "hsd_window_features": [C.c_int, _vp, C.c_int, C.POINTER(MetricParams), C.POINTER(NormBounds), _vp, _vp, _vp,
                                _vp, _vp, _vp],
        "hsd_quantize": [C.c_int, _vp, C.c_int64, _vp, _vp, C.c_int, _vp, _vp, _vp],
        "hsd_window_features_ex": [C.c_int, _vp, C.c_int, C.POINTER(MetricParams), C.POINTER(NormBounds), _vp, _vp,
                                   _vp, _vp, _vp, _vp, _vp],
        "hsd_engine_create": [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)],
        "hsd_engine_destroy": [_vp],
        "hsd_engine_enable_timing": [_vp, C.c_int],
        "hsd_engine_stage_times": [_vp, C.POINTER(C.c_int), C.POINTER(C.c_double * 5)],
        "hsd_step": [_vp, C.c_int, C.POINTER(StepIO), C.POINTER(VerifyParams), C.POINTER(MetricParams),
                     C.POINTER(NormBounds), C.c_int, _vp],
        "hsd_step_host": [_vp, C.c_int, C.POINTER(StepIO), C.POINTER(VerifyParams), C.POINTER(MetricParams),
                          C.POINTER(NormBounds), C.c_int, _vp],
        "hsd_step_host_async": [_vp, C.c_int, C.POINTER(StepIO), C.POINTER(VerifyParams), C.POINTER(MetricParams),
                                C.POINTER(NormBounds), C.c_int, _vp],
        "hsd_step_graph": [_vp, C.c_int, C.POINTER(StepIO), C.POINTER(VerifyParams), C.POINTER(MetricParams),
                           C.POINTER(NormBounds), C.c_int, _vp],
        "hsd_engine_sync": [_vp],
        "hsd_comm_unique_id": [_vp],
        "hsd_comm_create": [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)],
        "hsd_comm_destroy": [_vp],
        "hsd_comm_create_p2p": [C.c_int, C.c_int, C.c_int, C.POINTER(_vp)],
        "hsd_comm_p2p_export": [_vp, C.c_int, C.c_int, _vp],
        "hsd_comm_p2p_import": [_vp, _vp],
        "hsd_comm_p2p_status": [_vp, C.POINTER(C.c_int)],
        "hsd_shard_range": [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
        "hsd_search_topk_sharded": [_vp, _vp, C.c_int64, _vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp],
        "hsd_search_topk_sharded_ex": [_vp, _vp, C.c_int64, _vp, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int, _vp],
        "hsd_verify_round_drafts": [C.c_int, _vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int, _vp,
                                    C.c_int, _vp, C.c_int, _vp, _vp, _vp],
        "hsd_collection_generate_rows": [_vp, C.c_int, C.c_uint64, C.c_int64, C.c_int64],
        "hsd_debug_sim_scores": [_vp, _vp, C.c_int, C.c_int, _vp, _vp],
        "hsd_set_sim_path": [C.c_int],
        "hsd_search_plan": [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_void_p],
        "hsd_merge_topk": [C.c_int, _vp, _vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp],
        "hsd_gen_queries": [C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_int, C.c_int, _vp,
                            _vp],
        "hsd_gen_logits": [_vp, C.c_uint64, _vp, C.c_int, C.c_int, _vp, _vp],
        "hsd_gen_features": [C.c_int, C.c_uint64, C.c_int, C.c_int, _vp, _vp, _vp],
        "hsd_collection_generate_ex": [_vp, C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_int, C.c_int],
        "hsd_hybrid_create": [_vp, _vp, C.c_int64, C.c_int64, C.POINTER(HybridParams), C.c_int, C.POINTER(_vp)],
        "hsd_hybrid_destroy": [_vp],
        "hsd_hybrid_step": [_vp, C.c_int, _vp],
        "hsd_hybrid_positions": [_vp, _vp],
        "hsd_hybrid_reports": [_vp, _vp],
        "hsd_hybrid_trace": [_vp, _vp, C.POINTER(C.c_int)],
        "hsd_hybrid_counts": [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
        "hsd_hybrid_stage_times": [_vp, C.POINTER(C.c_int), C.POINTER(C.c_double * 5)],
        "hsd_jsonl_read": [C.c_char_p, C.c_int, C.POINTER(_vp)],
        "hsd_jsonl_free": [_vp],
        "hsd_jsonl_info": [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_char_p)],
        "hsd_jsonl_data": [_vp] + [C.POINTER(_vp)] * 6,
        "hsd_collection_from_jsonl": [_vp, C.c_int, C.c_int, C.POINTER(_vp)],
        "hsd_collection_load_jsonl": [C.c_char_p, C.c_int, C.c_int, C.POINTER(_vp)],
        "hsd_collection_save_image": [_vp, C.c_char_p],
        "hsd_calibrate_skip": [C.c_int, _vp, C.c_int, _vp, C.c_int, C.c_double, C.POINTER(C.c_double),
                               C.POINTER(C.c_int), _vp],
        "hsd_update_skip_state": [C.POINTER(SkipState), C.c_int, C.c_double, C.c_double],
        "hsd_collection_load_image": [C.c_char_p, C.c_int, C.POINTER(_vp)],
        "hsd_debug_last_cuda_error": [],
        "hsd_index_build": [_vp, C.POINTER(IvfParams), C.POINTER(_vp)],
        "hsd_index_destroy": [_vp],
        "hsd_index_info": [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_int), C.POINTER(C.c_int)],
        "hsd_index_lists": [_vp, _vp, _vp, _vp],
        "hsd_search_topk_index": [_vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    _lib = L
    return L


def check(status: int) -> None:
    if status != 0:
        msg = lib().hsd_last_error().decode(errors="replace")
        err = _STATUS.get(status, HsdError)(f"[hsd status {status}] {msg}")
        if status == 5:  # hsd::ParseError carries its line (errors.hpp:35-40)
            err.line_number = lib().hsd_last_error_line()
        raise err


def exported_symbols() -> list[str]:
    """Every entry point declared in include/hsd/hsd_gpu.h."""
    import re

    hdr = os.path.join(os.path.dirname(_HERE), "include", "hsd", "hsd_gpu.h")
    with open(hdr) as f:
        text = f.read()
    return sorted(set(re.findall(r"^(?:hsd_status|const char\*|int|long)\s+(hsd_\w+)\(", text, re.M)))


def device_count() -> int:
    n = C.c_int(0)
    check(lib().hsd_device_count(C.byref(n)))
    return n.value


# --------------------------------------------------------------------------- torch helpers
def _torch():
    import torch

    return torch


def _ptr(t):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


# --------------------------------------------------------------------------- Collection
class Collection:
    """Device-resident task shard; replaces hsd::Collection (store.hpp:59-96)."""

    def __init__(self, dim: int, capacity: int = 1, device: int = 0, dtype="f32"):
        """dtype: key storage, "f32" (default) or "bf16" (keys rounded once to bf16)."""
        self._h = C.c_void_p()
        if dtype not in _DTYPES:
            raise ConfigError(f"unknown key dtype {dtype!r}")
        self.dtype = _DTYPES[dtype]
        check(lib().hsd_collection_create_ex(device, dim, capacity, self.dtype, C.byref(self._h)))
        self.device = device
        self._dim = dim

    def close(self):
        idx = getattr(self, "_index", None)
        if idx is not None:  # the index refers to this collection's rows
            idx.close()
            self._index = None
        if self._h:
            lib().hsd_collection_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def dim(self) -> int:
        return self._dim

    def size(self) -> int:
        n = C.c_int64()
        check(lib().hsd_collection_size(self._h, C.byref(n)))
        return n.value

    def __len__(self):
        return self.size()

    def insert(self, embeddings, next_actions, episode_idx=None, step_idx=None) -> int:
        """Collection::insert (store.cpp:44-57) for a batch; returns the first id."""
        emb = np.ascontiguousarray(np.atleast_2d(embeddings), np.float32)
        act = np.ascontiguousarray(next_actions, np.float64).reshape(emb.shape[0], 21)
        if emb.shape[1] != self._dim:  # store.cpp:46-49
            raise SchemaError(f"embedding dim {emb.shape[1]} does not match collection dim {self._dim}")
        ep = None if episode_idx is None else np.ascontiguousarray(episode_idx, np.int32)
        st = None if step_idx is None else np.ascontiguousarray(step_idx, np.int32)
        first = C.c_int64()
        check(lib().hsd_collection_insert(self._h, emb.ctypes.data, act.ctypes.data,
                                          None if ep is None else ep.ctypes.data,
                                          None if st is None else st.ctypes.data, emb.shape[0], C.byref(first)))
        return first.value

    def generate(self, kind: int, db_seed: int, n: int, row0=None, payload=PAYLOAD_RANDOM, traj_T=0) -> None:
        """Append n counter-generated records; row0 selects global synthetic rows (DB shards);
        payload=PAYLOAD_TRAJ stores demonstration-policy drafts (row = e * traj_T + j)."""
        if payload != PAYLOAD_RANDOM:
            check(lib().hsd_collection_generate_ex(self._h, kind, db_seed, self.size() if row0 is None else row0, n,
                                                   payload, traj_T))
        elif row0 is None:
            check(lib().hsd_collection_generate(self._h, kind, db_seed, n))
        else:
            check(lib().hsd_collection_generate_rows(self._h, kind, db_seed, row0, n))

    def keys_view(self):
        """(keys, tokens) torch views of the resident arrays (keys float32 or bfloat16)."""
        torch = _torch()
        kp, tp = C.c_void_p(), C.c_void_p()
        check(lib().hsd_collection_data(self._h, C.byref(kp), C.byref(tp)))
        n = self.size()
        kt = torch.bfloat16 if self.dtype == BF16 else torch.float32
        keys = _from_ptr(kp.value, (n, self._dim), kt, self.device)
        toks = _from_ptr(tp.value, (n, TOKENS_STRIDE), torch.uint8, self.device)
        return keys, toks

    def search_topk_exact(self, queries, k: int, row_range=None, stream=None):
        """Batched Collection::search_topk_exact (store.cpp:59-73).

        queries: cuda float32 [B, dim] -> (scores float64 [B, k], ids int32 [B, k]).
        """
        torch = _torch()
        q = queries.contiguous()
        if q.dtype != torch.float32 or not q.is_cuda:
            raise InvalidInputError("queries must be a CUDA float32 tensor")
        if q.dim() == 1:
            q = q[None]
        if q.shape[1] != self._dim:
            raise InvalidInputError("embedding dim mismatch in cosine")  # store.cpp:30
        B = q.shape[0]
        kk = max(int(k), 1)
        scores = torch.empty((B, kk), dtype=torch.float64, device=q.device)
        ids = torch.empty((B, kk), dtype=torch.int32, device=q.device)
        if row_range is None:
            check(lib().hsd_search_topk_exact(self._h, _ptr(q), B, int(k), _ptr(scores), _ptr(ids), _stream(stream)))
        else:
            check(lib().hsd_search_topk_range(self._h, _ptr(q), B, int(k), int(row_range[0]), int(row_range[1]),
                                              _ptr(scores), _ptr(ids), _stream(stream)))
        return scores, ids

    # ---- approximate index (Collection::build_hnsw / search_topk, store.cpp:75-92) ----
    def build_hnsw(self, nlist: int = 1024, n_iter: int = 10, nprobe: int = 16) -> "Index":
        """Build the device approximate index (IVF-flat; the stand-in for the
        reference's HNSW) over the current records; search_topk then uses it
        until the next insert / generate (which makes it stale: exact again)."""
        self._index = Index(self, nlist=nlist, n_iter=n_iter)
        self._nprobe = int(nprobe)
        return self._index

    def has_hnsw(self) -> bool:
        idx = getattr(self, "_index", None)
        return idx is not None and not idx.info()["stale"]

    def search_topk(self, queries, k: int, stream=None):
        """Collection::search_topk (store.cpp:82-92): the index when built and
        current, else search_topk_exact."""
        if not self.has_hnsw():
            return self.search_topk_exact(queries, k, stream=stream)
        return self._index.search_topk(queries, k, nprobe=self._nprobe, stream=stream)

    def debug_sim_scores(self, queries, variant=1, stream=None):
        """Approximate tcgen05 filter scores float32 [B, size] (diagnostics; variant 1 = wide TF32/bf16
        filter of the default path, 2 = 64-query TF32, 3 = 3xTF32, 4 = the bf16 filter copy)."""
        torch = _torch()
        q = queries.contiguous()
        out = torch.empty((q.shape[0], self.size()), dtype=torch.float32, device=q.device)
        check(lib().hsd_debug_sim_scores(self._h, _ptr(q), q.shape[0], variant, _ptr(out), _stream(stream)))
        return out

    def set_filter(self, filter) -> None:
        """"native" (default) or "bf16_copy": keep a bf16 filter copy of fp32 keys (half the scan bytes; results
        stay bit-identical: the exact rescoring reads the fp32 keys)."""
        check(lib().hsd_collection_set_filter(self._h, {"native": 0, "bf16_copy": 1}.get(filter, filter)))

    def filter(self) -> str:
        f = C.c_int()
        check(lib().hsd_collection_get_filter(self._h, C.byref(f)))
        return "bf16_copy" if f.value == 1 else "native"

    def save_image(self, path: str) -> None:
        """Binary columnar device image (hsd_collection_save_image)."""
        check(lib().hsd_collection_save_image(self._h, os.fsencode(path)))

    def overflow_count(self, stream=None) -> int:
        """Queries that needed the exact range fallback on `stream` (results are exact either way)."""
        return self.search_stats(stream)["fallback_queries"]

    def set_features(self, features, has=None, row0=0) -> None:
        """Record::feature of records [row0, row0 + n) (host fp32 [n, d_f]; has uint8 [n] or None = all)."""
        f = np.ascontiguousarray(features, np.float32)
        h = None if has is None else np.ascontiguousarray(has, np.uint8)
        check(lib().hsd_collection_set_features(self._h, row0, f.shape[0], f.shape[1], f.ctypes.data_as(_vp),
                                                None if h is None else h.ctypes.data_as(_vp)))

    def features(self):
        """(features float32 [size, d_f], has uint8 [size]) device views, or None when no record carries one."""
        fp, hp, d = _vp(), _vp(), C.c_int()
        check(lib().hsd_collection_features(self._h, C.byref(fp), C.byref(hp), C.byref(d)))
        if not d.value:
            return None
        torch = _torch()
        n, dev = self.size(), self.device
        return (_from_ptr(fp.value, (n, d.value), torch.float32, dev), _from_ptr(hp.value, (n,), torch.uint8, dev))

    def search_plan(self, B: int, k: int, rows: int = -1) -> str:
        """The search path a batch of B queries takes: "scan" (K1x exact scan), "filter" (K1 + K2) or
        "filter_bf16_onchip" (K1 + K2, fp32 key tiles converted to bf16 on chip by the CTA-pair filter)."""
        v = C.c_int()
        check(lib().hsd_search_plan(self._h, int(B), int(k), int(rows), C.byref(v)))
        return {1: "scan", 2: "filter_bf16_onchip"}.get(v.value, "filter")

    def search_stats(self, stream=None, reset=False) -> dict:
        """Accumulated search statistics of `stream` (hsd_search_stats; synchronizes)."""
        v = (C.c_int * 3)()
        check(lib().hsd_search_stats(self._h, _stream(stream), int(reset), C.byref(v)))
        return {"fallback_queries": v[0], "candidates": v[1], "fallback_lists": v[2]}

    def verify_round(self, ids, logits, params, feat_now=None, feat_prev=None, history=None, gap_d=1, stream=None):
        """Fused gather + verify-skip + relaxed acceptance.

        ids int32 [E, k]; logits float32 [E, L, 256]; params: VerifyParams or a
        list (sweep).  Returns (outcomes structured np array [P, E], tokens
        uint8 tensor [P, E, L]).
        """
        torch = _torch()
        if isinstance(params, VerifyParams):
            params = [params]
        P = len(params)
        arr = (VerifyParams * P)(*params)
        ids = ids.contiguous()
        logits = logits.contiguous()
        E, k = ids.shape
        L = logits.shape[1]
        d_f = 0 if feat_now is None else feat_now.shape[1]
        out = torch.empty((P, E, C.sizeof(Outcome)), dtype=torch.uint8, device=ids.device)
        toks = torch.empty((P, E, L), dtype=torch.uint8, device=ids.device)
        check(lib().hsd_verify_round(self._h, _ptr(ids), E, k, L, _ptr(logits), _ptr(feat_now), _ptr(feat_prev), d_f,
                                     _ptr(history), gap_d, C.cast(arr, C.c_void_p), P, _ptr(out), _ptr(toks),
                                     _stream(stream)))
        o = out.cpu().numpy().view(OUTCOME_DTYPE).reshape(P, E)
        return o, toks


class Index:
    """IVF-flat approximate index over a Collection (hsd_index_*)."""

    def __init__(self, col: "Collection", nlist: int = 1024, n_iter: int = 10):
        self._col = col
        h = _vp()
        p = IvfParams(int(nlist), int(n_iter))
        check(lib().hsd_index_build(col.handle, C.byref(p), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().hsd_index_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        nl, n, ml, st = C.c_int(), C.c_int64(), C.c_int(), C.c_int()
        check(lib().hsd_index_info(self._h, C.byref(nl), C.byref(n), C.byref(ml), C.byref(st)))
        return {"nlist": nl.value, "n_rows": n.value, "max_list": ml.value, "stale": bool(st.value)}

    def lists(self):
        """(offs int32 [nlist+1], perm int32 [n], centroids float32 [nlist, dim]) on the host."""
        inf = self.info()
        offs = np.empty(inf["nlist"] + 1, np.int32)
        perm = np.empty(inf["n_rows"], np.int32)
        cent = np.empty((inf["nlist"], self._col._dim), np.float32)
        check(lib().hsd_index_lists(self._h, offs.ctypes.data, perm.ctypes.data, cent.ctypes.data))
        return offs, perm, cent

    def search_topk(self, queries, k: int, nprobe: int = 16, stream=None, return_probes=False):
        if not getattr(self, "_h", None) or not self._col._h:
            raise InvalidInputError("the index or its collection has been closed")
        torch = _torch()
        q = queries.contiguous()
        if q.dtype != torch.float32 or not q.is_cuda:
            raise InvalidInputError("queries must be a CUDA float32 tensor")
        if q.dim() == 1:
            q = q[None]
        if q.shape[1] != self._col._dim:
            raise InvalidInputError("embedding dim mismatch in cosine")  # store.cpp:30
        B = q.shape[0]
        kk = max(int(k), 1)
        scores = torch.empty((B, kk), dtype=torch.float64, device=q.device)
        ids = torch.empty((B, kk), dtype=torch.int32, device=q.device)
        probes = torch.full((B, max(int(nprobe), 1)), -1, dtype=torch.int32, device=q.device) if return_probes else None
        check(lib().hsd_search_topk_index(self._h, _ptr(q), B, int(k), int(nprobe), _ptr(scores), _ptr(ids),
                                          _ptr(probes) if probes is not None else None, _stream(stream)))
        if return_probes:
            return scores, ids, probes
        return scores, ids


def verify_round_drafts(ids, drafts, logits, params, feat_now=None, feat_prev=None, history=None, gap_d=1,
                        stream=None):
    """verify_round over pre-gathered draft records drafts uint8 [E, k, 32] (sharded search output)."""
    torch = _torch()
    if isinstance(params, VerifyParams):
        params = [params]
    P = len(params)
    arr = (VerifyParams * P)(*params)
    E, k = ids.shape
    L = logits.shape[1]
    d_f = 0 if feat_now is None else feat_now.shape[1]
    out = torch.empty((P, E, C.sizeof(Outcome)), dtype=torch.uint8, device=ids.device)
    toks = torch.empty((P, E, L), dtype=torch.uint8, device=ids.device)
    check(lib().hsd_verify_round_drafts(ids.device.index or 0, _ptr(ids), _ptr(drafts), E, k, L, _ptr(logits),
                                        _ptr(feat_now), _ptr(feat_prev), d_f, _ptr(history), gap_d,
                                        C.cast(arr, C.c_void_p), P, _ptr(out), _ptr(toks), _stream(stream)))
    return out.cpu().numpy().view(OUTCOME_DTYPE).reshape(P, E), toks


def enumerate_chains(ids, L, cap=64, col=None, drafts=None, stream=None):
    """The chains verify_tree visits (hsd_enumerate_chains): (n_chains int32 [E], chain_ab int16 [E, cap, 2],
    chain_tokens uint8 [E, cap, L]) — what a real verifier is run on."""
    torch = _torch()
    ids = ids.contiguous()
    E, k = ids.shape
    dev = ids.device
    n = torch.empty(E, dtype=torch.int32, device=dev)
    ab = torch.empty((E, cap, 2), dtype=torch.int16, device=dev)
    tok = torch.empty((E, cap, L), dtype=torch.uint8, device=dev)
    check(lib().hsd_enumerate_chains(col.handle if col is not None else None, dev.index or 0, _ptr(ids), _ptr(drafts),
                                     E, k, L, cap, _ptr(n), _ptr(ab), _ptr(tok), _stream(stream)))
    return n, ab, tok


def verify_round_chains(ids, params, greedy_ctx, chain_greedy=None, chain_logits=None, col=None, drafts=None,
                        feat_now=None, feat_prev=None, history=None, gap_d=1, stream=None):
    """verify_tree with per-chain teacher-forced verifier output (hsd_verify_round_chains): chain_greedy uint8
    [E, cap, L] or chain_logits float32 [E, cap, L, 256]; greedy_ctx int32 [E].  Returns (outcomes [E], tokens)."""
    torch = _torch()
    ids = ids.contiguous()
    E, k = ids.shape
    src = chain_greedy if chain_greedy is not None else chain_logits
    cap, L = src.shape[1], src.shape[2]
    d_f = 0 if feat_now is None else feat_now.shape[1]
    out = torch.empty((E, C.sizeof(Outcome)), dtype=torch.uint8, device=ids.device)
    toks = torch.empty((E, L), dtype=torch.uint8, device=ids.device)
    check(lib().hsd_verify_round_chains(col.handle if col is not None else None, ids.device.index or 0, _ptr(ids),
                                        _ptr(drafts), E, k, L, cap, _ptr(chain_greedy), _ptr(chain_logits),
                                        _ptr(greedy_ctx), _ptr(feat_now), _ptr(feat_prev), d_f, _ptr(history), gap_d,
                                        C.byref(params), _ptr(out), _ptr(toks), _stream(stream)))
    return out.cpu().numpy().view(OUTCOME_DTYPE).reshape(E), toks


def percentile_bounds(samples, stream=None):
    """compute_percentile_bounds (kinematics.cpp:238-247) of device fp64 samples -> (min, p95)."""
    samples = samples.contiguous()
    lo, hi = C.c_double(), C.c_double()
    check(lib().hsd_percentile_bounds(samples.device.index or 0, _ptr(samples), samples.numel(), C.byref(lo),
                                      C.byref(hi), _stream(stream)))
    return lo.value, hi.value


def norm_bounds_from_windows(xyz, params=None, stream=None) -> "NormBounds":
    """NormalizationBounds of a suite from its windows xyz fp64 [W, w, 3] (hsd_norm_bounds_from_windows)."""
    xyz = xyz.contiguous()
    mp = params if params is not None else DEFAULT_METRIC
    nb = NormBounds()
    check(lib().hsd_norm_bounds_from_windows(xyz.device.index or 0, _ptr(xyz), xyz.shape[0], C.byref(mp),
                                             C.byref(nb), _stream(stream)))
    return nb


class Comm:
    """NCCL communicator of a row-sharded DB (one process per GPU)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().hsd_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, uid, world: int, rank: int, device: int):
        """uid: an NCCL unique id (bytes) for the all-gather exchange, or None for a peer-memory-only
        communicator (call p2p_export / p2p_import before searching)."""
        self._h = C.c_void_p()
        if uid is None:
            check(lib().hsd_comm_create_p2p(world, rank, device, C.byref(self._h)))
        else:
            buf = (C.c_uint8 * 128).from_buffer_copy(uid)
            check(lib().hsd_comm_create(buf, world, rank, device, C.byref(self._h)))
        self.world, self.rank, self.device = world, rank, device

    def p2p_export(self, max_B: int, k_max: int) -> bytes:
        """CUDA IPC handle of this rank's receive window (all-gather it, then p2p_import)."""
        buf = (C.c_uint8 * 64)()
        check(lib().hsd_comm_p2p_export(self._h, max_B, k_max, buf))
        return bytes(buf)

    def p2p_import(self, handles) -> None:
        """handles: the world ranks' p2p_export() bytes, in rank order."""
        blob = b"".join(handles)
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        check(lib().hsd_comm_p2p_import(self._h, buf))

    def p2p_timed_out(self) -> bool:
        v = C.c_int()
        check(lib().hsd_comm_p2p_status(self._h, C.byref(v)))
        return bool(v.value)

    def close(self):
        if self._h:
            lib().hsd_comm_destroy(self._h)
            self._h = C.c_void_p()

    def search_topk(self, col: Collection, id_offset: int, queries, k: int, stream=None, out=None, reserve_sms=0):
        """Sharded search: local top-k + exchange + merge -> (scores, ids, drafts [B, k, 32]); `out` = preallocated
        (scores, ids, drafts); reserve_sms SMs are left to concurrent work on another stream."""
        torch = _torch()
        B = queries.shape[0]
        if out is None:
            out = (torch.empty((B, k), dtype=torch.float64, device=queries.device),
                   torch.empty((B, k), dtype=torch.int32, device=queries.device),
                   torch.empty((B, k, TOKENS_STRIDE), dtype=torch.uint8, device=queries.device))
        scores, ids, drafts = out
        check(lib().hsd_search_topk_sharded_ex(col.handle, self._h, id_offset, _ptr(queries), B, k, _ptr(scores),
                                               _ptr(ids), _ptr(drafts), reserve_sms, _stream(stream)))
        return scores, ids, drafts


def merge_topk(g_scores, g_ids, g_drafts=None, stream=None):
    """K3 device merge of G shard lists [G, B, k] (global ids) -> (scores, ids[, drafts]) [B, k]."""
    torch = _torch()
    G, B, k = g_ids.shape
    scores = torch.empty((B, k), dtype=torch.float64, device=g_ids.device)
    ids = torch.empty((B, k), dtype=torch.int32, device=g_ids.device)
    drafts = None if g_drafts is None else torch.empty((B, k, TOKENS_STRIDE), dtype=torch.uint8, device=g_ids.device)
    check(lib().hsd_merge_topk(g_ids.device.index or 0, _ptr(g_scores.contiguous()), _ptr(g_ids.contiguous()),
                               _ptr(None if g_drafts is None else g_drafts.contiguous()), G, B, k, _ptr(scores),
                               _ptr(ids), _ptr(drafts), _stream(stream)))
    return (scores, ids) if drafts is None else (scores, ids, drafts)


def _from_ptr(ptr, shape, dtype, device):
    """Non-owning torch view of device memory owned by the library."""
    torch = _torch()
    n = int(np.prod(shape))
    if n == 0:
        return torch.empty(shape, dtype=dtype, device=f"cuda:{device}")
    view_as = dtype
    if dtype == torch.bfloat16:  # numpy has no bf16: map as int16, reinterpret in torch
        dtype = torch.int16
    esz = torch.empty((), dtype=dtype).element_size()

    class _Arr:
        __cuda_array_interface__ = {"shape": (n,), "typestr": torch.empty((), dtype=dtype).numpy().dtype.str,
                                    "data": (ptr, False), "version": 3, "strides": (esz,)}

    return torch.as_tensor(_Arr(), device=f"cuda:{device}").view(view_as).view(shape)


# --------------------------------------------------------------------------- free functions
def window_features(xyz, params: MetricParams = DEFAULT_METRIC, bounds: NormBounds = LIBERO_GOAL, history=None,
                    stream=None, derivatives=False):
    """Batched window_features + classify_segment + decide_sd (kinematics.cpp:261-273).

    xyz: cuda float64 [W, w, 3] -> (R, D, F float64 [W], decision int32 [W]); with derivatives=True also
    vaj float64 [W, 3] = mean |velocity|, |acceleration|, |jerk| per step, computed in the same kernel.
    """
    torch = _torch()
    x = xyz.contiguous()
    if x.dtype != torch.float64:
        raise InvalidInputError("trajectory points must be float64")
    W, w = x.shape[0], x.shape[1]
    if w != params.w:
        raise InvalidInputError("window_features expects exactly w points")  # kinematics.cpp:264-266
    dev = x.device
    R = torch.empty(W, dtype=torch.float64, device=dev)
    D = torch.empty_like(R)
    F = torch.empty_like(R)
    dec = torch.empty(W, dtype=torch.int32, device=dev)
    if derivatives:
        vaj = torch.empty((W, 3), dtype=torch.float64, device=dev)
        check(lib().hsd_window_features_ex(dev.index or 0, _ptr(x), W, C.byref(params), C.byref(bounds),
                                           _ptr(history), _ptr(R), _ptr(D), _ptr(F), _ptr(dec), _ptr(vaj),
                                           _stream(stream)))
        return R, D, F, dec, vaj
    check(lib().hsd_window_features(dev.index or 0, _ptr(x), W, C.byref(params), C.byref(bounds), _ptr(history),
                                    _ptr(R), _ptr(D), _ptr(F), _ptr(dec), _stream(stream)))
    return R, D, F, dec


def quantize(actions, lo=-1.0, hi=1.0, k_bins=256, stream=None):
    """Batched quantize (actions.cpp:32-50): cuda float64 [n, 7] -> int32 bins [n, 7]."""
    torch = _torch()
    a = actions.contiguous()
    n = a.shape[0]
    lo7 = np.full(7, lo, np.float64) if np.isscalar(lo) else np.ascontiguousarray(lo, np.float64)
    hi7 = np.full(7, hi, np.float64) if np.isscalar(hi) else np.ascontiguousarray(hi, np.float64)
    bins = torch.empty((n, 7), dtype=torch.int32, device=a.device)
    status = torch.empty(n, dtype=torch.int32, device=a.device)
    check(lib().hsd_quantize(a.device.index or 0, _ptr(a), n, lo7.ctypes.data, hi7.ctypes.data, k_bins, _ptr(bins),
                             _ptr(status), _stream(stream)))
    if n and bool((status != 0).any()):
        raise InvalidInputError("non-finite action value")  # actions.cpp:38-40
    return bins


SIM_PATHS = {"auto": 0, "tc_single": 1, "filter": 2, "scan": 3}


def set_sim_path(name: str) -> None:
    """Search path switch: auto (cost model: exact scan of every row for small rows x batch, else the
    tensor-core filter + exact rescoring, CTA pairs above 128 queries) | tc_single (filter, single-CTA wide
    kernels only) | filter (filter + rescoring only) | scan (exact scan wherever it applies: B <= 4, k <= 32)."""
    check(lib().hsd_set_sim_path(SIM_PATHS[name]))


def classify_segment(F: float, threshold: float) -> str:
    """kinematics.cpp:257-259 (host helper; the device path fuses it into window_features)."""
    return "retrieval_sd" if F > threshold else "drafter_sd"


def gen_queries(kind, q_seed, db_seed, n_rows, q0, B, dim, device=0, stream=None):
    torch = _torch()
    out = torch.empty((B, dim), dtype=torch.float32, device=f"cuda:{device}")
    check(lib().hsd_gen_queries(device, kind, q_seed, db_seed, n_rows, q0, B, dim, _ptr(out), _stream(stream)))
    return out


def gen_logits(col: Collection, seed, rows, L, stream=None):
    torch = _torch()
    rows_t = torch.as_tensor(np.asarray(rows, np.int64), device=f"cuda:{col.device}")
    E = rows_t.numel()
    out = torch.empty((E, L, 256), dtype=torch.float32, device=f"cuda:{col.device}")
    check(lib().hsd_gen_logits(col.handle, seed, _ptr(rows_t), E, L, _ptr(out), _stream(stream)))
    return out


def gen_features(seed, E, d_f, device=0, stream=None):
    torch = _torch()
    now = torch.empty((E, d_f), dtype=torch.float32, device=f"cuda:{device}")
    prev = torch.empty_like(now)
    check(lib().hsd_gen_features(device, seed, E, d_f, _ptr(now), _ptr(prev), _stream(stream)))
    return now, prev


def query_rows(q_seed, kind, n_rows, q0, B):
    """Host mirror of hsd_query_row (include/hsd/hsd_synth.h): the DB row each synthetic query copies (-1 = none)."""
    from . import synth

    return synth.query_rows(q_seed, kind, n_rows, q0, B)


def shard_range(n_total, world, rank):
    b, e = C.c_int64(), C.c_int64()
    check(lib().hsd_shard_range(n_total, world, rank, C.byref(b), C.byref(e)))
    return b.value, e.value


# --------------------------------------------------------------------------- engine
@dataclass
class StepBuffers:
    """Caller-owned buffers of one decode round (device or pinned host)."""
    queries: object
    logits: object
    feat_now: object = None
    feat_prev: object = None
    xyz: object = None
    history: object = None
    scores: object = None
    ids: object = None
    out: object = None
    tokens: object = None
    R: object = None
    D: object = None
    F: object = None
    decision: object = None

    def io(self) -> StepIO:
        s = StepIO()
        for name, _ in StepIO._fields_:
            v = getattr(self, name)
            setattr(s, name, None if v is None else v.data_ptr())
        return s


class Engine:
    """Fused decode-round step (CS-5): kinematics -> search -> verify on one stream."""

    def __init__(self, col: Collection, max_B: int, k: int, L: int, d_f: int, w: int = 15):
        self._h = C.c_void_p()
        check(lib().hsd_engine_create(col.handle, max_B, k, L, d_f, w, C.byref(self._h)))
        self.col, self.max_B, self.k, self.L, self.d_f, self.w = col, max_B, k, L, d_f, w
        self._max_steps = 0

    def close(self):
        if self._h:
            lib().hsd_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def enable_timing(self, max_steps: int) -> None:
        check(lib().hsd_engine_enable_timing(self._h, max_steps))
        self._max_steps = max_steps

    def stage_marks(self, ref=None):
        """[n, 4] event times (ms) of the recorded steps (start, after similarity, after select, end) relative to
        the first recorded step of engine `ref` (default self)."""
        m = np.zeros((max(self._max_steps, 1), 4), np.float64)
        n = C.c_int()
        check(lib().hsd_engine_stage_marks(self._h, (ref or self)._h, m.shape[0], m.ctypes.data_as(_vp), C.byref(n)))
        return m[:n.value]

    def stage_times(self):
        """(steps, {stage: summed ms}) of the recorded steps (synchronizes)."""
        n = C.c_int()
        ms = (C.c_double * 5)()
        check(lib().hsd_engine_stage_times(self._h, C.byref(n), C.byref(ms)))
        names = ("kinematics", "similarity", "select", "verify", "total")
        return n.value, dict(zip(names, list(ms)))

    def step(self, B, bufs: StepBuffers, vp: VerifyParams, mp=DEFAULT_METRIC, nb=LIBERO_GOAL, gap_d=1, stream=None,
             graph=False):
        """One decode round on device buffers; graph=True replays a captured CUDA graph of the round (needs a
        non-default stream)."""
        io = bufs.io()
        fn = lib().hsd_step_graph if graph else lib().hsd_step
        check(fn(self._h, B, C.byref(io), C.byref(vp), C.byref(mp), C.byref(nb), gap_d, _stream(stream)))

    def step_host(self, B, bufs: StepBuffers, vp: VerifyParams, mp=DEFAULT_METRIC, nb=LIBERO_GOAL, gap_d=1,
                  stream=None):
        io = bufs.io()
        check(lib().hsd_step_host(self._h, B, C.byref(io), C.byref(vp), C.byref(mp), C.byref(nb), gap_d,
                                  _stream(stream)))

    def step_host_async(self, B, bufs: StepBuffers, vp: VerifyParams, mp=DEFAULT_METRIC, nb=LIBERO_GOAL, gap_d=1,
                        stream=None):
        """Enqueue one host-buffer step (pinned buffers; complete after sync())."""
        io = bufs.io()
        check(lib().hsd_step_host_async(self._h, B, C.byref(io), C.byref(vp), C.byref(mp), C.byref(nb), gap_d,
                                        _stream(stream)))

    def sync(self):
        check(lib().hsd_engine_sync(self._h))

    def search_stats(self, reset=False) -> dict:
        """The engine's accumulated search statistics (hsd_engine_stats; synchronizes the device)."""
        v = (C.c_int * 3)()
        check(lib().hsd_engine_stats(self._h, int(reset), C.byref(v)))
        return {"fallback_queries": v[0], "candidates": v[1], "fallback_lists": v[2]}


# --------------------------------------------------------------------------- hybrid loop (config 5)
def hybrid_params(robots, k=3, mode=MODE_HYBRID, traj_T=500, drafter_p_pct=85, drafter_L=7, gap_d=1, d_f=4096,
                  seed=1, db_seed=2026, key_kind=REAL, record_trace=True, verify=None, metric=None, bounds=None,
                  cost_verifier=1.0, cost_drafter_token=0.1, cost_retrieval=0.37) -> HybridParams:
    """HybridConfig defaults of the SPEC: K_top 3, p 0.85, L 7, relaxed 30/15,
    verify-skip min_S 0.95 / O_dist 5, cost 1.0 / 0.1 / 0.37."""
    if verify is None:
        verify = VerifyParams.make(relaxed=True, bias_seq_max=30, bias_token_max=15, skip_enabled=d_f > 0,
                                   min_S=0.95, O_dist=5)
    return HybridParams(robots, k, mode, traj_T, drafter_p_pct, drafter_L, gap_d, d_f, seed, db_seed, key_kind,
                        int(record_trace), verify, metric or DEFAULT_METRIC, bounds or LIBERO_GOAL, cost_verifier,
                        cost_drafter_token, cost_retrieval)


class HybridLoop:
    """Device-resident run_step / run_episode for many robots (hsd_hybrid_*)."""

    def __init__(self, col: Collection, params: HybridParams, n_total_rows=None, max_rounds=0, comm=None,
                 id_offset=0):
        self._h = C.c_void_p()
        self.params = params
        self.R = params.robots
        n_total = col.size() if n_total_rows is None else n_total_rows
        check(lib().hsd_hybrid_create(col.handle, None if comm is None else comm._h, id_offset, n_total,
                                      C.byref(params), max_rounds, C.byref(self._h)))
        self.col = col

    def close(self):
        if self._h:
            lib().hsd_hybrid_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, n_rounds=1, stream=None):
        check(lib().hsd_hybrid_step(self._h, n_rounds, _stream(stream)))

    def positions(self):
        out = np.zeros((self.R, 3), np.float64)
        check(lib().hsd_hybrid_positions(self._h, out.ctypes.data))
        return out

    def reports(self):
        out = np.zeros(self.R, EPISODE_REPORT_DTYPE)
        check(lib().hsd_hybrid_reports(self._h, out.ctypes.data))
        return out

    def trace(self):
        n = C.c_int()
        check(lib().hsd_hybrid_trace(self._h, None, C.byref(n)))
        out = np.zeros(n.value * self.R, STEP_RECORD_DTYPE)
        check(lib().hsd_hybrid_trace(self._h, out.ctypes.data if n.value else None, C.byref(n)))
        return out.reshape(n.value, self.R)

    def counts(self):
        a, b = C.c_int64(), C.c_int64()
        check(lib().hsd_hybrid_counts(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def stage_times(self):
        """{decide, search, verify, emit, total} ms per round (CUDA events) since the last call."""
        n, ms = C.c_int(), (C.c_double * 5)()
        check(lib().hsd_hybrid_stage_times(self._h, C.byref(n), C.byref(ms)))
        names = ("decide", "search", "verify", "emit", "total")
        return n.value, {k: v / max(n.value, 1) for k, v in zip(names, ms)}


# --------------------------------------------------------------------------- DB ingest (JSONL v1)
def jsonl_read(path: str, threads: int = 0) -> dict:
    """Host-side native parse of a reference JSONL v1 DB file (load_collection, store.cpp:152-191)."""
    h = C.c_void_p()
    check(lib().hsd_jsonl_read(os.fsencode(path), threads, C.byref(h)))
    try:
        n, dim, d_f, name = C.c_int64(), C.c_int(), C.c_int(), C.c_char_p()
        check(lib().hsd_jsonl_info(h, C.byref(n), C.byref(dim), C.byref(d_f), C.byref(name)))
        ptrs = [C.c_void_p() for _ in range(6)]
        check(lib().hsd_jsonl_data(h, *[C.byref(p) for p in ptrs]))
        n, dim, d_f = n.value, dim.value, d_f.value

        def arr(p, ct, shape):
            cnt = int(np.prod(shape))
            if not p.value or cnt == 0:
                return np.zeros(shape, np.dtype(ct))
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), (cnt,)).reshape(shape).copy()

        out = {"name": (name.value or b"").decode(), "n": n, "dim": dim, "d_f": d_f,
               "embedding": arr(ptrs[0], C.c_float, (n, dim)), "next_actions": arr(ptrs[1], C.c_double, (n, 3, 7)),
               "episode_idx": arr(ptrs[2], C.c_int32, (n,)), "step_idx": arr(ptrs[3], C.c_int32, (n,)),
               "feature": arr(ptrs[4], C.c_float, (n, d_f)) if d_f else None,
               "has_feature": arr(ptrs[5], C.c_uint8, (n,))}
        return out
    finally:
        lib().hsd_jsonl_free(h)


def _wrap_handle(h, device) -> Collection:
    col = Collection.__new__(Collection)
    col._h = h
    col.device = device
    d, t = C.c_int(), C.c_int()
    check(lib().hsd_collection_dim(h, C.byref(d)))
    check(lib().hsd_collection_dtype(h, C.byref(t)))
    col._dim, col.dtype = d.value, t.value
    return col


def load_jsonl(path: str, device: int = 0, dtype="f32") -> Collection:
    """load_collection (store.cpp:152-191) straight into HBM."""
    h = C.c_void_p()
    check(lib().hsd_collection_load_jsonl(os.fsencode(path), device, _DTYPES[dtype], C.byref(h)))
    return _wrap_handle(h, device)


def load_image(path: str, device: int = 0) -> Collection:
    """Reload a binary device image written by Collection.save_image."""
    h = C.c_void_p()
    check(lib().hsd_collection_load_image(os.fsencode(path), device, C.byref(h)))
    return _wrap_handle(h, device)


# --------------------------------------------------------------------------- verify-skip lifecycle (Alg. 1)
def calibrate_skip(features, offsets, T=0.9, stream=None):
    """offline_calibrate_skip: features cuda float32 [n, d_f], offsets int [n_traj + 1]
    (trajectory t = rows offsets[t]:offsets[t+1]) -> (min_S, O_dist); CalibrationError when no pair exceeds T."""
    f = features.contiguous()
    off = np.ascontiguousarray(offsets, np.int64)
    ms, od = C.c_double(), C.c_int()
    check(lib().hsd_calibrate_skip(f.device.index or 0, _ptr(f), f.shape[1], off.ctypes.data, off.size - 1,
                                   float(T), C.byref(ms), C.byref(od), _stream(stream)))
    return ms.value, od.value


def update_skip_state(state: SkipState, success: bool, S_c: float, min_S_h: float) -> SkipState:
    """update_skip_state, in place; returns the state."""
    check(lib().hsd_update_skip_state(C.byref(state), int(success), float(S_c), float(min_S_h)))
    return state


def trajectory_offsets(episode_idx) -> np.ndarray:
    """Offsets of maximal runs of equal episode_idx (per-episode feature lists in DB order)."""
    e = np.asarray(episode_idx)
    if e.size == 0:
        return np.zeros(1, np.int64)
    cuts = np.flatnonzero(np.diff(e) != 0) + 1
    return np.concatenate([[0], cuts, [e.size]]).astype(np.int64)
