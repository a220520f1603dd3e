"""Host-side synthetic workload pieces that are uploaded rather than generated
on the device: trajectory windows for the kinematic metric,
and the host mirror of hsd_query_row (include/hsd/hsd_synth.h) used to build
verifier logits whose greedy tokens track the query's source record.
"""
from __future__ import annotations

import numpy as np

_M = (1 << 64) - 1
TAG_QPICK = 8


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M
    return x ^ (x >> 31)


def _stream_base(seed: int, tag: int) -> int:
    return _splitmix64((seed * 0xD1342543DE82EF95 + tag * 0x2545F4914F6CDD1D) & _M)


def _hash_at(base: int, idx: int) -> int:
    return _splitmix64(base ^ ((idx * 0x9E3779B97F4A7C15) & _M))


def query_rows(q_seed: int, kind: int, n_rows: int, q0: int, B: int) -> np.ndarray:
    base = _stream_base(q_seed, TAG_QPICK)
    out = np.full(B, -1, np.int64)
    for b in range(B):
        h = _hash_at(base, q0 + b)
        sel = h & 0xFF
        hit = sel < 64 if kind == 0 else sel < 128
        if hit and n_rows > 0:
            out[b] = (h >> 8) % n_rows
    return out


KINDS = ("circle", "line", "helix", "stationary", "walk", "near_collinear")


def trajectory_windows(W: int, w: int = 15, seed: int = 4, kinds=KINDS) -> tuple[np.ndarray, np.ndarray]:
    """W windows of w xyz points (float64 [W, w, 3]) mixing the shapes the
    kinematic metric must separate: circle arcs (r in [.01, .5]), straight
    transport lines, helices, stationary grippers, noisy random walks and
    near-collinear arcs (SURVEY.md §8(d) 'Trajectories').  Returns (xyz, kind_index)."""
    rng = np.random.default_rng(seed)
    out = np.empty((W, w, 3), np.float64)
    kidx = np.empty(W, np.int32)
    for i in range(W):
        k = i % len(kinds)
        kind = kinds[k]
        kidx[i] = k
        c = rng.uniform(-0.5, 0.5, 3)
        Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        t = np.arange(w, dtype=np.float64)
        if kind == "circle":
            r = rng.uniform(0.01, 0.5)
            arc = rng.uniform(0.3, 2 * np.pi)
            ph = rng.uniform(0, 2 * np.pi)
            th = ph + t * arc / (w - 1)
            p = np.stack([r * np.cos(th), r * np.sin(th), np.zeros(w)], 1)
        elif kind == "line":
            step = rng.uniform(0.001, 0.02)
            p = np.stack([t * step, np.zeros(w), np.zeros(w)], 1)
        elif kind == "helix":
            r = rng.uniform(0.02, 0.1)
            th = t * rng.uniform(0.1, 0.5)
            p = np.stack([r * np.cos(th), r * np.sin(th), t * rng.uniform(0.001, 0.005)], 1)
        elif kind == "stationary":
            p = np.zeros((w, 3))
        elif kind == "walk":
            p = np.cumsum(rng.normal(0, 0.005, (w, 3)), 0)
        else:  # near-collinear arc: radius >> window extent
            r = rng.uniform(2.0, 20.0)
            th = t * 0.01 / r
            p = np.stack([r * np.sin(th), r * (1 - np.cos(th)), np.zeros(w)], 1)
        out[i] = p @ Q.T + c
    return out, kidx
