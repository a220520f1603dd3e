"""GPU side of DB ingest: a JSONL v1 file loaded straight into HBM searches
exactly like the reference Collection it describes; the binary device image
round-trips bit for bit."""
import json

import numpy as np
import pytest

import paper_2603_17573_b200 as H
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


def write_db(path, rng, n, dim):
    with open(path, "w") as f:
        f.write(json.dumps({"version": 1, "name": "t", "dim": dim, "metric": "cosine"}) + "\n")
        for i in range(n):
            rec = {"embedding": [float(x) for x in rng.standard_normal(dim)],
                   "payload": {"dataset_name": "d", "episode_idx": i // 50, "step_idx": i % 50,
                               "current_action": [0.0] * 7,
                               "next_actions": [[float(x) for x in rng.uniform(-1.2, 1.2, 7)] for _ in range(3)],
                               "language_instruction": "x"},
                   "feature": None}
            f.write(json.dumps(rec) + "\n")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_jsonl_to_hbm_search_matches_reference(torch, tmp_path, dtype):
    rng = np.random.default_rng(4)
    n, dim = 1500, 64
    path = str(tmp_path / "db.jsonl")
    write_db(path, rng, n, dim)
    col = H.load_jsonl(path, dtype=dtype)
    assert col.size() == n and col.dim() == dim
    db = H.jsonl_read(path)
    keys = db["embedding"] if dtype == "f32" else torch.as_tensor(db["embedding"]).bfloat16().float().numpy()
    q = torch.as_tensor(rng.standard_normal((37, dim)).astype(np.float32), device="cuda")
    sc, ids = col.search_topk_exact(q, 8)
    osc, oid = O.search_topk(keys, q.cpu().numpy(), 8)
    np.testing.assert_array_equal(ids.cpu().numpy(), oid)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    # payload tokens = quantize(next_actions) (actions.cpp:32-50), as insert does
    _, toks = col.keys_view()
    lo, hi = np.full(7, -1.0), np.full(7, 1.0)
    for r in (0, 17, n - 1):
        for s in range(3):
            np.testing.assert_array_equal(toks[r, s * 7:(s + 1) * 7].cpu().numpy(),
                                          O.quantize(db["next_actions"][r, s], lo, hi, 256)[1])
    # binary device image round trip
    img = str(tmp_path / "db.img")
    col.save_image(img)
    col2 = H.load_image(img)
    assert col2.size() == n and col2.dtype == col.dtype
    k1, t1 = col.keys_view()
    k2, t2 = col2.keys_view()
    assert torch.equal(k1.view(torch.int16) if dtype == "bf16" else k1, k2.view(torch.int16) if dtype == "bf16" else k2)
    assert torch.equal(t1, t2)
    sc2, ids2 = col2.search_topk_exact(q, 8)
    assert torch.equal(ids, ids2) and torch.equal(sc, sc2)


def test_image_errors(torch, tmp_path):
    bad = tmp_path / "bad.img"
    bad.write_bytes(b"NOTANIMG" + bytes(64))
    with pytest.raises(H.ParseError):
        H.load_image(str(bad))
    with pytest.raises(H.IoError):
        H.load_image(str(tmp_path / "missing.img"))


def test_jsonl_features_reach_the_device_and_calibrate(torch, tmp_path):
    """Record::feature (store.hpp:40-42) travels with the records: the device feature table equals the file's
    features (fp32), absent features stay zero, and offline Alg. 1 runs on it."""
    rng = np.random.default_rng(6)
    n, dim, d_f = 120, 16, 32
    path = str(tmp_path / "f.jsonl")
    feats = rng.standard_normal((n, d_f))
    feats /= np.linalg.norm(feats, axis=1, keepdims=True)
    with open(path, "w") as f:
        f.write(json.dumps({"version": 1, "name": "t", "dim": dim, "metric": "cosine"}) + "\n")
        for i in range(n):
            rec = {"embedding": [float(x) for x in rng.standard_normal(dim)],
                   "payload": {"dataset_name": "d", "episode_idx": i // 40, "step_idx": i % 40,
                               "current_action": [0.0] * 7, "next_actions": [[0.0] * 7] * 3,
                               "language_instruction": "x"},
                   "feature": None if i == 5 else [float(x) for x in feats[i]]}
            f.write(json.dumps(rec) + "\n")
    col = H.load_jsonl(path)
    fv = col.features()
    assert fv is not None
    ft, has = fv[0].cpu().numpy(), fv[1].cpu().numpy()
    want = feats.astype(np.float32)
    want[5] = 0
    np.testing.assert_array_equal(ft, want)
    assert has[5] == 0 and has.sum() == n - 1
    off = np.array([0, 40, 80, 120], np.int64)
    got = H.calibrate_skip(fv[0], off, T=-1.0)
    sims = [np.array([[O.feature_cos(want[a + i], want[a + j]) for j in range(40)] for i in range(40)])
            for a in (0, 40, 80)]
    assert got == O.calibrate(sims, -1.0)
    with pytest.raises(H.SchemaError):
        col.set_features(np.zeros((1, d_f + 1), np.float32), row0=0)
