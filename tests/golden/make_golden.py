"""Generate golden fixtures from the REFERENCE implementation itself.

Runs the reference's unmodified store.cpp / actions.cpp (compiled in place
into oracle/_ref/libhsdref.so by oracle/Makefile) on counter-generated inputs
and records its outputs as small .npz fixtures.  These pin the C restatement
(oracle/hsd_oracle.c) and, through it, the GPU path; they are committed so the
parity chain survives on hosts without /root/reference.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402


def search_fixture(name, kind, n, dim, B, k, db_seed, q_seed):
    R = O.ref()
    col = R.hsdref_collection_new(dim)
    rc = R.hsdref_insert_synth(col, kind, db_seed, 0, n, dim)
    assert rc == 0, rc
    q = O.gen_queries(kind, q_seed, db_seed, n, 0, B, dim)
    sc, ids, tok = O.ref_search(col, q, k, threads=8)
    R.hsdref_collection_free(col)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), kind=kind, n=n, dim=dim, B=B, k=k, db_seed=db_seed,
                        q_seed=q_seed, scores=sc, ids=ids, tokens=tok)
    print(name, sc.shape, ids[:2])


def quantize_fixture():
    rng = np.random.default_rng(7)
    acts = np.concatenate([
        rng.uniform(-1.5, 1.5, size=(2000, 7)),
        np.array([[-1.0] * 7, [1.0] * 7, [0.0] * 7, [1.0 - 1e-16] * 7, [-1.0 + 1e-16] * 7]),
        (np.arange(256)[:, None] / 255.0 * 2.0 - 1.0).repeat(7, axis=1),
    ])
    lo = np.full(7, -1.0)
    hi = np.full(7, 1.0)
    bins = np.zeros((acts.shape[0], 7), np.int32)
    out = np.zeros(7, np.int32)
    for i, a in enumerate(acts):
        rc = O.ref().hsdref_quantize(np.ascontiguousarray(a), lo, hi, 256, out)
        assert rc == 0
        bins[i] = out
    # non-uniform bounds
    lo2 = np.array([-0.9375, -0.9375, -0.9375, -0.1875, -0.1875, -0.1875, 0.0])
    hi2 = np.array([0.9375, 0.9375, 0.9375, 0.1875, 0.1875, 0.1875, 1.0])
    bins2 = np.zeros_like(bins)
    for i, a in enumerate(acts):
        O.ref().hsdref_quantize(np.ascontiguousarray(a), lo2, hi2, 256, out)
        bins2[i] = out
    np.savez_compressed(os.path.join(HERE, "quantize.npz"), acts=acts, bins=bins, lo2=lo2, hi2=hi2, bins2=bins2)
    print("quantize", bins.shape)


if __name__ == "__main__":
    assert O.ref_available(), "build oracle/_ref first: make -C oracle"
    search_fixture("search_exact_64", O.EXACT, 3000, 64, 24, 10, 11, 12)
    search_fixture("search_real_64", O.REAL, 3000, 64, 24, 10, 21, 22)
    search_fixture("search_exact_4096", O.EXACT, 2500, 4096, 8, 8, 31, 32)
    search_fixture("search_real_4096", O.REAL, 2500, 4096, 8, 8, 41, 42)
    quantize_fixture()
