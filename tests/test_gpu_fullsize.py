"""Full-size parity of the headline path (BASELINE config 2: 1M x 4096, B = 64)
and of the >128-query CTA-pair filter at 1M rows, bit-exact (ids and fp64
score bits) against the streaming CPU oracle on a sample of queries, plus
size-independent properties on every query.  ~25 GB of HBM per case."""
import numpy as np
import pytest

import paper_2603_17573_b200 as H
from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N, DIM, SEED = 1_000_000, 4096, 2026
SAMPLE16 = [0, 1, 2, 3, 5, 8, 13, 17, 21, 31, 34, 40, 48, 55, 60, 63]


@pytest.fixture(scope="module")
def torch():
    import torch

    return torch


def props(sc, ids, B, q_seed, family=O.REAL):
    s, i = sc.cpu().numpy(), ids.cpu().numpy()
    assert np.all((s[:, :-1] > s[:, 1:]) | ((s[:, :-1] == s[:, 1:]) & (i[:, :-1] < i[:, 1:])))
    if family == O.REAL:
        rows = H.query_rows(q_seed, O.REAL, N, 0, B)
        hit = rows >= 0
        assert np.all(i[hit, 0] == rows[hit])  # near-duplicate queries find their source row


def run_case(torch, dtype, filt, B, q_seed, sample, family=O.REAL, plan=None):
    col = H.Collection(DIM, capacity=N, dtype=dtype)
    try:
        col.generate(family, SEED, N)
        if filt == "bf16_copy":
            col.set_filter("bf16_copy")
        if plan is not None:
            assert col.search_plan(B, 8) == plan
        q = H.gen_queries(family, q_seed, SEED, N, 0, B, DIM)
        col.search_stats(reset=True)
        sc, ids = col.search_topk_exact(q, 8)
        st = col.search_stats()
        kind = family | (O.KEYS_BF16 if dtype == "bf16" else 0)
        osc, oid = O.search_synth(kind, SEED, N, q.cpu().numpy()[sample], 8, threads=0)
        np.testing.assert_array_equal(ids.cpu().numpy()[sample], oid)
        np.testing.assert_array_equal(sc.cpu().numpy()[sample], osc)
        props(sc, ids, B, q_seed, family)
        return st
    finally:
        col.close()
        torch.cuda.empty_cache()


def test_c2_bf16_filter_copy(torch):
    """The bench's default path: fp32 keys, bf16 filter copy, exact fp64 rescoring."""
    st = run_case(torch, "f32", "bf16_copy", 64, 7, SAMPLE16)
    assert st["fallback_queries"] == 0, st
    assert st["candidates"] / 64 < 256, st


def test_c2_native_tf32_filter(torch):
    run_case(torch, "f32", "native", 64, 7, SAMPLE16[::2])


def test_c2_bf16_collection(torch):
    run_case(torch, "bf16", "native", 64, 8, SAMPLE16)


def test_pair_kernel_b256_at_1m(torch):
    """B = 256: the CTA-pair filter (tcgen05.mma.cta_group::2) over 1M rows."""
    run_case(torch, "f32", "bf16_copy", 256, 9, [0, 37, 77, 128, 129, 200, 254, 255])


def test_pair_kernel_onchip_conversion_b256_at_1m(torch):
    """B = 256 over the fp32 keys without the copy: fp32 tiles converted to bf16 on chip (config 4's path)."""
    run_case(torch, "f32", "native", 256, 10, [0, 1, 63, 128, 129, 191, 254, 255], plan="filter_bf16_onchip")


def test_c2_cluster_family_at_1m(torch):
    """Runs of 64-512 near-duplicate / identical consecutive rows (CLUSTER) at the headline size and
    path: the range fallback keeps every result exact (the statistics may show it firing)."""
    st = run_case(torch, "f32", "bf16_copy", 64, 11, SAMPLE16[::2], family=O.CLUSTER)
    assert st["candidates"] > 0, st
