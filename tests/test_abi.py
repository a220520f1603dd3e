"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/hsd/hsd_gpu.h declares, fails loudly without a device (no CPU
fallback), and its pure host helpers behave."""
import ctypes as C

import pytest

import paper_2603_17573_b200 as H


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def test_library_exports_every_declared_symbol():
    L = H.lib()
    syms = H.exported_symbols()
    assert len(syms) >= 29
    for s in syms:
        assert hasattr(L, s), s
    assert L.hsd_abi_version() == 1


def test_status_codes_mirror_reference_taxonomy():
    # errors.hpp:10-50 -> hsd_status 1..7
    assert H._STATUS[1] is H.InvalidInputError and H._STATUS[2] is H.ConfigError
    assert H._STATUS[3] is H.SchemaError and H._STATUS[7] is H.CalibrationError


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device path")
def test_no_cpu_fallback():
    assert H.device_count() == 0
    with pytest.raises(H.NoDeviceError):
        H.Collection(64)


def test_argument_validation_without_device():
    L = H.lib()
    # config errors are detected before touching the device
    h = C.c_void_p()
    assert L.hsd_collection_create(0, 0, 1, C.byref(h)) == 2  # dim < 1 -> ConfigError (store.cpp:37)
    mp = H.MetricParams(1.5, 15, 0.5, 1.0)
    assert L.hsd_window_features(0, None, 1, C.byref(mp), C.byref(H.LIBERO_GOAL), None, None, None, None, None,
                                 None) == 2
    mp = H.MetricParams(0.5, 2, 0.5, 1.0)
    assert L.hsd_window_features(0, None, 1, C.byref(mp), C.byref(H.LIBERO_GOAL), None, None, None, None, None,
                                 None) == 2
    bad = H.NormBounds(0.2, 0.1, 0.0, 1.0)
    assert L.hsd_window_features(0, None, 1, C.byref(H.DEFAULT_METRIC), C.byref(bad), None, None, None, None, None,
                                 None) == 2


def test_shard_ranges_partition():
    for n in (0, 1, 7, 1000, 10_000_003):
        for world in (1, 2, 3, 8):
            prev = 0
            for r in range(world):
                b, e = H.shard_range(n, world, r)
                assert b == prev and e >= b
                prev = e
            assert prev == n
