"""pytest plugin (debug): report any pending CUDA runtime error after each test
(a cudaSetDevice / cudaGetLastError left behind by an entry point surfaces as a
bogus failure in a LATER test's launch check).
  PYTHONPATH=tools python -m pytest -p cuda_err_plugin tests -m gpu -s"""
import pytest

_rt = None


def _err():
    global _rt
    if _rt is None:
        import paper_2603_17573_b200 as H  # libhsd_gpu.so links libcudart: its cudaGetLastError is the one used
        _rt = H.lib()
    return _rt.hsd_debug_last_cuda_error()


@pytest.fixture(autouse=True)
def _cuda_error_check(request):
    yield
    import gc
    gc.collect()
    e = _err()
    if e:
        print(f"\n[cuda-err] pending CUDA error {e} after {request.node.nodeid}")
