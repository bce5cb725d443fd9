"""CPU-side checks of the drop-in boundary: the CUDA library and the C++ API
load and export every entry point include/eventscope_b200.h declares; with no
GPU the calls fail loudly (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "eventscope_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(es_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2506_02007_b200 import _build
    _build.build()
    import paper_2506_02007_b200 as es
    return es.load_library()


def test_header_declares_entry_points():
    names = declared()
    for must in ("es_gmm_fit", "es_gmm_score", "es_gmm_detect", "es_gmm_calibrate", "es_gmm_responsibilities",
                 "es_gmm_select_k_bic", "es_dataset_create", "es_ctx_create_nccl"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_cpp_api_symbols_exported():
    from paper_2506_02007_b200 import _build
    out = subprocess.run(["nm", "-DC", "--defined-only", _build.LIB], capture_output=True, text=True).stdout
    for sym in ("eventscope::fit_em(", "eventscope::detect(", "eventscope::calibrate_threshold(",
                "eventscope::component_log_density(", "eventscope::mixture_density(",
                "eventscope::responsibilities(", "eventscope::select_k_bic(", "eventscope::to_json"):
        assert sym in out, sym


def test_kernels_are_sm100a(lib):
    from paper_2506_02007_b200 import _build
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_2506_02007_b200 as es
    with pytest.raises(es.EventscopeError) as e:
        es.Context(0)
    assert e.value.kind == "Io" and e.value.name == "CudaError"
    assert lib.es_version()


def test_eacgm_seed_applies_only_without_explicit_seed(monkeypatch):
    import paper_2506_02007_b200 as es
    monkeypatch.setenv("EACGM_SEED", "77")
    assert es._seed(None) == 77 and es._seed(5) == 5 and es._seed(0) == 0
    assert es._opts("random", 0.0, 3, None, 5).seed == 5
    assert es._opts("random", 0.0, 3, None, None).seed == 77
    monkeypatch.delenv("EACGM_SEED")
    assert es._seed(None) == 0


def test_tensor_inputs_are_dtype_checked():
    import torch

    import paper_2506_02007_b200 as es
    with pytest.raises(es.EventscopeError) as e:
        es._check_tensor(torch.zeros(4, 2, dtype=torch.float32), "float64", 2)
    assert e.value.name == "InvalidDtype" and e.value.kind == "Data"
    with pytest.raises(es.EventscopeError) as e:
        es._check_tensor(torch.zeros(4, dtype=torch.float64), "float64", 2)
    assert e.value.name == "DimensionMismatch"
    es._check_tensor(torch.zeros(4, 2, dtype=torch.float64), "float64", 2)
