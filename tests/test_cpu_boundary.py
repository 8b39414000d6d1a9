"""CPU-side checks: the C-ABI library loads, exports every symbol that
include/salr_b200.h declares, validates arguments before touching the device,
and the host-side API logic mirrors the reference (no GPU needed)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO


def header_symbols():
    src = open(os.path.join(REPO, "include", "salr_b200.h")).read()
    return set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(salr_\w+)\s*\(", src, re.M))


def test_library_exports_every_header_symbol():
    from paper_2601_16991_b200 import _lib
    lib = _lib.load()
    declared = header_symbols()
    assert declared and declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.salr_version() == 1


def test_argument_validation_without_device():
    from paper_2601_16991_b200 import _lib
    import paper_2601_16991_b200 as S
    lib = _lib.load()
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    assert lib.salr_tb_geometry(0, 5, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)) == 1  # ShapeError
    with pytest.raises(S.ShapeError):
        _lib.check(1)
    assert "invalid dims" in lib.salr_last_error().decode()
    assert _lib.geometry(4096, 14336) == (64, 112, 7168)
    assert _lib.geometry(37, 53) == (1, 1, 1)
    # decode window outside the matrix -> BoundsError before any launch
    rc = lib.salr_decode(None, None, 0, 4, 8, 0, 5, 0, 8, None, 0, 8, None)
    assert rc == 3
    # r_pad other than 0/64/128 -> ConfigError
    rc = lib.salr_linear_forward(None, 1, 64, 64, None, None, 0, 128, None, None, 32, None, 0, 128, None, 0, 0, 0, 0, None)
    assert rc in (1, 4)


def test_pipeline_config_rules():
    import paper_2601_16991_b200 as S
    cfg = S.PipelineConfig()
    assert (cfg.tile_rows, cfg.tile_col_bytes, cfg.ring_capacity, cfg.overlap) == (64, 8, 4, True)
    for bad in (dict(tile_rows=0), dict(tile_col_bytes=0), dict(ring_capacity=0, overlap=False),
                dict(ring_capacity=1, overlap=True)):
        with pytest.raises(S.ConfigError):
            S.PipelineConfig(**bad)
    assert S.PipelineConfig(ring_capacity=1, overlap=False).device_stages == 1


def test_validate_transitions_auditor():
    import paper_2601_16991_b200 as S
    E, F, C = S.SlotState.EMPTY, S.SlotState.FILLED, S.SlotState.CONSUMED
    p = S.PipelineProbe(record=True, transitions=[(0, E, F), (0, F, C), (0, C, E)], produced=1, consumed=1)
    S.validate_transitions(p, 2)
    with pytest.raises(S.VerificationError):
        S.validate_transitions(S.PipelineProbe(transitions=[(0, E, C)], produced=0, consumed=0), 2)
    with pytest.raises(S.VerificationError):
        S.validate_transitions(S.PipelineProbe(transitions=[(0, E, F)], produced=1, consumed=1), 2)


def test_host_helpers_match_reference_formulas():
    import paper_2601_16991_b200 as S
    lut = S.build_lut()
    assert lut.shape == (256, 8) and lut.dtype == np.int8
    np.testing.assert_array_equal(lut[5], [0, -1, 1, -1, -1, -1, -1, -1])
    assert S.popcount8(255) == 8
    with pytest.raises(S.BoundsError):
        S.popcount8(256)
    assert S.header_bytes(0) == 41 and S.header_bytes(2) == 57
    assert S.compression_ratio(4096, 4096, 0.5, 2, 0) == pytest.approx(1.7778, abs=1e-3)
    assert S.kept_count(0.5, 4096 * 4096) == 8388608


def test_no_cpu_fallback():
    import torch
    import paper_2601_16991_b200 as S
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(S.SalrError):
        S.encode(np.ones((4, 4)))


def test_product_package_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_2601_16991_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
