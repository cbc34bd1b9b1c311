"""CPU-side checks of the C-ABI boundary: the library loads, exports every
symbol include/tdc.h declares, and validates descriptors without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "tdc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tdc_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def tdc():
    from paper_2211_03715_b200 import build
    build.build()
    from paper_2211_03715_b200 import tdc as mod
    return mod


def test_library_exports_every_declared_symbol(tdc):
    declared = _declared_symbols()
    assert "tdc_conv_plan" in declared and "tdc_conv_forward" in declared
    lib = ctypes.CDLL(tdc.LIB_PATH)
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(tdc.EXPORTED) == declared


def test_library_is_sm100a_only(tdc):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", tdc.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_binding_has_no_cpu_fallback():
    """The product package must not import the oracle or compute on the host."""
    pkg = os.path.join(ROOT, "paper_2211_03715_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "tdc_oracle" not in text, f


def test_version_and_status_strings(tdc):
    assert "sm_100a" in tdc.tdc_version()
    assert tdc.tdc_status_string(tdc.TDC_OK) == "ok"
    assert tdc.tdc_status_string(tdc.TDC_ERR_INVALID_ARGUMENT) == "invalid argument"
    assert tdc.tdc_status_string(99) == "unknown status"


@pytest.mark.parametrize("args,expect", [
    ((1, 16, 8, 8, 16, 4, 4, 3, 1, 1), (8, 8)),
    ((32, 64, 56, 56, 128, 32, 64, 3, 2, 1), (28, 28)),
    ((1, 3, 7, 5, 2, 1, 2, 5, 1, 2), (7, 5)),
    ((1, 8, 9, 9, 8, 2, 2, 3, 3, 0), (3, 3)),
])
def test_output_shape(tdc, args, expect):
    assert tdc.tdc_conv_output_shape(tdc.make_desc(*args)) == expect


@pytest.mark.parametrize("args,frag", [
    ((0, 16, 8, 8, 16, 4, 4, 3, 1, 1), "positive"),
    ((1, 16, 8, 8, 16, 17, 4, 3, 1, 1), "rank bounds"),
    ((1, 16, 8, 8, 16, 4, 20, 3, 1, 1), "rank bounds"),
    ((1, 16, 8, 8, 16, 4, 4, 3, 0, 1), "stride"),
    ((1, 16, 8, 8, 16, 4, 4, 3, 1, -1), "pad"),
    ((1, 16, 2, 8, 16, 4, 4, 5, 1, 0), "exceeds"),
])
def test_invalid_descriptors_are_rejected(tdc, args, frag):
    with pytest.raises(tdc.TdcError) as ei:
        tdc.tdc_conv_output_shape(tdc.make_desc(*args))
    assert ei.value.status == tdc.TDC_ERR_INVALID_ARGUMENT
    assert frag in str(ei.value)


def test_bad_layout_and_math(tdc):
    with pytest.raises(tdc.TdcError):
        tdc.tdc_conv_output_shape(tdc.make_desc(1, 4, 4, 4, 4, 2, 2, layout=7))
    with pytest.raises(tdc.TdcError):
        tdc.tdc_conv_output_shape(tdc.make_desc(1, 4, 4, 4, 4, 2, 2, math=9))


def test_plan_without_gpu_fails_cleanly(tdc):
    import numpy as np
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    d = tdc.make_desc(1, 4, 4, 4, 4, 2, 2)
    with pytest.raises(tdc.TdcError) as ei:
        tdc.tdc_conv_plan(d, np.zeros((2, 2, 3, 3), np.float32), np.zeros((4, 2), np.float32),
                          np.zeros((4, 2), np.float32))
    assert ei.value.status in (tdc.TDC_ERR_CUDA, tdc.TDC_ERR_INVALID_ARGUMENT)


def test_null_arguments(tdc):
    assert tdc.lib.tdc_conv_output_shape(None, None, None) == tdc.TDC_ERR_INVALID_ARGUMENT
    assert tdc.lib.tdc_conv_forward(None, None, None, 1, None) == tdc.TDC_ERR_INVALID_ARGUMENT
    assert tdc.lib.tdc_conv_plan_destroy(None) == tdc.TDC_OK
    assert "NULL" in tdc.tdc_last_error() or tdc.tdc_last_error()
