"""CPU: the C-ABI library loads, exports every symbol include/sftgpu.h declares, fails
loudly (no CPU fallback) when no CUDA device is present, and the product never imports
the oracle."""
import ast
import ctypes
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sftgpu.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(sftgpu_\w+)\s*\(", src, re.M)))


def test_header_declares_the_api():
    syms = declared_symbols()
    assert "sftgpu_transform_execute" in syms and "sftgpu_components_execute" in syms
    assert len(syms) >= 25


def test_library_exports_every_declared_symbol(sft):
    from paper_2110_11866_b200 import _abi

    lib = ctypes.CDLL(_abi.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(_abi.SIGNATURES), "ctypes binding out of sync with the header"


def test_nm_shows_sm100a_kernels(sft):
    from paper_2110_11866_b200 import _abi

    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device(sft):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    spec = sft.make_gauss_spec(4.0, 0, 3, 0)
    with pytest.raises(sft.SftGpuError):
        sft.TransformPlan(spec, 128, 1)
    with pytest.raises(sft.SftGpuError):
        sft.gauss_smooth(sft.Signal([1.0, 2.0, 3.0]), spec)


def test_invalid_arguments_map_to_value_error(sft):
    with pytest.raises(ValueError):
        sft.make_transform_spec("GMP3", 8.0, 1.0)
    with pytest.raises(ValueError):
        sft.Signal([])
    with pytest.raises(ValueError):
        sft.Signal([1.0, float("nan")])


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2110_11866_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dp, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert all(not a.name.startswith("oracle") for a in node.names), f
                    if isinstance(node, ast.ImportFrom) and node.module:
                        assert not node.module.startswith("oracle"), f
            if f.endswith((".cu", ".cpp", ".cuh", ".hpp")):
                assert "sft_oracle" not in open(os.path.join(dp, f)).read(), f


def test_product_library_does_not_link_oracle(sft):
    from paper_2110_11866_b200 import _abi

    out = subprocess.run(["ldd", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out
