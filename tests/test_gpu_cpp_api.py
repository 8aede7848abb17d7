"""GPU: the reference's engine/transform test cases written against the drop-in C++
API (include/sft_b200/sft.hpp) compile with g++, link libsftgpu.so, and pass."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_cpp_test(out):
    lib_dir = os.path.join(ROOT, "paper_2110_11866_b200")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_reference_api.cpp"), "-o", out, "-L", lib_dir, "-lsftgpu",
           f"-Wl,-rpath,{lib_dir}"]
    subprocess.check_call(cmd)


def test_cpp_api_compiles(tmp_path):
    """CPU: the drop-in header compiles warning-clean and links against the C ABI."""
    build_cpp_test(str(tmp_path / "t"))


@pytest.mark.gpu
def test_cpp_reference_suites_pass(tmp_path):
    exe = str(tmp_path / "t")
    build_cpp_test(exe)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(res.stdout[-3000:])
    assert res.returncode == 0, res.stdout[-3000:]
