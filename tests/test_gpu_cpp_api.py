"""The C++ drop-in API compiled against include/ and the in-tree .so, run on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_example(out):
    from paper_2506_02007_b200 import _build
    lib = _build.build()
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    env = dict(os.environ)
    env.pop("CXX", None)
    subprocess.run([cxx, "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "api_example.cpp"), lib,
                    f"-Wl,-rpath,{os.path.dirname(lib)}", "-o", out], check=True, env=env)


def test_cpp_example_compiles(tmp_path):
    build_example(str(tmp_path / "api_example"))


@pytest.mark.gpu
def test_cpp_example_runs(tmp_path):
    exe = str(tmp_path / "api_example")
    build_example(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("OK")
