"""The C++ host side (include/moe_b200.hpp, mirroring routing.hpp) compiled
against libmoe_b200.so and run: host-only cases on CPU, layer cases on GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "test_adapter")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


def test_cpp_adapter_host():
    _build()
    r = subprocess.run([EXE, "host"], capture_output=True, text=True)
    assert r.returncode == 0 and "OK host" in r.stdout, r.stderr


@pytest.mark.gpu
def test_cpp_adapter_gpu():
    _build()
    r = subprocess.run([EXE, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK host+gpu" in r.stdout, r.stdout + r.stderr
