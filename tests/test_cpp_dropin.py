"""Runs the C++ drop-in test program (tests/cpp/test_dropin.cpp): the reference's own
hot-path unit tests compiled against include/reattn/*.hpp (C-ABI -> sm_100a kernels)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")


def _build():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "liboracle.so"], check=True,
                   stdout=subprocess.DEVNULL)
    subprocess.run(["make", "-C", CPP], check=True, stdout=subprocess.DEVNULL)


def test_dropin_headers_compile():
    """CPU: the drop-in headers and the test program build (no GPU needed to compile)."""
    _build()
    assert os.access(os.path.join(CPP, "test_dropin"), os.X_OK)


@pytest.mark.gpu
def test_dropin_reference_unit_tests_on_gpu():
    _build()
    r = subprocess.run([os.path.join(CPP, "test_dropin")], capture_output=True, text=True,
                       timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " 0 failures" in r.stdout


@pytest.mark.gpu
def test_dropin_on_garbage_device_memory():
    """Same program after filling (and freeing) most device memory with 0xFF bytes: every
    buffer must be written before it is read and every copy ordered with the kernels that
    consume it (this run exposed a legacy-stream memset racing the context stream)."""
    _build()
    env = dict(os.environ, REATTN_TEST_GARBAGE="1")
    r = subprocess.run([os.path.join(CPP, "test_dropin")], capture_output=True, text=True,
                       timeout=600, env=env)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " 0 failures" in r.stdout
