"""The reference's own GoogleTest suites (proj/tests/test_selection.cpp, test_scope.cpp,
test_numerics.cpp, test_kv_cache.cpp, test_model.cpp, test_engine.cpp) compiled in place
against the drop-in headers in include/reattn -- not the reference's -- with the GoogleTest
shim in tests/reftests/gtest (tests/reftests/Makefile, run by __graft_entry__.build() where
/root/reference exists; the binaries travel to the GPU box).  Every reference test must pass
with the library doing the work on the GPU."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "reftests")
SUITES = ["test_selection", "test_scope", "test_numerics", "test_kv_cache", "test_model", "test_engine"]


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_the_drop_in(suite, tmp_path):
    exe = os.path.join(BIN, suite)
    if not os.path.exists(exe):
        pytest.skip(f"{suite} not built (build() compiles it where /root/reference exists)")
    env = dict(os.environ, TEST_TMPDIR=str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900, env=env)
    out = r.stdout + r.stderr
    m = re.search(r"\[==========\] (\d+) tests ran, (\d+) passed, (\d+) failed", out)
    assert m, out[-2000:]
    ran, passed, failed = map(int, m.groups())
    assert ran > 0 and failed == 0 and r.returncode == 0, out[-4000:]
