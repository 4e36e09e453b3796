"""The C++ drop-in (include/docp_gpu.hpp) against the reference functions,
run as the prebuilt Catch2-style binary tests/cpp/_bin/test_dropin (built by
build.py from the reference headers in this container; it reads nothing
under /root/reference at run time)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "test_dropin")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cpp/_bin/test_dropin not built (needs the reference headers)")
def test_cpp_dropin_suite():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    failed = [line for line in r.stdout.splitlines() if line.startswith("FAIL ")]
    passed = [line for line in r.stdout.splitlines() if line.startswith("PASS ")]
    assert r.returncode == 0 and not failed, r.stdout[-4000:] + r.stderr[-2000:]
    assert len(passed) >= 11
