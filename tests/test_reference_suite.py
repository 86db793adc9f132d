"""CPU: the reference's own test file, unchanged, against this package's
`fpx` (drop-in proof for `fpx.basis`).  Skipped where /root/reference is
absent (the GPU box)."""
import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests/test_basis.py"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists(REF_TESTS), reason="reference not mounted")
def test_reference_test_suite_passes_unchanged(tmp_path):
    probe = tmp_path / "conftest_probe.py"
    probe.write_text(
        "def pytest_sessionfinish(session):\n"
        "    import fpx.basis, sys\n"
        "    print('FPX_FROM', fpx.basis.__file__, file=sys.stderr)\n")
    env = dict(os.environ, PYTHONPATH=f"{ROOT}:{tmp_path}")
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        "-p", "conftest_probe", REF_TESTS, "--rootdir", str(tmp_path)],
                       cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=600)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-3000:]
    assert "94 passed" in out
    assert f"FPX_FROM {ROOT}/paper_2501_12349_b200/basis.py" in out
