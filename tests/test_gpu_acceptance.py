"""The reference's own acceptance gate (proj/tests/acceptance/acceptance.cpp,
unmodified) compiled against this repository's drop-in headers and linked to
libsigk.so (oracle/Makefile `acceptance`, built by build() where the reference
sources exist): all ten release criteria must pass on the GPU implementation,
criterion 10 through tools/sigbench (the reference CLI over the GPU library)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GATE = os.path.join(ROOT, "oracle", "_ref", "acceptance_dropin")
SIGBENCH = os.path.join(ROOT, "tools", "sigbench")


def test_reference_acceptance_gate_on_the_drop_in():
    if not os.path.exists(GATE):
        pytest.skip("oracle/_ref/acceptance_dropin not built (needs the reference sources at build time)")
    r = subprocess.run([GATE, "--sigbench", SIGBENCH], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all 10 acceptance criteria passed" in r.stdout
