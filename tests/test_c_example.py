"""The C ABI from plain C: examples/gft_example.c builds against include/gft.h + libgft (CPU
check), and on a GPU runs a cycle-graph forward / inverse with its own checks."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_example_builds():
    from paper_1907_07875_b200 import build as B
    B.build_library(verbose=False)
    exe = B.build_c_example(verbose=False)
    assert os.access(exe, os.X_OK)


@pytest.mark.gpu
@pytest.mark.parametrize("n,batch", [(64, 100000), (12, 1001), (80, 4097)])
def test_c_example_runs(n, batch):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = os.path.join(ROOT, "paper_1907_07875_b200", "_lib", "gft_example")
    if not os.access(exe, os.X_OK):
        from paper_1907_07875_b200 import build as B
        exe = B.build_c_example(verbose=False)
    out = subprocess.run([exe, str(n), str(batch)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("OK")
