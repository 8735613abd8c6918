"""The GEMM code paths selected by environment knobs, each in its own process (the knobs are
read once per process): single-CTA 3xTF32 tiles (CDFGNN_GEMM_PAIR=0; the default runs N >= 128
tiles on CTA pairs) and ∇W from transposed K-major copies (CDFGNN_WGRAD_KMAJOR=1), both through
tests/test_gpu_gemm.py's oracle checks (fp64 arithmetic, 1e-4 row-normwise)."""
import os
import subprocess
import sys

import pytest

from tests.gpu_util import require_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"CDFGNN_GEMM_PAIR": "0"}, {"CDFGNN_WGRAD_KMAJOR": "1"}])
def test_gemm_paths_under_knobs(env):
    require_gpu()
    out = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_gemm.py"), "-x", "-q",
                          "-p", "no:cacheprovider"], cwd=ROOT, env={**os.environ, **env}, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
