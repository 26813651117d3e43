"""compute-sanitizer on the kernels with hand-rolled synchronisation (needs
a B200): racecheck and synccheck on the TMA band half-sweep (mbarrier
producer/consumer rings and named barriers, 8- and 16-warp variants, the
fused-residual and <f, u> modes, tile regions), memcheck on a configs[0]
MG + CG solve and a four-part solve through the native multi-part driver
(tools/sanitize_case.py).

The GPU pool this repository is tested on has compute-sanitizer switched
off (its wrapper exits 86: runs under it left GPUs needing a reset); the
test then skips with that reason, and the kernels' synchronisation is
covered by the bit-for-bit parity tests instead (band vs exact solver at
256 ... 2048, tile regions vs whole sweeps, fused modes vs separate
passes)."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool,case", [("racecheck", "band"), ("synccheck", "band"),
                                       ("memcheck", "band"), ("memcheck", "solve")])
def test_sanitizer_clean(tool, case):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available() or not os.path.exists(SAN):
        pytest.skip("needs a CUDA device and compute-sanitizer")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "3", sys.executable,
           os.path.join(ROOT, "tools", "sanitize_case.py"), case]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    tail = (out.stdout + out.stderr)[-3000:]
    if out.returncode == 86 and "closed" in tail:
        pytest.skip("compute-sanitizer is disabled on this GPU pool: " + tail.strip()[:200])
    assert out.returncode == 0, tail
    assert "ERROR SUMMARY: 0 errors" in out.stdout + out.stderr, tail
