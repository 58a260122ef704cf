"""compute-sanitizer tier (SURVEY §5 race detection): every kernel family on tiny shapes under
memcheck, racecheck (shared-memory hazards) and synccheck (barrier misuse). The mbarrier/TMA/TMEM
pipelines of the persistent passes (kb_dmma.cuh, kb_tf32.cuh, kb_tc.cuh) synchronise through
mbarriers, so racecheck's shared-memory hazard tracking is their data-race check."""

import os
import re
import shutil
import subprocess
import sys

import pytest

from conftest import ROOT, cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
FAMILIES = {
    "dmma": {},                           # fp64 DMMA persistent passes (KB_PERSIST=0)
    "tf32": {},                           # 3xTF32 mma.sync persistent passes
    "tcgen05": {"KB_FP32_TC": "1"},       # tcgen05 / TMEM / TMA passes, forced at 256^2
    "ffma": {"KB_FP32_PATH": "ffma", "KB_FP32_TC": "0"},  # FFMA register-window passes
    "generic": {},                        # odd extents: generic cp.async tiles
    "persist": {"KB_PERSIST": "1"},       # whole-solve cooperative kernel
    "blur": {},
    "norms": {},                          # history path: resid norms + reduce partials
}


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("family", sorted(FAMILIES))
def test_kernel_family_is_clean_under_compute_sanitizer(family, tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    env = dict(os.environ, **FAMILIES[family])
    if family != "persist":
        env.setdefault("KB_PERSIST", "0")
    cmd = [SAN, f"--tool={tool}", "--error-exitcode=7", "--kernel-name", "regex:kb_",
           sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), family]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    text = out.stdout + out.stderr
    if "compute-sanitizer is closed" in text:
        # the GPU pool refuses compute-sanitizer (earlier runs by others left GPUs needing a
        # reset); the guard-band tests (test_gpu_guards.py) stand in for memcheck's write checks
        pytest.skip("compute-sanitizer is disabled on this GPU pool")
    assert f"ok {family}" in text, text[-3000:]
    m = re.search(r"ERROR SUMMARY: (\d+) error", text)
    assert m is not None and int(m.group(1)) == 0, text[-3000:]
    assert out.returncode == 0, text[-3000:]
