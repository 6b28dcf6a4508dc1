"""compute-sanitizer over the library's kernels: memcheck (out-of-bounds / misaligned device
accesses), racecheck (shared-memory hazards: the event pass, the scans with decoupled look-back, the merge
kernels all stage through shared memory) and synccheck (barrier misuse), on config 1 and two small seeded
traces that cover the lean and the general a2 paths and the crossing-span sweep (tests/sanitize_run.py)."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
HERE = os.path.dirname(os.path.abspath(__file__))


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "99", "--target-processes", "all"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(HERE, "sanitize_run.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=3000)
    out = p.stdout + p.stderr
    if "compute-sanitizer is closed" in out:
        # the pool's operators closed the tool (a wrapper refuses to run); the last runs under it are in
        # profiles/r02_gpu_tests_p.txt (all three tools green)
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    summ = re.findall(r"ERROR SUMMARY: (\d+) error", out) + re.findall(r"RACECHECK SUMMARY: \d+ hazards? displayed \((\d+) error", out)
    assert p.returncode == 0 and "sanitize workload ok" in out, out[-4000:]
    assert summ and all(int(x) == 0 for x in summ), out[-4000:]
