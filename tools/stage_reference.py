"""Stage the unmodified reference engine for the drop-in suite (tests/test_reference_suite_gpu.py).

Installs `mdkk` from /root/reference/pkg into baseline/_ref (git-ignored; it
travels to the GPU box with the repo snapshot) with the offline pip recipe,
and copies the reference's own test modules and input scripts next to it
(baseline/_ref/pkg/{tests,scripts}) so they can run against the drop-ins.
Nothing here is imported by the product package.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = "/root/reference/pkg"
DEST = os.path.join(ROOT, "baseline", "_ref")


def stage(force: bool = False) -> str:
    """Returns a one-line outcome (also recorded in DESIGN.md §9)."""
    if not os.path.isdir(REF_PKG):
        return "skipped: /root/reference is not present (GPU box uses the staged copy)"
    if not force and os.path.isdir(os.path.join(DEST, "mdkk")) and os.path.isdir(os.path.join(DEST, "pkg", "tests")):
        return "already staged"
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_PKG, src)   # the build writes egg-info into its source tree
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--find-links",
               "/opt/wheelhouse", "--target", DEST, "--no-deps", "--upgrade", src]
        out = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
        if out.returncode != 0:
            return "pip install failed: " + out.stdout.strip().splitlines()[-1]
    for sub in ("tests", "scripts"):
        dst = os.path.join(DEST, "pkg", sub)
        shutil.rmtree(dst, ignore_errors=True)
        shutil.copytree(os.path.join(REF_PKG, sub), dst, ignore=shutil.ignore_patterns("__pycache__"))
    return "installed mdkk into baseline/_ref; tests and scripts staged in baseline/_ref/pkg"


if __name__ == "__main__":
    print(stage(force="--force" in sys.argv))
