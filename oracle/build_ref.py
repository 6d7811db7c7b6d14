"""Build recipe for ``oracle/_ref``: the UNMODIFIED reference package, installed.

TEST / BASELINE INFRASTRUCTURE ONLY. ``oracle/_ref`` is what ``bench.py
--impl reference`` (and the ``cpu_baseline`` leg of our own arm) executes: the
reference's own ``tmcodec`` code path on the host cores, so those numbers are
``kind: "reference"`` rather than a port. The product package never imports it.

    python oracle/build_ref.py          # also run by __graft_entry__.build()

The reference is pure Python (+ one optional Cython file, off the hot path).
It is installed with pip, offline, from a scratch copy of
``/root/reference/pkg`` (the tree is read-only and the setuptools build writes
into its source directory), into ``oracle/_ref`` -- git-ignored, so no
reference source enters the history, but NOT gpurun-ignored, so the installed
package travels to the GPU box with the repository snapshot. On the GPU box
(no ``/root/reference``) this is a no-op and the prebuilt copy is used.
"""

from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

REF_PKG = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent / "_ref"
STAMP = OUT / ".built_from"
REF_TESTS = ("conftest.py", "test_tensor.py", "test_tucker.py", "test_pp.py", "test_color.py", "test_codec.py",
             "test_metrics.py")


def _source_mtime() -> float:
    return max(p.stat().st_mtime for p in (REF_PKG / "src").rglob("*") if p.is_file())


def build(force: bool = False) -> Path | None:
    """Install the reference into oracle/_ref; returns the path (None if unavailable)."""
    if not REF_PKG.exists():
        return OUT if (OUT / "tmcodec").exists() else None
    if not force and STAMP.exists() and (OUT / "tmcodec").exists() and (OUT / "reference_tests").exists():
        try:
            if float(STAMP.read_text().split()[0]) >= _source_mtime():
                return OUT
        except (ValueError, IndexError):
            pass
    with tempfile.TemporaryDirectory(prefix="tmb_refpkg_") as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(REF_PKG, src, ignore=shutil.ignore_patterns("__pycache__", "*.pyc", "build", "*.egg-info"))
        staging = Path(tmp) / "target"
        cmd = [sys.executable, "-m", "pip", "install", "--quiet", "--no-index", "--no-build-isolation", "--no-deps",
               "--target", str(staging), str(src)]
        res = subprocess.run(cmd, capture_output=True, text=True, cwd=tmp)
        if res.returncode != 0:
            raise RuntimeError(f"reference install failed:\n{res.stdout}\n{res.stderr}")
        if OUT.exists():
            shutil.rmtree(OUT)
        shutil.copytree(staging, OUT, ignore=shutil.ignore_patterns("__pycache__", "bin"))
        # the reference's own unit tests for the hot-path modules, run UNCHANGED against
        # the drop-in by tests/test_reference_suite.py
        tdir = OUT / "reference_tests"
        tdir.mkdir()
        for name in REF_TESTS:
            shutil.copy2(REF_PKG / "tests" / name, tdir / name)
    STAMP.write_text(f"{_source_mtime()} {REF_PKG}\n")
    return OUT


def import_reference():
    """Import the installed reference ``tmcodec`` (for bench.py's reference leg)."""
    if not (OUT / "tmcodec").exists():
        raise ImportError(f"{OUT} is not built (python oracle/build_ref.py in the build container)")
    if str(OUT) not in sys.path:
        sys.path.insert(0, str(OUT))
    import tmcodec  # noqa: PLC0415

    if not str(Path(tmcodec.__file__).resolve()).startswith(str(OUT)):
        raise ImportError(f"tmcodec resolved to {tmcodec.__file__}, not {OUT}")
    return tmcodec


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
