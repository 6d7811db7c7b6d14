"""The REFERENCE's own unit tests, unchanged, against the drop-in (SURVEY App.
C.6(i)): test_tensor.py, test_tucker.py, test_pp.py, test_color.py,
test_codec.py and test_metrics.py from the reference package (copied by
oracle/build_ref.py into the git-ignored oracle/_ref/reference_tests, which
travels to the GPU box), with ``tmcodec`` aliased to paper_2104_04726_b200
(tests/alias/tmcodec). Every tensor/solver/colour/quantiser call in them runs
through libtmb at the reference's own fp64 tolerances.

Deselected, out of scope: test_codec.py::TestFramesPath (the 3D-HEVC stand-in
frames codec and its external-encoder adapter; our
encode_stream raises NotImplementedError for path='frames').
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SUITE = ROOT / "oracle" / "_ref" / "reference_tests"
FILES = ["test_tensor.py", "test_tucker.py", "test_pp.py", "test_color.py", "test_codec.py", "test_metrics.py"]
DESELECT = "not TestFramesPath"


@pytest.mark.gpu
def test_reference_unit_tests_pass_against_drop_in():
    if not SUITE.exists():
        pytest.fail(f"{SUITE} missing: run python oracle/build_ref.py in the build container")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(ROOT / "tests" / "alias"), str(ROOT)]),
               PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "pytest", *FILES, "-q", "-p", "no:cacheprovider", "-k", DESELECT,
           "--rootdir", str(SUITE)]
    out = subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=1800)
    tail = "\n".join(out.stdout.splitlines()[-40:])
    print(tail)
    assert out.returncode == 0, tail + "\n" + out.stderr[-2000:]
    # and the module the suite imported as tmcodec.tensor is the drop-in, not the reference
    who = subprocess.run([sys.executable, "-c", "import tmcodec.tensor as t, tmcodec.tucker as u; "
                          "print(t.__name__, u.__name__)"], cwd=SUITE, env=env, capture_output=True, text=True)
    assert who.stdout.split() == ["paper_2104_04726_b200.tensor", "paper_2104_04726_b200.tucker"], who.stderr
