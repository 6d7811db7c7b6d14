"""``tmcodec`` -> ``paper_2104_04726_b200`` module alias, so the REFERENCE's own
unit tests (copied unchanged into oracle/_ref/reference_tests by
oracle/build_ref.py) import the drop-in instead of the reference:
``from tmcodec.tensor import ttm`` resolves to paper_2104_04726_b200.tensor.ttm.
Test infrastructure only (tests/test_reference_suite.py)."""

import sys

import paper_2104_04726_b200 as _pkg
from paper_2104_04726_b200 import codec, color, entropy, metrics, scene, tensor, tucker
from paper_2104_04726_b200 import *  # noqa: F401,F403

_ALIASES = {"tensor": tensor, "tucker": tucker, "color": color, "codec": codec, "entropy": entropy,
            "metrics": metrics, "sceneio": scene}
for _name, _mod in _ALIASES.items():
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod
__version__ = _pkg.__version__
