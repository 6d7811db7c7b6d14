"""CPU oracle for the Tucker-ALS hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in float64 numpy, the reference `tmcodec` algorithm for
the hot path (colour transform -> T-HOSVD -> HOOI sweeps -> core quantisation
-> reconstruction). Every function cites the reference file:line it follows
(paths relative to the reference's ``pkg/src/tmcodec/``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
(``cpu_baseline`` and ``--impl reference``) may import it, and only as the
checker / the timed CPU reference -- never as the thing measured or shipped.
The product package ``paper_2104_04726_b200`` never imports it and fails loudly
when its CUDA library is missing.

Pinning: ``tests/test_oracle.py`` checks this restatement against the
reference's own known-answer values and against golden
vectors produced by importing the reference itself in this container
(``scripts/make_golden.py`` -> ``tests/golden/*.npz``).
"""

from .tucker_oracle import *  # noqa: F401,F403
from .tucker_oracle import __all__  # noqa: F401
