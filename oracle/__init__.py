"""CPU oracle for the NeuralVDB hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package, and only
as the checker / the timed CPU reference.  The product package
(``paper_2208_04448_b200``) never imports it and has no CPU fallback.

Parity is pinned: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by running the reference package itself
(``tests/golden/make_golden.py``).
"""

from .svcodec_port import *  # noqa: F401,F403
