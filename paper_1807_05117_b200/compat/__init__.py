"""Host-facing (numpy) compatibility layer: ``sys.path.insert(0, <this dir>)``
makes ``import blreg`` resolve to ``compat/blreg``, a drop-in for the
reference package's hot-path modules whose arrays are numpy on the host and
whose numerics run on the B200 through ``paper_1807_05117_b200``.

SURVEY.md §8(b): "Expose these attributes (lazily copied to host when
accessed)".  Reference callers (``pkg/probe_hvp.py``, ``tests/test_objectives.py``)
run against it unmodified.
"""

import os

PATH = os.path.dirname(os.path.abspath(__file__))
