"""``blreg`` on the B200: numpy in / numpy out, sm_100a kernels underneath
(paper_1807_05117_b200).  Mirrors ``pkg/src/blreg/__init__.py``."""

from .domain import Domain

__version__ = "0.1.0"

__all__ = ["Domain", "__version__"]
