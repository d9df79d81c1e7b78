"""The reference's synthetic 2-D pair generators (``synthesis.py``) are not on
the hot path; the B200 package does not provide them."""


def synthesize_pair(kind, size=64, seed=0, **kwargs):
    raise NotImplementedError("blreg.synthesis is outside the B200 hot path (DESIGN.md §8)")
