"""SURVEY.md §8(d) / Appendix A.8 algorithmic byte model of the hot path.

One pad-field pass (realize a band block on the pad grid and consume it, or
produce a pad product and transform it back) moves c_pad = 2 S (P^3 + B^3)
bytes; a full-grid transform moves c_full = 2 S (N^3 + B^3); a full-grid
pointwise field read or write moves S N^3.  The de-duplicated per-call counts
assume no cross-HVP caching (the base trajectory is re-integrated).

    python tools/bytes_model.py            # table for BASELINE configs 1-4

bench.py reports the same model for its workload as roofline_hvp.survey_model_*.
"""

from __future__ import annotations

import sys


def counts(call: str, nt: int):
    """(pad passes, full-grid transforms, full-grid fields) per call (Appendix A.8)."""
    if call == "energy":
        return 4 * nt * 12 + 3, 6, 10
    if call == "state_gradient":
        return (4 * nt * 12 + 3) + (4 * nt * 17 + 4), 3 + 10 * (nt + 1), 19 * (nt + 1)
    if call == "deformation_gradient":
        return (4 * nt * 12 + 3) + (4 * nt * 12 + 3) + 15 * (nt + 1), 6 + 3 * (nt + 1), 29
    if call == "state_gn_hvp":
        return 4 * nt * 24 + 6, 3 + 3 * (nt + 1), 6 + 12 * (nt + 1)
    if call == "deformation_gn_hvp":
        return (4 * nt * 24 + 6) + (4 * nt * 12 + 3) + 15 * (nt + 1), 6, 12
    raise ValueError(call)


def model_bytes(call: str, d: int, n: int, k: int, p: int, nt: int, real_bytes: int = 8) -> float:
    b = 2 * k + 1
    f, x, g = counts(call, nt)
    S = real_bytes
    return float(f * 2 * S * (p ** d + b ** d) + x * 2 * S * (n ** d + b ** d) + g * S * n ** d)


def reference_pad(k: int) -> int:
    """next_fast_len(4K+1) (spectral.py:142-145): the smallest 2,3,5,7,11-smooth length."""
    p = 4 * k + 1
    while True:
        r = p
        for f in (2, 3, 5, 7, 11):
            while r % f == 0:
                r //= f
        if r == 1:
            return p
        p += 1


CONFIGS = {1: (2, 64, 16, 10), 2: (3, 64, 16, 10), 3: (3, 128, 32, 10), 4: (3, 256, 64, 20)}


def main(argv=None):
    sys.path.insert(0, ".")
    from paper_1807_05117_b200.domain import default_pad

    peak = 6544.0
    print(f"{'config':>6} {'call':>20} {'P ref':>6} {'GB @ref P':>10} {'P eng':>6} {'GB @eng P':>10} "
          f"{'HVP/s bound @eng':>17}")
    for c, (d, n, k, nt) in CONFIGS.items():
        pref = reference_pad(k)
        peng = default_pad((k,) * d)[0]
        for call in ("state_gn_hvp", "deformation_gn_hvp"):
            a = model_bytes(call, d, n, k, pref, nt)
            e = model_bytes(call, d, n, k, peng, nt)
            print(f"{c:>6} {call:>20} {pref:>6} {a / 1e9:>10.2f} {peng:>6} {e / 1e9:>10.2f} "
                  f"{peak * 1e9 / e:>17.1f}")


if __name__ == "__main__":
    main()
