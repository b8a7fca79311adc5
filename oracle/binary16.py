"""IEEE 754 binary16 codec for the communication wire (oracle; test infrastructure).

PAPER.md:85-87 (section 3, Software): "While computation was generally done in
single precision, in order to reduce the communication overhead during all-reduce
operations, we used half-precision floats for communication."

The paper does not state the rounding mode or overflow behaviour.  Reading R7
(DESIGN.md): round-to-nearest-even (the IEEE default), magnitudes above the largest
finite binary16 value 65504 saturate to +-65504 and are counted, non-finite input is
an error carrying the first offending index.

Written from the format definition (1 sign bit, 5 exponent bits with bias 15,
10 fraction bits; subnormals have exponent field 0 and value f * 2^-24), not from a
library conversion routine.  Vectorised NumPy; every step is exact in float64.
"""
from __future__ import annotations

import numpy as np

MAX_FINITE = 65504.0  # (2 - 2^-10) * 2^15


class NonFiniteError(ValueError):
    """Non-finite value handed to the codec; ``index`` is the first offending
    flat index (SPEC error convention: error carrying the first offending index)."""

    def __init__(self, index: int):
        super().__init__(f"non-finite value at index {index}")
        self.index = int(index)


def to_binary16(x, return_saturation: bool = False):
    """Encode float values as binary16 bit patterns (uint16), RNE, saturating.

    Steps: take |x|; clamp to 65504 (saturation, counted when |x| > 65504);
    find the binade exponent e with 2^e <= |x| < 2^(e+1) (frexp);  the binary16
    quantum is 2^(max(e,-14) - 10) (normal numbers carry 10 fraction bits,
    subnormals are multiples of 2^-24);  n = |x| / quantum rounded to the nearest
    integer, ties to even (np.rint);  the pattern is
    (max(e,-14) + 14) << 10  +  n   (n in [0, 2048]; n = 2048 carries into the
    exponent field, n = 1024 in the subnormal binade is the smallest normal), with
    the sign bit 0x8000 for negative x (including -0.0).
    """
    x = np.asarray(x, dtype=np.float64)
    flat = x.reshape(-1)
    bad = ~np.isfinite(flat)
    if bad.any():
        raise NonFiniteError(int(np.argmax(bad)))
    neg = np.signbit(flat)
    a = np.abs(flat)
    sat = a > MAX_FINITE
    a = np.minimum(a, MAX_FINITE)
    _, E = np.frexp(a)               # a = f * 2^E, f in [0.5, 1)
    e = E.astype(np.int64) - 1       # 2^e <= a < 2^(e+1)
    e = np.where(a == 0.0, -25, e)   # zero goes to the subnormal binade
    eq = np.maximum(e, -14)
    n = np.rint(np.ldexp(a, -(eq - 10)))        # exact scaling, RNE to integer
    bits = ((eq + 14) << 10) + n.astype(np.int64)
    bits = bits | np.where(neg, 0x8000, 0)
    out = bits.astype(np.uint16).reshape(x.shape)
    if return_saturation:
        return out, int(sat.sum())
    return out


def from_binary16(bits) -> np.ndarray:
    """Exact widening of binary16 patterns to float64 (SPEC from_binary16).

    exponent field 0: (-1)^s * f * 2^-24;  1..30: (-1)^s * (1024 + f) * 2^(E-25);
    31 with f != 0 (NaN): error;  31 with f == 0: +-inf.
    """
    b = np.asarray(bits, dtype=np.uint16).astype(np.int64)
    s = (b >> 15) & 1
    E = (b >> 10) & 0x1F
    f = b & 0x3FF
    nan = (E == 31) & (f != 0)
    if nan.any():
        raise NonFiniteError(int(np.argmax(nan.reshape(-1))))
    mag = np.where(E == 0, np.ldexp(f.astype(np.float64), -24),
                   np.ldexp((1024 + f).astype(np.float64), (E - 25).astype(np.int64)))
    mag = np.where(E == 31, np.inf, mag)
    return np.where(s == 1, -mag, mag)
