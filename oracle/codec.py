"""Software FP8 E4M3 and BF16 codecs (oracle; TEST INFRASTRUCTURE ONLY).

The paper names E4M3 as its FP8 format (§4.1) and fixes its maximum
magnitude through Algorithm 1 step 7, ``sigma_p = m / 448.0``.  It is
silent on rounding, overflow and the sign of zero; reading R3 adopts
round-to-nearest-even, saturation to +-448 (never a NaN code) and -0 -> 0x80.

E4M3 layout: 1 sign bit, 4 exponent bits (bias 7), 3 mantissa bits.
  E == 0      : subnormal, value = q * 2^-9
  1 <= E <= 15: value = (1 + q/8) * 2^(E-7), except E == 15, q == 7 (NaN)
  max finite  = 1.75 * 2^8 = 448 (code 0x7E)

All arithmetic below is exact in float64 (inputs are float32), so the only
rounding is the explicit RNE step (numpy ``rint`` rounds half to even).
"""
import numpy as np

E4M3_MAX = 448.0          # P:696 (Alg.1 step 7 divides by 448.0)
_MIN_NORMAL = 2.0 ** -6   # smallest normal E4M3 magnitude (E = 1, q = 0)
_SUBNORMAL_ULP = 2.0 ** -9


def encode_e4m3(x):
    """float32 array -> uint8 E4M3 codes, RNE, saturating, sign of zero kept.

    Reading R3: |x| >= 448 saturates to 0x7E | sign; a negative
    value that rounds to zero returns 0x80.  Non-finite input raises.
    """
    x = np.asarray(x, dtype=np.float32)
    if not np.all(np.isfinite(x)):
        raise ValueError("encode_e4m3: non-finite operand")
    xd = x.astype(np.float64)
    sign = np.signbit(xd).astype(np.uint8) << 7
    a = np.abs(xd)
    code = np.zeros(a.shape, dtype=np.int64)

    sub = a < _MIN_NORMAL
    # subnormal range: multiples of 2^-9; q == 8 is exactly the smallest normal
    # (code 0x08), so the integer q is already the code.
    code[sub] = np.rint(a[sub] / _SUBNORMAL_ULP).astype(np.int64)

    nrm = ~sub
    if np.any(nrm):
        an = a[nrm]
        f, e2 = np.frexp(an)            # an = f * 2^e2, f in [0.5, 1)
        e = e2 - 1                       # an = (2f) * 2^e, 2f in [1, 2)
        q = np.rint((2.0 * f - 1.0) * 8.0).astype(np.int64)
        carry = q == 8
        e = np.where(carry, e + 1, e)
        q = np.where(carry, 0, q)
        cn = ((e + 7) << 3) | q
        cn = np.where((an >= E4M3_MAX) | (cn > 0x7E), 0x7E, cn)
        code[nrm] = cn
    return (code.astype(np.uint8) | sign).astype(np.uint8)


def decode_e4m3(code):
    """uint8 E4M3 codes -> exact float64 values; NaN codes (0x7F, 0xFF) raise."""
    c = np.asarray(code, dtype=np.uint8).astype(np.int64)
    if np.any((c & 0x7F) == 0x7F):
        raise ValueError("decode_e4m3: invalid fp8 code (NaN pattern)")
    s = np.where(c & 0x80, -1.0, 1.0)
    E = (c >> 3) & 0xF
    q = (c & 7).astype(np.float64)
    mag = np.where(E == 0, q * _SUBNORMAL_ULP,
                   (1.0 + q / 8.0) * np.exp2((E - 7).astype(np.float64)))
    return s * mag


def bf16_rne_bits(x):
    """float32 array -> uint16 BF16 bit patterns, round-to-nearest-even.

    BF16 keeps the top 16 bits of the IEEE float32 pattern; RNE adds
    0x7FFF + lsb(kept part) before truncating.  Finite inputs only.
    """
    x = np.asarray(x, dtype=np.float32)
    if not np.all(np.isfinite(x)):
        raise ValueError("bf16_rne_bits: non-finite operand")
    u = x.view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return (r & 0xFFFF).astype(np.uint16)


def bf16_bits_to_f64(b):
    """uint16 BF16 bit patterns -> exact float64 values."""
    b = np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


def bf16_round(x):
    """float32 array -> float64 values on the BF16 grid (RNE)."""
    return bf16_bits_to_f64(bf16_rne_bits(x))
