"""Pins for oracle/codec.py: E4M3 and BF16 codecs.

Pinned against (a) independent libraries (torch.float8_e4m3fn, torch.bfloat16,
ml_dtypes), (b) brute-force nearest-value search over the finite code set,
(c) closed-form facts of the format and the paper's 448.
"""
import json
import os

import ml_dtypes
import numpy as np
import torch

from oracle.codec import (bf16_bits_to_f64, bf16_rne_bits, decode_e4m3,
                          encode_e4m3)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
ALL = np.arange(256, dtype=np.uint8)
FINITE = ALL[(ALL & 0x7F) != 0x7F]


def _torch_dec(codes):
    return torch.from_numpy(np.asarray(codes, np.uint8)).view(torch.float8_e4m3fn).to(torch.float64).numpy()


def test_code_table_vs_torch_fp8():
    # independent library decode of every finite bit pattern
    np.testing.assert_array_equal(decode_e4m3(FINITE), _torch_dec(FINITE))


def test_code_table_closed_form_facts():
    v = decode_e4m3(FINITE)
    assert len(FINITE) == 254                     # 256 minus the two NaN patterns
    assert v.max() == GOLD["e4m3_max"]["value"]
    pos = decode_e4m3(np.arange(0, 0x7F, dtype=np.uint8))
    assert np.all(np.diff(pos) > 0)               # codes 0..126 strictly increasing
    assert pos[1] == 2.0 ** -9                    # min subnormal
    assert pos[8] == 2.0 ** -6                    # min normal
    assert decode_e4m3(np.uint8(0x80)) == 0.0 and np.signbit(decode_e4m3(np.uint8(0x80)))


def test_nan_codes_rejected():
    for c in (0x7F, 0xFF):
        try:
            decode_e4m3(np.uint8(c))
        except ValueError:
            continue
        raise AssertionError("NaN code accepted")


def test_round_trip_all_codes():
    np.testing.assert_array_equal(encode_e4m3(decode_e4m3(FINITE).astype(np.float32)), FINITE)


def _brute_nearest(x):
    """nearest finite E4M3 value by exhaustive search; ties -> even mantissa."""
    vals = decode_e4m3(np.arange(0, 0x7F, dtype=np.uint8))
    out = np.empty(x.shape, dtype=np.uint8)
    for i, xv in enumerate(x.astype(np.float64)):
        a = min(abs(xv), 448.0)
        d = np.abs(vals - a)
        best = np.flatnonzero(d == d.min())
        c = best[0] if len(best) == 1 else [b for b in best if b % 2 == 0][0]
        out[i] = c | (0x80 if np.signbit(xv) else 0)
    return out


def test_encode_brute_force_nearest_even():
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.standard_normal(3000) * np.exp2(rng.integers(-14, 10, 3000)),
        decode_e4m3(FINITE),                                  # exact grid points
        (decode_e4m3(np.arange(0, 0x7E, dtype=np.uint8)) +    # exact midpoints
         decode_e4m3(np.arange(1, 0x7F, dtype=np.uint8))) / 2,
        [460.0, 464.0, 500.0, 1e30, -1e30, -1e-9, 0.0, -0.0],
    ]).astype(np.float32)
    np.testing.assert_array_equal(encode_e4m3(x), _brute_nearest(x))


def test_encode_vs_torch_and_ml_dtypes():
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(200000) * np.exp2(rng.integers(-16, 9, 200000))).astype(np.float32)
    x = x[np.abs(x) <= 448.0]
    ref_t = torch.from_numpy(x).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    ref_m = x.astype(ml_dtypes.float8_e4m3fn).view(np.uint8)
    got = encode_e4m3(x)
    np.testing.assert_array_equal(got, ref_t)
    np.testing.assert_array_equal(got, ref_m)


def test_saturation_and_special_ties():
    cases = {
        448.0: 0x7E, 460.0: 0x7E, 464.0: 0x7E, 1e30: 0x7E, -1e30: 0xFE, -448.0: 0xFE,
        1.0625: 0x38,              # tie between 1.0 and 1.125 -> 1.0 (even)
        1.1875: 0x3A,              # tie between 1.125 and 1.25 -> 1.25 (even)
        2.0 ** -10: 0x00,          # half the min subnormal -> 0 (even)
        3 * 2.0 ** -10: 0x02,      # tie between 2^-9 and 2^-8 -> 2^-8 (even)
        -1e-9: 0x80,               # negative underflow keeps the sign
    }
    for x, c in cases.items():
        assert int(encode_e4m3(np.float32(x))) == c, (x, c)


def test_relative_error_bound():
    rng = np.random.default_rng(2)
    x = (rng.uniform(2.0 ** -6, 448.0, 100000) * rng.choice([-1, 1], 100000)).astype(np.float32)
    err = np.abs(decode_e4m3(encode_e4m3(x)) - x.astype(np.float64))
    assert np.all(err <= 2.0 ** -4 * np.abs(x.astype(np.float64)))


def test_bf16_vs_torch():
    rng = np.random.default_rng(3)
    u = rng.integers(0, 2 ** 32, 500000, dtype=np.uint64).astype(np.uint32)
    x = u.view(np.float32)
    x = x[np.isfinite(x)]
    # add exact ties (low 16 bits == 0x8000) around both parities
    ties = ((rng.integers(0, 2 ** 16, 2000, dtype=np.uint64).astype(np.uint32) << 16) | 0x8000).view(np.float32)
    x = np.concatenate([x, ties[np.isfinite(ties) & (np.abs(ties) < 3e38)]])
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(bf16_rne_bits(x), ref)


def test_bf16_examples():
    # 1 + 2^-8 is exactly halfway between 1.0 and 1 + 2^-7; RNE -> 1.0 (corrects S:62)
    assert bf16_bits_to_f64(bf16_rne_bits(np.float32(1 + 2 ** -8))) == 1.0
    assert bf16_bits_to_f64(bf16_rne_bits(np.float32(1 + 3 * 2 ** -8))) == 1 + 2 ** -6
    assert bf16_bits_to_f64(bf16_rne_bits(np.float32(1 + 2 ** -9))) == 1.0
