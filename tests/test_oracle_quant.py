"""Pins for oracle/quant.py (§5)."""
import numpy as np
import pytest

from oracle.quant import (dequantize, dequantize_f32, error_bound, message_bits, quantize,
                          quantize_f32)


def test_spec_examples(spec_examples):
    for ex in spec_examples["quantize"]:
        q, lo, hi = quantize(np.array(ex["m"]), ex["B"])
        assert q[0].tolist() == ex["codes"]
        if "restored" in ex:
            np.testing.assert_array_equal(dequantize(q, lo, hi, ex["B"])[0], ex["restored"])
        qf, lf, hf = quantize_f32(np.array(ex["m"], np.float32), ex["B"])
        assert qf[0].tolist() == ex["codes"]
        if "restored" in ex:
            np.testing.assert_array_equal(dequantize_f32(qf, lf, hf, ex["B"])[0], ex["restored"])


def test_unclamped_formula_reaches_2_pow_B():
    # the printed formula maps max(m) to 2^B; reading R15 clamps it
    q, _, _ = quantize(np.array([0.0, 1.0]), 3, clamp=False)
    assert q[0].tolist() == [0, 8]


def test_message_size(spec_examples):
    ex = spec_examples["message_size"]
    assert message_bits(ex["L"], ex["B"], ex["T"]) == ex["quantized_bits"]
    assert ex["T"] * ex["L"] == ex["original_bits"]


@pytest.mark.parametrize("B", [1, 2, 4, 8, 16])
def test_error_bound_fp64(B):
    rng = np.random.default_rng(B)
    m = rng.standard_normal((10000, 17)) * rng.uniform(1e-3, 1e3, size=(10000, 1))
    q, lo, hi = quantize(m, B)
    rec = dequantize(q, lo, hi, B)
    err = np.abs(rec - m)
    bound = error_bound(lo, hi, B)[:, None]
    clamped = q == 2 ** B - 1
    # P:L604 for unclamped codes; (max−min)/2^B where the top code was clamped (R15)
    slack = 1e-12 * np.maximum(np.abs(lo), np.abs(hi))[:, None]
    assert np.all(np.where(clamped, err <= 2 * bound + slack, err <= bound + slack))
    assert q.min() >= 0 and q.max() <= 2 ** B - 1


@pytest.mark.parametrize("B", [1, 2, 4, 8, 16])
def test_error_bound_fp32_with_rounding_slack(B):
    rng = np.random.default_rng(100 + B)
    m = (rng.standard_normal((10000, 33)) * rng.uniform(1e-2, 1e2, size=(10000, 1))).astype(np.float32)
    q, lo, hi = quantize_f32(m, B)
    rec = dequantize_f32(q, lo, hi, B).astype(np.float64)
    err = np.abs(rec - m.astype(np.float64))
    rng_ = hi.astype(np.float64) - lo.astype(np.float64)
    ulp = np.spacing(np.maximum(np.abs(lo), np.abs(hi)).astype(np.float32)).astype(np.float64)
    clamped = q == 2 ** B - 1
    bound = np.where(clamped, rng_[:, None] / 2 ** B, rng_[:, None] / 2 ** (B + 1))
    assert np.all(err <= bound + 3 * ulp[:, None])


def test_order_preserving():
    rng = np.random.default_rng(7)
    m = rng.standard_normal((2000, 9))
    for B in (2, 8):
        q, _, _ = quantize(m, B)
        for r in range(m.shape[0]):
            o = np.argsort(m[r])
            assert np.all(np.diff(q[r][o]) >= 0)


def test_fp32_and_fp64_codes_agree_away_from_ties():
    rng = np.random.default_rng(3)
    m = rng.standard_normal((3000, 64)).astype(np.float32)
    q32, _, _ = quantize_f32(m, 8)
    q64, _, _ = quantize(m.astype(np.float64), 8)
    assert np.mean(q32 == q64) > 0.9999
    assert np.max(np.abs(q32 - q64)) <= 1
