"""B-bit linear quantisation of vertex messages (oracle, §5 of the paper).

P:L592-595: q_i = ⌊ 2^B (m_i − min m) / (max m − min m) + 0.5 ⌋
P:L596:     message size T·L bits → B·L + 2T bits (min and max header)
P:L598-601: m̃_i = (max m − min m) / 2^B · q_i + min m
P:L602-604: error ≤ (max m − min m) / 2^(B+1)

Readings (R15): B = 8 stored as uint8, so the printed formula's value
2^B at m_i = max is clamped to 2^B − 1 (error ≤ (max−min)/2^B for clamped
elements); a constant vector (max = min) quantises to all zeros.
``quantize_f32`` / ``dequantize_f32`` follow the canonical fp32 op sequence of
R15 (every op rounded to nearest, no FMA) — the sequence the CUDA kernels use,
so codes can be compared bit-for-bit on identical fp32 inputs.
Pins: tests/test_oracle_quant.py (SPEC S:L458-468 worked values, the P:L604
bound over 10^4 vectors per B, order preservation, S:L476 message size).
"""
import numpy as np


def quantize(m, B: int, clamp: bool = True):
    """Row-wise quantisation (rows = vertices).  Returns (q int64, lo, hi) in fp64."""
    m = np.atleast_2d(np.asarray(m, dtype=np.float64))
    lo = m.min(axis=1)
    hi = m.max(axis=1)
    rng = hi - lo
    q = np.zeros(m.shape, dtype=np.int64)
    nz = rng > 0
    if nz.any():
        x = (2.0 ** B) * (m[nz] - lo[nz, None]) / rng[nz, None] + 0.5
        q[nz] = np.floor(x).astype(np.int64)
    if clamp:
        np.minimum(q, 2 ** B - 1, out=q)
    return q, lo, hi


def dequantize(q, lo, hi, B: int):
    """m̃ = (max − min)/2^B · q + min, fp64."""
    q = np.atleast_2d(q)
    return ((np.asarray(hi) - np.asarray(lo)) / (2.0 ** B))[:, None] * q + np.asarray(lo)[:, None]


def message_bits(L: int, B: int, T: int = 32) -> int:
    """Quantised message size B·L + 2T bits."""
    return B * L + 2 * T


def error_bound(lo, hi, B: int):
    """(max − min) / 2^(B+1)."""
    return (np.asarray(hi) - np.asarray(lo)) / (2.0 ** (B + 1))


def quantize_f32(d, B: int):
    """R15 canonical fp32 sequence.  d: float32 [rows, F].
    rng = hi − lo; q = 0 if rng == 0 else min(⌊RN(RN(RN(RN(d − lo)·2^B) / rng) + 0.5)⌋, 2^B − 1)."""
    d = np.atleast_2d(np.asarray(d, dtype=np.float32))
    lo = d.min(axis=1).astype(np.float32)
    hi = d.max(axis=1).astype(np.float32)
    rng = (hi - lo).astype(np.float32)
    scale = np.float32(2.0 ** B)
    with np.errstate(divide="ignore", invalid="ignore"):
        t = (d - lo[:, None]).astype(np.float32)
        t = (t * scale).astype(np.float32)
        t = (t / rng[:, None]).astype(np.float32)
        t = (t + np.float32(0.5)).astype(np.float32)
    q = np.where(rng[:, None] == 0, 0, np.floor(np.where(rng[:, None] == 0, 0, t)))
    q = np.minimum(q, 2 ** B - 1).astype(np.int64)
    return q, lo, hi


def dequantize_f32(q, lo, hi, B: int):
    """R15: deq = RN(RN(RN(rng·2^-B)·q) + lo), rng = RN(hi − lo), all fp32."""
    lo = np.asarray(lo, dtype=np.float32)
    hi = np.asarray(hi, dtype=np.float32)
    rng = (hi - lo).astype(np.float32)
    step = (rng * np.float32(2.0 ** -B)).astype(np.float32)
    v = (step[:, None] * np.atleast_2d(q).astype(np.float32)).astype(np.float32)
    return (v + lo[:, None]).astype(np.float32)
