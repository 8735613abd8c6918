"""Helpers shared by the GPU tests (no method arithmetic)."""
import numpy as np
import pytest


def require_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def ws_view(workspace, ptr, rows, ld, dtype=np.float32):
    """numpy copy of a buffer inside the caller-owned workspace (pointer from the C ABI)."""
    import torch
    itemsize = np.dtype(dtype).itemsize
    n = rows * ld * itemsize
    if n == 0:
        return np.zeros((rows, ld), dtype=dtype)
    off = ptr - workspace.data_ptr()
    assert 0 <= off and off + n <= workspace.numel()
    torch.cuda.synchronize()
    return workspace[off:off + n].cpu().numpy().view(dtype).reshape(rows, ld).copy()


def rownorm_err(x, y, floor=1e-6):
    """max_r ‖x_r − y_r‖∞ / max(‖y_r‖∞, floor·‖y‖∞)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    if y.size == 0:
        return 0.0
    den = np.maximum(np.abs(y).max(axis=1), floor * max(np.abs(y).max(), 1e-300))
    return float((np.abs(x - y).max(axis=1) / den).max())
