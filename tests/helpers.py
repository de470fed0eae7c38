"""Shared test helpers (tolerances, bf16 decoding)."""

import numpy as np

# north-star tolerances (BASELINE.json): relative Frobenius error
TOL_BF16 = 1e-2
TOL_F32 = 1e-4


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(float(np.linalg.norm(a)), float(np.linalg.norm(b)))
    return 0.0 if scale == 0.0 else float(np.linalg.norm(a - b) / scale)


def bf16_bits_to_f64(bits):
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return u.view(np.float32).astype(np.float64)
