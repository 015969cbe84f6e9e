"""Rotary position encoding, fp64 (oracle; test infrastructure only).

The paper uses a *decoupled* RoPE key for MLA/GLA ("concatenating a small
decoupled Rotary Position Encoding (RoPE) with the latent") and a separate
single-head RoPE half for GTA.  It never states the base or the
channel pairing; the reading (R5) is base 10000,
interleaved pairs (2i, 2i+1), theta_i = base^(-2i/d).
"""

import numpy as np


def rope_angles(pos, d, base=10000.0):
    """Angles pos * theta_i for pairs i in [0, d/2); theta_i = base^(-2i/d)."""
    assert d % 2 == 0
    i = np.arange(d // 2, dtype=np.float64)
    theta = base ** (-2.0 * i / d)
    return np.asarray(pos, dtype=np.float64)[..., None] * theta


def rope_rotate(x, pos, base=10000.0):
    """Rotate the last axis of ``x`` (even width d) at position(s) ``pos``.

    ``pos`` broadcasts against ``x.shape[:-1]``.  Pair (2i, 2i+1) is rotated by
    angle pos*theta_i:  [x0 cos - x1 sin, x0 sin + x1 cos].
    """
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    ang = rope_angles(pos, d, base)
    cos, sin = np.cos(ang), np.sin(ang)
    x0 = x[..., 0::2]
    x1 = x[..., 1::2]
    out = np.empty(np.broadcast_shapes(x.shape, ang.shape[:-1] + (d,)), dtype=np.float64)
    out[..., 0::2] = x0 * cos - x1 * sin
    out[..., 1::2] = x0 * sin + x1 * cos
    return out


def rope_unrotate(x, pos, base=10000.0):
    """Inverse rotation (angle -pos*theta_i)."""
    return rope_rotate(x, -np.asarray(pos, dtype=np.float64), base)
