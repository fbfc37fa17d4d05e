"""TEST INFRASTRUCTURE (never imported by the product): numpy restatement of
the on-device terrain segment generator (paper_2209_02878_b200/csrc/rs_gen.cu,
rs_generate_segments) for bit-exact parity of the rows it writes.

The generator itself restates the DISTRIBUTION of the reference's
generate_scene segments (/root/reference/pkg/src/raysurf/oracle.py:219-271)
with a counter-based RNG (Philox-4x32-10, the Salmon et al. 2011 constants)
instead of numpy's PCG64 stream, so that any shard of a 1B-segment batch can
be generated on the GPU that queries it.  The ground-truth flags it emits are
independently checked against the C oracle / the reference kernel in the
tests (a generated crossing segment crosses exactly once, a miss never).
"""

from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)
MARGIN = 0.05  # oracle.py:27 _GRAZE_MARGIN


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox-4x32-10 (uint32 arrays in, four uint32 arrays out)."""
    c = [np.asarray(x, dtype=np.uint32).copy() for x in (c0, c1, c2, c3)]
    k0, k1 = np.uint32(k0), np.uint32(k1)
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = M0 * c[0].astype(np.uint64)
            p1 = M1 * c[2].astype(np.uint64)
            hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & MASK).astype(np.uint32)
            hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & MASK).astype(np.uint32)
            c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
            k0 = np.uint32(k0 + W0)
            k1 = np.uint32(k1 + W1)
    return c


def _u53(a, b):
    return ((a >> np.uint32(5)).astype(np.float64) * 67108864.0
            + (b >> np.uint32(6)).astype(np.float64)) / 9007199254740992.0


def _uni(a, b, u):
    return a + (b - a) * u


def generate_segments(vertices, triangles, n, seed=2022, first=0, crossing_fraction=0.5):
    """Rows [first, first+n) exactly as rs_generate_segments writes them:
    (starts (n,3) f32, ends (n,3) f32, flags (n,) u8)."""
    V = np.asarray(vertices, dtype=np.float32)
    T = np.asarray(triangles, dtype=np.int32)
    n_t = T.shape[0]
    z_lo, z_hi = float(V[:, 2].min()), float(V[:, 2].max())
    x_hi, y_hi = float(V[:, 0].max()) + 1.0, float(V[:, 1].max()) + 1.0
    z_pad = 0.5 + 0.1 * (z_hi - z_lo)
    g = np.arange(first, first + n, dtype=np.uint64)
    glo = (g & MASK).astype(np.uint32)
    ghi = (g >> np.uint64(32)).astype(np.uint32)
    k0 = np.uint32(seed & 0xFFFFFFFF)
    k1 = np.uint32(((seed >> 32) & 0xFFFFFFFF) ^ 0x5EED)
    words = []
    for c in range(4):
        words += philox4x32_10(glo, ghi, np.full(n, c, np.uint32), np.zeros(n, np.uint32), k0, k1)
    u = [_u53(words[2 * k], words[2 * k + 1]) for k in range(8)]
    cross = u[0] < crossing_fraction
    S = np.zeros((n, 3))
    E = np.zeros((n, 3))

    # crossers (oracle.py:228-249)
    t = np.minimum((u[1] * float(n_t)).astype(np.int64), n_t - 1)
    w0, w1 = u[2].copy(), u[3].copy()
    fold = (w0 + w1) > 1.0
    w0[fold] = 1.0 - w0[fold]
    w1[fold] = 1.0 - w1[fold]
    scale = 1.0 - 3.0 * MARGIN
    b0 = MARGIN + scale * (1.0 - (w0 + w1))
    b1 = MARGIN + scale * w0
    b2 = MARGIN + scale * w1
    c = V[T[t]].astype(np.float64)  # (n,3 corners,3)
    px = (b0 * c[:, 0, 0] + b1 * c[:, 1, 0]) + b2 * c[:, 2, 0]
    py = (b0 * c[:, 0, 1] + b1 * c[:, 1, 1]) + b2 * c[:, 2, 1]
    below = z_lo - z_pad * (1.0 + u[4])
    above = z_hi + z_pad * (1.0 + u[5])
    up = u[6] < 0.5
    cs = np.column_stack([px, py, np.where(up, below, above)])
    ce = np.column_stack([px, py, np.where(up, above, below)])

    # misses (oracle.py:251-271)
    kind = (u[1] * 3.0).astype(np.int64)
    ms = np.empty((n, 3))
    me = np.empty((n, 3))
    ms[:, 1] = _uni(-1.0, y_hi, u[4])
    me[:, 1] = _uni(-1.0, y_hi, u[5])
    side = kind == 2
    ms[:, 0] = np.where(side, _uni(-6.0, -1.0, u[2]), _uni(-1.0, x_hi, u[2]))
    me[:, 0] = np.where(side, _uni(-6.0, -1.0, u[3]), _uni(-1.0, x_hi, u[3]))
    span = 2.0 * z_pad
    top, bot = z_hi + z_pad, z_lo - z_pad
    ms[:, 2] = np.select([kind == 0, kind == 1], [top + _uni(0.0, span, u[6]), bot - _uni(0.0, span, u[6])],
                         _uni(bot, top, u[6]))
    me[:, 2] = np.select([kind == 0, kind == 1], [top + _uni(0.0, span, u[7]), bot - _uni(0.0, span, u[7])],
                         _uni(bot, top, u[7]))
    S = np.where(cross[:, None], cs, ms).astype(np.float32)
    E = np.where(cross[:, None], ce, me).astype(np.float32)
    return S, E, cross.astype(np.uint8)
