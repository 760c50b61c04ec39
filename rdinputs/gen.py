"""Counter-based generator for the config-4/5 initial states.

SM(z) is the SplitMix64 finaliser used as a hash (Steele, Lea & Flood 2014):
    z += 0x9E3779B97F4A7C15
    z  = (z ^ z>>30) * 0xBF58476D1CE4E5B9
    z  = (z ^ z>>27) * 0x94D049BB133111EB
    return z ^ z>>31
The n-th value of stream s is R(s, n) = SM(SM(s) + n), all mod 2^64.
Everything is in GLOBAL coordinates, so a row slab of rank r of G generates
exactly the rows the single-GPU grid has (the inputs are independent of G).
"""
from __future__ import annotations

import numpy as np

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(z):
    """SM(z) on a uint64 scalar or array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def stream(s: int, n):
    """R(s, n) = SM(SM(s) + n)."""
    base = splitmix64(np.uint64(s))
    with np.errstate(over="ignore"):
        return splitmix64(base + np.asarray(n, dtype=np.uint64))


def noise_plane(H: int, W: int, plane: int, seed: int = 1, dtype=np.float32, row0: int = 0,
                W_global: int | None = None, amplitude: float = 0.1) -> np.ndarray:
    """i.i.d. U[0, amplitude) noise for plane p (0: u, 1: v) of rows [row0, row0+H).

    value = ((x >> 40) * 2^-24) * amplitude in fp64, rounded once to dtype, with
    x = R(seed, (p << 62) | (i * W_global + j)) for GLOBAL cell (i, j).
    """
    Wg = W if W_global is None else W_global
    out = np.empty((H, W), dtype=dtype)
    base = splitmix64(np.uint64(seed))
    tag = np.uint64(plane) << np.uint64(62)
    j = np.arange(W, dtype=np.uint64)
    rows_per = max(1, (1 << 22) // max(W, 1))
    for i0 in range(0, H, rows_per):
        i1 = min(H, i0 + rows_per)
        i = np.arange(row0 + i0, row0 + i1, dtype=np.uint64)[:, None]
        with np.errstate(over="ignore"):
            idx = tag | (i * np.uint64(Wg) + j[None, :])
            x = splitmix64(base + idx)
        val = (x >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)
        val = val * amplitude
        out[i0:i1] = val.astype(dtype)
    return out


def half_discs(H: int, W: int, count: int = 64, seed: int = 2, radius: int = 8,
               mask_phi: float | None = None) -> list[dict]:
    """`count` broken-wavefront seeds: cy = R(s,3k) mod H, cx = R(s,3k+1) mod W,
    dir = R(s,3k+2) mod 4 (0:+x 1:+y 2:-x 3:-y); u := 1 on the half-disc of
    radius `radius` facing dir (BASELINE.json configs[3]). With mask_phi the
    write is restricted to cells whose phi equals it (R-22)."""
    k = np.arange(count, dtype=np.uint64)
    cy = stream(seed, 3 * k) % np.uint64(H)
    cx = stream(seed, 3 * k + np.uint64(1)) % np.uint64(W)
    d = stream(seed, 3 * k + np.uint64(2)) % np.uint64(4)
    out = []
    for a, b, c in zip(cy.tolist(), cx.tolist(), d.tolist()):
        s = {"kind": "half_disc", "cy2": 2 * int(a), "cx2": 2 * int(b), "r": radius, "dir": int(c)}
        if mask_phi is not None:
            s["mask_phi"] = mask_phi
        out.append(s)
    return out


def obstacles(H: int, W: int, count: int = 256, seed: int = 3) -> list[tuple[int, int, int, int]]:
    """Rectangles [y0,y0+h) x [x0,x0+w) clipped to the grid, h,w in 32..1024:
    y0 = R(s,4k) mod H, x0 = R(s,4k+1) mod W, h = 32 + R(s,4k+2) mod 993,
    w = 32 + R(s,4k+3) mod 993 (BASELINE.json configs[4])."""
    k = np.arange(count, dtype=np.uint64)
    y0 = (stream(seed, 4 * k) % np.uint64(H)).astype(np.int64)
    x0 = (stream(seed, 4 * k + np.uint64(1)) % np.uint64(W)).astype(np.int64)
    h = 32 + (stream(seed, 4 * k + np.uint64(2)) % np.uint64(993)).astype(np.int64)
    w = 32 + (stream(seed, 4 * k + np.uint64(3)) % np.uint64(993)).astype(np.int64)
    return [(int(a), int(b), int(min(H, a + c)), int(min(W, b + d))) for a, b, c, d in zip(y0, x0, h, w)]
