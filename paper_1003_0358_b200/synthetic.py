"""Seeded synthetic 28x28 digit generator (MNIST is unavailable offline).

Each digit class 0-9 is a fixed set of pen strokes (polylines in the unit
box).  Per image we jitter the control points, apply a random scale, slant,
rotation and offset, pick a pen thickness, and rasterise with a one-pixel
anti-aliasing ramp onto the 20x20 MNIST digit box centred in 28x28.  uint8
background 0, strokes up to 255.  Output is a pure function of (n, seed),
so both the CUDA path and the CPU oracle read identical bytes.  The writers
produce the IDX containers the reference parses (mnist_io.py:79-129).
"""

from __future__ import annotations

import struct

import numpy as np

_ELL = lambda cx, cy, rx, ry, k=14: [  # noqa: E731
    (cx + rx * np.cos(t), cy + ry * np.sin(t)) for t in np.linspace(0, 2 * np.pi, k)
]

STROKES: dict[int, list[list[tuple[float, float]]]] = {
    0: [_ELL(0.5, 0.5, 0.24, 0.36, 16)],
    1: [[(0.38, 0.28), (0.52, 0.14), (0.52, 0.86)]],
    2: [[(0.25, 0.3), (0.35, 0.17), (0.55, 0.14), (0.7, 0.25), (0.68, 0.42), (0.25, 0.85),
         (0.77, 0.85)]],
    3: [[(0.25, 0.2), (0.55, 0.14), (0.72, 0.28), (0.62, 0.44), (0.42, 0.48)],
        [(0.62, 0.48), (0.74, 0.64), (0.64, 0.82), (0.25, 0.84)], [(0.42, 0.48), (0.62, 0.48)]],
    4: [[(0.62, 0.86), (0.62, 0.14), (0.22, 0.62), (0.8, 0.62)]],
    5: [[(0.72, 0.15), (0.32, 0.15), (0.29, 0.45), (0.6, 0.42), (0.73, 0.6), (0.63, 0.82),
         (0.27, 0.83)]],
    6: [[(0.66, 0.14), (0.38, 0.38), (0.28, 0.64), (0.38, 0.85), (0.62, 0.83), (0.71, 0.63),
         (0.55, 0.5), (0.3, 0.6)]],
    7: [[(0.24, 0.17), (0.76, 0.17), (0.44, 0.86)], [(0.4, 0.5), (0.66, 0.5)]],
    8: [_ELL(0.5, 0.31, 0.17, 0.16, 12), _ELL(0.5, 0.67, 0.21, 0.18, 12)],
    9: [_ELL(0.5, 0.34, 0.18, 0.18, 12), [(0.68, 0.36), (0.6, 0.86)]],
}


def _segments(digit: int) -> np.ndarray:
    segs = []
    for line in STROKES[digit]:
        for p, q in zip(line[:-1], line[1:]):
            segs.append((p, q))
    return np.asarray(segs, dtype=np.float64)  # (S, 2, 2)


_PIX = np.stack(np.meshgrid(np.arange(28) + 0.5, np.arange(28) + 0.5, indexing="xy"),
                axis=-1).reshape(-1, 2)  # (784, 2) as (x, y)
_PIX32 = _PIX.astype(np.float32)


def _render(digit: int, rng: np.random.Generator, n: int) -> np.ndarray:
    segs = _segments(digit)  # (S, 2, 2)
    S = segs.shape[0]
    pts = np.broadcast_to(segs, (n, S, 2, 2)).copy()
    pts += rng.uniform(-0.025, 0.025, size=pts.shape)
    scale = rng.uniform(0.85, 1.1, size=(n, 1, 1))
    aspect = rng.uniform(0.85, 1.15, size=(n, 1, 1))
    slant = rng.uniform(-0.25, 0.25, size=(n, 1, 1))
    rot = np.deg2rad(rng.uniform(-10, 10, size=(n, 1, 1)))
    off = rng.uniform(-2.0, 2.0, size=(n, 1, 1, 2))
    thick = rng.uniform(1.0, 2.0, size=(n, 1, 1))
    x = (pts[..., 0] - 0.5) * scale * aspect
    y = (pts[..., 1] - 0.5) * scale
    x = x - slant * y
    c, s = np.cos(rot), np.sin(rot)
    xr = c * x - s * y
    yr = s * x + c * y
    P = (np.stack([14.0 + 20.0 * xr, 14.0 + 20.0 * yr], axis=-1) + off).astype(np.float32)
    ax, ay = P[:, None, :, 0, 0], P[:, None, :, 0, 1]  # (n,1,S)
    bx, by = P[:, None, :, 1, 0] - ax, P[:, None, :, 1, 1] - ay
    px = _PIX32[None, :, 0:1] - ax  # (n,784,S)
    py = _PIX32[None, :, 1:2] - ay
    inv = 1.0 / np.maximum(bx * bx + by * by, 1e-9)
    t = np.clip((px * bx + py * by) * inv, 0.0, 1.0)
    px -= t * bx
    py -= t * by
    dist = np.sqrt((px * px + py * py).min(-1))  # (n,784)
    inten = np.clip(thick[:, 0].astype(np.float32) - dist + 0.5, 0.0, 1.0)
    return np.rint(inten * 255.0).astype(np.uint8).reshape(n, 28, 28)


def make_digits(n: int, seed: int = 12345, chunk: int = 1024) -> tuple[np.ndarray, np.ndarray]:
    """(images (n,28,28) u8, labels (n,) u8), deterministic in (n, seed)."""
    rng = np.random.Generator(np.random.Philox(key=np.array([seed, 0xD161], dtype=np.uint64)))
    labels = rng.integers(0, 10, size=n).astype(np.uint8)
    images = np.zeros((n, 28, 28), dtype=np.uint8)
    for d in range(10):
        idx = np.nonzero(labels == d)[0]
        sub = np.random.Generator(np.random.Philox(
            key=np.array([seed, 0xD161 + 1 + d], dtype=np.uint64)))
        for lo in range(0, len(idx), chunk):
            part = idx[lo:lo + chunk]
            images[part] = _render(d, sub, len(part))
    return images, labels


def write_idx_images(images: np.ndarray) -> bytes:
    images = np.ascontiguousarray(images, dtype=np.uint8)
    return struct.pack(">4I", 0x803, images.shape[0], 28, 28) + images.tobytes()


def write_idx_labels(labels: np.ndarray) -> bytes:
    labels = np.ascontiguousarray(labels, dtype=np.uint8)
    return struct.pack(">2I", 0x801, labels.shape[0]) + labels.tobytes()
