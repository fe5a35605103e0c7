"""Synthetic inputs shared by the GPU tests and bench.py's config lines
(test infrastructure, not product code)."""
import numpy as np


def dense_touching(seed, h, w, fg=0.36):
    """BASELINE config C3's mask: clusters of 2-4 overlapping discs (radius
    4-8 px) until `fg` of the tile is foreground, so most nuclei touch a
    neighbour.  Returns (mask u8, number of discs)."""
    rng = np.random.default_rng(seed)
    m = np.zeros((h, w), np.uint8)
    yy, xx = np.mgrid[-9:10, -9:10]
    stamps = {r: (yy * yy + xx * xx <= r * r).astype(np.uint8) for r in range(4, 9)}
    discs = 0
    while True:
        for _ in range(2000):
            cy, cx = rng.integers(9, h - 9), rng.integers(9, w - 9)
            for _ in range(rng.integers(2, 5)):
                r = int(rng.integers(4, 9))
                oy = int(np.clip(cy + rng.integers(-r, r + 1), 9, h - 10))
                ox = int(np.clip(cx + rng.integers(-r, r + 1), 9, w - 10))
                m[oy - 9:oy + 10, ox - 9:ox + 10] |= stamps[r]
                discs += 1
        if m.mean() >= fg:
            return m, discs


def serpentine_maze(h, w, level=200):
    """A 1-px corridor snaking through every other row (C2's adversarial
    long-wavefront reconstruction) and its single seed at (0, 0)."""
    maze = np.zeros((h, w), np.uint8)
    maze[0::2, :] = level
    maze[1::4, w - 1] = level
    maze[3::4, 0] = level
    seed = np.zeros_like(maze)
    seed[0, 0] = level
    return maze, seed
