"""Image files of the splat renderer ("writes binary PPM (P6, 8-bit, sRGB with gamma 2.2) and a linear
float sidecar").  I/O only: the radiance and the 8-bit codes come from spoly_render."""
from __future__ import annotations

import numpy as np


def write_ppm(path: str, rgb) -> None:
    """rgb: (H, W, 3) uint8 (numpy or a torch tensor on any device), row 0 = first row of pixels."""
    a = rgb.cpu().numpy() if hasattr(rgb, "cpu") else np.asarray(rgb)
    a = np.ascontiguousarray(a, dtype=np.uint8)
    h, w = a.shape[:2]
    with open(path, "wb") as f:
        f.write(b"P6\n%d %d\n255\n" % (w, h))
        f.write(a.tobytes())


def write_pfm(path: str, radiance) -> None:
    """radiance: (H, W) linear values, stored as a gray little-endian PFM (rows bottom-to-top by the format)."""
    a = radiance.cpu().numpy() if hasattr(radiance, "cpu") else np.asarray(radiance)
    a = np.ascontiguousarray(a[::-1], dtype="<f4")
    h, w = a.shape
    with open(path, "wb") as f:
        f.write(b"Pf\n%d %d\n-1.0\n" % (w, h))
        f.write(a.tobytes())


def read_pfm(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        assert f.readline().strip() == b"Pf"
        w, h = map(int, f.readline().split())
        scale = float(f.readline())
        a = np.frombuffer(f.read(), dtype="<f4" if scale < 0 else ">f4").reshape(h, w)
    return a[::-1].astype(np.float64)
