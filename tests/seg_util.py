"""Seeded phantom B-scans for the segmentation tests (SPEC segment examples): Rayleigh speckle,
a bright fascia band at 15 mm, a bone-cortex arc with an acoustic shadow beneath it."""
import numpy as np


def phantom_frame(rng, w=256, h=600, sy=0.1, bone_mm=35.0, tilt_deg=0.0, fascia_mm=15.0,
                  sigma=40.0, shadow=True):
    img = np.minimum(sigma * np.sqrt(-2.0 * np.log1p(-rng.random((h, w)))), 255.0)
    cols = np.arange(w)
    # tilt: the arc depth varies linearly across columns (+ a slight curvature)
    depth = bone_mm + np.tan(np.radians(tilt_deg)) * (cols - w / 2) * sy + 0.5 * ((cols - w / 2) / w) ** 2
    f0 = int(round(fascia_mm / sy))
    img[f0:f0 + 8, :] = 150 + 30 * rng.random((8, w))
    for c in cols:
        r = int(round(depth[c] / sy))
        if 0 <= r < h - 3:
            img[r:r + 3, c] = 220 + 35 * rng.random(3)
            if shadow:
                img[r + 3:, c] *= 0.15
    return img.astype(np.uint8), depth


def speckle_frame(rng, w=256, h=600, sigma=40.0):
    return np.minimum(sigma * np.sqrt(-2.0 * np.log1p(-rng.random((h, w)))), 255.0).astype(np.uint8)
