"""CPU restatement of the ray-marcher's compositing (TEST INFRASTRUCTURE ONLY: imported by
tests/ as the checker, never by the product).

The reference does not ship a renderer; SPEC.md render_volume fixes the rule: front-to-back
alpha compositing along each ray with a piecewise-linear (value, r, g, b, alpha) transfer
function, colour += T * alpha * rgb, T *= 1 - alpha, background blended by the final T.
"""
import numpy as np


def transfer(points, v: np.ndarray):
    """(rgb (..., 3), alpha (...)) of values v, clamped to the control-point range."""
    tab = np.asarray(points, dtype=np.float64)
    xs = tab[:, 0]
    vc = np.clip(v, xs[0], xs[-1])
    i = np.clip(np.searchsorted(xs, vc, side="right"), 1, len(xs) - 1)
    w = ((vc - xs[i - 1]) / (xs[i] - xs[i - 1]))[..., None]
    out = tab[i - 1, 1:] + w * (tab[i, 1:] - tab[i - 1, 1:])
    return out[..., :3], out[..., 3]


def composite(values: np.ndarray, points, state=None):
    """Fold a slab of values (pixels, steps) into state = (colour (pixels, 3), T (pixels,))."""
    rgb, a = transfer(points, np.asarray(values, dtype=np.float64))
    npx = values.shape[0]
    if state is None:
        state = (np.zeros((npx, 3)), np.ones(npx))
    col, tr = state[0].copy(), state[1].copy()
    for s in range(values.shape[1]):
        col += (tr * a[:, s])[:, None] * rgb[:, s]
        tr = tr * (1.0 - a[:, s])
    return col, tr


def finish(state, background, height: int, width: int):
    col, tr = state
    rad = (col + tr[:, None] * np.asarray(background, dtype=np.float64)).reshape(height, width, 3)
    img = np.floor(np.clip(rad, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
    return rad, img
