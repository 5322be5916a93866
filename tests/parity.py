"""Parity metrics.

* loss: scalar relative error.
* gradients, Adam m: per tensor max|gpu - ref| / max|ref|.
* Adam v (a square of the gradient): same metric against twice the tolerance.
* post-Adam parameters: same metric, over the elements whose reference
  gradient is determined at the run's precision (|g_ref| > tol * max|g_ref|
  of the tensor). Adam's first steps are ~lr*sign(g), so where g is below the
  precision of the path the sign (and hence a 2*lr move) is not determined;
  those elements are instead checked to differ by at most 2*lr*steps.
"""
import numpy as np

TOL = {"bf16": 1e-2, "fp32": 1e-5}


def tensor_slices(lay, lo, hi):
    """[(name, start, end)] of the canonical tensors inside [lo, hi)."""
    out = []
    for _, name, shape, off in lay.entries:
        n = int(np.prod(shape))
        if lo <= off < hi:
            out.append((name, off - lo, off - lo + n))
    return out


def normwise(a, b):
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / den) if den > 0 else float(np.abs(a - b).max())


def check_tensors(lay, lo, hi, gpu, ref, tol, what):
    worst = 0.0
    for name, a, b in tensor_slices(lay, lo, hi):
        e = normwise(gpu[a:b], ref[a:b])
        assert e <= tol, f"{what} {name}: {e:.3e} > {tol:.1e}"
        worst = max(worst, e)
    return worst


def check_params(lay, lo, hi, gpu, ref, ref_grad, tol, lr, steps):
    worst = 0.0
    for name, a, b in tensor_slices(lay, lo, hi):
        g = np.abs(ref_grad[a:b])
        mask = g > tol * g.max() if g.max() > 0 else np.zeros_like(g, bool)
        d = np.abs(gpu[a:b] - ref[a:b])
        assert np.all(d[~mask] <= 2 * lr * steps * 1.001 + 1e-7), f"param {name} unmasked drift"
        if mask.any():
            den = np.abs(ref[a:b]).max()
            e = float(d[mask].max() / den) if den > 0 else float(d[mask].max())
            assert e <= tol, f"param {name}: {e:.3e} > {tol:.1e}"
            worst = max(worst, e)
    return worst
