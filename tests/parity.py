"""Parity metrics.

* loss: scalar relative error.
* gradients, Adam m: per tensor relative error. fp32 check mode (tol 1e-5):
  max|gpu - ref| / max|ref|. bf16 (tol 1e-2): relative Frobenius error
  ||gpu - ref||_2 / ||ref||_2 — the max-based ratio sits at the bf16 noise
  floor (~1e-2 for weight gradients behind 3-4 bf16 roundings, DESIGN.md
  "Tolerances"), so it is reported, not gated, in bf16.
* Adam v (a square of the gradient): same metric against twice the tolerance.
* post-Adam parameters: same metric, over the elements whose reference
  gradient is well determined at the run's precision and large against
  Adam's eps (|g_ref| > mask * max|g_ref| of the tensor, mask 1e-3 in fp32,
  1e-2 in bf16). Adam's update is ~lr*g/(|g|+eps): where g is below the path's
  precision its sign (and hence a 2*lr move) is not determined, and for small
  |g| the ratio amplifies g's relative error; those elements are instead
  checked to differ by at most 2*lr*steps. After more than one step only
  that drift bound is checked (an earlier undetermined sign has moved the
  element by ~2*lr whatever the later gradients are).
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


def frobenius(a, b):
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a - b))


def metric_for(tol):
    return frobenius if tol >= 1e-3 else normwise


def check_tensors(lay, lo, hi, gpu, ref, tol, what):
    worst = 0.0
    f = metric_for(tol)
    for name, a, b in tensor_slices(lay, lo, hi):
        e = f(gpu[a:b], ref[a:b])
        assert e <= tol, f"{what} {name}: {e:.3e} > {tol:.1e}"
        worst = max(worst, e)
    return worst


def check_params(lay, lo, hi, gpu, ref, ref_grad, tol, lr, steps):
    """ref_grad: the reference gradient of the (single) step taken. For
    steps > 1 only the drift bound |p_gpu - p_ref| <= 2*lr*steps is checked:
    an element whose earlier-step gradient was undetermined moved by ~2*lr
    regardless of the current gradient (Adam's update is ~lr*sign(g))."""
    worst = 0.0
    mask_frac = 1e-3 if tol < 1e-3 else 1e-2
    for name, a, b in tensor_slices(lay, lo, hi):
        g = np.abs(ref_grad[a:b])
        mask = g > mask_frac * g.max() if g.max() > 0 else np.zeros_like(g, bool)
        d = np.abs(gpu[a:b] - ref[a:b])
        if steps > 1:
            assert np.all(d <= 2 * lr * steps * 1.001 + 1e-7), f"param {name} drift"
            continue
        assert np.all(d[~mask] <= 2 * lr * steps * 1.001 + 1e-7), f"param {name} unmasked drift"
        if mask.any():
            e = metric_for(tol)(gpu[a:b][mask], ref[a:b][mask])
            assert e <= tol, f"param {name}: {e:.3e} > {tol:.1e}"
            worst = max(worst, e)
    return worst
