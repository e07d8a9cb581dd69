"""The marginalised data term phi and the problem container
(spcp objective.py:20-117), backed by the GPU.

`ProblemSpec` keeps the reference's fields and validation; on first use it
uploads X (fp32 and/or fp64 copies) and the bit-packed mask to HBM once
(`ProblemSpec.device`).  `phi_value_grad` evaluates phi, grad phi and S* on
the device.  `shrink` / `huber` are the scalar/elementwise helpers of the
reference API.
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import DimensionError
from .validation import as_mask, as_matrix

__all__ = ["ProblemSpec", "shrink", "huber", "phi_value_grad", "set_default_precision",
           "get_default_precision"]

_DEFAULT_PRECISION = {"value": "fp64"}


def set_default_precision(p):
    """Precision used by split_objective / phi_value_grad when none is given:
    "fp64" (default, reference-exact), "fp32" (fused fp32 kernel)."""
    if p not in ("fp32", "fp64"):
        raise ValueError(f"precision must be 'fp32' or 'fp64', got {p!r}")
    _DEFAULT_PRECISION["value"] = p


def get_default_precision():
    return _DEFAULT_PRECISION["value"]


def _is_torch(x):
    mod = type(x).__module__
    return mod.startswith("torch")


@dataclass(frozen=True)
class ProblemSpec:
    """Observations X (off-mask entries ignored), optional boolean mask and the
    two penalties (objective.py:20-59).  `x` may also be a CUDA tensor (data
    generated on the device, e.g. the 200000 x 20000 benchmark shape)."""

    x: object
    lambda_l: float
    lambda_s: float
    mask: np.ndarray | None = field(default=None)

    def __post_init__(self):
        if _is_torch(self.x):
            import torch

            xt = self.x
            if xt.dim() != 2:
                raise DimensionError(f"x must be a 2-D matrix, got ndim={xt.dim()}")
            if not bool(torch.isfinite(xt).all()):
                raise ValueError("x contains NaN or Inf entries")
            shape = tuple(xt.shape)
        else:
            object.__setattr__(self, "x", as_matrix(self.x, "x"))
            shape = self.x.shape
        object.__setattr__(self, "mask", as_mask(self.mask, shape))
        object.__setattr__(self, "lambda_l", float(self.lambda_l))
        object.__setattr__(self, "lambda_s", float(self.lambda_s))
        if not self.lambda_l > 0.0:
            raise ValueError(f"lambda_l must be positive, got {self.lambda_l}")
        if not self.lambda_s > 0.0:
            raise ValueError(f"lambda_s must be positive, got {self.lambda_s}")
        object.__setattr__(self, "_dev", None)
        object.__setattr__(self, "_exact32", None)

    @property
    def shape(self):
        return tuple(self.x.shape)

    def observed(self):
        """Zero-filled observations (objective.py:49-53)."""
        if self.mask is None:
            return self.x
        return np.where(self.mask, self.x, 0.0)

    def project(self, a):
        """Zero the unobserved entries of a (objective.py:55-59)."""
        if self.mask is None:
            return a
        return np.where(self.mask, a, 0.0)

    # ---------------------------------------------------------------- device
    def fp32_exact(self):
        """True when every X entry is exactly representable in float32, so one
        fp32 copy in HBM serves both the fp32 and the fp64 kernels."""
        if self._exact32 is None:
            if _is_torch(self.x):
                import torch

                ex = self.x.dtype == torch.float32 or bool(
                    (self.x.float().double() == self.x).all())
            else:
                ex = bool(np.array_equal(self.x.astype(np.float32).astype(np.float64), self.x))
            object.__setattr__(self, "_exact32", ex)
        return self._exact32

    def device(self, precision="fp64"):
        """The DeviceProblem holding this spec in HBM, with the X copies the
        requested precision ("fp32" | "fp64" | "mixed") needs."""
        from .device import DeviceProblem

        if precision not in ("fp32", "fp64", "mixed"):
            raise ValueError(f"unknown precision {precision!r}")
        exact = self.fp32_exact()
        need = set()
        if precision in ("fp32", "mixed"):
            need.add("f32")
        if precision in ("fp64", "mixed"):
            need.add("f32" if exact else "f64")
        dev = self._dev
        if dev is not None and need <= dev.store:
            return dev
        store = set(need) | (set(dev.store) if dev is not None else set())
        # the replaced problem is not closed here: callers may still hold it;
        # it frees its HBM when the last reference goes away
        dev = DeviceProblem(self.x, self.lambda_l, self.lambda_s, self.mask,
                            store=tuple(sorted(store)))
        object.__setattr__(self, "_dev", dev)
        return dev

    def release_device(self):
        if self._dev is not None:
            self._dev.close()
            object.__setattr__(self, "_dev", None)


def shrink(z, tau):
    """sign(z) max(|z| - tau, 0), the prox of tau|.| (objective.py:62-72)."""
    if tau <= 0.0:
        raise ValueError(f"tau must be positive, got {tau}")
    z = np.asarray(z, dtype=np.float64)
    out = np.sign(z) * np.maximum(np.abs(z) - tau, 0.0)
    return out if out.ndim else float(out)


def huber(z, tau):
    """z^2/2 for |z| <= tau else tau|z| - tau^2/2 (objective.py:75-87)."""
    if tau <= 0.0:
        raise ValueError(f"tau must be positive, got {tau}")
    z = np.asarray(z, dtype=np.float64)
    az = np.abs(z)
    out = np.where(az <= tau, 0.5 * z * z, tau * az - 0.5 * tau * tau)
    return out if out.ndim else float(out)


def phi_value_grad(l, spec):
    """(value, grad, s_star) of phi at a dense L, computed on the GPU
    (objective.py:90-117): r = x - l on the mask, S* = shrink(r), grad =
    -clip(r, +-lambda_s), value = sum of Huber(r)."""
    l = as_matrix(l, "l")
    if l.shape != spec.shape:
        raise DimensionError(f"l shape {l.shape} does not match data shape {spec.shape}")
    return spec.device("fp64").phi_dense_host(l)
