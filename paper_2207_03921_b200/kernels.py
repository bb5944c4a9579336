"""Kernel descriptions consumed by the assembly boundary.

``KernelSpec`` and the built-in factories restate
``/root/reference/pkg/src/nlfem/kernels.py`` (``KernelSpec`` :21-54,
``fractional_kernel`` :57-79, ``peridynamic_kernel`` :82-103,
``constant_kernel_infinity`` :106-118).  The device evaluates built-in
kernels by id (``csrc/nlg_kernels.cuh``):

====  =======================================  ==========================
id    value(x, y)                              reference
====  =======================================  ==========================
0     c |x-y|^(-2-2s)                           _engine._kernel_mat :33-34
1     c (x-y)(x-y)^T / |x-y|^3   (n = 2)        _engine._kernel_mat :35-41
2     c                                         _engine._kernel_mat :42-43
3     (1 + a x_0) c   (nonsymmetric)            _pyengine._pq :38-45 with
                                                BASELINE config 5's kernel
====  =======================================  ==========================

Label-dependent kernels (``value``'s ``label_x, label_y`` arguments,
reference kernels.py:21-35) run on the device as a built-in times a symmetric
3 x 3 table over the element labels (:func:`label_scaled_kernel`): interface
problems with one coefficient per pair of subdomains.

Id 3 is new: the reference reaches nonsymmetric kernels only through a
Python callable on its interpreted engine, which cannot run on a GPU.
Kernels with ``builtin_id < 0`` (arbitrary callables) are rejected by the
device path with :class:`ConfigurationError`; there is no CPU fallback.
``value`` is kept for API compatibility (the reference's ``local_contribution``
and user code call it) and agrees with the device formula bit for bit.
"""

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigurationError
from .geometry import BALL_KINDS
from .mesh import Label


@dataclass(frozen=True)
class KernelSpec:
    """Horizon, singularity exponent s, output dimension n, symmetry flag,
    ball kind, host value callable, built-in id, scale constant and the
    extra parameters of parametrised built-ins (``params``)."""

    delta: float
    s: float
    n: int
    symmetric: bool
    ball: str
    value: callable = field(compare=False)
    builtin_id: int = -1
    scale: float = math.nan
    params: tuple = ()
    label_scale: tuple = ()  # 3 x 3 factors over the element labels (label_scaled_kernel)

    def __post_init__(self):
        if self.delta <= 0.0:
            raise ConfigurationError("kernel horizon delta must be positive")
        if self.s >= 1.0:
            raise ConfigurationError(f"singularity exponent s={self.s} must be below 1")
        if self.n not in (1, 2):
            raise ConfigurationError("kernel output dimension n must be 1 or 2")
        if self.ball not in BALL_KINDS:
            raise ConfigurationError(f"ball must be one of {BALL_KINDS}, got {self.ball!r}")


def _require_delta(delta):
    if delta <= 0.0:
        raise ConfigurationError("delta must be positive")


def fractional_kernel(s, delta, ball="nocaps"):
    """c |x-y|^(-2-2s), c = (2-2s) / (pi delta^(2-2s)), 0 < s < 1 (id 0)."""
    if not 0.0 < s < 1.0:
        raise ConfigurationError(f"fractional kernel needs 0 < s < 1, got s={s}")
    _require_delta(delta)
    c = (2.0 - 2.0 * s) / (math.pi * delta ** (2.0 - 2.0 * s))
    e = -1.0 - s

    def value(x, y, label_x=Label.DOMAIN, label_y=Label.DOMAIN):
        r2 = (x[0] - y[0]) * (x[0] - y[0]) + (x[1] - y[1]) * (x[1] - y[1])
        return np.array([[c * r2 ** e]])

    return KernelSpec(delta=delta, s=s, n=1, symmetric=True, ball=ball, value=value,
                      builtin_id=0, scale=c)


def peridynamic_kernel(delta, ball="nocaps"):
    """Bond-based peridynamics c (x-y)(x-y)^T / |x-y|^3, c = 3/delta^3 (id 1, n = 2)."""
    _require_delta(delta)
    c = 3.0 / delta ** 3

    def value(x, y, label_x=Label.DOMAIN, label_y=Label.DOMAIN):
        d0, d1 = x[0] - y[0], x[1] - y[1]
        r2 = d0 * d0 + d1 * d1
        f = c / (r2 * math.sqrt(r2))
        return np.array([[f * d0 * d0, f * d0 * d1], [f * d0 * d1, f * d1 * d1]])

    return KernelSpec(delta=delta, s=-0.5, n=2, symmetric=True, ball=ball, value=value,
                      builtin_id=1, scale=c)


def constant_kernel(delta, ball="approxcaps", scale=None):
    """Constant kernel (id 2) on any ball; default scale 4/(pi delta^4).

    BASELINE configs 1 and 4 use it on the Euclidean ball, which the
    reference has no factory for (SURVEY.md App. A builds the KernelSpec by
    hand with builtin_id=2).
    """
    _require_delta(delta)
    c = 4.0 / (math.pi * delta ** 4) if scale is None else float(scale)

    def value(x, y, label_x=Label.DOMAIN, label_y=Label.DOMAIN):
        return np.array([[c]])

    return KernelSpec(delta=delta, s=-1.0, n=1, symmetric=True, ball=ball, value=value,
                      builtin_id=2, scale=c)


def constant_kernel_infinity(delta):
    """3/(4 delta^4) truncated by the square of half width delta (id 2)."""
    _require_delta(delta)
    return constant_kernel(delta, ball="infinity", scale=3.0 / (4.0 * delta ** 4))


def affine_kernel(delta, alpha=0.5, scale=None, ball="approxcaps"):
    """Nonsymmetric (1 + alpha x_0) c, c = 4/(pi delta^4) by default (id 3).

    BASELINE config 5's kernel.  ``value(x, y)`` depends on its first
    argument, so gamma(x, y) != gamma(y, x) and the device accumulates the
    P = value(x, y) and Q = value(y, x) terms separately, as the reference's
    interpreted engine does (_pyengine.py:124-151, :259-262).
    """
    _require_delta(delta)
    c = 4.0 / (math.pi * delta ** 4) if scale is None else float(scale)
    a = float(alpha)

    def value(x, y, label_x=Label.DOMAIN, label_y=Label.DOMAIN):
        return np.array([[(1.0 + a * x[0]) * c]])

    return KernelSpec(delta=delta, s=-1.0, n=1, symmetric=False, ball=ball, value=value,
                      builtin_id=3, scale=c, params=(a, c))


def label_scaled_kernel(base, table):
    """``table[label_x][label_y] * base.value(x, y)``: a built-in kernel whose
    strength depends on the labels of the two host elements (interface
    problems; the reference reaches these only through a Python callable on
    its interpreted engine, kernels.py:21-35, _pyengine.py:38-45).

    ``table`` is indexed by :class:`~.mesh.Label` (a 3 x 3 array over labels
    0..2, or a 2 x 2 array over DOMAIN, DIRICHLET) and must be symmetric: the
    device integrates each unordered element pair once and scales it when it
    is emitted.  The returned spec's ``value`` is the same formula on the
    host, so the reference's engines evaluate it identically.
    """
    t = np.asarray(table, dtype=np.float64)
    if t.shape == (2, 2):
        full = np.zeros((3, 3))
        full[1:, 1:] = t
        t = full
    if t.shape != (3, 3):
        raise ConfigurationError("label table must be 2 x 2 (DOMAIN, DIRICHLET) or 3 x 3 (labels 0..2)")
    if not np.array_equal(t, t.T):
        raise ConfigurationError("label table must be symmetric")
    if base.builtin_id < 0:
        raise ConfigurationError("label_scaled_kernel needs a built-in base kernel")
    tab = tuple(tuple(float(v) for v in row) for row in t)
    bval = base.value

    def value(x, y, label_x=Label.DOMAIN, label_y=Label.DOMAIN):
        return tab[int(label_x)][int(label_y)] * bval(x, y)

    return KernelSpec(delta=base.delta, s=base.s, n=base.n, symmetric=base.symmetric, ball=base.ball,
                      value=value, builtin_id=base.builtin_id, scale=base.scale,
                      params=tuple(getattr(base, "params", ()) or ()), label_scale=tab)
