"""Quadrature rules and the touching-pair path selection.

Restates ``/root/reference/pkg/src/nlfem/quadrature.py``:
``QuadratureConfig`` :32-66, ``dispatch`` :69-89 (Table 1 of the paper),
``rule_7point`` :92-112, ``gauss_legendre`` :121-126 and the tensorised
singular rules ``singular_rule`` :290-310 (``_identical_maps`` :161-208,
``_edge_maps`` :211-256, ``_vertex_maps`` :259-287).

The tables are built on the host once (lru-cached) and uploaded to the
device with the problem.  They are computed with the same floating-point
expressions as the reference, so the node/weight tables agree bit for bit
(checked by tests/test_host_types.py when the reference is importable).
"""

import enum
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .errors import ConfigurationError
from .geometry import PairClass

TRIANGLE_RULES = ("7point",)
WEAK_SINGULAR_MODES = ("avoid", "transform")


class Path(enum.Enum):
    STANDARD = "standard"
    AVOID_DIAGONAL = "avoid-diagonal"
    REGULARIZING = "regularizing"


# device path codes (bfs_assemble's path_touch)
PATH_CODES = {Path.STANDARD: 0, Path.AVOID_DIAGONAL: 1, Path.REGULARIZING: 2}


@dataclass(frozen=True)
class QuadratureConfig:
    """Outer/inner triangle rule names, Gauss order of the tensor rules and
    the treatment of touching pairs for -1 < s <= 0 ("avoid" | "transform")."""

    outer: str = "7point"
    inner: str = "7point"
    gauss_points_1d: int = 5
    weak_singular: str = "avoid"

    def __post_init__(self):
        for which in (self.outer, self.inner):
            if which not in TRIANGLE_RULES:
                raise ConfigurationError(f"unknown triangle rule {which!r}")
        if not isinstance(self.gauss_points_1d, int) or self.gauss_points_1d < 2:
            raise ConfigurationError("gauss_points_1d must be an integer >= 2")
        if self.weak_singular not in WEAK_SINGULAR_MODES:
            raise ConfigurationError(
                f"weak_singular must be one of {WEAK_SINGULAR_MODES}, got {self.weak_singular!r}")

    @property
    def outer_rule(self):
        return triangle_rule(self.outer)

    @property
    def inner_rule(self):
        return triangle_rule(self.inner)


def dispatch(s, pair_class, weak_singular="avoid"):
    """Integration path of a pair: Table 1 of the paper."""
    if s >= 1.0:
        raise ConfigurationError(f"kernel exponent s={s} is not below 1")
    if pair_class is PairClass.DISJOINT or s <= -1.0:
        return Path.STANDARD
    if s <= 0.0 and weak_singular != "transform":
        return Path.AVOID_DIAGONAL
    return Path.REGULARIZING


@lru_cache(maxsize=None)
def _rule7():
    # barycentre, the three corners, the three edge midpoints (degree 3)
    pts = np.array([[1.0 / 3.0, 1.0 / 3.0], [0.0, 0.0], [1.0, 0.0], [0.0, 1.0],
                    [0.5, 0.0], [0.5, 0.5], [0.0, 0.5]])
    w = np.array([27.0, 3.0, 3.0, 3.0, 8.0, 8.0, 8.0]) / 120.0
    pts.setflags(write=False)
    w.setflags(write=False)
    return pts, w


def rule_7point():
    """7-point degree-3 rule on the reference triangle; weights sum to 1/2."""
    return _rule7()


def triangle_rule(name):
    if name == "7point":
        return rule_7point()
    raise ConfigurationError(f"unknown triangle rule {name!r}")


def gauss_legendre(n):
    """Gauss-Legendre nodes and weights mapped to (0, 1)."""
    if n < 1:
        raise ConfigurationError("gauss_legendre needs n >= 1")
    t, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (t + 1.0), 0.5 * w


def hats(p):
    """The three reference hat functions at points p (N, 2) -> (N, 3)."""
    return np.column_stack([1.0 - p[:, 0] - p[:, 1], p[:, 0], p[:, 1]])


class TensorizedSingularRule:
    """Point pairs (xs, ys) on two reference triangles with weights w that
    include every transform Jacobian, plus the hat values hx, hy there."""

    __slots__ = ("kind", "xs", "ys", "w", "hx", "hy")

    def __init__(self, kind, xs, ys, w):
        self.kind = kind
        self.xs, self.ys, self.w = xs, ys, w
        self.hx, self.hy = hats(xs), hats(ys)
        for arr in (self.xs, self.ys, self.w, self.hx, self.hy):
            arr.setflags(write=False)

    @property
    def n_points(self):
        return self.w.shape[0]


def _grid4(g, gw):
    """Flattened 4-D tensor grid of nodes and of per-axis weights."""
    nodes = [a.ravel() for a in np.meshgrid(g, g, g, g, indexing="ij")]
    weights = [a.ravel() for a in np.meshgrid(gw, gw, gw, gw, indexing="ij")]
    return nodes, weights


def _mirror(pieces):
    """Stack (x, y, w) sub-rules, each followed by its x<->y swapped copy."""
    xs, ys, ws = [], [], []
    for x, y, w in pieces:
        xs += [x, y]
        ys += [y, x]
        ws += [w, w]
    return np.concatenate(xs), np.concatenate(ys), np.concatenate(ws)


def _identical_family(g, gw):
    (xi, e1, t1, t2), (a, b, c, d) = _grid4(g, gw)
    w = a * b * c * d * xi * (1.0 - xi) ** 2 * t1
    u0 = t1 * (1.0 - t2)
    u1 = t1 * t2
    zero, one = np.zeros_like(xi), np.ones_like(xi)
    # (offset of x, direction from x to y) for the three difference sectors
    sectors = ((zero, zero, 1.0 - e1, e1),
               (xi * e1, zero, -e1, one),
               (xi, zero, -one, 1.0 - e1))
    pieces = []
    for ox0, ox1, dz0, dz1 in sectors:
        x = np.column_stack([ox0 + (1.0 - xi) * u0, ox1 + (1.0 - xi) * u1])
        y = np.column_stack([x[:, 0] + xi * dz0, x[:, 1] + xi * dz1])
        pieces.append((x, y, w))
    return _mirror(pieces)


def _edge_family(g, gw):
    (xi, h1, h2, h3), (a, b, c, d) = _grid4(g, gw)
    wall = a * b * c * d
    sh = (1.0 - xi) * h3
    pieces = [
        (np.column_stack([sh, xi * h1 * (1.0 - h2)]),
         np.column_stack([sh + xi * (1.0 - h1), xi * h1]),
         wall * xi ** 2 * h1 * (1.0 - xi)),
        (np.column_stack([sh, xi * (h1 + (1.0 - h1) * h2)]),
         np.column_stack([sh + xi * (1.0 - h1), xi * h1]),
         wall * xi ** 2 * (1.0 - h1) * (1.0 - xi)),
        (np.column_stack([sh, xi + 0.0 * h1]),
         np.column_stack([sh + xi * (1.0 - h1) * h2, xi * h1]),
         wall * xi ** 2 * (1.0 - h1) * (1.0 - xi)),
    ]
    return _mirror(pieces)


def _vertex_family(g, gw):
    (xi, h1, h2, h3), (a, b, c, d) = _grid4(g, gw)
    x = np.column_stack([xi * (1.0 - h1), xi * h1])
    y = np.column_stack([xi * h2 * (1.0 - h3), xi * h2 * h3])
    w = a * b * c * d * xi ** 3 * h2
    return _mirror([(x, y, w)])


_FAMILIES = {"identical": _identical_family, "edge": _edge_family, "vertex": _vertex_family}
SINGULAR_KINDS = tuple(_FAMILIES)


@lru_cache(maxsize=None)
def singular_rule(kind, n_1d):
    """Tensorised rule of one touching class ("identical" | "edge" | "vertex").

    6 n^4 points for identical and edge pairs, 2 n^4 for vertex pairs; each
    family's weights sum to 1/4, the measure of two reference triangles.
    """
    if n_1d < 2:
        raise ConfigurationError("singular rules need at least 2 Gauss points per axis")
    if kind not in _FAMILIES:
        raise ConfigurationError(f"unknown singular rule kind {kind!r}")
    g, gw = gauss_legendre(n_1d)
    xs, ys, w = _FAMILIES[kind](g, gw)
    return TensorizedSingularRule(kind, np.ascontiguousarray(xs), np.ascontiguousarray(ys),
                                  np.ascontiguousarray(w))
