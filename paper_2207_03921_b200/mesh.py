"""Labeled triangulations: the input value type of the assembly boundary.

Host-side restatement of ``/root/reference/pkg/src/nlfem/mesh.py``:
``Label`` :18-21, ``Mesh`` :35-115 (validation, CCW check, measured h),
``AdjacencyGraph`` :118-139, ``build_adjacency_graph`` :142-167,
``generate_structured_mesh`` :170-219 and ``perturb`` :222-256.  The
adjacency graph is still accepted and validated by :func:`bfs_assemble`
(it is part of the reference's entry-point signature), but the device path
finds interaction neighbours with a uniform-grid hash instead of a BFS.

Besides the reference's generators this module provides the BASELINE.json
mesh constructions: :func:`grid_mesh` for the padded
uniform grids of configs 1-4 and :func:`lshape_mesh` for config 5.
Everything is vectorised numpy so config 4 (8.4M triangles) builds in
seconds rather than the reference's per-element Python loops.
"""

import enum
import math

import numpy as np
from scipy import sparse

from .errors import ConfigurationError


class Label(enum.IntEnum):
    INACTIVE = 0
    DOMAIN = 1
    DIRICHLET = 2


_LABEL_VALUES = np.array(sorted(int(v) for v in Label))


def signed_areas(vertices, elements):
    """Half the cross product of the two edges leaving vertex 0 of each element."""
    p0 = vertices[elements[:, 0]]
    p1 = vertices[elements[:, 1]]
    p2 = vertices[elements[:, 2]]
    return 0.5 * ((p1[:, 0] - p0[:, 0]) * (p2[:, 1] - p0[:, 1])
                  - (p1[:, 1] - p0[:, 1]) * (p2[:, 0] - p0[:, 0]))


def _longest_edge(vertices, elements):
    if elements.shape[0] == 0:
        return 0.0
    best = 0.0
    for a, b in ((0, 1), (1, 2), (2, 0)):
        d = vertices[elements[:, a]] - vertices[elements[:, b]]
        best = max(best, float(np.hypot(d[:, 0], d[:, 1]).max()))
    return best


class Mesh:
    """Triangulation of the base domain with per-element labels.

    ``vertices`` (V, 2) float64, ``elements`` (K, 3) counterclockwise vertex
    ids, ``labels`` (K,) :class:`Label` values.  ``h`` is the longest edge,
    measured from the data; a declared ``h`` is only cross-checked.  Arrays
    are made read-only, so a mesh can be shared between threads and devices.
    """

    __slots__ = ("vertices", "elements", "labels", "h", "delta", "parse_report")

    def __init__(self, vertices, elements, labels, delta=0.0, h=None, parse_report=None):
        V = np.ascontiguousarray(vertices, dtype=np.float64)
        E = np.ascontiguousarray(elements, dtype=np.int64)
        L = np.ascontiguousarray(labels, dtype=np.int64)
        if V.ndim != 2 or V.shape[1] != 2:
            raise ConfigurationError("vertices must be (V, 2)")
        if E.ndim != 2 or E.shape[1] != 3:
            raise ConfigurationError("elements must be (K, 3)")
        if L.shape != (E.shape[0],):
            raise ConfigurationError("labels must be (K,)")
        if not np.isfinite(V).all():
            raise ConfigurationError("vertex coordinates must be finite")
        if E.size:
            if E.min() < 0 or E.max() >= V.shape[0]:
                raise ConfigurationError("element vertex index out of range")
        bad = np.setdiff1d(np.unique(L), _LABEL_VALUES)
        if bad.size:
            raise ConfigurationError(f"unknown element label {int(bad[0])}")
        if E.size:
            srt = np.sort(E, axis=1)
            if (srt[:, 0] == srt[:, 1]).any() or (srt[:, 1] == srt[:, 2]).any():
                raise ConfigurationError("element with repeated vertex")
            nonpos = signed_areas(V, E) <= 0.0
            if nonpos.any():
                raise ConfigurationError(
                    f"element {int(np.argmax(nonpos))} has non-positive area; "
                    "orient counterclockwise")
        measured = _longest_edge(V, E)
        if h is not None and measured > 0.0 and abs(h - measured) > 1e-12 * measured:
            raise ConfigurationError(f"declared h={h} does not match measured diameter {measured}")
        for arr in (V, E, L):
            arr.setflags(write=False)
        self.vertices = V
        self.elements = E
        self.labels = L
        self.h = measured
        self.delta = float(delta)
        self.parse_report = parse_report

    @property
    def n_vertices(self):
        return self.vertices.shape[0]

    @property
    def n_elements(self):
        return self.elements.shape[0]

    def element_coords(self, k):
        return self.vertices[self.elements[k]]

    def areas(self):
        return signed_areas(self.vertices, self.elements)


class AdjacencyGraph:
    """Vertex-sharing element neighbours in CSR form (sorted, no self loops)."""

    __slots__ = ("ptr", "idx")

    def __init__(self, ptr, idx):
        self.ptr = np.ascontiguousarray(ptr, dtype=np.int64)
        self.idx = np.ascontiguousarray(idx, dtype=np.int64)
        self.ptr.setflags(write=False)
        self.idx.setflags(write=False)

    @property
    def n_elements(self):
        return self.ptr.shape[0] - 1

    def neighbors(self, k):
        return self.idx[self.ptr[k]:self.ptr[k + 1]]


def build_adjacency_graph(mesh):
    """Neighbours sharing at least one vertex, via incidence @ incidence^T."""
    K, V = mesh.n_elements, mesh.n_vertices
    inc = sparse.csr_matrix(
        (np.ones(3 * K, dtype=np.int32), mesh.elements.ravel(),
         np.arange(0, 3 * K + 1, 3, dtype=np.int64)), shape=(K, V))
    both = (inc @ inc.T).tocsr()
    both.setdiag(0)
    both.eliminate_zeros()
    both.sort_indices()
    return AdjacencyGraph(both.indptr.astype(np.int64), both.indices.astype(np.int64))


def _split_cells(N, keep=None):
    """Row-major cell list -> two CCW triangles per cell on an (N+1)^2 grid.

    Cell (i, j) gives (p00, p10, p11) and (p00, p11, p01), the diagonal
    and numbering of the reference generator (mesh.py:198-218).
    """
    j, i = np.divmod(np.arange(N * N, dtype=np.int64), N)
    if keep is not None:
        i, j = i[keep], j[keep]
    p00 = j * (N + 1) + i
    p10, p01 = p00 + 1, p00 + N + 1
    p11 = p01 + 1
    tri = np.empty((2 * i.size, 3), dtype=np.int64)
    tri[0::2] = np.stack([p00, p10, p11], axis=1)
    tri[1::2] = np.stack([p00, p11, p01], axis=1)
    return tri


def generate_structured_mesh(half_width, delta, n_div):
    """Reference generator: (0, half_width)^2 padded by an integer number of cells."""
    if not isinstance(n_div, (int, np.integer)) or n_div < 2:
        raise ConfigurationError("n_div must be an integer >= 2")
    if half_width <= 0.0:
        raise ConfigurationError("half_width must be positive")
    if delta < 0.0:
        raise ConfigurationError("delta must be nonnegative")
    g = half_width / n_div
    m = int(round(delta / g))
    if abs(delta - m * g) > 1e-12 * max(delta, g):
        raise ConfigurationError(f"delta={delta} is not an integer multiple of the grid spacing {g}")
    N = n_div + 2 * m
    coords = (np.arange(N + 1, dtype=np.float64) - m) * g
    xx, yy = np.meshgrid(coords, coords, indexing="xy")
    verts = np.column_stack([xx.ravel(), yy.ravel()])
    tri = _split_cells(N)
    cj, ci = np.divmod(np.arange(N * N), N)
    inside = (ci >= m) & (ci < m + n_div) & (cj >= m) & (cj < m + n_div)
    labels = np.repeat(np.where(inside, int(Label.DOMAIN), int(Label.DIRICHLET)), 2)
    return Mesh(verts, tri, labels, delta=delta)


def grid_mesh(N, lo, hi, delta=0.0, domain=(0.0, 1.0)):
    """BASELINE configs 1-4: uniform N-cell grid on [lo, hi]^2.

    Vertex (i, j) sits at (lo + i g, lo + j g), g = (hi - lo) / N.  An element
    is DOMAIN iff its barycentre lies in the open square ``domain``^2, else
    DIRICHLET (the interaction layer).
    """
    g = (hi - lo) / N
    c = lo + np.arange(N + 1, dtype=np.float64) * g
    xx, yy = np.meshgrid(c, c, indexing="xy")
    verts = np.column_stack([xx.ravel(), yy.ravel()])
    tri = _split_cells(N)
    bc = verts[tri].mean(axis=1)
    a, b = domain
    inside = (bc[:, 0] > a) & (bc[:, 0] < b) & (bc[:, 1] > a) & (bc[:, 1] < b)
    labels = np.where(inside, int(Label.DOMAIN), int(Label.DIRICHLET))
    return Mesh(verts, tri, labels, delta=delta)


def lshape_mesh(N, lo=-0.1, hi=1.1, cut=0.6, delta=0.1):
    """BASELINE config 5 base mesh: the N-cell grid on [lo, hi]^2 minus the
    cells whose centre has x > cut and y > cut, kept cells numbered row-major
    and vertex ids compacted; every element DOMAIN (pure Neumann)."""
    g = (hi - lo) / N
    cj, ci = np.divmod(np.arange(N * N, dtype=np.int64), N)
    cx = lo + (ci + 0.5) * g
    cy = lo + (cj + 0.5) * g
    keep = ~((cx > cut) & (cy > cut))
    tri = _split_cells(N, keep)
    used = np.unique(tri)
    remap = np.full((N + 1) * (N + 1), -1, dtype=np.int64)
    remap[used] = np.arange(used.size)
    c = lo + np.arange(N + 1, dtype=np.float64) * g
    xx, yy = np.meshgrid(c, c, indexing="xy")
    verts = np.column_stack([xx.ravel(), yy.ravel()])[used]
    labels = np.full(tri.shape[0], int(Label.DOMAIN), dtype=np.int64)
    return Mesh(verts, remap[tri], labels, delta=delta)


def perturb(mesh, amplitude=0.2, seed=0):
    """Seeded interior-vertex jitter (reference mesh.py:222-256).

    Boundary vertices (endpoints of edges owned by one element) stay put;
    the others move uniformly inside a disk of radius amplitude * shortest
    edge; the amplitude halves until every element keeps positive area.
    Same random stream as the reference, so the same seed gives the same mesh.
    """
    E = mesh.elements
    ends = np.concatenate([E[:, [0, 1]], E[:, [1, 2]], E[:, [2, 0]]])
    ends.sort(axis=1)
    edges, counts = np.unique(ends, axis=0, return_counts=True)
    fixed = np.zeros(mesh.n_vertices, dtype=bool)
    fixed[edges[counts == 1].ravel()] = True
    d = mesh.vertices[edges[:, 0]] - mesh.vertices[edges[:, 1]]
    emin = math.inf
    for dx, dy in d.tolist():
        emin = min(emin, math.hypot(dx, dy))
    rng = np.random.default_rng(seed)
    theta = rng.uniform(0.0, 2.0 * math.pi, mesh.n_vertices)
    rad = np.sqrt(rng.uniform(0.0, 1.0, mesh.n_vertices))
    disp = np.column_stack([rad * np.cos(theta), rad * np.sin(theta)])
    disp[fixed] = 0.0
    a = amplitude * emin
    for _ in range(20):
        moved = mesh.vertices + a * disp
        if (signed_areas(moved, E) > 0.0).all():
            return Mesh(moved, E, mesh.labels, delta=mesh.delta)
        a *= 0.5
    raise ConfigurationError("could not perturb mesh without inverting elements")
