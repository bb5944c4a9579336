"""Validation and marshalling of the assembly inputs.

Mirrors the prologue of the reference's ``bfs_assemble``
(``/root/reference/pkg/src/nlfem/assembly.py:212-264``): the same checks in
the same order with the same :class:`ConfigurationError` messages, the
touching-pair path of Table 1 (``_touch_path`` :187-193), the outer-element
mask for ``rows`` (:232-235), the 7-point tables (``_quad_arrays`` :123-127),
the tensor rules (:237-238) and the h-relative thresholds (:240-241).  The
result, :class:`AssemblyInputs`, is what the C ABI's ``nlg_problem`` carries.
"""

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError
from .geometry import BALL_IDS, PairClass
from .mesh import Label
from .quadrature import PATH_CODES, SINGULAR_KINDS, QuadratureConfig, dispatch, singular_rule

SPAN = 64          # reference span size, assembly.py:31 (used by the CPU oracle)
DROP_REL = 2e-14   # assembly.py:35
SKIP_REL = 1e-13   # assembly.py:38


@dataclass
class AssemblyInputs:
    vertices: np.ndarray
    elements: np.ndarray
    labels: np.ndarray
    outer_mask: np.ndarray
    dof_map: np.ndarray
    n_dofs: int
    nc: int
    is_dg: int
    kernel_id: int
    symmetric: int
    s: float
    scale: float
    delta: float
    ball_id: int
    path_touch: int
    rskip2: float
    drop2: float
    kp0: float
    kp1: float
    op: np.ndarray
    ow: np.ndarray
    oh: np.ndarray
    ip: np.ndarray
    iw: np.ndarray
    rules: tuple  # (identical, edge, vertex) TensorizedSingularRule
    label_scale: tuple = ()  # 9 factors over labels 0..2 (row-major), or () for none


def touch_path(kernel, ansatz, quad):
    """Path code of touching pairs: 0 standard, 1 avoid-diagonal, 2 regularizing."""
    path = dispatch(kernel.s, PairClass.IDENTICAL, quad.weak_singular)
    if ansatz.kind == "dg" and kernel.s > 0.5:
        raise ConfigurationError(
            "the transformed singular rule needs a continuous ansatz for s > 0.5; "
            f"got a DG ansatz with s = {kernel.s}")
    return PATH_CODES[path]


def quad_arrays(quad):
    op, ow = quad.outer_rule
    ip, iw = quad.inner_rule
    oh = np.column_stack([1.0 - op[:, 0] - op[:, 1], op[:, 0], op[:, 1]])
    return op, ow, oh, ip, iw


KERNEL_FIELDS = ("delta", "s", "n", "symmetric", "ball", "builtin_id", "scale")


def is_kernel_spec(kernel):
    """A kernel description by its fields, not its class: this package's
    :class:`~.kernels.KernelSpec` and the reference's
    ``nlfem.kernels.KernelSpec`` (kernels.py:21-54) both qualify, so a caller
    that swaps only the assembly import keeps its kernel objects."""
    return all(hasattr(kernel, f) for f in KERNEL_FIELDS)


def kernel_label_scale(kernel):
    """The 3 x 3 label table of a label-dependent kernel
    (:func:`~.kernels.label_scaled_kernel`) as 9 floats, or ()."""
    tab = getattr(kernel, "label_scale", ()) or ()
    if not len(tab):
        return ()
    t = np.asarray(tab, dtype=np.float64)
    if t.shape != (3, 3):
        raise ConfigurationError("label_scale must be a 3 x 3 table over the labels 0..2")
    if not np.array_equal(t, t.T):
        raise ConfigurationError(
            "label_scale must be symmetric: the device scales each element pair once")
    return tuple(float(v) for v in t.ravel())


def kernel_params(kernel):
    """Extra parameters of a parametrised built-in (id 3: (alpha, c))."""
    return tuple(getattr(kernel, "params", ()) or ())


def validate(mesh, adjacency, kernel, ansatz, quad, n_threads, rows, traversal):
    if quad is None:
        quad = QuadratureConfig()
    if not is_kernel_spec(kernel):
        raise ConfigurationError("kernel must be a KernelSpec")
    if kernel.n != ansatz.n:
        raise ConfigurationError(
            f"kernel has {kernel.n} output component(s) but the ansatz has {ansatz.n}")
    if rows not in ("all", "domain"):
        raise ConfigurationError(f"rows must be 'all' or 'domain', got {rows!r}")
    if traversal not in ("bfs", "brute"):
        raise ConfigurationError(f"traversal must be 'bfs' or 'brute', got {traversal!r}")
    if not isinstance(n_threads, int) or n_threads < 1:
        raise ConfigurationError(f"n_threads must be a positive integer, got {n_threads!r}")
    if adjacency is not None and adjacency.n_elements != mesh.n_elements:
        raise ConfigurationError("adjacency graph does not match the mesh")
    return quad


def marshal(mesh, adjacency, kernel, ansatz, quad=None, n_threads=1, rows="all",
            traversal="bfs"):
    """Validate like the reference and flatten into :class:`AssemblyInputs`."""
    quad = validate(mesh, adjacency, kernel, ansatz, quad, n_threads, rows, traversal)
    path_touch = touch_path(kernel, ansatz, quad)
    if kernel.builtin_id < 0:
        raise ConfigurationError(
            "the B200 assembly evaluates built-in kernels only (builtin_id 0-3); a Python "
            "callable kernel cannot run on the device and there is no CPU fallback")
    if kernel.builtin_id > 3:
        raise ConfigurationError(f"unknown built-in kernel id {kernel.builtin_id}")
    if kernel.builtin_id == 3 and len(kernel_params(kernel)) != 2:
        raise ConfigurationError("kernel id 3 needs params (alpha, c)")
    labels = mesh.labels
    outer = labels == Label.DOMAIN if rows == "domain" else labels != Label.INACTIVE
    op, ow, oh, ip, iw = quad_arrays(quad)
    h = mesh.h
    kp = kernel_params(kernel) + (0.0, 0.0)
    return AssemblyInputs(
        vertices=np.ascontiguousarray(mesh.vertices, dtype=np.float64),
        elements=np.ascontiguousarray(mesh.elements, dtype=np.int64),
        labels=np.ascontiguousarray(labels, dtype=np.int64),
        outer_mask=np.ascontiguousarray(outer, dtype=np.int64),
        dof_map=np.ascontiguousarray(ansatz.dof_map, dtype=np.int64),
        n_dofs=int(ansatz.dof_count), nc=int(ansatz.n),
        is_dg=1 if ansatz.kind == "dg" else 0,
        kernel_id=int(kernel.builtin_id), symmetric=1 if kernel.symmetric else 0,
        s=float(kernel.s), scale=float(kernel.scale), delta=float(kernel.delta),
        ball_id=BALL_IDS[kernel.ball], path_touch=path_touch,
        rskip2=(SKIP_REL * h) ** 2, drop2=DROP_REL * h * h,
        kp0=float(kp[0]), kp1=float(kp[1]),
        op=np.ascontiguousarray(op), ow=np.ascontiguousarray(ow), oh=np.ascontiguousarray(oh),
        ip=np.ascontiguousarray(ip), iw=np.ascontiguousarray(iw),
        rules=tuple(singular_rule(kind, quad.gauss_points_1d) for kind in SINGULAR_KINDS),
        label_scale=kernel_label_scale(kernel),
    )
