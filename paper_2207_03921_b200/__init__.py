"""B200-native nonlocal FE stiffness assembly (drop-in for nlfem's
bfs_assemble / assemble_load hot path, arXiv 2207.03921)."""

from .assembly import (AnsatzSpace, DevicePlan, LocalStiffness, SparseSystem, assemble_load, assemble_mass,
                       bfs_assemble, build_ansatz, local_contribution)
from .errors import ConfigurationError, DeviceError, MeshFormatError, NumericalError
from .geometry import BALL_IDS, BALL_KINDS, PairClass, classify_pair
from .kernels import (KernelSpec, affine_kernel, constant_kernel, constant_kernel_infinity,
                      fractional_kernel, label_scaled_kernel, peridynamic_kernel)
from .mesh import (AdjacencyGraph, Label, Mesh, build_adjacency_graph, generate_structured_mesh,
                   grid_mesh, lshape_mesh, perturb)
from .nlio import read_mesh, read_nlcsr, write_mesh, write_nlcsr, write_nlcsr_blocks
from .quadrature import Path, QuadratureConfig, dispatch, gauss_legendre, rule_7point, singular_rule

__all__ = [
    "AnsatzSpace", "DevicePlan", "LocalStiffness", "SparseSystem", "assemble_load", "assemble_mass", "bfs_assemble",
    "build_ansatz", "local_contribution",
    "ConfigurationError", "DeviceError", "MeshFormatError", "NumericalError",
    "BALL_IDS", "BALL_KINDS", "PairClass", "classify_pair",
    "KernelSpec", "affine_kernel", "constant_kernel", "constant_kernel_infinity",
    "fractional_kernel", "label_scaled_kernel", "peridynamic_kernel",
    "AdjacencyGraph", "Label", "Mesh", "build_adjacency_graph", "generate_structured_mesh",
    "grid_mesh", "lshape_mesh", "perturb",
    "read_mesh", "read_nlcsr", "write_mesh", "write_nlcsr", "write_nlcsr_blocks",
    "Path", "QuadratureConfig", "dispatch", "gauss_legendre", "rule_7point", "singular_rule",
]
