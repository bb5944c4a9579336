"""Ball kinds and pair classes shared by the host layer and the device code.

Mirrors the public constants of ``/root/reference/pkg/src/nlfem/geometry.py``
(``BALL_KINDS``/``BALL_IDS`` :18-20, ``PairClass`` :23-29,
``classify_pair`` :32-37).  The clipping itself runs on the GPU
(``csrc/nlg_geom.cuh``); no host clipping code exists on the product path.
"""

import enum

BALL_KINDS = ("nocaps", "approxcaps", "infinity")
BALL_IDS = {name: i for i, name in enumerate(BALL_KINDS)}


class PairClass(enum.Enum):
    """Contact of two elements, by the number of vertex ids they share."""

    DISJOINT = 0
    VERTEX_TOUCHING = 1
    EDGE_TOUCHING = 2
    IDENTICAL = 3


def classify_pair(mesh, k, l):
    """Pair class of elements ``k`` and ``l`` of ``mesh``."""
    shared = set(mesh.elements[k].tolist()) & set(mesh.elements[l].tolist())
    return PairClass(len(shared))
