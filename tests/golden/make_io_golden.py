"""Golden nlcsr / nlmesh files written by the REFERENCE's own writers.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_io_golden.py

Takes the reference-assembled matrix and mesh of the lshape16_const fixture
and writes them with nlfem.assembly.write_nlcsr and nlfem.mesh.write_mesh
(assembly.py:509-516, mesh.py:259-266); tests/test_io.py requires this
repo's writers to produce the same bytes.

write_mesh formats numpy scalars with !r; under numpy >= 2 that prints
"np.float64(-0.1)", which the reference's own read_mesh cannot parse, so the
fixture is written with numpy's 1.25 scalar repr (the text the reference
writes under the numpy 1.x its pyproject allows).
"""
import os
import sys

import numpy as np
from scipy import sparse

sys.path.insert(0, "/root/reference/pkg/src")
from nlfem import assembly as A  # noqa: E402
from nlfem import mesh as M  # noqa: E402

np.set_printoptions(legacy="1.25")
HERE = os.path.dirname(os.path.abspath(__file__))
z = np.load(os.path.join(HERE, "lshape16_const.npz"), allow_pickle=True)
n = len(z["indptr"]) - 1
A.write_nlcsr(os.path.join(HERE, "io_lshape16.nlcsr"),
              sparse.csr_matrix((z["data"], z["indices"], z["indptr"]), shape=(n, n)))
M.write_mesh(M.Mesh(z["vertices"], z["elements"], z["labels"]), os.path.join(HERE, "io_lshape16.nlmesh"))
print("wrote io_lshape16.nlcsr, io_lshape16.nlmesh")
