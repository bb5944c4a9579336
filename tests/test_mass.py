"""Mass matrix (assembly.py:484-506): the oracle restatement is
pinned against the reference itself (CPU, where the reference tree exists);
the device assembly against the oracle (GPU)."""

import numpy as np
import pytest

from golden_io import Case, rel_fro, same_pattern
from oracle import oracle

CASES = ["cfg1_approxcaps", "peri_nocaps_avoid", "lshape16_const", "frac_s04_nocaps_dg"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_mass_matches_reference(name, reference):
    import sys
    c = Case(name)
    rmesh = sys.modules["nlfem.mesh"].Mesh(c.mesh.vertices, c.mesh.elements, c.mesh.labels)
    ref = reference.assemble_mass(rmesh, reference.build_ansatz(rmesh, c.spec["ansatz"], c.spec["n"]))
    ours = oracle.assemble_mass(c.mesh, c.ansatz)
    assert same_pattern(ours, ref)
    assert rel_fro(ours, ref) <= 1e-15


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_mass_matches_oracle(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_03921_b200 import assemble_mass
    c = Case(name)
    M = assemble_mass(c.mesh, c.ansatz)
    R = oracle.assemble_mass(c.mesh, c.ansatz)
    assert M.shape == R.shape
    assert same_pattern(M, R)
    assert rel_fro(M, R) <= 1e-14
    # exact P1 mass: the entries of the active elements' rows sum to their area / 3 shares
    total = M.sum()
    assert abs(total - c.ansatz.n * c.mesh.areas()[c.mesh.labels != 0].sum()) <= 1e-12 * abs(total)
