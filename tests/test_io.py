"""nlcsr / nlmesh text I/O against the reference's
writers: golden files written by nlfem's own write_nlcsr / write_mesh
(tests/golden/make_io_golden.py), Python repr/int token formatting, round
trips and the readers' error behaviour (assembly.py:519-570, mesh.py:269-347).
CPU only (the formatter is host code in libnlg.so)."""

import os

import numpy as np
import pytest
from scipy import sparse

from paper_2207_03921_b200 import Mesh, MeshFormatError, nlio

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def _golden():
    z = np.load(os.path.join(GOLD, "lshape16_const.npz"), allow_pickle=True)
    n = len(z["indptr"]) - 1
    return z, sparse.csr_matrix((z["data"], z["indices"], z["indptr"]), shape=(n, n))


def _repr_line(a):
    return " ".join(repr(float(v)) for v in a)


def test_float_tokens_match_python_repr():
    rng = np.random.default_rng(7)
    parts = [
        rng.standard_normal(20000), rng.standard_normal(20000) * 1e-300, rng.standard_normal(20000) * 1e300,
        np.exp(rng.uniform(-745, 709, 40000)) * rng.choice([-1.0, 1.0], 40000),
        rng.integers(-10**6, 10**6, 5000).astype(np.float64),
        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e16, 1e15, 9999999999999998.0, 1e-4, 1e-5, 0.1, 0.5,
                  123456789012345678.0, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 1.5e-5,
                  0.00012345, 1.0 / 3.0, 2.0 / 3.0, 100.0, 1e22, 1e23]),
        rng.random(20000).view(np.uint64).astype(np.uint64).view(np.float64),  # arbitrary bit patterns
    ]
    v = np.concatenate(parts)
    v = v[np.isfinite(v) | np.isnan(v)]
    got = nlio.format_tokens(v, threads=4).decode("ascii")
    assert got == _repr_line(v)


def test_int_tokens():
    a = np.array([0, -1, 7, 2**62, -2**63, 123456789], dtype=np.int64)
    assert nlio.format_tokens(a).decode() == " ".join(str(int(x)) for x in a)
    b = np.arange(-5, 200000, 3, dtype=np.int32)
    assert nlio.format_tokens(b, threads=8).decode() == " ".join(str(int(x)) for x in b)


def test_write_nlcsr_matches_reference_bytes(tmp_path):
    _, m = _golden()
    p = tmp_path / "m.nlcsr"
    nlio.write_nlcsr(p, m)
    assert p.read_bytes() == open(os.path.join(GOLD, "io_lshape16.nlcsr"), "rb").read()


def test_block_writer_equals_whole_writer(tmp_path, monkeypatch):
    _, m = _golden()
    monkeypatch.setattr(nlio, "_CHUNK", 97)  # many chunks per block
    cuts = [0, 1, 60, 61, 150, m.shape[0]]
    blocks = [m[a:b] for a, b in zip(cuts[:-1], cuts[1:])]
    p = tmp_path / "b.nlcsr"
    nlio.write_nlcsr_blocks(p, m.shape, blocks, threads=3)
    assert p.read_bytes() == open(os.path.join(GOLD, "io_lshape16.nlcsr"), "rb").read()
    with pytest.raises(ValueError):
        nlio.write_nlcsr_blocks(tmp_path / "x.nlcsr", m.shape, blocks[:-1])


def test_nlcsr_round_trip_and_empty(tmp_path):
    _, m = _golden()
    p = tmp_path / "m.nlcsr"
    nlio.write_nlcsr(p, m)
    r = nlio.read_nlcsr(p)
    assert np.array_equal(r.indptr, m.indptr) and np.array_equal(r.indices, m.indices)
    assert np.array_equal(r.data, m.data)  # repr round-trips exactly
    e = sparse.csr_matrix((3, 4))
    nlio.write_nlcsr(tmp_path / "e.nlcsr", e)
    assert (tmp_path / "e.nlcsr").read_text() == "nlcsr 1 3 4 0\n0 0 0 0\n\n\n"
    # like the reference reader, blank (empty-array) lines do not count as data lines
    with pytest.raises(MeshFormatError, match="expected exactly 3 data lines"):
        nlio.read_nlcsr(tmp_path / "e.nlcsr")


@pytest.mark.parametrize("text,msg", [
    ("", "empty file"),
    ("nlcsr 2 1 1 0\n0 0\n\n\n", "unsupported nlcsr version"),
    ("matrix 1 1 1 0\n0 0\n\n\n", "expected header"),
    ("nlcsr 1 a 1 0\n0 0\n\n\n", "header counts must be integers"),
    ("nlcsr 1 1 1 1\n0 1\n0\n", "expected exactly 3 data lines"),
    ("nlcsr 1 1 1 1\n0 1 2\n0\n1.0\n", "expected 2 row pointer entries"),
    ("nlcsr 1 1 1 1\n0 1\nx\n1.0\n", "column index entries must be integers"),
    ("nlcsr 1 1 1 1\n0 1\n0\nfoo\n", "value entries must be numbers"),
    ("nlcsr 1 1 1 1\n0 0\n0\n1.0\n", "not a valid monotone offset array"),
    ("nlcsr 1 1 1 1\n0 1\n5\n1.0\n", "column index out of range"),
])
def test_read_nlcsr_errors(tmp_path, text, msg):
    p = tmp_path / "bad.nlcsr"
    p.write_text(text)
    with pytest.raises(MeshFormatError, match=msg):
        nlio.read_nlcsr(p)


def test_write_mesh_matches_reference_bytes(tmp_path):
    z, _ = _golden()
    mesh = Mesh(z["vertices"], z["elements"], z["labels"])
    p = tmp_path / "m.nlmesh"
    nlio.write_mesh(mesh, p)
    assert p.read_bytes() == open(os.path.join(GOLD, "io_lshape16.nlmesh"), "rb").read()
    back = nlio.read_mesh(p, delta=0.1)
    assert np.array_equal(back.vertices, mesh.vertices) and np.array_equal(back.elements, mesh.elements)
    assert np.array_equal(back.labels, mesh.labels) and back.delta == 0.1
    assert back.parse_report == {"reoriented": []}


def test_read_mesh_comments_and_reorientation(tmp_path):
    p = tmp_path / "cw.nlmesh"
    p.write_text("# a comment\nnlmesh 1 4 2  # header\n0.0 0.0\n1.0 0.0\n0.0 1.0\n1.0 1.0\n\n"
                 "0 2 1 1  # clockwise\n1 3 2 2\n")
    m = nlio.read_mesh(p)
    assert m.parse_report == {"reoriented": [0]}
    assert m.elements[0].tolist() == [0, 1, 2] and (m.areas() > 0).all()


@pytest.mark.parametrize("text,msg", [
    ("", "line 1: empty mesh file"),
    ("nlmesh 2 0 0\n", "expected header"),
    ("nlmesh 1 x 0\n", "header counts must be integers"),
    ("nlmesh 1 -1 0\n", "nonnegative"),
    ("nlmesh 1 3 1\n0 0\n1 0\n", "unexpected end of file"),
    ("nlmesh 1 1 0\n0 0\n5 5\n", "line 3: unexpected extra content"),
    ("nlmesh 1 1 0\n0\n", "line 2: expected '<x> <y>'"),
    ("nlmesh 1 1 0\n0 a\n", "invalid vertex coordinate"),
    ("nlmesh 1 1 0\n0 inf\n", "vertex coordinate not finite"),
    ("nlmesh 1 3 1\n0 0\n1 0\n0 1\n0 1 3 1\n", "line 5: vertex index 3 out of range"),
    ("nlmesh 1 3 1\n0 0\n1 0\n0 1\n0 1 1 1\n", "repeated vertex"),
    ("nlmesh 1 3 1\n0 0\n1 0\n0 1\n0 1 2 7\n", "unknown label 7"),
    ("nlmesh 1 3 1\n0 0\n1 0\n2 0\n0 1 2 1\n", "non-positive area"),
    ("nlmesh 1 3 1\n0 0\n1 0\n0 1\n0 1 2\n", "expected '<i> <j> <k> <label>'"),
    ("nlmesh 1 3 1\n0 0\n1 0\n0 1\n0 1 b 1\n", "element entries must be integers"),
])
def test_read_mesh_errors(tmp_path, text, msg):
    p = tmp_path / "bad.nlmesh"
    p.write_text(text)
    with pytest.raises(MeshFormatError, match=msg):
        nlio.read_mesh(p)
