"""Text I/O of the assembly's inputs and outputs.

* nlcsr matrices: :func:`write_nlcsr` / :func:`read_nlcsr` mirror the
  reference's ``write_nlcsr`` / ``read_nlcsr`` (``assembly.py:509-570``):
  header ``nlcsr 1 <rows> <cols> <nnz>``, then one line each of row
  pointers, column indices and values.  The tokens are formatted by the
  native ``nlg_format_*`` functions (``csrc/nlg_io.cpp``: Python ``int()`` /
  ``repr(float)`` bytes, multi-threaded), and :func:`write_nlcsr_blocks`
  streams a matrix given as CSR row blocks (e.g. the per-rank pieces of a
  sharded config-4 assembly, ~264 GB of text) without ever holding the
  whole text or the whole matrix: each block is formatted in bounded chunks.
* nlmesh meshes: :func:`write_mesh` / :func:`read_mesh` mirror
  ``mesh.py:259-347`` (same layout, comment handling, reorientation of
  clockwise triangles and error messages).

The files are byte-identical to the reference writers' (tests/test_io.py
checks them against ``repr``/``int`` formatting and round trips).
"""

import ctypes
import os

import numpy as np
from scipy import sparse

from . import _native
from .errors import MeshFormatError
from .mesh import Label, Mesh

_CHUNK = 1 << 22  # tokens formatted per native call (bounded buffers)
_FMT = {np.dtype(np.float64): "nlg_format_f64", np.dtype(np.int64): "nlg_format_i64",
        np.dtype(np.int32): "nlg_format_i32"}


def format_tokens(arr, threads=0):
    """Space-separated text of a 1-D float64 / int64 / int32 array (bytes)."""
    a = np.ascontiguousarray(arr)
    if a.dtype not in _FMT:
        a = a.astype(np.float64 if a.dtype.kind == "f" else np.int64)
    n = int(a.size)
    if n == 0:
        return b""
    fn = getattr(_native.load_library(), _FMT[a.dtype])
    cap = 33 * n + 1
    buf = np.empty(cap, dtype=np.uint8)
    ln = fn(a.ctypes.data, n, buf.ctypes.data, cap, int(threads))
    if ln < 0:
        raise RuntimeError("token buffer too small")
    return buf[:ln].tobytes()


def _write_array(fh, parts, threads):
    """One text line: the concatenated arrays of `parts`, chunked."""
    first = True
    for arr in parts:
        for s in range(0, int(arr.size), _CHUNK):
            txt = format_tokens(arr[s:s + _CHUNK], threads)
            if not txt:
                continue
            if not first:
                fh.write(b" ")
            fh.write(txt)
            first = False
    fh.write(b"\n")


def _as_block(b):
    if sparse.issparse(b):
        m = b.tocsr()
        return m.indptr, m.indices, m.data
    if hasattr(b, "matrix"):
        m = b.matrix
        return m.indptr, m.indices, m.data
    indptr, indices, data = b
    return indptr, indices, data


def write_nlcsr_blocks(path, shape, blocks, threads=0):
    """Stream a CSR matrix given as consecutive row blocks to nlcsr text.

    ``blocks``: a sequence (it is traversed three times) of CSR row blocks in
    row order, each a scipy matrix or an ``(indptr, indices, data)`` triple
    whose indptr starts at 0; together they cover ``shape[0]`` rows.
    """
    rows, cols = (int(x) for x in shape)
    blks = [_as_block(b) for b in blocks]
    nnz = sum(int(ip[-1] - ip[0]) for ip, _, _ in blks)
    nrow = sum(len(ip) - 1 for ip, _, _ in blks)
    if nrow != rows:
        raise ValueError(f"row blocks cover {nrow} rows, expected {rows}")
    with open(path, "wb") as fh:
        fh.write(f"nlcsr 1 {rows} {cols} {nnz}\n".encode("ascii"))
        ptr_parts, off = [np.zeros(1, dtype=np.int64)], 0
        for ip, _, _ in blks:
            ip = np.asarray(ip, dtype=np.int64)
            ptr_parts.append(ip[1:] - ip[0] + off)
            off += int(ip[-1] - ip[0])
        _write_array(fh, ptr_parts, threads)
        _write_array(fh, [np.asarray(ix)[ip[0]:ip[-1]] for ip, ix, _ in blks], threads)
        _write_array(fh, [np.asarray(dv, dtype=np.float64)[ip[0]:ip[-1]] for ip, _, dv in blks], threads)


def write_nlcsr(path, system, threads=0):
    """Write a sparse matrix (or SparseSystem) as nlcsr text (assembly.py:509-516)."""
    matrix = system.matrix if hasattr(system, "matrix") else system.tocsr()
    write_nlcsr_blocks(path, matrix.shape, [matrix], threads)


def _content_lines(raw):
    out = []
    for i, line in enumerate(raw, start=1):
        body = line.split("#", 1)[0].strip()
        if body:
            out.append((i, body))
    return out


def read_nlcsr(path):
    """Read nlcsr text back into a CSR matrix, validating like assembly.py:519-570."""
    with open(path, "r", encoding="ascii") as fh:
        lines = _content_lines(fh)
    if not lines:
        raise MeshFormatError(f"{path}: empty file")
    ln, header = lines[0]
    head = header.split()
    if len(head) != 5 or head[0] != "nlcsr":
        raise MeshFormatError(f"{path}:{ln}: expected header 'nlcsr 1 <rows> <cols> <nnz>'")
    if head[1] != "1":
        raise MeshFormatError(f"{path}:{ln}: unsupported nlcsr version {head[1]!r}")
    try:
        rows, cols, nnz = (int(p) for p in head[2:])
    except ValueError:
        raise MeshFormatError(f"{path}:{ln}: header counts must be integers") from None
    if min(rows, cols, nnz) < 0:
        raise MeshFormatError(f"{path}:{ln}: header counts must be nonnegative")
    if len(lines) != 4:
        raise MeshFormatError(f"{path}: expected exactly 3 data lines after the header")

    def parse(entry, count, what, dtype):
        ln, body = entry
        toks = body.split()
        if len(toks) != count:
            raise MeshFormatError(f"{path}:{ln}: expected {count} {what} entries, got {len(toks)}")
        try:
            if dtype is np.int64:
                return np.array([int(t) for t in toks], dtype=np.int64)
            return np.array([float(t) for t in toks], dtype=np.float64)
        except ValueError:
            kind = "integers" if dtype is np.int64 else "numbers"
            raise MeshFormatError(f"{path}:{ln}: {what} entries must be {kind}") from None

    indptr = parse(lines[1], rows + 1, "row pointer", np.int64)
    indices = parse(lines[2], nnz, "column index", np.int64)
    data = parse(lines[3], nnz, "value", np.float64)
    if indptr[0] != 0 or indptr[-1] != nnz or np.any(np.diff(indptr) < 0):
        raise MeshFormatError(f"{path}: row pointer is not a valid monotone offset array")
    if nnz and (indices.min() < 0 or indices.max() >= cols):
        raise MeshFormatError(f"{path}: column index out of range")
    return sparse.csr_matrix((data, indices, indptr), shape=(rows, cols))


def write_mesh(mesh, path, threads=0):
    """nlmesh text (mesh.py:259-266): header, 'x y' vertex lines, 'i j k label' element lines."""
    with open(path, "wb") as fh:
        fh.write(f"nlmesh 1 {mesh.n_vertices} {mesh.n_elements}\n".encode("ascii"))
        if mesh.n_vertices:
            xy = format_tokens(mesh.vertices.reshape(-1), threads).split(b" ")
            fh.write(b"".join(xy[2 * i] + b" " + xy[2 * i + 1] + b"\n" for i in range(mesh.n_vertices)))
        if mesh.n_elements:
            cols = np.concatenate([mesh.elements, mesh.labels[:, None]], axis=1).reshape(-1)
            tk = format_tokens(cols.astype(np.int64), threads).split(b" ")
            fh.write(b"".join(b" ".join(tk[4 * i:4 * i + 4]) + b"\n" for i in range(mesh.n_elements)))


_LABELS = {int(v) for v in Label}


def read_mesh(path, delta=0.0):
    """Read nlmesh text (mesh.py:269-347): '#' comments, clockwise triangles
    reoriented (their indices in parse_report["reoriented"]), malformed
    content -> MeshFormatError naming the line."""
    with open(path) as fh:
        content = _content_lines(fh)
    if not content:
        raise MeshFormatError("line 1: empty mesh file")
    ln, text = content[0]
    head = text.split()
    if len(head) != 4 or head[0] != "nlmesh" or head[1] != "1":
        raise MeshFormatError(f"line {ln}: expected header 'nlmesh 1 <n_vertices> <n_elements>'")
    try:
        nv, ne = int(head[2]), int(head[3])
    except ValueError:
        raise MeshFormatError(f"line {ln}: header counts must be integers") from None
    if nv < 0 or ne < 0:
        raise MeshFormatError(f"line {ln}: header counts must be nonnegative")
    need = 1 + nv + ne
    if len(content) < need:
        raise MeshFormatError(f"line {content[-1][0]}: unexpected end of file, "
                              f"need {nv} vertex and {ne} element lines")
    if len(content) > need:
        raise MeshFormatError(f"line {content[need][0]}: unexpected extra content")
    vertices = np.empty((nv, 2), dtype=np.float64)
    for r, (ln, text) in enumerate(content[1:1 + nv]):
        toks = text.split()
        if len(toks) != 2:
            raise MeshFormatError(f"line {ln}: expected '<x> <y>'")
        try:
            vertices[r] = (float(toks[0]), float(toks[1]))
        except ValueError:
            raise MeshFormatError(f"line {ln}: invalid vertex coordinate") from None
        if not np.isfinite(vertices[r]).all():
            raise MeshFormatError(f"line {ln}: vertex coordinate not finite")
    elements = np.empty((ne, 3), dtype=np.int64)
    labels = np.empty(ne, dtype=np.int64)
    reoriented = []
    for r, (ln, text) in enumerate(content[1 + nv:]):
        toks = text.split()
        if len(toks) != 4:
            raise MeshFormatError(f"line {ln}: expected '<i> <j> <k> <label>'")
        try:
            i, j, k, lab = (int(t) for t in toks)
        except ValueError:
            raise MeshFormatError(f"line {ln}: element entries must be integers") from None
        for v in (i, j, k):
            if not 0 <= v < nv:
                raise MeshFormatError(f"line {ln}: vertex index {v} out of range")
        if len({i, j, k}) < 3:
            raise MeshFormatError(f"line {ln}: repeated vertex in element")
        if lab not in _LABELS:
            raise MeshFormatError(f"line {ln}: unknown label {lab}")
        p0, p1, p2 = vertices[i], vertices[j], vertices[k]
        area = 0.5 * ((p1[0] - p0[0]) * (p2[1] - p0[1]) - (p1[1] - p0[1]) * (p2[0] - p0[0]))
        if area < 0.0:
            j, k = k, j
            reoriented.append(r)
        elif area == 0.0:
            raise MeshFormatError(f"line {ln}: triangle has non-positive area")
        elements[r] = (i, j, k)
        labels[r] = lab
    return Mesh(vertices, elements, labels, delta=delta, parse_report={"reoriented": reoriented})
