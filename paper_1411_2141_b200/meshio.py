"""Mesh file formats of the reference (meshgen.py:400-452): a Triangle-style
``<stem>.node`` / ``<stem>.ele`` text pair and a single JSON file, both with
0-based ids.  The package's mesher (meshgen.generate_mesh) and the
reference's ``meshreg mesh`` both write them; the writers here produce the
reference's bytes.
"""

from __future__ import annotations

import json

import numpy as np

from .image import FileFormatError
from .mesh import TriMesh

__all__ = ["save_mesh", "load_mesh", "save_mesh_json", "load_mesh_json", "load_mesh_arg"]


def save_mesh(mesh, stem):
    """``<stem>.node``: count, then ``i x y`` with Python float repr;
    ``<stem>.ele``: count, then ``i a b c`` (meshgen.py:405-414)."""
    with open(f"{stem}.node", "w", encoding="ascii") as fh:
        fh.write(f"{mesh.n_vertices}\n")
        fh.writelines(f"{i} {float(x)!r} {float(y)!r}\n" for i, (x, y) in enumerate(mesh.vertices))
    with open(f"{stem}.ele", "w", encoding="ascii") as fh:
        fh.write(f"{mesh.n_triangles}\n")
        fh.writelines(f"{i} {a} {b} {c}\n" for i, (a, b, c) in enumerate(mesh.triangles))


def load_mesh(stem):
    """Read a .node/.ele pair; rows may come in any order, the leading id
    places them (meshgen.py:417-432)."""
    try:
        with open(f"{stem}.node", "r", encoding="ascii") as fh:
            tok = fh.read().split()
        n = int(tok[0])
        rows = np.array(tok[1:1 + 3 * n], dtype=np.float64).reshape(n, 3)
        V = rows[np.argsort(rows[:, 0].astype(int))][:, 1:]
        with open(f"{stem}.ele", "r", encoding="ascii") as fh:
            tok = fh.read().split()
        m = int(tok[0])
        rows = np.array(tok[1:1 + 4 * m], dtype=np.int64).reshape(m, 4)
        T = rows[np.argsort(rows[:, 0])][:, 1:]
    except (ValueError, IndexError) as exc:
        raise FileFormatError(f"malformed mesh files {stem}.node/.ele: {exc}") from exc
    return TriMesh(V, T)


def save_mesh_json(mesh, path):
    """``{"nodes": [[x, y], ...], "triangles": [[a, b, c], ...]}``
    (meshgen.py:435-441)."""
    doc = {"nodes": [[float(x), float(y)] for x, y in mesh.vertices],
           "triangles": [[int(a), int(b), int(c)] for a, b, c in mesh.triangles]}
    with open(path, "w", encoding="ascii") as fh:
        json.dump(doc, fh)


def load_mesh_json(path):
    try:
        with open(path, "r", encoding="ascii") as fh:
            doc = json.load(fh)
        V = np.array(doc["nodes"], dtype=np.float64)
        T = np.array(doc["triangles"], dtype=np.int64)
    except (ValueError, KeyError, TypeError) as exc:
        raise FileFormatError(f"malformed mesh file {path!r}: {exc}") from exc
    return TriMesh(V, T)


def load_mesh_arg(path):
    """--mesh argument: a .json file, or a .node/.ele stem (cli.py:202-206)."""
    path = str(path)
    if path.endswith(".json"):
        return load_mesh_json(path)
    return load_mesh(path[:-5] if path.endswith(".node") else path)
