"""Deferred mesh handles (mrb_mesh_create_many) on the host: the checks
TriMesh.__init__ runs before connectivity (mesh.py:61-86) with the
reference's messages, and the host build a deferred handle falls back to
(exports) equal to mrb_mesh_build's bit for bit.  No GPU needed."""
import numpy as np
import pytest

import paper_1411_2141_b200 as mrb
from conftest import golden
from paper_1411_2141_b200 import _lib


def create(V, T):
    return mrb.DeferredMesh.create_many([(V, T)])[0]


def test_create_validation_messages_match_reference():
    with pytest.raises(ValueError, match=r"vertices must be \(n, 2\)"):
        create(np.zeros((3, 3)), [(0, 1, 2)])
    with pytest.raises(ValueError, match="with m >= 1"):
        create(np.zeros((3, 2)), np.zeros((0, 3)))
    with pytest.raises(ValueError, match="vertex coordinates must be finite"):
        create([(0, 0), (1, np.nan), (0, 1)], [(0, 1, 2)])
    with pytest.raises(ValueError, match="triangle index out of range"):
        create([(0, 0), (1, 0), (0, 1)], [(0, 1, 3)])
    with pytest.raises(ValueError, match="repeated vertex"):
        create([(0, 0), (1, 0), (0, 1)], [(0, 1, 1)])
    with pytest.raises(ValueError) as e:
        create([(0, 0), (1, 0), (2, 0)], [(0, 1, 2)])
    assert str(e.value) == "degenerate triangle 0 (area 0)"


def test_create_many_is_all_or_nothing():
    g = golden("gen64")
    good = (g["V"], g["T_in"])
    with pytest.raises(ValueError, match="repeated vertex"):
        mrb.DeferredMesh.create_many([good, good, ([(0, 0), (1, 0), (0, 1)], [(0, 1, 1)])])
    ms = mrb.DeferredMesh.create_many([good, good])
    assert [m.n_vertices for m in ms] == [len(g["V"])] * 2


def _export(h, n, m, ne):
    lib = _lib.load()
    arrs = [np.empty((m, 3), np.int64), np.empty((ne, 2), np.int64), np.empty(n, np.int64),
            np.empty(n, np.uint8), np.empty(n + 1, np.int64), np.empty(2 * ne, np.int64),
            np.empty(n + 1, np.int64), np.empty(3 * m, np.int64)]
    assert lib.mrb_mesh_export_connectivity(h, *(_lib.ptr(a) for a in arrs)) == _lib.OK
    geo = [np.empty(m), np.empty((m, 3, 2)), np.empty(n)]
    assert lib.mrb_mesh_export_geometry(h, *(_lib.ptr(a) for a in geo)) == _lib.OK
    return arrs + geo


@pytest.mark.parametrize("name", ["gen64", "c1", "accept_c3"])
def test_deferred_host_fallback_equals_build(name):
    """A host consumer of a deferred handle gets the full host build: the
    exported connectivity and geometry equal TriMesh's (with clockwise input
    triangles, so the creation's reorientation is covered)."""
    g = golden(name)
    V, T = g["V"], g["T_in"].astype(np.int64).copy()
    T[::3] = T[::3][:, [0, 2, 1]]  # every third triangle clockwise
    ref = mrb.TriMesh(V, T)
    d = create(V, T)
    lib = _lib.load()
    counts = np.zeros(6, np.int64)
    assert lib.mrb_mesh_counts(d._h, _lib.ptr(counts)) == _lib.OK
    assert np.array_equal(counts, ref._counts)
    n, m, ne = (int(c) for c in counts[:3])
    for a, b in zip(_export(d._h, n, m, ne), _export(ref._h, n, m, ne)):
        assert np.array_equal(a, b)


def test_deferred_connectivity_errors_surface_at_first_use():
    """Checks that need connectivity run with the host (or device) build: a
    non-manifold edge and a lone vertex raise the reference's messages there."""
    lib = _lib.load()
    d = create([(0, 0), (1, 0), (0, 1), (0, -1), (0.3, 0.7)], [(0, 1, 2), (0, 1, 3), (0, 1, 4)])
    counts = np.zeros(6, np.int64)
    assert lib.mrb_mesh_counts(d._h, _lib.ptr(counts)) == _lib.E_VALUE
    with pytest.raises(ValueError, match="non-manifold edge shared by more than two triangles"):
        mrb.TriMesh([(0, 0), (1, 0), (0, 1), (0, -1), (0.3, 0.7)],
                    [(0, 1, 2), (0, 1, 3), (0, 1, 4)])
    lone = create([(0, 0), (1, 0), (0, 1), (5, 5)], [(0, 1, 2)])
    assert lib.mrb_mesh_counts(lone._h, _lib.ptr(counts)) == _lib.E_VALUE
    with pytest.raises(ValueError, match=r"vertex 3 has valence 0 \(< 2\)"):
        mrb.TriMesh([(0, 0), (1, 0), (0, 1), (5, 5)], [(0, 1, 2)])
