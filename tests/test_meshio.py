"""Mesh writers/readers (occmesh.meshio, meshio.py:22-140): the libodc
writers must produce the reference writer's bytes.  Pinned two ways: the
sha256 of the reference's own output on golden meshes (tests/golden/
meshio.json, made by make_meshio_golden.py), and a restated f-string
formatter on random meshes.  Host-only: no GPU needed."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2409_13418_b200 import TriangleMesh
from paper_2409_13418_b200.meshio import MeshParseError, export_obj, export_ply, import_obj, import_ply

GOLDEN = Path(__file__).resolve().parent / "golden"


def _mesh(name):
    if name == "awkward":
        d = np.load(GOLDEN / "meshio_awkward.npz")
    elif name == "empty":
        return TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64))
    else:
        d = np.load(GOLDEN / f"{name}.npz")
    return TriangleMesh.trusted(np.ascontiguousarray(d["vertices"], np.float64),
                                np.ascontiguousarray(d["triangles"], np.int64))


def _sha(p):
    b = Path(p).read_bytes()
    return hashlib.sha256(b).hexdigest(), len(b)


GOLD = json.loads((GOLDEN / "meshio.json").read_text())


@pytest.mark.parametrize("name", sorted(GOLD))
@pytest.mark.parametrize("ext", ["obj", "ply"])
def test_writer_matches_reference_bytes(tmp_path, name, ext):
    m = _mesh(name)
    p = tmp_path / f"m.{ext}"
    (export_obj if ext == "obj" else export_ply)(m, p)
    sha, n = _sha(p)
    assert (sha, n) == (GOLD[name][ext]["sha256"], GOLD[name][ext]["bytes"])


def _obj_restated(v, t):
    lines = [f"v {a:.17g} {b:.17g} {c:.17g}" for a, b, c in v.tolist()]
    lines += [f"f {a + 1} {b + 1} {c + 1}" for a, b, c in t.tolist()]
    return ("\n".join(lines) + ("\n" if lines else "")).encode()


@pytest.mark.parametrize("seed", range(4))
def test_obj_random_against_fstring(tmp_path, seed):
    rng = np.random.default_rng(seed)
    n = 70000  # spans several parallel chunks
    v = rng.normal(size=(n, 3)) * 10.0 ** rng.integers(-300, 300, size=(n, 1))
    v[::97] = np.round(v[::97])
    v[::101, 1] = -0.0
    t = rng.integers(0, n, size=(n // 2, 3))
    p = tmp_path / "r.obj"
    export_obj(TriangleMesh.trusted(v, t), p)
    assert p.read_bytes() == _obj_restated(v, t)


def test_round_trips(tmp_path):
    m = _mesh("torus_32")
    export_obj(m, tmp_path / "a.obj")
    back = import_obj(tmp_path / "a.obj")
    assert np.array_equal(back.vertices, m.vertices) and np.array_equal(back.triangles, m.triangles)
    export_ply(m, tmp_path / "a.ply")
    back = import_ply(tmp_path / "a.ply")
    assert np.array_equal(back.vertices, m.vertices.astype(np.float32).astype(np.float64))
    assert np.array_equal(back.triangles, m.triangles)


@pytest.mark.parametrize("text,msg", [
    ("v 1 2\n", "vertex needs 3 coordinates"),
    ("v 1 2 x\n", "bad vertex"),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2\n", "only triangular"),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 q\n", "bad face index"),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 0 1 2\n", "negative or zero"),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 4\n", "out of range"),
    ("p 1\n", "unknown directive"),
])
def test_obj_parse_errors(tmp_path, text, msg):
    p = tmp_path / "bad.obj"
    p.write_text(text)
    with pytest.raises(MeshParseError, match=msg):
        import_obj(p)


def test_obj_reader_accepts_reference_extras(tmp_path):
    p = tmp_path / "ok.obj"
    p.write_text("# c\n\nv 0 0 0\nv 1 0 0\nv 0 1 0\nvn 0 0 1\ng x\nf 1/1 2/2 3/3\n")
    m = import_obj(p)
    assert m.n_vertices == 3 and m.triangles.tolist() == [[0, 1, 2]]


def test_ply_parse_errors(tmp_path):
    m = _mesh("sphere_32")
    export_ply(m, tmp_path / "a.ply")
    data = (tmp_path / "a.ply").read_bytes()
    cases = {
        "missing PLY header": data.replace(b"end_header\n", b"end_headr\n"),
        "not a PLY": b"plx" + data[3:],
        "trailing bytes": data + b"\x00",
        "shorter than the declared face": data[:-5],
    }
    hdr_end = data.find(b"end_header\n") + len(b"end_header\n")
    face0 = hdr_end + 12 * m.n_vertices
    cases["not a triangle"] = data[:face0] + b"\x04" + data[face0 + 1:]
    for msg, blob in cases.items():
        p = tmp_path / "b.ply"
        p.write_bytes(blob)
        with pytest.raises(MeshParseError, match=msg):
            import_ply(p)
