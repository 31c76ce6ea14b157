"""fcs-mesh v1 JSON (DomainDecomposition::to_json / from_json,
src/geometry.cpp:17-31,71-135,573-629): the builder writes the reference's
mesh files and reads them.

Checked against the compiled reference (oracle/_ref): the JSON the builder
writes for a geometry equals the reference's JSON of the same geometry key
for key and value for value; the reference reads the builder's files and
writes them back unchanged; the builder reads the reference's files into
patches that produce the reference's decomposition again.
"""
import json
import math

import numpy as np
import pytest

from oracle import ref
from paper_2506_19370_b200 import multipatch as M, problems as PR

from .test_multipatch import N0, NV, _bcs, _geometry

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
GEOMS = [pytest.param(0, id="annulus"), pytest.param(1, id="two-patch"), pytest.param(2, id="corner")]


@pytest.mark.parametrize("which", GEOMS)
def test_written_mesh_equals_reference_mesh(which):
    patches, _ = _geometry(which)
    ours = M.mesh_to_json(patches, NV, n0=N0)
    R = ref.RefEngine.testgeom(which, N0, weight_path="")
    assert ours == R.mesh_json()
    # and through text (what a mesh file holds)
    assert json.loads(json.dumps(ours)) == ours


@pytest.mark.parametrize("which", GEOMS)
def test_reference_reads_written_mesh(which):
    patches, _ = _geometry(which)
    ours = M.mesh_to_json(patches, NV, n0=N0)
    assert ref.mesh_roundtrip(ours) == ours


@pytest.mark.parametrize("which", GEOMS)
def test_read_reference_mesh_rebuilds_decomposition(which, tmp_path):
    R = ref.RefEngine.testgeom(which, N0, weight_path="")
    path = tmp_path / "mesh.json"
    path.write_text(json.dumps(R.mesh_json()))
    patches, meta = M.load_mesh(str(path))
    assert meta == {"nv": NV, "n0": N0, "n1": 43, "nf": 5}
    assert M.mesh_to_json(patches, **meta) == R.mesh_json()
    D = M.build_decomposition(patches, _bcs(), NV, validate_overlap=which != 2)
    assert len(D.subs) == R.nsubs
    for k, d in enumerate(D.subs):
        assert np.array_equal(d.mask, R.get(k, "mask").astype(np.uint8)), k
        assert float(np.abs(d.w_norm - R.get(k, "w_norm")).max()) < 1e-13, k
    # save_mesh writes the same file back
    M.save_mesh(str(tmp_path / "again.json"), patches, **meta)
    assert json.loads((tmp_path / "again.json").read_text()) == R.mesh_json()


def test_config4_layout_mesh_equals_reference():
    """the forward-facing-step layout (problems.step_flow: convex C1 corner at
    the step top, concave C2 corner at its foot, S and I patches of 256 x 256
    subpatches) as a mesh file equals the reference's"""
    R = ref.RefEngine.testgeom(5, 0, weight_path="")
    j = R.mesh_json()
    patches, meta = M.mesh_from_json(j)
    assert [p.kind for p in patches] == ["C1", "I", "I", "S", "C2"]
    assert M.mesh_to_json(patches, **meta) == j
    assert sum(len(p.subpatches) for p in patches) == R.nsubs


def test_arc_curves_and_bilinear_round_trip():
    """a C1 patch between two circular arcs and a bilinear patch: keys the
    test geometries do not use, read back by the reference unchanged"""
    SI = M.SideInfo
    # two arcs crossing at (1, 0) at t = 1/2 with perpendicular tangents
    A = M.CircularArc((0.0, 0.0), 1.0, math.pi / 6, -math.pi / 6)
    B = M.CircularArc((1.0, 1.0), 1.0, 1.5 * math.pi - math.pi / 6, 1.5 * math.pi + math.pi / 6)
    c1 = M.build_c1_patch(A, B, (1.0, 0.0), "hull")
    c1.sides = [SI(True, "far") for _ in range(4)]
    c1.index = 0
    M.subdivide_L(c1, 2, 21, NV)
    q = M.Patch(M.S, M.BilinearMap((0.1, 0.0), (1.3, 0.2), (0.0, 0.9), (1.1, 1.3)),
                [SI(), SI(True, "out"), SI(True, "wall"), SI()])
    q.index = 1
    M.subdivide_Q(q, 3, 2, 25, NV)
    ours = M.mesh_to_json([c1, q], NV, n0=25, n1=21)
    assert ref.mesh_roundtrip(ours) == ours
    back, meta = M.mesh_from_json(ours)
    assert M.mesh_to_json(back, **meta) == ours
    # the arc mapping evaluates as the reference's CurveSumMap: l_A(q1) + l_B(q2) - C
    x, y = back[0].map(0.3, 0.6)
    ax, ay = A.point(0.3)
    bx, by = B.point(0.6)
    assert (x, y) == ((ax + bx) - 1.0, (ay + by) - 0.0)


def test_corner_patch_checks():
    """build_c1_patch / build_c2_patch input checks (src/geometry.cpp:351-389)"""
    seg = M.Segment
    c2 = M.build_c2_patch(seg((0.3, 0.0), (0.6, 0.0)), seg((0.6, 0.2), (0.6, 0.0)), (0.6, 0.0), "wall")
    assert c2.kind == "C2" and [sd.on_gamma for sd in c2.sides] == [False, True, False, True]
    with pytest.raises(M.GeometryError, match="end at the corner"):
        M.build_c2_patch(seg((0.3, 0.0), (0.6, 0.0)), seg((0.6, 0.0), (0.6, 0.2)), (0.6, 0.0))
    with pytest.raises(M.GeometryError, match="parallel"):
        M.build_c2_patch(seg((0.3, 0.0), (0.6, 0.0)), seg((0.9, 0.0), (0.6, 0.0)), (0.6, 0.0))
    with pytest.raises(M.GeometryError, match="t=1/2"):
        M.build_c1_patch(seg((0.0, 0.0), (1.0, 0.0)), seg((0.5, -0.5), (0.5, 0.5)), (0.4, 0.0))


def test_mesh_errors_match_reference():
    patches, _ = _geometry(1)
    j = M.mesh_to_json(patches, NV, n0=N0)
    bad = dict(j, version=2)
    with pytest.raises(M.GeometryError, match="unknown format/version"):
        M.mesh_from_json(bad)
    with pytest.raises(ref.RefError, match="unknown format/version"):
        ref.mesh_roundtrip(bad)
    short = json.loads(json.dumps(j))
    short["patches"][1]["subpatches"] = short["patches"][1]["subpatches"][:1]
    with pytest.raises(M.GeometryError, match="subpatch table"):
        M.mesh_from_json(short)
    with pytest.raises(ref.RefError, match="subpatch table"):
        ref.mesh_roundtrip(short)


def test_config3_layout_mesh_matches_reference_geometry():
    """problems.cylinder_flow's patches (medium resolution) against the
    reference's build of the same layout: identical but for the body wall's
    tag ("body" here, "wall" in ref_engine_testgeom 3)"""
    dec, _, _ = PR.cylinder_flow(full=False)
    ours = M.mesh_to_json(dec.patches, NV, n0=0)
    R = ref.RefEngine.testgeom(3, 0, workers=2, weight_path="")
    theirs = R.mesh_json()
    ours["patches"][0]["sides"][2]["tag"] = "wall"
    assert ours == theirs
