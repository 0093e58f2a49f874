"""GPU pack_mesh (geometry.cpp:73-195).

CPU: the oracle restatement equals the reference's own compiled pack_mesh
(oracle/_ref) bit for bit on synthetic closed meshes (the bunny asset is not in
the container) and on its error paths. GPU: the CUDA ray-parity kernel equals
the oracle bit for bit (centers in grid order, candidate and ambiguous counts).
"""
import numpy as np
import pytest

from paper_2603_14634_b200 import pbdr as P

import meshes as M

CASES = [("icosphere", lambda: M.icosphere(0.05, 2), 0.005),
         ("torus", lambda: M.torus(), 0.004),
         ("cube_on_grid_edges", lambda: M.cube(0.05), 0.005)]


@pytest.mark.parametrize("name,make,radius", CASES)
def test_oracle_pack_mesh_matches_reference(pyoracle, name, make, radius):
    v, t = make()
    ref = pyoracle.ref_pack_mesh(v, t, radius)
    if ref is None:
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    got = pyoracle.pack_mesh(v, t, radius)
    assert got[0] == ref[0] == 0
    assert np.array_equal(got[1], ref[1]), name
    assert got[2:] == ref[2:]
    assert len(got[1]) > 0


def test_oracle_pack_mesh_errors(pyoracle):
    v, t = M.icosphere(0.05, 1)
    assert pyoracle.pack_mesh(v, t, 0.2)[0] == 3      # radius too large: EmptyPackingError
    assert pyoracle.pack_mesh(v, t, -1.0)[0] == 9     # pbdr::Error
    bad = t.copy()
    bad[0, 0] = len(v)
    assert pyoracle.pack_mesh(v, bad, 0.005)[0] == 9  # index out of range
    ref = pyoracle.ref_pack_mesh(v, t, 0.2)
    if ref is not None:
        assert ref[0] == 3 and pyoracle.ref_pack_mesh(v, bad, 0.005)[0] == 9


def test_pack_box_mesh_volume(pyoracle):
    # Sanity of the restatement on a shape with a known answer: the grid points
    # inside an axis-aligned cube of half extent 0.05 at radius 0.005 are all
    # 10^3 of them (none sits on a face).
    v, t = M.cube(0.05)
    st, c, cand, amb = pyoracle.pack_mesh(v, t, 0.005)
    assert st == 0 and len(c) == 1000 and cand == 1000 and amb == 0


@pytest.mark.gpu
@pytest.mark.parametrize("name,make,radius", CASES + [("torus_fine", lambda: M.torus(0.06, 0.025, 48, 24), 0.0015)])
def test_gpu_pack_mesh_bit_exact(pbdr, pyoracle, name, make, radius):
    v, t = make()
    centers, cand, amb = P.pack_mesh(v, t, radius)
    st, oc, ocand, oamb = pyoracle.pack_mesh(v, t, radius)
    assert st == 0
    assert np.array_equal(centers, oc), name
    assert (cand, amb) == (ocand, oamb)


@pytest.mark.gpu
def test_gpu_pack_mesh_errors(pbdr):
    v, t = M.icosphere(0.05, 1)
    with pytest.raises(P.EmptyPackingError):
        P.pack_mesh(v, t, 0.2)
    with pytest.raises(P.Error):
        P.pack_mesh(v, t, -1.0)
