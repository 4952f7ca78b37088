"""CPU checks of the native boundary: the C-ABI library loads, exports every symbol
include/grip_ipc.h declares, and the host-side packing reproduces the reference layout."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    h = (ROOT / "include" / "grip_ipc.h").read_text()
    return sorted(set(re.findall(r"\b(grip_[a-z_]+)\s*\(", h)))


def test_library_exports_every_declared_symbol():
    import __graft_entry__
    lib_path = __graft_entry__.build_native()
    lib = ctypes.CDLL(str(lib_path))
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    lib.grip_abi_version.restype = ctypes.c_int
    from paper_2503_05020_b200 import _native as nv
    assert lib.grip_abi_version() == nv.ABI_VERSION == 4


def test_struct_layouts_match_header():
    from paper_2503_05020_b200 import _native as nv
    h = (ROOT / "include" / "grip_ipc.h").read_text()
    body = h[h.index("typedef struct GripSceneDesc"):h.index("} GripSceneDesc;")]
    fields = re.findall(r"\*\s*([A-Za-z0-9_]+);", body)
    assert fields == [f for f, _ in nv.GripSceneDesc._fields_[2:]]
    assert ctypes.sizeof(nv.GripStepReport) == 72
    assert nv.NPARAM == 14


def test_product_never_imports_oracle():
    for p in (ROOT / "paper_2503_05020_b200").rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p


@pytest.mark.parametrize("name", ["cfg1", "sphere", "soft"])
def test_packing_matches_oracle_layout(golden, name):
    """DOF layout, masses, surface map and collision soup equal the restated reference build."""
    from oracle import solver as osv
    from paper_2503_05020_b200 import packing
    from paper_2503_05020_b200 import scene as sc

    d = np.load(golden / f"traj_{name}.npz")
    scene = sc.build_trial_scene(sc.ObjectSpec(kind=str(d["kind"]), soft=bool(d["soft_object"])),
                                 sc.GripperSpec(soft_fingers=bool(d["soft_fingers"])),
                                 d["cand_R"], d["cand_T"], float(d["cand_opening"]))
    lay = packing.layout_env(scene.bodies, scene.collide_pairs_off)
    ref = osv.OracleEnv(scene.bodies, collide_pairs_off=scene.collide_pairs_off)
    assert lay.n_node * 3 == ref.n_dofs and lay.n_sv == ref.n_sv
    np.testing.assert_array_equal(lay.x0.reshape(-1), ref.x)
    np.testing.assert_array_equal(lay.tris, ref.tris)
    np.testing.assert_array_equal(lay.edges, ref.edges)
    np.testing.assert_array_equal(lay.vbody, ref.vbody)
    np.testing.assert_array_equal(lay.pair_ok, ref.pair_ok)
    np.testing.assert_array_equal(np.repeat(lay.free, 3), ref.free)
    M = lay._arrays["Mb"]
    Mref = ref.M.toarray()
    for n in range(lay.n_node):
        np.testing.assert_array_equal(M[n], Mref[3 * n:3 * n + 3, 3 * n:3 * n + 3])
    # G x == surface positions
    sv = ref.surface_positions()
    nodes = lay.x0
    for r in lay.records:
        sl = slice(r.surf0, r.surf0 + r.n_sv)
        if r.kind == "soft":
            np.testing.assert_array_equal(nodes[r.node0 + r.vmap], sv[sl])
        elif r.kind == "affine":
            np.testing.assert_allclose(nodes[r.node0][None] + r.xi @ nodes[r.node0 + 1:r.node0 + 4].T, sv[sl],
                                       rtol=0, atol=1e-15)
        else:
            np.testing.assert_array_equal(lay.kin0[sl], sv[sl])
    packed = packing.Packed([lay], [packing.env_params(sc.ContactParams(), sc.SolverParams())], [np.zeros(3)],
                            packing.body_velocities(scene.bodies))
    np.testing.assert_array_equal(packed.edge_rest_sq, ref.edge_rest_sq)
