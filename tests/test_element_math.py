"""Pin the CUDA element math (csrc/grip_elements.cuh) on the CPU.

The same __host__ __device__ routines the kernels run are compiled for the host
(libgrip_hostcheck.so, built by __graft_entry__.build()) and compared with the
reference's golden vectors and the oracle.  Runs without a GPU.
"""

import ctypes
from pathlib import Path

import numpy as np
import pytest

from oracle import energies as en
from oracle import geometry as geo

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "build" / "libgrip_hostcheck.so"

dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


@pytest.fixture(scope="module")
def hc():
    if not LIB.exists():
        import __graft_entry__
        __graft_entry__.build_hostcheck()
    lib = ctypes.CDLL(str(LIB))
    d, i = ctypes.c_double, ctypes.c_int
    pi = ctypes.POINTER(ctypes.c_int)
    lib.hc_pt_closest.argtypes = [dp, dp, pi]; lib.hc_pt_closest.restype = d
    lib.hc_ee_closest.argtypes = [dp, dp, dp]; lib.hc_ee_closest.restype = d
    lib.hc_pt_element.argtypes = [dp, d, d, dp, dp, dp, i]; lib.hc_pt_element.restype = i
    lib.hc_ee_element.argtypes = [dp, d, d, d, dp, dp, dp, i]; lib.hc_ee_element.restype = i
    lib.hc_nh_element.argtypes = [dp, dp, d, d, d, dp, dp, dp]; lib.hc_nh_element.restype = i
    lib.hc_abd_element.argtypes = [dp, d, dp, dp]; lib.hc_abd_element.restype = d
    lib.hc_friction.argtypes = [dp, dp, dp, dp, d, d, d, d, dp, dp]; lib.hc_friction.restype = d
    lib.hc_ccd.argtypes = [dp, dp, i, d, i, d, pi]; lib.hc_ccd.restype = d
    lib.hc_cubic.argtypes = [d, d, d, d]; lib.hc_cubic.restype = d
    lib.hc_pencil.argtypes = [dp, dp]; lib.hc_pencil.restype = d
    lib.hc_clamp_stencil.argtypes = [dp]; lib.hc_clamp12.argtypes = [dp]
    lib.hc_stress.argtypes = [dp, dp, d, d, dp]; lib.hc_stress.restype = i
    return lib


@pytest.fixture(scope="module")
def K(golden):
    return dict(np.load(golden / "kernels.npz"))


def test_closest_points(hc, K):
    tri, p = K["ptc_tri"], K["ptc_p"]
    for n in range(0, len(p), 7):
        x = np.ascontiguousarray(np.concatenate([p[n], tri[n].ravel()]))
        b = np.zeros(3)
        r = ctypes.c_int()
        D = hc.hc_pt_closest(x, b, ctypes.byref(r))
        # the first 900 cases sit exactly on vertices / edges / the plane: their region is
        # decided by the sign of a rounding-level quantity, so only D is compared there
        if n >= 900:
            assert r.value == K["ptc_region"][n]
        assert abs(D - K["ptc_D"][n]) <= 1e-12 * max(1.0, K["ptc_D"][n])
    xe = K["eec_x"]
    for n in range(0, len(xe), 7):
        s, t = np.zeros(1), np.zeros(1)
        D = hc.hc_ee_closest(np.ascontiguousarray(xe[n].ravel()), s, t)
        assert abs(D - K["eec_D"][n]) <= 1e-12 * max(1.0, K["eec_D"][n])
        if n >= 300:  # the first 300 pairs are parallel: (s, t) is not unique there, D is
            assert abs(s[0] - K["eec_s"][n]) <= 1e-12 and abs(t[0] - K["eec_t"][n]) <= 1e-12


def test_contact_elements_vs_reference(hc, K):
    """Per-stencil energy/grad/projected Hessian vs the reference's ContactSet.potential."""
    X, pt, ee, epsx = K["pot_x"], K["pot_pt"], K["pot_ee"], K["pot_epsx"]
    idx, H_ref = K["pot_idx"], K["pot_H"]
    rows = {tuple(r): k for k, r in enumerate(idx)}
    E_sum = 0.0
    g_sum = np.zeros_like(X)
    checked = 0
    for kind, stencils in (("pt", pt), ("ee", ee)):
        for n, row in enumerate(stencils):
            x = np.ascontiguousarray(X[row].ravel())
            E, g, H = np.zeros(1), np.zeros(12), np.zeros(144)
            if kind == "pt":
                fl = hc.hc_pt_element(x, 3e6, 1e-3, E, g, H, 1)
            else:
                fl = hc.hc_ee_element(x, epsx[n], 3e6, 1e-3, E, g, H, 1)
            assert not (fl & 2)
            if fl & 1:
                E_sum += E[0]
                np.add.at(g_sum, row, g.reshape(4, 3))
                Hr = H_ref[rows[tuple(row)]]
                scale = np.abs(Hr).max()
                assert np.abs(H.reshape(12, 12) - Hr).max() <= 1e-9 * scale, (kind, n)
                checked += 1
    assert checked == len(idx)
    np.testing.assert_allclose(E_sum, K["pot_E"], rtol=1e-12)
    np.testing.assert_allclose(g_sum, K["pot_g"], rtol=1e-9, atol=1e-11 * np.abs(K["pot_g"]).max())


def test_neo_hookean_vs_reference(hc, K):
    rest, cur = K["nh_rest"], K["nh_cur"]
    Dmi, V0, _ = en.tet_rest(rest.reshape(-1, 3), np.arange(4 * len(rest)).reshape(-1, 4))
    Es = 0.0
    for n in range(len(rest)):
        E, g, H = np.zeros(1), np.zeros(12), np.zeros(144)
        fl = hc.hc_nh_element(np.ascontiguousarray(cur[n].ravel()), np.ascontiguousarray(Dmi[n].ravel()), V0[n],
                              float(K["nh_mu"]), float(K["nh_lam"]), E, g, H)
        assert fl == 0
        Es += E[0]
        np.testing.assert_allclose(E[0], K["nh_Ee"][n], rtol=1e-11, atol=1e-18)
        np.testing.assert_allclose(g.reshape(4, 3), K["nh_g"][4 * n:4 * n + 4], rtol=1e-9,
                                   atol=1e-10 * np.abs(K["nh_g"][4 * n:4 * n + 4]).max())
        Hr = K["nh_H"][n]
        assert np.abs(H.reshape(12, 12) - Hr).max() <= 1e-9 * np.abs(Hr).max(), n
        row = np.zeros(7)
        assert hc.hc_stress(np.ascontiguousarray(cur[n].ravel()), np.ascontiguousarray(Dmi[n].ravel()),
                            *en.lame(9.4e6, 0.3), row) == 1
        c = K["stress_cauchy"][n]
        ref = [c[0, 0], c[1, 1], c[2, 2], c[0, 1], c[1, 2], c[0, 2], K["stress_vm"][n]]
        np.testing.assert_allclose(row, ref, rtol=1e-9, atol=1e-6)
    np.testing.assert_allclose(Es, K["nh_E"], rtol=1e-12)


def test_abd_vs_reference(hc, K):
    for A, E, g, H in zip(K["abd_A"], K["abd_E"], K["abd_g"], K["abd_H"]):
        gg, HH = np.zeros(12), np.zeros(144)
        e = hc.hc_abd_element(np.ascontiguousarray(A.ravel()), 1e8 * 1.25e-4, gg, HH)
        np.testing.assert_allclose(e, E, rtol=1e-12)
        np.testing.assert_allclose(gg, g, rtol=1e-10, atol=1e-6)
        assert np.abs(HH.reshape(12, 12) - H).max() <= 1e-9 * np.abs(H).max()


def test_clamp_generic(hc, K):
    for A, ref in zip(K["spd_in"], K["spd_out"]):
        H = np.ascontiguousarray(A.ravel().copy())
        hc.hc_clamp12(H)
        assert np.abs(H.reshape(12, 12) - ref).max() <= 1e-10 * max(1.0, np.abs(ref).max())


def test_ccd_vs_reference(hc, K):
    cx, cp, ref = K["ccd_x"], K["ccd_p"], K["ccd_alpha"]
    bad = ctypes.c_int()
    for n in range(len(cx)):
        x, p = np.ascontiguousarray(cx[n].ravel()), np.ascontiguousarray(cp[n].ravel())
        a = [hc.hc_ccd(x, p, 0, 0.9, 32, 0.0, ctypes.byref(bad)), hc.hc_ccd(x, p, 1, 0.9, 32, 0.0, ctypes.byref(bad)),
             hc.hc_ccd(x, p, 0, 0.9, 32, 0.1, ctypes.byref(bad))]
        np.testing.assert_allclose(a, ref[n], rtol=1e-12, atol=1e-15)


def test_pencil_and_cubic_vs_reference(hc, K):
    c = K["cub_c"]
    got = np.array([hc.hc_cubic(*row) for row in c])
    np.testing.assert_allclose(got, K["cub_root"], rtol=1e-12)
    for M0, dM, ref in zip(K["pen_M0"], K["pen_dM"], K["pen_alpha"]):
        t = hc.hc_pencil(np.ascontiguousarray(M0.ravel()), np.ascontiguousarray(dM.ravel()))
        if t > 1.0:
            a = 1.0
        else:
            a = 0.9 * t
            for _ in range(60):
                if np.linalg.det(M0 + a * dM) > 0.0:
                    break
                a *= 0.5
        np.testing.assert_allclose(a, ref, rtol=1e-9)  # near-double roots amplify det rounding


def test_friction_vs_oracle(hc):
    rng = np.random.default_rng(3)
    for _ in range(100):
        x = rng.normal(size=(4, 3)) * 1e-3
        xp = x - rng.normal(size=(4, 3)) * rng.choice([1e-7, 1e-5, 1e-4])
        bary = rng.dirichlet(np.ones(3))
        gam = np.concatenate([[1.0], -bary])
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        T = en.tangent_basis(n[None])[0]
        anc = {"verts": np.arange(4)[None], "gamma": gam[None], "tangent": T[None], "lam": np.array([2.5]),
               "mu": np.array([0.7]), "bodies": np.zeros((1, 2), np.int64)}
        E, g, _, H = en.friction_potential(anc, x, xp, 1e-3, 0.01, order=2)
        gg, HH = np.zeros(12), np.zeros(144)
        e = hc.hc_friction(np.ascontiguousarray(x.ravel()), np.ascontiguousarray(xp.ravel()), gam,
                           np.ascontiguousarray(T.ravel()), 2.5, 0.7, 1e-3, 0.01, gg, HH)
        np.testing.assert_allclose(e, E, rtol=1e-12, atol=1e-20)
        np.testing.assert_allclose(gg.reshape(4, 3), g, rtol=1e-10, atol=1e-12 * np.abs(g).max())
        np.testing.assert_allclose(HH.reshape(12, 12), H[0], rtol=1e-10, atol=1e-12 * np.abs(H).max())


def test_friction_vs_reference_golden(hc, golden):
    """The host build of the friction element (grip_elements.cuh) and the oracle against the
    reference's own friction_potential (contact.py:475-524) on tests/golden/friction.npz."""
    F = np.load(golden / "friction.npz")
    eps_v, dt = float(F["eps_v"]), float(F["dt"])
    for k in range(len(F["fr_E"])):
        x, xp, gam, T = F["fr_x"][k], F["fr_xp"][k], F["fr_gamma"][k], F["fr_T"][k]
        lam, mu = float(F["fr_lam"][k]), float(F["fr_mu"][k])
        Er, gr, Hr = F["fr_E"][k], F["fr_g"][k], F["fr_H"][k]
        anc = {"verts": np.arange(4)[None], "gamma": gam[None], "tangent": T[None], "lam": np.array([lam]),
               "mu": np.array([mu]), "bodies": np.zeros((1, 2), np.int64)}
        E, g, _, H = en.friction_potential(anc, x, xp, eps_v, dt, order=2)
        np.testing.assert_allclose(E, Er, rtol=1e-12, atol=1e-20)
        np.testing.assert_allclose(g, gr, rtol=1e-10, atol=1e-12 * max(np.abs(gr).max(), 1e-300))
        np.testing.assert_allclose(H[0], Hr, rtol=1e-10, atol=1e-12 * max(np.abs(Hr).max(), 1e-300))
        gg, HH = np.zeros(12), np.zeros(144)
        e = hc.hc_friction(np.ascontiguousarray(x.ravel()), np.ascontiguousarray(xp.ravel()), np.ascontiguousarray(gam),
                           np.ascontiguousarray(T.ravel()), lam, mu, eps_v, dt, gg, HH)
        np.testing.assert_allclose(e, Er, rtol=1e-12, atol=1e-20)
        np.testing.assert_allclose(gg.reshape(4, 3), gr, rtol=1e-10, atol=1e-12 * max(np.abs(gr).max(), 1e-300))
        np.testing.assert_allclose(HH.reshape(12, 12), Hr, rtol=1e-10, atol=1e-12 * max(np.abs(Hr).max(), 1e-300))
