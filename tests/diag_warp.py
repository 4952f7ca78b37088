"""Diagnostic (not collected): device warp element kernels vs host-check per-thread math."""
import ctypes, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2503_05020_b200._native import debug_elements
from oracle import energies as oen
from oracle import geometry as geo
K = dict(np.load(ROOT / "tests/golden/kernels.npz"))
X, pt, ee, epsx = K["pot_x"], K["pot_pt"], K["pot_ee"], K["pot_epsx"]
inp = np.array([np.concatenate([X[r].ravel(), [3e6, 1e-3]]) for r in pt])
E, g, H, fl = debug_elements(0, inp)
_, _, reg = geo.pt_closest(X[pt[:, 0]], X[pt[:, 1]], X[pt[:, 2]], X[pt[:, 3]])
D, gD, HD, _ = oen.pt_terms(X[pt], 2)
ok = 0
for n in range(len(pt)):
    if not fl[n] & 1:
        continue
    b, f1, f2 = oen.barrier_D(D[n:n+1], 1e-3)
    Hraw = 3e6 * (f2[0] * np.outer(gD[n], gD[n]) + f1[0] * HD[n])
    Hp = oen.spd_clamp(Hraw[None])[0]
    err = np.abs(H[n] - Hp).max() / np.abs(Hp).max()
    gerr = np.abs(g[n] - 3e6 * f1[0] * gD[n]).max() / np.abs(gD[n]).max() / abs(3e6 * f1[0])
    if err > 1e-9 and ok < 4:
        ok += 1
        ev = np.linalg.eigvalsh(0.5 * (Hraw + Hraw.T))
        print("PT", n, "region", reg[n], "Herr", err, "gerr", gerr, "eig min/max", ev.min(), ev.max())
        print(" gpu row0", np.round(H[n][0, :6], 3))
        print(" ref row0", np.round(Hp[0, :6], 3))
        print(" raw row0", np.round(Hraw[0, :6], 3))
errs = []
for n in range(len(pt)):
    if fl[n] & 1:
        b, f1, f2 = oen.barrier_D(D[n:n+1], 1e-3)
        Hraw = 3e6 * (f2[0] * np.outer(gD[n], gD[n]) + f1[0] * HD[n])
        Hp = oen.spd_clamp(Hraw[None])[0]
        errs.append((reg[n], np.abs(H[n] - Hp).max() / np.abs(Hp).max()))
errs = np.array(errs)
for r in range(7):
    m = errs[:, 0] == r
    if m.any():
        print("region", r, "count", m.sum(), "max err", errs[m, 1].max())
rest, cur = K["nh_rest"], K["nh_cur"]
Dmi, V0, _ = oen.tet_rest(rest.reshape(-1, 3), np.arange(4 * len(rest)).reshape(-1, 4))
inp = np.array([np.concatenate([cur[n].ravel(), Dmi[n].ravel(), [V0[n], K["nh_mu"], K["nh_lam"]]]) for n in range(len(rest))])
E, g, H, fl = debug_elements(2, inp)
e1 = [np.abs(H[n] - K["nh_H"][n]).max() / np.abs(K["nh_H"][n]).max() for n in range(len(rest))]
e2 = [np.abs(H[n] - K["nh_Hraw"][n]).max() / np.abs(K["nh_Hraw"][n]).max() for n in range(len(rest))]
print("NH proj err max", max(e1), "vs raw", min(e2), "E err", np.abs(E - K["nh_Ee"]).max())
inp = np.array([np.concatenate([A.ravel(), [1e8 * 1.25e-4]]) for A in K["abd_A"]])
E, g, H, _ = debug_elements(3, inp)
print("ABD err", max(np.abs(H[n] - K["abd_H"][n]).max() / np.abs(K["abd_H"][n]).max() for n in range(len(inp))))
