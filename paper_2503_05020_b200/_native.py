"""ctypes binding of the C ABI in include/grip_ipc.h (libgripipc.so, built in-tree).

There is no fallback: if the shared library is missing or no CUDA device is
visible, loading raises.  The oracle under oracle/ is test infrastructure
and is never imported here.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_DIR = Path(__file__).resolve().parent / "_lib"
LIB_PATH = Path(os.environ["GRIP_LIB"]) if os.environ.get("GRIP_LIB") else LIB_DIR / "libgripipc.so"  # GRIP_LIB: A/B builds
ABI_VERSION = 4
NPARAM = 14
(P_DT, P_KAPPA, P_DHAT, P_EPSV, P_RELTOL, P_MAXIT, P_ELLFLOOR, P_MAXLS, P_CCDSCALE, P_CCDIT, P_KINGUARD, P_MURULE,
 P_PCGRTOL, P_SPARE) = range(NPARAM)

NS_RUNNING, NS_CONVERGED, NS_FAILED = 0, 1, 2
REASONS = {
    0: "",
    1: "non-convergence",
    2: "line-search-failure",
    3: "ValueError: inverted element passed to elastic energy",
    4: "ValueError: contact stencil at non-positive distance",
    5: "FloatingPointError: non-finite assembly",
    6: "SolveBreakdown: linear solve failed after regularization",
    7: "IntersectionError: CCD called from an intersecting or touching state",
    8: "IntersectionError: step filter called with non-positive determinant state",
    9: "non-finite state",
    10: "device buffer capacity exceeded",
}

_P = ctypes.c_void_p


class GripSceneDesc(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_int32), ("n_env", ctypes.c_int32)] + [
        (name, _P) for name in (
            "node_off", "sv_off", "tri_off", "edge_off", "tet_off", "abd_off", "body_off",
            "node_x0", "node_M", "node_free", "node_body", "node_kind", "node_sv",
            "sv_kind", "sv_node", "sv_xi", "sv_body", "sv_kin0",
            "tris", "edges", "edge_rest_sq", "tet_nodes", "tet_Dmi", "tet_V0", "tet_mu", "tet_lam",
            "abd_node", "abd_kV", "abd_body",
            "body_kind", "body_mu", "body_pairmask", "body_vel0",
            "body_tri_lo", "body_tri_hi", "body_edge_lo", "body_edge_hi",
            "env_params", "env_gravity", "env_cell_hint")]


class GripStepReport(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("reason", ctypes.c_int32), ("iterations", ctypes.c_int32),
                ("n_alphas", ctypes.c_int32), ("residual", ctypes.c_double), ("min_distance", ctypes.c_double),
                ("energy", ctypes.c_double), ("time", ctypes.c_double), ("step_index", ctypes.c_int32),
                ("kinematic_blocked", ctypes.c_int32), ("regularized", ctypes.c_int32),
                ("newton_calls", ctypes.c_int32), ("pcg_iters", ctypes.c_int32), ("pad", ctypes.c_int32)]


REPORT_DTYPE = np.dtype([("status", "<i4"), ("reason", "<i4"), ("iterations", "<i4"), ("n_alphas", "<i4"),
                         ("residual", "<f8"), ("min_distance", "<f8"), ("energy", "<f8"), ("time", "<f8"),
                         ("step_index", "<i4"), ("kinematic_blocked", "<i4"), ("regularized", "<i4"),
                         ("newton_calls", "<i4"), ("pcg_iters", "<i4"), ("pad", "<i4")])
assert REPORT_DTYPE.itemsize == ctypes.sizeof(GripStepReport)

_lib = None


def load():
    """Load libgripipc.so; raises (never falls back) if it or a CUDA device is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} not built: run __graft_entry__.build() (nvcc, sm_100a)")
    lib = ctypes.CDLL(str(LIB_PATH))
    vp, i32, dbl = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    pb = ctypes.POINTER(ctypes.c_void_p)
    lib.grip_abi_version.restype = i32
    lib.grip_last_error.restype = ctypes.c_char_p
    lib.grip_create.argtypes = [ctypes.POINTER(GripSceneDesc), i32, pb]
    for name, args in (
        ("grip_destroy", [vp]), ("grip_set_controls", [vp, vp, vp]), ("grip_begin_step", [vp, vp]),
        ("grip_newton_iteration", [vp, vp]), ("grip_finalize_step", [vp, vp, vp, vp]),
        ("grip_step", [vp, vp, vp, vp]), ("grip_get_state", [vp, vp, vp, vp]),
        ("grip_set_state", [vp, vp, vp, vp]), ("grip_get_surface", [vp, vp]),
        ("grip_get_contacts", [vp, vp, vp, vp]),
        ("grip_query_candidates", [vp, i32, dbl, vp, i32, vp, vp, i32, vp]),
        ("grip_stress", [vp, vp]), ("grip_last_step_stats", [vp, vp, vp, vp]),
        ("grip_get_body_state", [vp, vp, vp]), ("grip_set_profiling", [vp, i32]),
        ("grip_kernel_stats", [vp, i32, vp, vp, vp]), ("grip_stream_timer", [vp, i32, vp]),
        ("grip_round", [vp, vp, vp, vp, vp, vp]),
        ("grip_debug_elements", [i32, i32, vp, i32, vp, vp, vp, vp]),
        ("grip_debug_chain", [i32, i32, vp, i32, vp, vp, vp, vp, vp]),
        ("grip_reset_envs", [vp, vp, ctypes.POINTER(GripSceneDesc)]), ("grip_set_recording", [vp, i32]),
        ("grip_get_events", [vp, vp, vp, vp, vp, ctypes.c_int64]),
        ("grip_sdf_exact", [vp, ctypes.c_int64, vp, i32, vp, i32, vp, vp, vp, vp]),
        ("grip_get_frames", [vp, vp, vp, vp, vp, vp]),
        ("grip_sdf_nn", [vp, ctypes.c_int64, vp, ctypes.c_int64, vp, vp, i32, vp]),
        ("grip_set_priority", [vp, i32]), ("grip_contacts_now", [vp, vp, dbl, vp]),
        ("grip_check_finite", [vp, vp]), ("grip_set_stream", [vp, vp]),
        ("grip_get_state_device", [vp, vp, vp, vp]), ("grip_set_controls_device", [vp, vp, vp]), ("grip_cta_records", [vp, vp, ctypes.c_int64, vp, i32]),
        ("grip_protocol_setup", [vp, vp, vp, vp, vp, vp, vp]), ("grip_protocol_reset", [vp, vp, vp, vp]),
        ("grip_run_rounds", [vp, i32, vp]), ("grip_protocol_read", [vp, vp]),
        ("grip_run_rounds_async", [vp, i32, vp]), ("grip_rounds_wait", [vp, i32, vp, vp]),
        ("grip_sdf_query", [vp, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int64, vp, vp])):
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = i32
    if lib.grip_abi_version() != ABI_VERSION:
        raise RuntimeError("libgripipc.so ABI version mismatch; rebuild")
    _lib = lib
    return lib


def check(rc):
    if rc != 0:
        raise RuntimeError("grip: " + (_lib.grip_last_error() or b"").decode())


def ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def debug_elements(etype, inputs):
    """Evaluate standalone elements with the device kernels (see grip_debug_elements)."""
    lib = load()
    a = np.ascontiguousarray(inputs, np.float64)
    n, stride = a.shape
    E, g, H, fl = np.zeros(n), np.zeros((n, 12)), np.zeros((n, 144)), np.zeros(n, np.int32)
    check(lib.grip_debug_elements(int(etype), n, ptr(a), stride, ptr(E), ptr(g), ptr(H), ptr(fl)))
    return E, g, H.reshape(n, 12, 12), fl


def debug_chain(etype, inputs, eig=None):
    """The same elements through the production element chain of a sweep (grip_debug_chain);
    eig (n, 9, 9) warm starts for NH tets are updated in place."""
    lib = load()
    a = np.ascontiguousarray(inputs, np.float64)
    n, stride = a.shape
    E, g, H, fl = np.zeros(n), np.zeros((n, 12)), np.zeros((n, 144)), np.zeros(n, np.int32)
    if eig is not None:
        assert eig.flags.c_contiguous and eig.dtype == np.float64 and eig.shape == (n, 9, 9)
    check(lib.grip_debug_chain(int(etype), n, ptr(a), stride, ptr(E), ptr(g), ptr(H), ptr(eig), ptr(fl)))
    return E, g, H.reshape(n, 12, 12), fl


class GripTrialOut(ctypes.Structure):
    """include/grip_ipc.h GripTrialOut (device protocol record of one env)."""
    _fields_ = [("halt_force", ctypes.c_double * 2), ("com_disp", ctypes.c_double * 6),
                ("final_disp", ctypes.c_double), ("threshold", ctypes.c_double), ("phase", ctypes.c_int32),
                ("verdict", ctypes.c_int32), ("n_steps", ctypes.c_int32), ("fail_phase", ctypes.c_int32),
                ("fail_reason", ctypes.c_int32), ("fail_step", ctypes.c_int32), ("halted", ctypes.c_int32),
                ("final_contact", ctypes.c_int32), ("halt_step", ctypes.c_int32 * 2), ("markers", ctypes.c_int32 * 18),
                ("min_distance", ctypes.c_double), ("min_J", ctypes.c_double)]


def sdf_exact(pts, verts, tris, face_n, edge_n, vert_n):
    """Signed exact distances of pts to a triangle surface (grip_sdf_exact)."""
    lib = load()
    f = lambda a: np.ascontiguousarray(a, np.float64)  # noqa: E731
    pts, verts, face_n, edge_n, vert_n = f(pts), f(verts), f(face_n), f(edge_n), f(vert_n)
    tris = np.ascontiguousarray(tris, np.int32)
    out = np.empty(len(pts))
    check(lib.grip_sdf_exact(ptr(pts), len(pts), ptr(verts), len(verts), ptr(tris), len(tris), ptr(face_n),
                             ptr(edge_n), ptr(vert_n), ptr(out)))
    return out


def sdf_nn(pts, cloud):
    """Exact nearest-neighbour distances of pts to cloud (grip_sdf_nn): the cloud is Morton-sorted
    into leaves of 8 under an implicit complete binary tree of boxes built here."""
    lib = load()
    pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    cloud = np.asarray(cloud, np.float64).reshape(-1, 3)
    lo, hi = cloud.min(axis=0), cloud.max(axis=0)
    g = np.clip(((cloud - lo) / np.maximum(hi - lo, 1e-300) * 1023.0).astype(np.int64), 0, 1023)
    code = np.zeros(len(cloud), np.int64)
    for b in range(10):   # 30-bit Morton code
        for a in range(3):
            code |= ((g[:, a] >> b) & 1) << (3 * b + a)
    cloud = np.ascontiguousarray(cloud[np.argsort(code, kind="stable")])
    m = len(cloud)
    n_leaf = max(1, -(-m // 8))
    levels = int(np.ceil(np.log2(n_leaf))) if n_leaf > 1 else 0
    L = 1 << levels
    # padding slots: +inf for the minima, -inf for the maxima (empty leaves: inverted boxes)
    llo = np.concatenate([cloud, np.full((L * 8 - m, 3), np.inf)]).reshape(L, 8, 3).min(axis=1)
    lhi = np.concatenate([cloud, np.full((L * 8 - m, 3), -np.inf)]).reshape(L, 8, 3).max(axis=1)
    lv_lo, lv_hi = [llo], [lhi]
    while len(lv_lo[-1]) > 1:
        a, b = lv_lo[-1], lv_hi[-1]
        lv_lo.append(np.minimum(a[0::2], a[1::2]))
        lv_hi.append(np.maximum(b[0::2], b[1::2]))
    box_lo = np.ascontiguousarray(np.concatenate(lv_lo[::-1]))
    box_hi = np.ascontiguousarray(np.concatenate(lv_hi[::-1]))
    out = np.empty(len(pts))
    check(lib.grip_sdf_nn(ptr(pts), len(pts), ptr(cloud), m, ptr(box_lo), ptr(box_hi), levels, ptr(out)))
    return out


def sdf_query(values, origin, spacing, pts, rot=None, trans=None, world_lo=None, world_hi=None, want_values=False):
    """max d_o over pts (and every d_o if want_values) of a grid SDF (grip_sdf_query)."""
    lib = load()
    f = lambda a: None if a is None else np.ascontiguousarray(a, np.float64)  # noqa: E731
    values, pts = f(values), f(pts).reshape(-1, 3)
    dims = np.asarray(values.shape, np.int32)
    origin, spacing, rot, trans, world_lo, world_hi = map(f, (origin, spacing, rot, trans, world_lo, world_hi))
    d_o = np.empty(len(pts)) if want_values else None
    dmax = ctypes.c_double()
    check(lib.grip_sdf_query(ptr(values), ptr(dims), ptr(origin), ptr(spacing), ptr(rot), ptr(trans), ptr(world_lo),
                             ptr(world_hi), ptr(pts), len(pts), ptr(d_o), ctypes.byref(dmax)))
    return dmax.value, d_o


class EventBlock:
    """One step's contact events of one env, as arrays (contact.py:348-372 stencil_forces rows)."""

    __slots__ = ("i", "d")
    KINDS = ("point-triangle", "edge-edge")

    def __init__(self, i, d):
        self.i, self.d = i, d

    def __len__(self):
        return len(self.i)

    def as_dicts(self):
        return [{"kind": self.KINDS[r[0]], "bodies": (int(r[1]), int(r[2])), "verts": [int(v) for v in r[3:7]],
                 "d": float(dd[0]), "lambda": float(dd[1])} for r, dd in zip(self.i.tolist(), self.d)]

    def force_on(self, body):
        """Summed lambda of the events touching `body` (protocol.py:78-86); 0 (int) when none."""
        sel = (self.i[:, 1] == body) | (self.i[:, 2] == body)
        return sum(self.d[sel, 1].tolist()) if sel.any() else 0


class DeviceBatch:
    """Owns one GripBatch handle (device memory + stream) built from a packed scene."""

    def __init__(self, packed, device=None):
        lib = load()
        self.packed = packed
        self._keep = []
        desc = GripSceneDesc()
        desc.abi_version = ABI_VERSION
        desc.n_env = packed.n_env
        for name, _ in GripSceneDesc._fields_[2:]:
            arr = np.ascontiguousarray(getattr(packed, name))
            self._keep.append(arr)
            setattr(desc, name, arr.ctypes.data)
        h = ctypes.c_void_p()
        dev = int(os.environ.get("LOCAL_RANK", "0")) if device is None else int(device)
        check(lib.grip_create(ctypes.byref(desc), dev, ctypes.byref(h)))
        self.h = h
        self.n_env = packed.n_env
        self.lib = lib
        self.max_alpha = int(max(packed.env_params[:, P_MAXIT].max(), 1)) + 1

    def close(self):
        if getattr(self, "h", None):
            self.lib.grip_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_controls(self, gravity=None, body_vel=None):
        g = None if gravity is None else np.ascontiguousarray(gravity, np.float64)
        v = None if body_vel is None else np.ascontiguousarray(body_vel, np.float64)
        check(self.lib.grip_set_controls(self.h, ptr(g), ptr(v)))

    def step(self, active):
        act = np.ascontiguousarray(active, np.uint8)
        rep = np.zeros(self.n_env, REPORT_DTYPE)
        alphas = np.zeros((self.n_env, self.max_alpha))
        check(self.lib.grip_step(self.h, ptr(act), rep.ctypes.data_as(ctypes.c_void_p), ptr(alphas)))
        return rep, alphas

    def round(self, begin, iterating):
        b = np.ascontiguousarray(begin, np.uint8)
        it = np.ascontiguousarray(iterating, np.uint8)
        fin = np.zeros(self.n_env, np.uint8)
        rep = np.zeros(self.n_env, REPORT_DTYPE)
        alphas = np.zeros((self.n_env, self.max_alpha))
        check(self.lib.grip_round(self.h, ptr(b), ptr(it), ptr(fin), rep.ctypes.data_as(ctypes.c_void_p), ptr(alphas)))
        return fin.astype(bool), rep, alphas

    # per-env arrays a slot refill replaces (everything pose- or material-dependent; the topology
    # arrays and offsets must stay): (name, values per entity, offset array)
    RESET_FIELDS = (("node_x0", 3, "node_off"), ("node_M", 9, "node_off"), ("sv_kin0", 3, "sv_off"),
                    ("sv_xi", 3, "sv_off"), ("tet_Dmi", 9, "tet_off"), ("tet_V0", 1, "tet_off"),
                    ("tet_mu", 1, "tet_off"), ("tet_lam", 1, "tet_off"), ("body_mu", 1, "body_off"),
                    ("edge_rest_sq", 1, "edge_off"), ("abd_kV", 1, "abd_off"))

    def reset_envs(self, mask, packed):
        """Slot refill (grip_reset_envs): the masked envs take their pose, rest shape and materials
        from `packed` (a full-size Packed of the same topology), every other per-env state returns
        to a fresh batch's."""
        m = np.ascontiguousarray(mask, np.uint8)
        desc = GripSceneDesc()
        desc.abi_version = ABI_VERSION
        desc.n_env = packed.n_env
        keep = []
        for name, _ in GripSceneDesc._fields_[2:]:
            arr = np.ascontiguousarray(getattr(packed, name))
            keep.append(arr)
            setattr(desc, name, arr.ctypes.data)
        check(self.lib.grip_reset_envs(self.h, ptr(m), ctypes.byref(desc)))
        del keep

    def begin_step(self, active):
        act = np.ascontiguousarray(active, np.uint8)
        check(self.lib.grip_begin_step(self.h, ptr(act)))

    def newton_iteration(self, pending):
        pend = np.ascontiguousarray(pending, np.uint8)
        check(self.lib.grip_newton_iteration(self.h, ptr(pend)))
        return pend.astype(bool)

    def finalize_step(self, active):
        act = np.ascontiguousarray(active, np.uint8)
        rep = np.zeros(self.n_env, REPORT_DTYPE)
        alphas = np.zeros((self.n_env, self.max_alpha))
        check(self.lib.grip_finalize_step(self.h, ptr(act), rep.ctypes.data_as(ctypes.c_void_p), ptr(alphas)))
        return rep, alphas

    def get_state(self, with_kin=True):
        p = self.packed
        x = np.empty((p.n_node_total, 3))
        v = np.empty((p.n_node_total, 3))
        kin = np.empty((p.n_sv_total, 3)) if with_kin else None
        check(self.lib.grip_get_state(self.h, ptr(x), ptr(v), ptr(kin)))
        return x, v, kin

    # -- torch interop: a caller's stream and device tensors (no host round trip) ---------------
    def set_stream(self, stream=None):
        """Run on a torch.cuda.Stream (or a raw cudaStream_t int); None: the library's own stream."""
        handle = None if stream is None else (stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        check(self.lib.grip_set_stream(self.h, ctypes.c_void_p(handle) if handle else None))

    def state_tensors(self, out=None):
        """x, v (n_node, 3) and kinematic positions (n_sv, 3) as float64 CUDA tensors, copied
        device-to-device on the batch's stream (grip_get_state_device)."""
        import torch
        p = self.packed
        dev = torch.device("cuda", torch.cuda.current_device())
        x, v, kin = out or (torch.empty((p.n_node_total, 3), dtype=torch.float64, device=dev),
                            torch.empty((p.n_node_total, 3), dtype=torch.float64, device=dev),
                            torch.empty((p.n_sv_total, 3), dtype=torch.float64, device=dev))
        for t in (x, v, kin):
            if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
                raise ValueError("state tensors must be contiguous float64 CUDA tensors")
        check(self.lib.grip_get_state_device(self.h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(v.data_ptr()),
                                             ctypes.c_void_p(kin.data_ptr())))
        return x, v, kin

    def set_controls_tensors(self, gravity=None, body_vel=None):
        """Per-env gravity (n_env, 3) and per-body velocities (n_body, 3) from float64 CUDA tensors."""
        def dp(t):
            if t is None:
                return None
            if t.dtype.is_floating_point is False or not t.is_cuda or not t.is_contiguous() or t.element_size() != 8:
                raise ValueError("control tensors must be contiguous float64 CUDA tensors")
            return ctypes.c_void_p(t.data_ptr())
        check(self.lib.grip_set_controls_device(self.h, dp(gravity), dp(body_vel)))

    def set_state(self, x=None, v=None, kin=None):
        f = lambda a: None if a is None else np.ascontiguousarray(a, np.float64)  # noqa: E731
        x, v, kin = f(x), f(v), f(kin)
        check(self.lib.grip_set_state(self.h, ptr(x), ptr(v), ptr(kin)))

    def surface(self):
        sv = np.empty((self.packed.n_sv_total, 3))
        check(self.lib.grip_get_surface(self.h, ptr(sv)))
        return sv

    def contacts(self):
        p = self.packed
        force = np.empty(p.n_body_total)
        mask = np.empty(p.n_body_total, np.uint32)
        md = np.empty(p.n_env)
        check(self.lib.grip_get_contacts(self.h, ptr(force), ptr(mask), ptr(md)))
        return force, mask, md

    def contacts_now(self, mask, radius_factor=1.05):
        """Contact readout at the current state (grip_contacts_now): per-env min stencil distance at
        radius_factor * dhat; the active stencils become the event rows of event_blocks()."""
        m = np.ascontiguousarray(mask, np.uint8)
        md = np.full(self.n_env, np.inf)
        check(self.lib.grip_contacts_now(self.h, ptr(m), float(radius_factor), ptr(md)))
        return md

    CTA_KERNELS = ("begin", "candidates", "assemble_direct", "line_search", "finalize", "bound")

    def cta_records(self, reset=True, cap=1 << 21):
        """Per-CTA timing records (GRIP_CTA_TIMING builds): structured array seq, kernel, env, sm,
        t0 (ns, low 32 bits of the global timer), dur (ns)."""
        raw = np.zeros((cap, 4), np.uint64)
        n = ctypes.c_int64()
        check(self.lib.grip_cta_records(self.h, ptr(raw), cap, ctypes.byref(n), int(reset)))
        r = raw[:n.value]
        out = np.zeros(len(r), [("seq", "<u8"), ("kernel", "<i4"), ("env", "<i4"), ("sm", "<i4"), ("info", "<u4"),
                                ("t0", "<u8"), ("dur", "<u8")])
        out["seq"], out["kernel"], out["env"] = r[:, 0], (r[:, 1] >> np.uint64(32)), r[:, 1] & np.uint64(0xffffffff)
        out["sm"], out["info"] = r[:, 2] & np.uint64(0xffff), r[:, 2] >> np.uint64(16)
        out["t0"], out["dur"] = r[:, 3] >> np.uint64(32), r[:, 3] & np.uint64(0xffffffff)
        return out

    def check_finite(self):
        """Per env: True when its state holds a NaN / inf (grip_check_finite)."""
        bad = np.zeros(self.n_env, np.uint8)
        check(self.lib.grip_check_finite(self.h, ptr(bad)))
        return bad.astype(bool)

    def candidates(self, env, radius):
        n_pt, n_ee = ctypes.c_int32(), ctypes.c_int32()
        check(self.lib.grip_query_candidates(self.h, int(env), float(radius), None, 0, ctypes.byref(n_pt), None, 0,
                                             ctypes.byref(n_ee)))
        pt = np.empty((max(n_pt.value, 1), 4), np.int32)
        ee = np.empty((max(n_ee.value, 1), 4), np.int32)
        check(self.lib.grip_query_candidates(self.h, int(env), float(radius), ptr(pt), n_pt.value, ctypes.byref(n_pt),
                                             ptr(ee), n_ee.value, ctypes.byref(n_ee)))
        return pt[:n_pt.value].astype(np.int64), ee[:n_ee.value].astype(np.int64)

    def stress(self):
        out = np.empty((max(self.packed.n_tet_total, 1), 7))
        check(self.lib.grip_stress(self.h, ptr(out)))
        return out[:self.packed.n_tet_total]

    def frames(self, mask):
        """Packed recorder frame of the masked envs (grip_get_frames): x, v (nodes x 3),
        kin (surface vertices x 3), stress (tets x 7), each in env order."""
        p = self.packed
        m = np.ascontiguousarray(mask, np.uint8)
        sel = np.nonzero(m)[0]
        nn = int(sum(p.node_off[e + 1] - p.node_off[e] for e in sel))
        ns = int(sum(p.sv_off[e + 1] - p.sv_off[e] for e in sel))
        nt = int(sum(p.tet_off[e + 1] - p.tet_off[e] for e in sel))
        x, v, kin, st = np.empty((nn, 3)), np.empty((nn, 3)), np.empty((ns, 3)), np.empty((nt, 7))
        check(self.lib.grip_get_frames(self.h, ptr(m), ptr(x), ptr(v), ptr(kin), ptr(st)))
        return x, v, kin, st

    def body_state(self):
        com = np.empty((self.packed.n_body_total, 3))
        sp = np.empty(self.n_env)
        check(self.lib.grip_get_body_state(self.h, ptr(com), ptr(sp)))
        return com, sp

    def set_priority(self, priority):
        """Stream priority among concurrent batches (grip_set_priority)."""
        check(self.lib.grip_set_priority(self.h, int(priority)))

    def set_recording(self, on=True):
        """Contact-event recording in every finalize (grip_set_recording)."""
        check(self.lib.grip_set_recording(self.h, int(on)))

    EVENT_KINDS = ("point-triangle", "edge-edge")

    def event_blocks(self, mask):
        """Contact events of the last finalize for envs with mask[e] (protocol.py:72-75):
        env -> EventBlock (int rows kind, body a, body b, 4 verts; float rows d, lambda)."""
        m = np.ascontiguousarray(mask, np.uint8)
        counts = np.zeros(self.n_env, np.int32)
        cap = int(max(1, m.sum()) * 64)
        while True:
            ei = np.zeros((cap, 7), np.int32)
            ed = np.zeros((cap, 2))
            rc = self.lib.grip_get_events(self.h, ptr(m), ptr(counts), ptr(ei), ptr(ed), cap)
            if rc == 0:
                break
            if b"capacity" not in self.lib.grip_last_error():
                check(rc)
            cap *= 2
        out, off = {}, 0
        for e in np.nonzero(m)[0]:
            n = int(counts[e])
            out[int(e)] = EventBlock(ei[off:off + n], ed[off:off + n])
            off += n
        return out

    def events(self, mask):
        """As event_blocks, as the reference's lists of {kind, bodies, verts, d, lambda} dicts."""
        return {e: b.as_dicts() for e, b in self.event_blocks(mask).items()}

    # -- device-resident protocol (grip_protocol_*, grip_run_rounds) --------------------------
    def protocol_setup(self, finger_body, closing_dir, object_body, gripper_bits, max_close, cfg):
        i32a = lambda a: np.ascontiguousarray(a, np.int32)  # noqa: E731
        self._pr_keep = [i32a(finger_body), np.ascontiguousarray(closing_dir, np.float64), i32a(object_body),
                         i32a(gripper_bits), i32a(max_close), np.ascontiguousarray(cfg, np.float64)]
        check(self.lib.grip_protocol_setup(self.h, *[ptr(a) for a in self._pr_keep]))

    def protocol_reset(self, mask, closing_dir, max_close):
        m = np.ascontiguousarray(mask, np.uint8)
        cd = np.ascontiguousarray(closing_dir, np.float64)
        mc = np.ascontiguousarray(max_close, np.int32)
        check(self.lib.grip_protocol_reset(self.h, ptr(m), ptr(cd), ptr(mc)))

    def run_rounds(self, rounds):
        n = ctypes.c_int64()
        check(self.lib.grip_run_rounds(self.h, int(rounds), ctypes.byref(n)))
        return n.value

    def run_rounds_async(self, rounds):
        """Enqueue `rounds` rounds + an async readout (grip_run_rounds_async); returns a ticket."""
        t = ctypes.c_int32()
        check(self.lib.grip_run_rounds_async(self.h, int(rounds), ctypes.byref(t)))
        return t.value

    def rounds_wait(self, ticket, records=True):
        """(env-steps, GripTrialOut array or None) of an enqueued call (grip_rounds_wait)."""
        n = ctypes.c_int64()
        out = (GripTrialOut * self.n_env)() if records else None
        check(self.lib.grip_rounds_wait(self.h, int(ticket), ctypes.byref(n), out))
        return n.value, out

    def protocol_read(self):
        out = (GripTrialOut * self.n_env)()
        check(self.lib.grip_protocol_read(self.h, out))
        return out

    def set_profiling(self, on=True):
        check(self.lib.grip_set_profiling(self.h, int(on)))

    KERNELS = ("begin", "candidates", "work_scan", "elements", "assemble_pcg", "line_search", "finalize", "tets")

    def kernel_stats(self):
        out = {}
        units = np.zeros(8)
        for k, name in enumerate(self.KERNELS):
            ms, n = ctypes.c_double(), ctypes.c_int64()
            check(self.lib.grip_kernel_stats(self.h, k, ctypes.byref(ms), ctypes.byref(n),
                                             ptr(units) if k == 3 else None))
            out[name] = {"ms": ms.value, "launches": n.value}
        out["elements"]["units"] = {"tets": units[0], "affine": units[1], "contacts": units[2], "anchors": units[3]}
        out["assemble_pcg"]["pcg_iterations"] = units[4]
        out["assemble_pcg"]["solves"] = units[5]
        out["assemble_pcg"]["mean_unknowns"] = units[6] / max(units[5], 1.0)
        out["elements"]["env_iterations"] = units[7]   # newton_iteration calls (env sweeps)
        return out

    def timer_start(self):
        check(self.lib.grip_stream_timer(self.h, 1, None))

    def timer_stop(self):
        ms = ctypes.c_double()
        check(self.lib.grip_stream_timer(self.h, 0, ctypes.byref(ms)))
        return ms.value

    def stats(self):
        ms, la, sw = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
        check(self.lib.grip_last_step_stats(self.h, ctypes.byref(ms), ctypes.byref(la), ctypes.byref(sw)))
        return ms.value, la.value, sw.value
