"""torch interop of the C ABI (device pointers from torch tensors plus a cudaStream_t):
a batch run on a caller's torch stream with its controls pushed from CUDA tensors and its state
read into CUDA tensors is bitwise the same as the host-pointer path."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _group(ids):
    from paper_2503_05020_b200 import scene as sc
    from paper_2503_05020_b200.multienv import DeviceEnvGroup
    from paper_2503_05020_b200.solver import Environment
    c = sc.load_cfg2_candidates()
    scenes = [sc.cfg2_scene(i, c) for i in ids]
    envs = [Environment(s.bodies, collide_pairs_off=s.collide_pairs_off) for s in scenes]
    return DeviceEnvGroup(envs), scenes


def test_torch_stream_and_device_tensors_match_host_path():
    import torch
    from paper_2503_05020_b200 import packing
    ids = [0, 1, 2]
    host, scenes = _group(ids)
    devg, _ = _group(ids)
    p = host.packed
    vel = np.zeros((p.n_body_total, 3))
    for e, s in enumerate(scenes):
        for f, b_ids in s.finger_links.items():
            for b in b_ids:
                vel[p.body_off[e] + b] = s.closing_dirs[f] * 0.05
    grav = np.tile([0.0, 0.0, -9.8], (p.n_env, 1))
    stream = torch.cuda.Stream()
    devg.dev.set_stream(stream)
    with torch.cuda.stream(stream):
        g_t = torch.as_tensor(grav, device="cuda")
        v_t = torch.as_tensor(vel, device="cuda")
    devg.dev.set_controls_tensors(g_t, v_t)
    host.dev.set_controls(grav, vel)
    act = np.ones(p.n_env, np.uint8)
    for _ in range(4):
        r_h, _ = host.dev.step(act)
        r_d, _ = devg.dev.step(act)
        assert np.array_equal(r_h["iterations"], r_d["iterations"])
    with torch.cuda.stream(stream):
        x_t, v_t2, kin_t = devg.dev.state_tensors()
    stream.synchronize()
    x_h, v_h, kin_h = host.dev.get_state(True)
    assert np.array_equal(x_t.cpu().numpy(), x_h)
    assert np.array_equal(v_t2.cpu().numpy(), v_h)
    assert np.array_equal(kin_t.cpu().numpy(), kin_h)
    devg.dev.set_stream(None)   # back to the library's stream
    r_h, _ = host.dev.step(act)
    r_d, _ = devg.dev.step(act)
    assert np.array_equal(host.dev.get_state(False)[0], devg.dev.get_state(False)[0])
    assert packing is not None
