"""World-size-2 multi-rank path on CPU (gloo): env sharding and the final outcome gather.

The GPU run uses the same code with NCCL; per-step there is no collective (envs are
independent), so this covers every piece of cross-rank logic.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as tmp

from paper_2503_05020_b200.distributed import OUTCOME_FIELDS, gather_outcomes, pack_outcomes, shard
from paper_2503_05020_b200.protocol import TrialRecord


def test_shard_covers_all_envs_once():
    for n in (1, 7, 400, 3200):
        for world in (1, 2, 4, 8):
            got = []
            for r in range(world):
                lo, hi = shard(n, world, r)
                got.extend(range(lo, hi))
            assert got == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_envs, q, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard(n_envs, world, rank)
    recs = []
    for e in range(lo, hi):
        r = TrialRecord(verdict=("stable", "unstable", "sim-failed")[e % 3], n_steps=70 + e)
        r.metrics = {"final_phase_com_disp": 1e-5 * e, "final_contact": e % 2 == 0}
        r.halt_forces = {"finger0": {"step": e, "force": 50.0 + e}}
        recs.append(r)
    # rank 1 finished one trial more than its shard (variable counts per rank are gathered)
    jobs = list(range(lo, hi))
    if rank == 1:
        extra = TrialRecord(verdict="stable", n_steps=1)
        recs.append(extra)
        jobs.append(lo)
    allr = gather_outcomes(pack_outcomes(recs, jobs, rank=rank))
    # dataset shards: every rank writes its own directory, rank 0 merges the manifests
    from paper_2503_05020_b200 import dataset as ds
    from paper_2503_05020_b200.distributed import merge_manifests, rank_dir
    w = ds.ShardWriter(rank_dir(out_dir, rank))
    for j, r in zip(jobs, recs):
        w.put(j, r)
    w.close()
    dist.barrier()
    man = merge_manifests(out_dir, world, ds.FORMAT) if rank == 0 else None
    q.put((rank, allr, man))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_envs", [7, 10])
def test_gather_outcomes_world2_gloo(n_envs, tmp_path):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_envs, q, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res = {r: a for r, a, _ in got}
    man = [m for r, _, m in got if r == 0][0]
    lo1 = shard(n_envs, 2, 1)[0]
    for rank in (0, 1):
        a = res[rank]
        assert a.shape == (n_envs + 1, len(OUTCOME_FIELDS))
        main = a[a[:, 2] != 1]                     # the extra trial has n_steps 1
        np.testing.assert_array_equal(main[:, 0], np.arange(n_envs))
        np.testing.assert_array_equal(main[:, 1], np.arange(n_envs) % 3)
        np.testing.assert_array_equal(main[:, 2], 70 + np.arange(n_envs))
        np.testing.assert_allclose(main[:, 6], 50.0 + np.arange(n_envs))
        np.testing.assert_array_equal(main[:, 12], (np.arange(n_envs) >= lo1).astype(float))
        extra = a[a[:, 2] == 1]
        assert extra.shape[0] == 1 and extra[0, 0] == lo1 and extra[0, 12] == 1
    np.testing.assert_array_equal(res[0], res[1])
    # merged manifest: every trial of both ranks, dirs under the rank shards
    assert man["n_trials"] == n_envs + 1
    dirs = [t["dir"] for t in man["trials"]]
    assert all(d.startswith("rank00/") or d.startswith("rank01/") for d in dirs)
    assert sum(d.startswith("rank01/") for d in dirs) == n_envs - lo1 + 1
    for t in man["trials"]:
        assert (tmp_path / t["dir"] / "meta.json").exists()


def test_pack_outcomes_running_trial():
    """A trial still running when the outcomes are gathered (the device protocol's records mid
    trial) packs as verdict -1 instead of failing."""
    r = TrialRecord(verdict="running", n_steps=12)
    a = pack_outcomes([r], [5])
    assert a[0, 0] == 5 and a[0, 1] == -1 and a[0, 2] == 12


def _bench_worker(rank, world, port, q, out_dir):
    """bench.py's end-of-run path (gather_timed) on a world-2 gloo group: each rank finished a
    different number of trials (its own candidates), recorded into its own dataset shard."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2503_05020_b200 import dataset as ds
    from paper_2503_05020_b200._native import REASONS
    from paper_2503_05020_b200.distributed import rank_dir
    jobs = [rank * 400 + k for k in range(3 + rank)]
    timed = []
    for j in jobs:
        r = TrialRecord(verdict="sim-failed" if j % 2 else "stable", n_steps=j % 150)
        if j % 2:
            r.failure = {"phase": "close", "reason": "non-convergence", "step": 3}
        r.min_distance, r.min_J = 1e-4, 0.9
        timed.append((j, r))
    w = ds.ShardWriter(rank_dir(out_dir, rank))
    for j, r in timed:
        w.put(j, r)
    w.close()
    out = bench.gather_timed(timed, rank, world, dist, out_dir, REASONS)
    q.put((rank, out))
    dist.destroy_process_group()


def test_bench_gather_world2_gloo(tmp_path):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank in (0, 1):
        o = got[rank]
        assert o["trials"] == 7 and o["ranks"] == [0, 1] and o["backend"] == "gloo"
        assert o["verdicts"] == {"stable": 4, "unstable": 0, "sim-failed": 3}
    assert got[0]["merged_trials"] == 7
    import json
    man = json.loads((tmp_path / "manifest.json").read_text())
    assert sorted(t["id"] for t in man["trials"]) == [0, 1, 2, 400, 401, 402, 403]
