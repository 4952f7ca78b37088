"""Benchmark: env-steps/s of the batched grasp protocol (BASELINE config 2) on B200.

Workload (BASELINE.json configs[1]): 400 environments per GPU, each a soft UMI-style
two-pad gripper grasping a rigid (ABD) box / cylinder / sphere (slot s: kind s % 3,
reference-sampled antipodal candidates), stepped through the reference's validation
protocol (settle, force-halted closing, hold, six gravity phases; protocol.py:152-277).
Slots are kept full the way a dataset-generation run keeps them full: when a trial ends,
its slot restarts with the next candidate of the same object kind.  A bench "step" is one
device round: one Newton sweep of every unfinished env plus begin/finalize for envs at a
time-step boundary.  W warm-up rounds bring the slots to steady state, then K timed
rounds; value counts the env time steps (solver.py:764-771 newton_step calls) that
completed in the timed rounds.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Reports (one JSON line on rank 0): value = env-steps/s from CUDA events on the
library stream (max over ranks), e2e = the same through the public Python API
with host buffers (controls H2D, reports/forces D2H every step, wall clock),
roofline of the dominant kernel from live per-launch CUDA events, and a CPU
baseline: the oracle port (oracle/, the reference's algorithm restated in numpy)
timed on this host's cores on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "env-steps/sec at 400 envs (1/2/4/8 B200) vs CPU ref; ms per Newton iteration"
UNIT = "env-steps/s"
ENVS_PER_GPU = 400

# Algorithmic bytes per element of the element kernel (fp64 8 B, index 4 B; each input
# read once, each output written once): inputs + (E 8 + grad 96 + 12x12 Hessian 1152 + idx 16).
EL_OUT = 8 + 96 + 1152 + 16
EL_BYTES = {"tets": 16 + 96 + 72 + 24 + EL_OUT,        # node ids, 4 positions, Dm^-1, V0/mu/lam
            "affine": 96 + 8 + EL_OUT,                  # q, kappa*V
            "contacts": 16 + 4 + 96 + 8 + 8 + EL_OUT,   # row, code, 4 positions, rest lengths
            "anchors": 16 + 32 + 48 + 16 + 192 + EL_OUT}  # verts, gamma, T, lam/mu, x and x_prev


# kernel groups as timed live (grip_kernel_stats) -> the kernels of the committed ncu capture
KGROUPS = {"elements": ["k_tet_front", "k_elements_w", "k_tet_jacobi2", "k_tet_back", "k_tet_finish"],
           "assemble_pcg": ["k_contact_K", "k_assemble_direct"], "candidates": ["k_candidates"],
           "line_search": ["k_linesearch"], "begin": ["k_begin"], "finalize": ["k_finalize"]}
NCU_FULL = ROOT / "profiles" / "r1_ncu_full_v5.json"


def _ncu_group(group):
    """dram read + write bytes and fp64 FLOPs per launch of a kernel group, from the committed
    ncu --set full capture (one round: each kernel of the group once)."""
    try:
        rows = json.loads(NCU_FULL.read_text())
    except (OSError, ValueError):
        return None, None, None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    want = {k: 2 if k == "k_tet_jacobi2" else 1 for k in KGROUPS.get(group, [])}   # launches per round
    seen, traffic, flop = {}, 0.0, 0.0
    for d in rows:
        k = d["kernel"].split("::")[-1]
        if seen.get(k, 0) >= want.get(k, 0):
            continue
        seen[k] = seen.get(k, 0) + 1
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, unit = d[m].split()
            traffic += float(v.replace(",", "")) * scale[unit]
        flop += d.get("fp64_flop", 0.0)
    if not seen:
        return None, None, None
    return traffic, flop, f"{NCU_FULL.relative_to(ROOT)} (ncu --set full, one round)"


def _fp64_peak():
    """fp64 DFMA peak: the microbenchmark (tools/fp64_peak.cu) run live, else its committed B200 run."""
    exe = ROOT / "build" / "fp64_peak"
    if exe.exists():
        try:
            out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60).stdout
            return float(json.loads(out)["fp64_tflops"]), "measured live (tools/fp64_peak.cu)"
        except Exception:
            pass
    try:
        d = json.loads((ROOT / "profiles" / "fp64_peak_b200.json").read_text())
        return float(d["fp64_tflops"]), "profiles/fp64_peak_b200.json (tools/fp64_peak.cu on B200)"
    except (OSError, ValueError, KeyError):
        return None, None


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.rows.append([c.strip() for c in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 7 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 7 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows if len(r) > 7 for n, v in zip(names, r[4:8]) if v.strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU side (oracle port): bounded sample of the same workload on the host cores
# ---------------------------------------------------------------------------


def _cpu_worker(args):
    """One env through W untimed + K timed protocol steps with the oracle; returns timings."""
    i, warmup, steps = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import solver as osv   # CPU baseline leg only
    from paper_2503_05020_b200 import scene as sc
    s = sc.cfg2_scene(i % 400)
    env = osv.OracleEnv(s.bodies, collide_pairs_off=s.collide_pairs_off)
    sm = _OracleProtocol(env, s)
    for _ in range(warmup):
        if not sm.advance():
            break
    t0 = time.perf_counter()
    n = 0
    calls = 0
    for _ in range(steps):
        c0 = getattr(env, "n_calls", 0)
        if not sm.advance():
            break
        calls += getattr(env, "n_calls", 0) - c0
        n += 1
    return n, time.perf_counter() - t0, calls


class _OracleProtocol:
    """The protocol state machine (protocol.py:152-277) driving one oracle env."""

    def __init__(self, env, scene, halt=50.0, speed=0.05):
        self.env, self.s = env, scene
        self.phase, self.k, self.g, self.quiet = 0, 0, 0, 0
        self.halted = {f: False for f in scene.finger_links}
        dt = env.dt
        self.n = [int(np.ceil(0.05 / dt)), int(np.ceil((scene.opening / 2.0) / (speed * dt))) + 5,
                  int(np.ceil(1.0 / dt)), int(np.ceil(0.1 / dt))]
        self.halt, self.speed = halt, speed

    def advance(self):
        from oracle import solver as osv
        env, s = self.env, self.s
        if self.phase >= 4:
            return False
        if env.status != "active":
            return False
        rep = env.step()
        ev = env.events_now()
        forces = {f: osv.finger_force(ev, ids) for f, ids in s.finger_links.items()}
        self.k += 1
        if self.phase == 1:
            for f, ids in s.finger_links.items():
                if not self.halted[f] and forces[f] > self.halt:
                    self.halted[f] = True
                    for b in ids:
                        env.bodies[b].velocity = np.zeros(3)
        if rep["status"] == "failed":
            self.phase = 4
            return True
        end = False
        if self.phase == 0:
            end = self.k >= self.n[0]
        elif self.phase == 1:
            end = all(self.halted.values()) or self.k >= self.n[1]
        elif self.phase == 2:
            self.quiet = self.quiet + 1 if env.max_point_speed() < env.eps_v else 0
            end = self.quiet >= 5 or self.k >= self.n[2]
        else:
            end = self.k >= self.n[3]
        if end:
            self.k = 0
            if self.phase == 0:
                for f, ids in s.finger_links.items():
                    for b in ids:
                        env.bodies[b].velocity = np.asarray(s.closing_dirs[f]) * self.speed
                self.phase = 1
            elif self.phase == 1:
                for ids in s.finger_links.values():
                    for b in ids:
                        env.bodies[b].velocity = np.zeros(3)
                self.phase = 2
            elif self.phase == 2:
                self.phase, self.g = 3, 0
                env.gravity = 9.8 * np.array([1.0, 0, 0])
            else:
                self.g += 1
                if self.g >= 6:
                    self.phase = 4
                else:
                    d = np.zeros(3)
                    d[self.g // 2] = 1.0 if self.g % 2 == 0 else -1.0
                    env.gravity = 9.8 * d
        return True


def cpu_measure(n_envs, warmup, steps, cores):
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        res = pool.map(_cpu_worker, [(i, warmup, steps) for i in range(n_envs)], chunksize=1)
    wall = time.perf_counter() - t0
    n = sum(r[0] for r in res)
    busy = sum(r[1] for r in res)
    calls = sum(r[2] for r in res)
    # each worker is single threaded: aggregate rate = env-steps / (busy core-seconds / cores)
    rate = n / (busy / min(cores, n_envs)) if busy > 0 else 0.0
    return {"value": rate, "env_steps": n, "core_seconds": busy, "wall_s": wall, "newton_calls": calls,
            "ms_per_newton_iteration": 1e3 * busy / max(calls, 1)}


def run_reference(args, rank, world):
    """--impl reference: the oracle port of the reference path on all host cores."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    n_envs = cores
    t_all = time.perf_counter()
    # each worker runs one env's full protocol trial (capped at 150 steps): the same phase mix
    # as the GPU's steady state; W / K are reported but the sample is the bounded trial set
    r = cpu_measure(n_envs, 0, min(args.steps, 150), cores)
    steps_done = r["env_steps"]
    value = r["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * r["core_seconds"] / max(args.steps, 1) / max(min(cores, n_envs), 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2: soft 2-pad gripper on rigid box/cylinder/sphere, full grasp protocol",
                   "envs": n_envs, "sample": f"{n_envs} envs, full protocol trials (<= {min(args.steps, 150)} steps)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(cores, n_envs), "kind": "port",
                         "sample": f"oracle/ numpy port, {n_envs} envs, {steps_done} env-steps, "
                                   f"{r['ms_per_newton_iteration']:.1f} ms per newton_iteration"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t_all,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=300)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--envs", type=int, default=ENVS_PER_GPU, help="envs per GPU")
    ap.add_argument("--cpu-envs", type=int, default=0, help="CPU baseline sample envs (0 = host cores)")
    ap.add_argument("--cpu-steps", type=int, default=150, help="CPU baseline: max protocol steps per env (full trial)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--lockstep", action="store_true", help="lockstep Batch.step rounds instead of continuous batching")
    ap.add_argument("--record", default=None, help="record every trial (frames, stress, contact events) and "
                                                   "emit it to this directory in the reference's dataset format")
    ap.add_argument("--protocol", default="device", choices=["host", "device"],
                    help="grasp-protocol state machine on the host (per round) or on the device (k_protocol)")
    ap.add_argument("--rounds-per-call", type=int, default=4, help="device protocol: rounds per host call")
    ap.add_argument("--lane-priority", default="0,1,2",
                    help="stream priority per object kind (box, cylinder, sphere): the heavier envs first")
    ap.add_argument("--only-kind", type=int, default=-1, help="diagnostic: run only the lanes of this object kind")
    ap.add_argument("--lanes", type=int, default=3,
                    help="1: one device batch; 3k: k device batches (own stream + host thread) per object kind")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.record is not None or args.lockstep:
        args.protocol = "host"   # recording and lockstep rounds drive the host state machine
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2503_05020_b200 import scene as sc
    from paper_2503_05020_b200.multienv import DeviceEnvGroup
    from paper_2503_05020_b200.protocol import BatchedGraspTrials
    from paper_2503_05020_b200.solver import Environment

    cands = sc.load_cfg2_candidates()
    ids = [rank * args.envs + i for i in range(args.envs)]       # weak scaling: 400 envs per GPU
    kinds = np.asarray(cands["kind"])
    slot_kind = np.array([kinds[i % 400] for i in ids])
    # lanes: one device batch (own CUDA stream, own host thread) per object kind, so the light
    # box / cylinder envs are not held at every kernel boundary by the heavy sphere envs; --lanes 1
    # puts all envs of this rank in one batch
    if args.lanes == 1:
        lane_ids = [ids]
    else:
        per_kind = max(1, args.lanes // 3)
        lane_ids = []
        for kk in range(3):
            of_kind = [i for i, k in zip(ids, slot_kind) if k == kk]
            lane_ids += [of_kind[j::per_kind] for j in range(per_kind)]
        lane_ids = [l for l in lane_ids if l]
        if args.only_kind >= 0:   # diagnostic: one kind's lane(s) alone
            lane_ids = [l for l in lane_ids if slot_kind[ids.index(l[0])] == args.only_kind]
    payloads = {j: BatchedGraspTrials.scene_payload(sc.cfg2_scene(j, cands)) for j in range(400)}  # outside timing
    queue = {k: [j for j in range(400) if kinds[j] == k] for k in range(3)}
    qlock = threading.Lock()
    qpos = {k: 0 for k in range(3)}

    class Lane:
        def __init__(self, lids):
            scenes = [sc.cfg2_scene(i % 400, cands) for i in lids]
            envs = [Environment(s.bodies, collide_pairs_off=s.collide_pairs_off) for s in scenes]
            self.group = DeviceEnvGroup(envs, device=local)
            self.device = args.protocol == "device"
            if self.device:
                from paper_2503_05020_b200.protocol import DeviceProtocolTrials
                self.trials = DeviceProtocolTrials(self.group, scenes)
            else:
                self.trials = BatchedGraspTrials(self.group, scenes, record=args.record is not None)
            self.dev = self.group.dev
            self.kind = np.array([kinds[i % 400] for i in lids])
            self.done_trials = []
            self.advance = None if self.device else (self.trials.advance if args.lockstep else self.trials.advance_round)
            self.env_steps = 0
            self.rounds = 0
            self.h2d = self.d2h = 0

        def refill_device(self):
            out = self.trials.dev.protocol_read()
            E, B = self.group.packed.n_env, self.group.packed.n_body_total
            rec = 4 * 39 + 8 * 19                                  # per-env protocol state (GripTrialOut source)
            self.d2h += rec * E
            fin = [e for e in range(len(out)) if out[e].phase == 4]
            if not fin:
                return
            p = self.group.packed
            for e in fin:                                        # grip_reset_envs slices of the new candidate
                self.h2d += 8 * (3 * (p.node_off[e + 1] - p.node_off[e]) + 3 * (p.sv_off[e + 1] - p.sv_off[e])
                                 + 10 * (p.tet_off[e + 1] - p.tet_off[e]))
            self.h2d += (rec + 24) * E + 24 * B                    # grip_protocol_reset round trip
            self.d2h += (rec + 24) * E + 24 * B
            pls = []
            with qlock:
                for e in fin:
                    self.done_trials.append(self.trials.record(e, out).verdict)
                    k = int(self.kind[e])
                    pls.append(payloads[queue[k][qpos[k] % len(queue[k])]])
                    qpos[k] += 1
            self.trials.refill(fin, pls)

        def refill(self):
            if self.device:
                return self.refill_device()
            fin = np.nonzero(self.trials.phase == 4)[0]
            if len(fin) == 0:
                return
            pls = []
            with qlock:
                for e in fin:
                    self.done_trials.append(self.trials.records[e].verdict)
                    if writer is not None:
                        writer.put(self.trials.records[e])
                    k = int(self.kind[e])
                    pls.append(payloads[queue[k][qpos[k] % len(queue[k])]])
                    qpos[k] += 1
            self.trials.refill(fin, pls)

        def round(self):
            t0 = time.perf_counter()
            self._round()
            self.call_ms_max = max(getattr(self, "call_ms_max", 0.0), 1e3 * (time.perf_counter() - t0))

        def _round(self):
            t0 = time.perf_counter()
            if self.device:   # R device rounds per host call, protocol decisions on the device
                n = self.trials.advance(args.rounds_per_call)
                self.rounds += args.rounds_per_call
                self.d2h += 8 + 4 * self.group.packed.n_env       # env-step counter, overflow flags
            else:
                n = self.advance()
                self.rounds += 1
            t1 = time.perf_counter()
            self.refill()
            self.t_step = getattr(self, "t_step", 0.0) + t1 - t0
            self.t_refill = getattr(self, "t_refill", 0.0) + time.perf_counter() - t1
            self.env_steps += n

    writer = None
    if args.record is not None:
        # dataset emission: finished trials go to a writer thread (dataset.py)
        import queue as queue_mod
        from paper_2503_05020_b200 import dataset as ds
        writer = queue_mod.Queue()
        out_dir = Path(args.record)
        n_written = [0]

        def write_loop():
            while True:
                rec = writer.get()
                if rec is None:
                    return
                ds.emit_trial(rec, out_dir / f"trial_{n_written[0]:05d}")
                n_written[0] += 1

        wthread = threading.Thread(target=write_loop, daemon=True)
        wthread.start()
    lanes = [Lane(l) for l in lane_ids]
    if args.lane_priority:   # e.g. "0,1,2": box, cylinder, sphere lanes
        pr = [int(v) for v in args.lane_priority.split(",")]
        for ln in lanes:
            ln.dev.set_priority(pr[int(ln.kind[0])] if len(pr) > int(ln.kind[0]) else 0)

    def run_lanes(n_rounds, timed):
        """Every lane runs rounds on its own thread; the lane with the most envs runs exactly
        n_rounds, the others keep going until it is done (their streams stay busy)."""
        main_lane = max(range(len(lanes)), key=lambda i: len(lane_ids[i]))
        stop = threading.Event()

        errors = []

        def work(i):
            try:
                work_lane(i)
            except BaseException as exc:   # surface a lane's failure in the main thread
                errors.append(exc)
                stop.set()

        def work_lane(i):
            ln = lanes[i]
            if timed:
                ln.dev.timer_start()
            if i == main_lane:
                r0 = ln.rounds
                while ln.rounds - r0 < n_rounds:
                    ln.round()
                stop.set()
            else:
                while not stop.is_set():
                    ln.round()
            if timed:
                ln.ms = ln.dev.timer_stop()

        th = [threading.Thread(target=work, args=(i,)) for i in range(len(lanes))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errors:
            raise errors[0]

    run_lanes(args.warmup, False)
    for ln in lanes:
        ln.dev.set_profiling(True)
        ln.l0 = ln.dev.stats()[1]
        ln.sw0 = ln.dev.stats()[2]
        ln.env_steps = 0
        ln.rounds = 0
        ln.nd0 = len(ln.done_trials)
    h2d = d2h = 0
    if args.protocol == "host":
        for ln in lanes:
            E, B = ln.group.packed.n_env, ln.group.packed.n_body_total
            maxa = ln.dev.max_alpha
            h2d += 8 * 3 * E + 8 * 3 * B + 2 * E                                # gravity, body velocities, round masks
            d2h += 72 * E + 8 * maxa * E + (8 + 4) * B + 8 * E + 24 * B + 8 * E + E  # reports, alphas, forces+masks+min_d, com, speed, finalized
    for ln in lanes:
        ln.h2d = ln.d2h = 0
        ln.call_ms_max = 0.0
        ln.t_step = ln.t_refill = 0.0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        run_lanes(args.steps, True)
        wall = time.perf_counter() - t0
    torch.cuda.synchronize()
    ms = max(ln.ms for ln in lanes)
    if args.protocol == "device":   # counted: per bench step (round of the largest lane)
        h2d = sum(ln.h2d for ln in lanes) / max(args.steps, 1)
        d2h = sum(ln.d2h for ln in lanes) / max(args.steps, 1)
    env_steps = sum(ln.env_steps for ln in lanes)
    nsweeps = sum(ln.dev.stats()[2] - ln.sw0 for ln in lanes)
    launches = sum(ln.dev.stats()[1] - ln.l0 for ln in lanes)
    kss = [ln.dev.kernel_stats() for ln in lanes]
    ks = {}
    for name in kss[0]:
        ks[name] = {"ms": sum(k[name]["ms"] for k in kss), "launches": sum(k[name]["launches"] for k in kss)}
    ks["elements"]["units"] = {u: sum(k["elements"]["units"][u] for k in kss) for u in kss[0]["elements"]["units"]}
    env_iters = sum(k["elements"].get("env_iterations", 0.0) for k in kss)
    for f in ("pcg_iterations", "solves"):
        ks["assemble_pcg"][f] = sum(k["assemble_pcg"][f] for k in kss)
    ks["assemble_pcg"]["mean_unknowns"] = 0.0
    if world > 1:
        t = torch.tensor([ms, wall, float(env_steps), float(nsweeps)], dtype=torch.float64, device="cuda")
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm_ = t.clone()
        dist.all_reduce(sm_, op=dist.ReduceOp.SUM)
        ms_max, wall_max, total_steps = float(mx[0]), float(mx[1]), float(sm_[2])
    else:
        ms_max, wall_max, total_steps = ms, wall, float(env_steps)
    value = total_steps / (ms_max / 1e3)
    e2e = total_steps / wall_max
    # roofline of the dominant kernel group (live CUDA events per launch, this rank)
    dom = max((k for k in ks if k != "work_scan"), key=lambda k: ks[k]["ms"])
    peak, peak_kind = _peaks()
    roof = {"kernel": dom, "kernels": KGROUPS.get(dom, []), "bound": "hbm", "peak": peak, "unit": "GB/s",
            "peak_source": peak_kind, "traffic": None}
    u = ks["elements"]["units"]
    nlaunch = max(ks[dom]["launches"], 1)
    sec_per_launch = ks[dom]["ms"] / 1e3 / nlaunch
    if dom == "elements":
        alg = sum(EL_BYTES[k] * u[k] for k in EL_BYTES) / nlaunch
    elif dom == "assemble_pcg":
        # every element's Hessian, gradient and energy read once (1152 + 96 + 8 B)
        alg = 1256.0 * sum(u.values()) / nlaunch
    else:
        alg = None
    if alg is not None:
        roof["alg_bytes_per_launch"] = alg
        roof["achieved"] = alg / sec_per_launch / 1e9
        roof["frac"] = roof["achieved"] / peak
    else:
        roof["achieved"] = roof["frac"] = None
    traffic, flop, src = _ncu_group(dom)
    if traffic is not None:
        roof["traffic"] = traffic
        roof["traffic_source"] = src
        roof["traffic_note"] = ("ncu capture = one launch over a single 400-env batch (--lanes 1); "
                                f"the bench's launches cover {args.envs / len(lanes):.0f} envs each")
    fpk, fpk_src = _fp64_peak()
    if flop and fpk:
        roof["fp64"] = {"flop_per_launch": flop, "achieved_tflops": flop / sec_per_launch / 1e12, "peak_tflops": fpk,
                        "frac": flop / sec_per_launch / 1e12 / fpk, "peak_source": fpk_src,
                        "flop_source": "ncu (2 dfma + dadd + dmul thread instructions), " + (src or "")}
    roof["kernel_ms"] = {k: round(v["ms"], 3) for k, v in ks.items()}
    roof["kernel_launches"] = {k: v["launches"] for k, v in ks.items()}
    pk = ks["assemble_pcg"]
    roof["pcg"] = {"iterations_per_solve": pk["pcg_iterations"] / max(pk["solves"], 1.0),
                   "mean_unknowns": pk["mean_unknowns"], "solves": pk["solves"]}
    roof["element_counts"] = ks["elements"]["units"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2: soft 2-pad UMI-style gripper on rigid (ABD) box/cylinder/sphere, "
                               "full grasp protocol, antipodal candidate seed i",
                   "envs_per_gpu": args.envs, "global_envs": args.envs * world, "parallelism": f"env-shard x{world}",
                   "l2": "working set > L2 (element Hessians alone ~0.5 GB per GPU)",
                   "env_steps_timed": total_steps, "newton_sweeps": int(nsweeps),
                   "ms_per_newton_sweep": ms_max / max(nsweeps, 1),
                   # the metric's second half: one batched Newton iteration = one round of
                   # a lane over its active envs; env_iterations = newton_iteration calls of all envs
                   "newton": {"env_iterations_per_s": env_iters / (ms_max / 1e3),
                              "ms_per_batched_iteration": ms_max / max(args.steps, 1),
                              "envs_per_batched_iteration": env_iters / max(sum(ln.rounds for ln in lanes), 1),
                              "note": "profiling on: env_iterations counted in k_work_scan since set_profiling"},
                   "mode": ("lockstep Batch.step" if args.lockstep else "continuous batching, steady-state refill")
                           + (f", protocol on the device ({args.rounds_per_call} rounds per host call)"
                              if args.protocol == "device" else ", protocol on the host"),
                   "trials_completed_timed": sum(len(ln.done_trials) - ln.nd0 for ln in lanes),
                   "lanes": [{"envs": len(l), "rounds": ln.rounds, "env_steps": ln.env_steps, "ms": round(ln.ms, 3),
                              "max_call_ms": round(getattr(ln, "call_ms_max", 0.0), 2),
                              "host_refill_ms": round(1e3 * getattr(ln, "t_refill", 0.0), 1),
                              "step_call_ms": round(1e3 * getattr(ln, "t_step", 0.0), 1)}
                             for l, ln in zip(lane_ids, lanes)]},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "roofline": roof,
        "gpu_launches": int(launches),
        "recording": None if writer is None else {"dir": str(args.record), "trials_written": n_written[0],
                                                  "format": "gripsim-dataset-v1 (traj.bin, stress.bin, jsonl, meta)"},
        "clocks": clk.summary(),
    }
    if world > 1:
        # the path's one collective: fixed-size per-env outcome records, gathered once at the end
        from paper_2503_05020_b200.distributed import gather_outcomes, pack_outcomes
        tg = time.perf_counter()
        recs = {}
        for l, ln in zip(lane_ids, lanes):
            if ln.device:   # the device protocol's current trial records
                out = ln.trials.dev.protocol_read()
                recs.update({i: ln.trials.record(k, out) for k, i in enumerate(l)})
            else:
                recs.update({i: r for i, r in zip(l, ln.trials.records)})
        allr = gather_outcomes(pack_outcomes([recs[i] for i in ids], ids), args.envs * world, device="cuda")
        line["outcome_gather"] = {"envs": int(len(allr)), "ms": 1e3 * (time.perf_counter() - tg), "backend": "nccl"}
    if rank == 0 and not args.no_cpu:
        cores = os.cpu_count() or 1
        n_cpu = args.cpu_envs or cores
        r = cpu_measure(n_cpu, 0, args.cpu_steps, cores)
        line["cpu_baseline"] = {"value": r["value"], "unit": UNIT, "cores": min(cores, n_cpu), "kind": "port",
                                "sample": f"oracle/ numpy port of the reference step, {n_cpu} cfg2 envs, "
                                          f"full protocol trials (<= {args.cpu_steps} steps each), "
                                          f"{r['env_steps']} env-steps, {r['core_seconds']:.1f} core-s, "
                                          f"{r['ms_per_newton_iteration']:.1f} ms per newton_iteration"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
