"""Benchmark: env-steps/s of batched grasp trials (BASELINE configs 2-5) on B200.

Workload (BASELINE.json configs[1], the default): 400 environments per GPU, each a soft
UMI-style two-pad gripper grasping a rigid (ABD) box / cylinder / sphere (env i: kind i % 3,
the reference-sampled antipodal candidate of seed i), run through the reference's validation
protocol (settle, force-halted closing, hold, six gravity phases; protocol.py:152-277) by
``runner.TrialRunner``: three device batches ("lanes") per object kind, each with its own CUDA
streams and host thread, the protocol state machine on the device, one round per host call with
the next call already queued (pipelined), and every finished trial's slot refilled in place with
the rank's next candidate (dataset-generation steady state).
``--config 3`` runs 400 soft Neo-Hookean objects with kinematic fingers and the reference's
randomized material; ``--config 4`` 200 bimanual envs (two soft grippers, one soft object) with
the recorder's stress field output every step; ``--sweep`` the config-5 env-count sweep.

A bench "step" is ``--rounds-per-step`` (32) continuous-batching rounds of the lane with the most
envs (one round = one Newton sweep of every unfinished env plus begin / finalize / protocol for
the envs at a time-step boundary); the other lanes keep running until it is done.  Before the
W timed-out warm-up steps end, every slot must also have finished one trial (steady phase mix,
all buffers grown), whatever W says.  value = env time steps (solver.py:764-771 newton_step
calls) completed in the K timed steps / device time (CUDA events on each lane's stream, max over
lanes, max over ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2|3|4]

Also reported (one JSON line on rank 0): e2e (the same through the public runner API, host wall
clock, with every refill's candidate payload H2D and every trial readout D2H inside the timed
region), the north star's safety report (intersections, inverted elements, min distance, min J,
label / failure mix of the timed trials), the roofline of the dominant kernel group and a
whole-round byte model, and the CPU baseline: the UNMODIFIED reference (baseline/_ref gripsim)
timed on this host's cores on a bounded sample of the same workload (the oracle port if the
reference is not installed).
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os

# 9 runner lanes x 3 streams: 32 hardware work queues instead of the default 8 (before any CUDA use;
# the package sets the same default)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# 9 lane threads + the main thread per rank: sleep instead of spinning on a call's readout when the
# ranks' threads would outnumber the host cores
if int(os.environ.get("WORLD_SIZE", "1")) * 10 > (os.cpu_count() or 1):
    os.environ.setdefault("GRIP_BLOCKING_SYNC", "1")
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
REF_DIR = ROOT / "baseline" / "_ref"

WORKLOADS = {
    2: dict(envs=400, mode="device", lanes=3, workload="cfg2: soft 2-pad UMI-style gripper on rigid (ABD) box/cylinder/sphere, "
                                              "full grasp protocol, antipodal candidate seed i (kind i % 3)"),
    3: dict(envs=400, mode="device", lanes=6, workload="cfg3: soft Neo-Hookean box/sphere (kind i % 2) with kinematic fingers, "
                                              "randomized material (E log-uniform 1e4-1e7, mu 0.1-1), friction, full "
                                              "grasp protocol"),
    4: dict(envs=200, mode="host", lanes=5, workload="cfg4: bimanual, two soft 2-pad grippers on one soft cube (yaw i), full "
                                            "grasp protocol with 4 halting pads, recorder frames incl. stress field "
                                            "every step"),
}

# Algorithmic bytes per element of the element kernels (fp64 8 B, index 4 B; each input read once,
# each output written once): inputs + (E 8 + grad 96 + 12x12 Hessian 1152 + idx 16).
EL_OUT = 8 + 96 + 1152 + 16
EL_BYTES = {"tets": 16 + 96 + 72 + 24 + EL_OUT,        # node ids, 4 positions, Dm^-1, V0/mu/lam
            "affine": 96 + 8 + EL_OUT,                  # q, kappa*V
            "contacts": 16 + 4 + 96 + 8 + 8 + EL_OUT,   # row, code, 4 positions, rest lengths
            "anchors": 16 + 32 + 48 + 16 + 192 + EL_OUT}  # verts, gamma, T, lam/mu, x and x_prev
ASM_BYTES = 1256.0   # per element: its Hessian, gradient and energy read once by the assembly

# kernel groups as timed live (grip_kernel_stats) -> the kernels of the ncu capture; launches per round
# (k_tet_jacobi2 runs twice per round: the tets' launch on the second stream with the tet grid, the
# contacts' on the main stream with 148 blocks -- told apart by grid size in the capture)
KGROUPS = {"tets": {"k_tet_scan": 1, "k_tet_front": 1, "k_tet_jacobi2@tet": 1, "k_tet_back": 1},
           "elements": {"k_elements_w": 1, "k_tet_jacobi2@contact": 1, "k_tet_finish": 1},
           "assemble_pcg": {"k_contact_K": 1, "k_assemble_direct": 1}, "candidates": {"k_candidates": 1},
           "line_search": {"k_linesearch": 1}, "begin": {"k_begin": 1},
           "finalize": {"k_finalize": 1, "k_finalize_protocol": 1}}
EL_GROUP = {"tets": ("tets",), "elements": ("affine", "contacts", "anchors")}
NCU_FULL = [ROOT / "profiles" / "r2_ncu_full.json", ROOT / "profiles" / "r1_ncu_full_v5.json"]


# ---------------------------------------------------------------------------
# helpers: peaks, ncu capture, clocks
# ---------------------------------------------------------------------------


def _ncu_group(group):
    """DRAM read + write bytes and fp64 FLOPs per round of a kernel group (each kernel's average
    per launch in the committed ncu --set full capture x its launches per round), the capture's
    element units per round (for rescaling to the timed launches) and its source."""
    for path in NCU_FULL:
        try:
            doc = json.loads(path.read_text())
        except (OSError, ValueError):
            continue
        rows = doc["rows"] if isinstance(doc, dict) else doc
        meta = doc.get("meta", {}) if isinstance(doc, dict) else {"units_per_round": {"tets": 76800.0},
                                                                  "note": "one --lanes 1 round, 400 envs per launch"}
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        acc = {}
        for d in rows:
            k = d["kernel"].split("::")[-1].split("(")[0]
            if k == "k_tet_jacobi2":
                grid = int(float(str(d.get("launch__grid_size", "0")).split()[0].replace(",", "")))
                k += "@contact" if grid == 148 else "@tet"
            if k not in KGROUPS.get(group, {}):
                continue
            b = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v, unit = d[m].split()
                b += float(v.replace(",", "")) * scale[unit]
            a = acc.setdefault(k, [0, 0.0, 0.0])
            a[0] += 1
            a[1] += b
            a[2] += d.get("fp64_flop", 0.0)
        if not acc:
            continue
        w = KGROUPS[group]
        traffic = sum(w[k] * a[1] / a[0] for k, a in acc.items())
        flop = sum(w[k] * a[2] / a[0] for k, a in acc.items())
        return traffic, flop, meta, str(path.relative_to(ROOT))
    return None, None, None, None


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
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


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
# workloads: jobs (candidate indices), scenes, lane keys
# ---------------------------------------------------------------------------


def workload(cfg):
    """(valid candidate ids, scene_of(job), key_of(job), lane priority per key)."""
    from paper_2503_05020_b200 import scene as sc
    if cfg == 2:
        c = sc.load_cfg2_candidates()
        kinds = np.asarray(c["kind"])
        return (list(np.nonzero(c["ok"])[0]), (lambda j: sc.cfg2_scene(j, c)), (lambda j: int(kinds[j])),
                {0: 0, 1: 1, 2: 2})
    if cfg == 3:
        c = sc.load_cfg3_candidates()
        kinds = np.asarray(c["kind"])
        return list(np.nonzero(c["ok"])[0]), (lambda j: sc.cfg3_scene(j, c)), (lambda j: int(kinds[j])), {0: 0, 1: 1}
    if cfg == 4:
        return list(range(1 << 16)), (lambda j: sc.bimanual_scene(yaw=2.0 * np.pi * ((j * 0.6180339887498949) % 1.0))), \
            (lambda j: 0), {0: 0}
    raise ValueError(f"unknown config {cfg}")


def rank_jobs(pool, envs, world, rank, global_envs=None):
    """Jobs (candidate ids) of this rank.  Weak scaling: `envs` per rank, rank r takes the pool's
    candidates [r*envs, (r+1)*envs) (distinct across ranks while the pool lasts).  Strong
    scaling (global_envs): the contiguous shard of the first global_envs candidates."""
    from paper_2503_05020_b200.distributed import shard
    if global_envs:
        lo, hi = shard(global_envs, world, rank)
        return [int(pool[j % len(pool)]) for j in range(lo, hi)]
    return [int(pool[(rank * envs + i) % len(pool)]) for i in range(envs)]


# ---------------------------------------------------------------------------
# CPU side: the reference (baseline/_ref) or the oracle port, on the host cores
# ---------------------------------------------------------------------------

_CPU_COUNTER = None


def _ref_available():
    try:
        sys.path.insert(0, str(REF_DIR))
        import gripsim.pipeline.protocol  # noqa: F401
        return True
    except Exception:
        return False
    finally:
        if sys.path and sys.path[0] == str(REF_DIR):
            sys.path.pop(0)


def _ref_trial(args):
    """One full reference trial (pipeline/__init__.py:25-49 _validation_worker minus metrics): the
    reference's own build_trial_env + run_grasp_trial, unmodified; env.step is wrapped on the
    instance only to count completed env-steps into a shared counter."""
    cfg, j = args
    os.environ["OMP_NUM_THREADS"] = "1"
    sys.path.insert(0, str(REF_DIR))
    from gripsim.geometry import mesh as gm
    from gripsim.pipeline import config as rcfg
    from gripsim.pipeline import protocol as rproto
    from gripsim.synth import GraspCandidate
    from paper_2503_05020_b200 import scene as sc
    sc_ = rcfg.SceneConfig()
    override = None
    if cfg == 2:
        c = sc.load_cfg2_candidates()
        kind = [str(k) for k in c["kinds"]][int(c["kind"][j])]
        sc_.gripper.soft_fingers = True
        if kind == "cylinder":
            r, h, seg = c["cyl"]
            path = Path(f"/tmp/grip_bench_cyl_{os.getpid()}.obj")
            if not path.exists():
                gm.save_obj(gm.revolved_surface([(0.0, 0.0), (r, 0.0), (r, h), (0.0, h)], segments=int(seg),
                                                center=(0.0, 0.0, -0.5 * h)), path)
            sc_.object.kind, sc_.object.mesh_path = "mesh", str(path)
        else:
            sc_.object.kind = kind
    else:
        c = sc.load_cfg3_candidates()
        kind = [str(k) for k in c["kinds"]][int(c["kind"][j])]
        sc_.object.kind, sc_.object.soft = kind, True
        sc_.gripper.soft_fingers = False
        from gripsim.materials import MaterialParams
        override = MaterialParams(young_modulus=float(c["E"][j]), poisson_ratio=float(c["nu"][j]),
                                  density=float(c["rho"][j]), friction_coefficient=float(c["mu"][j]))
    cand = GraspCandidate("parallel", c["R"][j], c["T"][j], [c["opening"][j]], [])
    env, ob, fl = rcfg.build_trial_env(sc_, cand, env_id=j, material_override=override)
    step = env.step

    def counted():
        rep = step()
        with _CPU_COUNTER.get_lock():
            _CPU_COUNTER.value += 1
        return rep

    env.step = counted
    rec = rproto.run_grasp_trial(env, sc_.protocol, ob, fl)
    return rec.n_steps


def _port_trial(args):
    """The same trial through the oracle port (oracle/, the reference's algorithm restated)."""
    cfg, j = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import solver as osv   # CPU baseline leg only
    from paper_2503_05020_b200 import scene as sc
    s = sc.cfg2_scene(j) if cfg == 2 else sc.cfg3_scene(j)
    env = osv.OracleEnv(s.bodies, collide_pairs_off=s.collide_pairs_off)
    step = env.step

    def counted():
        rep = step()
        with _CPU_COUNTER.get_lock():
            _CPU_COUNTER.value += 1
        return rep

    env.step = counted
    sm = _OracleProtocol(env, s)
    while sm.advance():
        pass
    return sm.k


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
        if self.phase >= 4 or env.status != "active":
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


def _init_counter(counter):
    global _CPU_COUNTER
    _CPU_COUNTER = counter


def cpu_measure(cfg, jobs, seconds, cores, warm=5.0):
    """Steady-state CPU throughput: `cores` worker processes (fork, OMP_NUM_THREADS=1) run full
    trials of `jobs` back to back (more jobs than cores, so no core idles); every completed
    env-step bumps a shared counter.  After `warm` s the counter is read over `seconds` of wall
    time: env-steps / s on all cores, partial trials included, no tail effect."""
    use_ref = cfg in (2, 3) and _ref_available()
    fn = _ref_trial if use_ref else _port_trial
    ctx = mp.get_context("fork")
    counter = ctx.Value("q", 0)
    pool = ctx.Pool(cores, initializer=_init_counter, initargs=(counter,))
    res = pool.imap_unordered(fn, [(cfg, j) for j in jobs], chunksize=1)
    time.sleep(warm)
    c0, t0 = counter.value, time.perf_counter()
    time.sleep(seconds)
    c1, t1 = counter.value, time.perf_counter()
    pool.terminate()
    pool.join()
    del res
    return {"value": (c1 - c0) / (t1 - t0), "env_steps": int(c1 - c0), "wall_s": t1 - t0, "cores": cores,
            "kind": "reference" if use_ref else "port",
            "impl": "baseline/_ref gripsim 0.1.0 (unmodified): build_trial_env + run_grasp_trial" if use_ref
            else "oracle/ numpy port of the reference path"}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU path on all host cores, same config / metric."""
    if rank != 0:
        return
    cfg = 2 if args.config in (2, 5) else args.config
    cores = os.cpu_count() or 1
    seconds = float(min(120.0, max(20.0, 3.0 * args.steps)))
    pool, _, _, _ = workload(cfg) if cfg != 4 else (0, None, None, None)
    if cfg == 4:
        print(json.dumps({"impl": "reference", "unavailable": "config 4 (bimanual) has no reference trial driver"}))
        return
    jobs = rank_jobs(pool, WORKLOADS[cfg]["envs"], 1, 0)[:8 * cores]
    t_all = time.perf_counter()
    r = cpu_measure(cfg, jobs, seconds, cores)
    value = r["value"]
    sample = (f"{r['impl']}; {cores} worker processes, full protocol trials of bench candidates "
              f"{jobs[0]}..{jobs[-1]} back to back; env-steps counted over {r['wall_s']:.0f} s of wall time "
              f"after 5 s warm-up: {r['env_steps']} env-steps")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * r["wall_s"] / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[cfg]["workload"], "envs": len(jobs), "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": r["kind"], "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t_all,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------


def build_runner(args, cfg, envs, rank, world, writer=None):
    from paper_2503_05020_b200.runner import TrialRunner
    pool, scene_of, key_of, prio = workload(cfg)
    jobs = rank_jobs(pool, envs, world, rank, args.global_envs)
    mode = WORKLOADS[cfg]["mode"] if args.protocol == "auto" else args.protocol
    record = cfg == 4 or args.record is not None
    if record:
        mode = "host"
    on_record = None if writer is None else (lambda j, r: writer.put(j, r))
    lanes = args.lanes_per_kind or WORKLOADS[cfg]["lanes"]   # measured best per config
    runner = TrialRunner(jobs, scene_of, key_of, slots=None, lanes_per_key=lanes,
                         rounds_per_call=args.rounds_per_call, priority=prio if args.lane_priority else None,
                         cycle=True, device=None, mode=mode, record=record, on_record=on_record,
                         pipeline=not getattr(args, "no_pipeline", False))
    distinct = len(set(jobs)) == len(jobs) and bool(args.global_envs or (world * envs <= len(pool)))
    return runner, jobs, mode, bool(distinct)


def safety_report(trials, reasons):
    """The north star's report over the trials finished in the timed region: intersections
    (CCD / determinant / non-positive-distance failures, or a completed step at distance <= 0),
    inverted elements (inversion failures, or a completed step with J <= 0), min distance, min J,
    label and failure-reason mix (ccd.py:19, materials.py:125, solver.py:727-731)."""
    inter_reasons = {reasons[7], reasons[8], reasons[4]}
    inv_reasons = {reasons[3]}
    mix, fails = {}, {}
    inter = inv = 0
    md, mj = np.inf, np.inf
    for _, r in trials:
        mix[r.verdict] = mix.get(r.verdict, 0) + 1
        reason = r.failure.get("reason") if r.failure else None
        if reason:
            fails[reason] = fails.get(reason, 0) + 1
        inter += int(reason in inter_reasons or r.min_distance <= 0.0)
        inv += int(reason in inv_reasons or r.min_J <= 0.0)
        md, mj = min(md, r.min_distance), min(mj, r.min_J)
    return {"trials": len(trials), "intersections": inter, "inverted_elements": inv,
            "min_distance_m": None if not np.isfinite(md) else md, "min_J": None if not np.isfinite(mj) else mj,
            "verdicts": mix, "failure_reasons": fails,
            "source": "device protocol records (k_finalize: min stencil distance, min det F / det A per step)"}


def kernel_report(runner, env_steps_s, ms_max, peak):
    """Per-group device time, the roofline of the dominant group and a whole-round byte model."""
    lanes = runner.lanes
    kss = [ln.dev.kernel_stats() for ln in lanes]
    ks = {}
    for name in kss[0]:
        ks[name] = {"ms": sum(k[name]["ms"] for k in kss), "launches": sum(k[name]["launches"] for k in kss)}
    units = {u: sum(k["elements"]["units"][u] for k in kss) for u in kss[0]["elements"]["units"]}
    env_iters = sum(k["elements"].get("env_iterations", 0.0) for k in kss)
    dom = max((k for k in ks if k != "work_scan"), key=lambda k: ks[k]["ms"])
    roof = {"kernel": dom, "kernels": list(KGROUPS.get(dom, {})), "bound": "hbm", "peak": peak[0], "unit": "GB/s",
            "peak_source": peak[1], "traffic": None}
    nl = max(ks[dom]["launches"], 1)
    sec_per_launch = ks[dom]["ms"] / 1e3 / nl
    el_alg = sum(EL_BYTES[k] * units[k] for k in EL_BYTES)
    alg = {g: sum(EL_BYTES[k] * units[k] for k in ks_) for g, ks_ in EL_GROUP.items()}
    alg["assemble_pcg"] = ASM_BYTES * sum(units.values())
    alg = alg.get(dom)
    if alg is not None:
        roof["alg_bytes_per_launch"] = alg / nl
        roof["achieved"] = alg / nl / sec_per_launch / 1e9
        roof["frac"] = roof["achieved"] / peak[0]
    else:
        roof["achieved"] = roof["frac"] = None
    traffic, flop, meta, src = _ncu_group(dom)
    if traffic is not None:
        # the capture's per-round figures rescaled to the timed launches by element units per launch
        cap_units = sum(((meta or {}).get("units_per_round") or {}).values()) or None
        timed_units = sum(units.values()) / nl if dom in ("elements", "tets", "assemble_pcg") else None
        s = (timed_units / cap_units) if (cap_units and timed_units) else 1.0
        roof["traffic"] = traffic * s
        roof["traffic_source"] = src
        roof["traffic_scale"] = {"capture_units_per_launch": cap_units, "timed_units_per_launch": timed_units,
                                 "factor": s, "note": (meta or {}).get("note")}
        fpk, fpk_src = _fp64_peak()
        if flop and fpk:
            f = flop * s
            roof["fp64"] = {"flop_per_launch": f, "achieved_tflops": f / sec_per_launch / 1e12, "peak_tflops": fpk,
                            "frac": f / sec_per_launch / 1e12 / fpk, "peak_source": fpk_src,
                            "flop_source": "ncu (2 dfma + dadd + dmul thread instructions), " + src}
    roof["kernel_ms"] = {k: round(v["ms"], 3) for k, v in ks.items()}
    roof["kernel_launches"] = {k: v["launches"] for k, v in ks.items()}
    roof["element_counts"] = units
    # whole-round algorithmic bytes (SURVEY §8d's per-kernel figures with the counts this run has):
    # elements + assembly exact from the element counters; broad phase 2 x (24 N_sv + 12 N_tri +
    # 8 N_e) and line search / begin / finalize 200 N_t + 72 N_n (one energy pass) + 48 B per node,
    # per env-iteration, from each lane's mean env sizes
    other = 0.0
    for ln, k in zip(lanes, kss):
        p = ln.group.packed
        E = max(p.n_env, 1)
        nsv, ntri, ne = p.n_sv_total / E, float(p.tri_off[-1]) / E, float(p.edge_off[-1]) / E
        nt, nn = p.n_tet_total / E, p.n_node_total / E
        it = k["elements"].get("env_iterations", 0.0)
        other += it * (2 * (24 * nsv + 12 * ntri + 8 * ne) + 200 * nt + 72 * nn + 48 * nn)
    total = el_alg + ASM_BYTES * sum(units.values()) + other
    roof["round_model"] = {"alg_bytes": total, "device_ms": ms_max, "achieved_gbs": total / (ms_max / 1e3) / 1e9,
                           "frac": total / (ms_max / 1e3) / 1e9 / peak[0], "env_iterations": env_iters,
                           "parts_bytes": {"elements": el_alg, "assembly": ASM_BYTES * sum(units.values()),
                                           "broad_phase+line_search+begin/finalize": other}}
    return roof, ks, env_iters


def gather_timed(timed, rank, world, dist, record_dir, reasons, device=None):
    """The path's one collective: every rank's finished trials (job, TrialRecord) as fixed-size
    outcome rows, all-gathered once at the end (NCCL on the GPU box, gloo in the CPU test);
    with recording, rank 0 then merges the rank-local dataset shard manifests."""
    from paper_2503_05020_b200.distributed import gather_outcomes, merge_manifests, pack_outcomes
    tg = time.perf_counter()
    allr = gather_outcomes(pack_outcomes([r for _, r in timed], [j for j, _ in timed], rank=rank, reasons=reasons),
                           device=device)
    out = {"trials": int(len(allr)), "ms": 1e3 * (time.perf_counter() - tg),
           "backend": dist.get_backend() if dist is not None else None,
           "ranks": sorted({int(x) for x in allr[:, 12]}) if len(allr) else [],
           "verdicts": {v: int((allr[:, 1] == k).sum()) for k, v in enumerate(("stable", "unstable", "sim-failed"))}}
    if record_dir is not None and dist is not None:
        dist.barrier()
        if rank == 0:
            from paper_2503_05020_b200 import dataset as ds
            out["merged_trials"] = merge_manifests(record_dir, world, ds.FORMAT)["n_trials"]
    return out


def run_gpu(args, rank, world, local, cfg, envs, dist=None, quiet=False):
    import torch
    from paper_2503_05020_b200._native import REASONS
    writer = None
    if args.record is not None:
        from paper_2503_05020_b200 import dataset as ds
        from paper_2503_05020_b200.distributed import rank_dir
        writer = ds.ShardWriter(rank_dir(args.record, rank), params={"config": cfg})
    t_build = time.perf_counter()
    runner, jobs, mode, distinct = build_runner(args, cfg, envs, rank, world, writer)
    build_s = time.perf_counter() - t_build
    rps = args.rounds_per_step
    cps = max(1, rps // args.rounds_per_call) if mode == "device" else rps
    # warm-up: W steps, and at least every slot through one trial (steady phase mix, buffers grown)
    t_w = time.perf_counter()
    runner.run(main_calls=args.warmup * cps, min_trials=runner.n_slots)
    warm_s = time.perf_counter() - t_w
    warm_trials = len(runner.finished_order)
    runner.reset_stats()
    runner.set_profiling(True)
    l0 = [ln.dev.stats()[1] for ln in runner.lanes]
    n0 = len(runner.finished)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        runner.run(main_calls=args.steps * cps, timed=True)
        wall = time.perf_counter() - t0
    torch.cuda.synchronize()
    st = [ln.stats for ln in runner.lanes]
    ms = max(s.device_ms for s in st)
    env_steps = sum(s.env_steps for s in st)
    launches = sum(ln.dev.stats()[1] - a for ln, a in zip(runner.lanes, l0))
    if dist is not None:
        t = torch.tensor([ms, wall, float(env_steps)], dtype=torch.float64, device="cuda")
        mx, sm_ = t.clone(), t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm_, op=dist.ReduceOp.SUM)
        ms_max, wall_max, total_steps = float(mx[0]), float(mx[1]), float(sm_[2])
    else:
        ms_max, wall_max, total_steps = ms, wall, float(env_steps)
    value = total_steps / (ms_max / 1e3)
    e2e = total_steps / wall_max
    roof, ks, env_iters = kernel_report(runner, env_steps, ms, _peaks())
    timed = runner.finished[n0:]
    h2d = sum(s.h2d_bytes for s in st) / max(args.steps, 1)
    d2h = sum(s.d2h_bytes for s in st) / max(args.steps, 1)
    main = runner.main_lane
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.global_envs else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[cfg]["workload"], "config": cfg, "envs_per_gpu": runner.n_slots,
                   "global_envs": args.global_envs or envs * world, "parallelism": f"env-shard x{world}",
                   "distinct_candidates_across_ranks": distinct,
                   "l2": "inputs > L2: working set ~1.3 GB per 400 envs (element Hessians alone ~0.5 GB)",
                   "step": f"{rps} continuous-batching rounds of the largest lane",
                   "protocol": "device (k_protocol), %d rounds per host call" % args.rounds_per_call
                               if mode == "device" else "host (BatchedGraspTrials), one round per host call",
                   "lanes": [{"key": int(ln.key), "slots": s.slots, "calls": s.calls, "rounds": s.rounds,
                              "env_steps": s.env_steps, "trials_done": s.trials_done, "device_ms": round(s.device_ms, 2),
                              "max_call_ms": round(s.max_call_ms, 2), "host_refill_ms": round(1e3 * s.refill_s, 1),
                              "host_step_ms": round(1e3 * s.step_s, 1)} for ln, s in zip(runner.lanes, st)],
                   "env_steps_timed": total_steps, "trials_completed_timed": len(timed),
                   "warmup": {"trials": warm_trials, "s": round(warm_s, 2), "build_s": round(build_s, 2)},
                   # the metric's second half: one batched Newton iteration = one round of
                   # the largest lane over its active envs; env_iterations = newton_iteration calls
                   "newton": {"env_iterations_per_s": env_iters / (ms / 1e3),
                              "ms_per_batched_iteration": ms / max(st[main].rounds, 1),
                              "envs_per_batched_iteration": env_iters / max(sum(s.rounds for s in st), 1)}},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "what": "TrialRunner.run (public API) wall clock: every refill's candidate payload H2D (pinned "
                        "staging) and every call's trial-record readout D2H inside the timed region"},
        "safety": safety_report(timed, REASONS),
        "roofline": roof,
        "gpu_launches": int(launches),
        "recording": None,
        "clocks": clk.summary(),
    }
    if writer is not None:
        man = writer.close()
        line["recording"] = {"dir": str(args.record), "rank_trials": man["n_trials"],
                             "format": "gripsim-dataset-v1 (traj.bin, stress.bin, jsonl, meta), per-rank shards"}
    if dist is not None:
        line["outcome_gather"] = gather_timed(timed, rank, world, dist, args.record, REASONS, device="cuda")
        if line["recording"] is not None and "merged_trials" in line["outcome_gather"]:
            line["recording"]["merged_trials"] = line["outcome_gather"].pop("merged_trials")
    return line, jobs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5],
                    help="BASELINE configs[config-1]; 5 = the env-count sweep of config 2 (see --sweep)")
    ap.add_argument("--envs", type=int, default=0, help="envs per GPU (default: the config's)")
    ap.add_argument("--global-envs", type=int, default=0, help="strong scaling: total envs split over the ranks")
    ap.add_argument("--sweep", default="", help="config 5: comma-separated env counts, one JSON line each")
    ap.add_argument("--rounds-per-step", type=int, default=32)
    ap.add_argument("--rounds-per-call", type=int, default=1, help="device protocol: rounds per host call")
    ap.add_argument("--lanes-per-kind", type=int, default=0,
                    help="device batches per object kind (default: the config's measured best, 3 / 6 / 5)")
    ap.add_argument("--no-pipeline", action="store_true", help="device protocol: wait for each call before "
                    "enqueuing the next (no host / device overlap)")
    ap.add_argument("--no-lane-priority", dest="lane_priority", action="store_false")
    ap.add_argument("--protocol", default="auto", choices=["auto", "host", "device"])
    ap.add_argument("--record", default=None, help="record every trial and emit it here (dataset format), "
                                                    "rank-local shards + merged manifest")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as tdist
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist
    if args.config == 5 or args.sweep:
        counts = [int(v) for v in (args.sweep or "1,2,4,8,16,32,64,128,256,400,800,1600,3200").split(",")]
        for n in counts:
            line, _ = run_gpu(args, rank, world, local, 2, n, dist)
            line["config"]["sweep"] = True
            line["vs_baseline"] = None
            if rank == 0:
                print(json.dumps(line), flush=True)
        if dist is not None:
            dist.destroy_process_group()
        return
    cfg = args.config
    envs = args.envs or WORKLOADS[cfg]["envs"]
    line, jobs = run_gpu(args, rank, world, local, cfg, envs, dist)
    if rank == 0 and not args.no_cpu and cfg in (2, 3):
        cores = os.cpu_count() or 1
        r = cpu_measure(cfg, jobs[:8 * cores], args.cpu_seconds, cores)
        line["cpu_baseline"] = {"value": r["value"], "unit": UNIT, "cores": cores, "kind": r["kind"],
                                "sample": f"{r['impl']}; {cores} worker processes, full protocol trials of this "
                                          f"rank's candidates back to back, env-steps counted over "
                                          f"{r['wall_s']:.0f} s after 5 s warm-up: {r['env_steps']} env-steps"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
