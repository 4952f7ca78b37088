"""Grasp-trial generation on one GPU: many trials, few device batches, continuous slot refill.

The reference validates a candidate list by ``validate_candidates`` (pipeline/__init__.py:51-70):
one ``_validation_worker`` trial per candidate, fanned out over a fork pool by
``run_batch_trials`` (multienv.py:204-216), each trial a full ``run_grasp_trial``
(protocol.py:152-277) on its own Environment.  Here the trials of one GPU share a few device
batches ("lanes"): a lane is one ``DeviceEnvGroup`` of ``slots`` environments with the protocol
state machine on the device (``DeviceProtocolTrials``, ``grip_run_rounds``), its own CUDA stream
and its own host thread.  When a slot's trial ends, its record is collected and the slot is
re-initialised in place (``grip_reset_envs`` + ``grip_protocol_reset``) with the next candidate of
the lane's queue, so the batch stays full without rebuilding anything.

Lanes are keyed by topology (a refill must keep the slot's meshes; e.g. the object kind): every
job of a key goes to that key's lanes.  Results are per job and independent of the lane layout,
slot count and refill order (every slot reset returns the env to a fresh state, which the GPU
tests check bitwise), so the same records come out of 1 lane of 400 slots or 3 lanes of 40.

Each host call runs one device round and is pipelined: the lane enqueues the next call
(``grip_run_rounds_async``) before it waits for the previous one's readout (``grip_rounds_wait``),
so recording finished trials and refilling their slots overlaps the device; refills queue behind
the call in flight, whose readout then predates them (those slots are skipped once).

``cycle=True`` wraps each key's queue around (steady-state throughput: the bench); otherwise a
lane stops once its queue is empty and all its slots are idle.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field

import numpy as np

from paper_2503_05020_b200.multienv import AssetCache, DeviceEnvGroup
from paper_2503_05020_b200.protocol import BatchedGraspTrials, DeviceProtocolTrials
from paper_2503_05020_b200.solver import Environment


@dataclass
class LaneStats:
    slots: int = 0
    calls: int = 0
    rounds: int = 0
    env_steps: int = 0
    trials_done: int = 0
    device_ms: float = 0.0
    step_s: float = 0.0
    refill_s: float = 0.0
    max_call_ms: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0


class Lane:
    """One device batch of `slots` environments fed from a job queue (see module docstring)."""

    def __init__(self, runner, key, jobs, n_slots, device, priority):
        self.runner, self.key = runner, key
        self.queue = list(jobs)
        self.qpos = 0
        first = [self._next_job() for _ in range(n_slots)]
        first = [j for j in first if j is not None]
        scenes = [runner.scene(j) for j in first]
        envs = [Environment(s.bodies, collide_pairs_off=s.collide_pairs_off) for s in scenes]
        self.group = DeviceEnvGroup(envs, device=device)
        self.dev = self.group.dev
        self.mode = runner.mode
        if self.mode == "device":
            self.trials = DeviceProtocolTrials(self.group, scenes, runner.protocol)
        else:
            self.trials = BatchedGraspTrials(self.group, scenes, runner.protocol, record=runner.record)
        if priority:
            self.dev.set_priority(priority)
        self.slot_job = list(first)
        self.stats = LaneStats(slots=len(first))
        self.started = [True] * len(first)
        self._stop = False
        self.pending = None   # ticket of the device call in flight (pipelined runner)
        self.stale = set()    # slots refilled behind the call in flight: its readout predates the refill

    def _next_job(self):
        if self.qpos >= len(self.queue):
            if not self.runner.cycle or not self.queue:
                return None
            self.qpos = 0
        j = self.queue[self.qpos]
        self.qpos += 1
        return j

    @property
    def idle(self):
        return all(j is None for j in self.slot_job)

    def call(self, last=False):
        """One host call: R device rounds (device protocol) or one round (host protocol), then
        collect the finished trials and refill their slots.

        Pipelined (device protocol, runner.pipeline): the next call's rounds are enqueued before
        this call's results are waited for, so the host's collect-and-refill overlaps the
        device; refills queue behind the call in flight (a finished slot idles one call longer).
        last: complete the call in flight without enqueuing another."""
        r = self.runner
        t0 = time.perf_counter()
        out = None
        if self.mode == "device":
            E = self.group.packed.n_env
            if r.pipeline:
                if self.pending is None:
                    self.pending = self.trials.advance_async(r.rounds_per_call)
                nxt = None if last else self.trials.advance_async(r.rounds_per_call)
                n, out = self.trials.wait(self.pending)
                self.pending = nxt
                skip, self.stale = self.stale, set()
                self.stats.d2h_bytes += 192 * E                     # the call's protocol records
            else:
                n = self.trials.advance(r.rounds_per_call)
                skip = set()
            self.stats.rounds += r.rounds_per_call
            self.stats.d2h_bytes += 8 + 4 * E                       # env-step counter, overflow flags
        else:
            n = self.trials.advance_round()
            self.stats.rounds += 1
            skip = set()
        t1 = time.perf_counter()
        refilled = self._collect_and_refill(out, skip)
        if self.pending is not None:
            self.stale = set(refilled)
        t2 = time.perf_counter()
        self.stats.calls += 1
        self.stats.env_steps += int(n)
        self.stats.step_s += t1 - t0
        self.stats.refill_s += t2 - t1
        self.stats.max_call_ms = max(self.stats.max_call_ms, 1e3 * (t2 - t0))

    def drain(self):
        """Complete the pipelined call in flight (its trials are collected and refilled)."""
        if self.pending is not None:
            self.call(last=True)

    def _collect_and_refill(self, out=None, skip=()):
        """Finished trials of the readout `out` (slots in `skip` excluded: their readout predates
        a refill) are recorded and their slots refilled; returns the refilled slots."""
        r = self.runner
        if self.mode == "device":
            E = self.group.packed.n_env
            if out is None:
                out = self.trials.dev.protocol_read()
                self.stats.d2h_bytes += 192 * E
            fin = [e for e in range(E) if out[e].phase == 4 and self.slot_job[e] is not None and e not in skip]
            recs = {e: self.trials.record(e, out) for e in fin}
        else:
            fin = [int(e) for e in np.nonzero(self.trials.phase == 4)[0] if self.slot_job[e] is not None]
            recs = {e: self.trials.records[e] for e in fin}
        if not fin:
            return []
        refill, payloads = [], []
        for e in fin:
            job = self.slot_job[e]
            r._finish(job, recs[e])
            self.stats.trials_done += 1
            nxt = self._next_job()
            self.slot_job[e] = nxt
            if nxt is not None:
                refill.append(e)
                payloads.append(r.payload(nxt))
        if refill:
            p = self.group.packed
            for e in refill:
                cnt = lambda off: int(getattr(p, off)[e + 1] - getattr(p, off)[e])  # noqa: E731
                # grip_reset_envs staging (x0, M, kin0, xi, Dm^-1, V0, mu, lam, body mu, rest lengths,
                # kappa V, cell hint + list / offset) and the protocol restart (closing dirs + 6 ints)
                self.stats.h2d_bytes += 8 * (12 * cnt("node_off") + 6 * cnt("sv_off") + 12 * cnt("tet_off")
                                             + cnt("body_off") + cnt("edge_off") + cnt("abd_off") + 1) + 12
                self.stats.h2d_bytes += 48 + 24
            self.trials.refill(refill, payloads)
        return refill


class TrialRunner:
    """Runs grasp trials for `jobs` on one GPU (see module docstring).

    jobs:        job ids (any hashable, e.g. candidate indices)
    scene_of:    job -> GraspScene (scene.build_trial_scene / cfg2_scene / ...)
    key_of:      job -> topology key; jobs of one key share lanes (refills keep topology)
    slots:       slots per key: int, {key: int}, or None (one slot per job, no refill)
    lanes_per_key: lanes (device batches) each key's slots are split over
    priority:    {key: stream priority} (heavier envs first among concurrent lanes)
    cycle:       wrap the queues around (steady state) instead of stopping when they run out
    mode:        "device" (protocol kernel, R rounds per call) or "host" (BatchedGraspTrials)
    on_record:   callback(job, TrialRecord) for every finished trial (e.g. a dataset writer)
    pipeline:    device protocol: keep the next call enqueued while the host collects and refills
    """

    def __init__(self, jobs, scene_of, key_of, slots=None, lanes_per_key=1, rounds_per_call=1, priority=None,
                 cycle=False, device=None, protocol=None, mode="device", record=False, on_record=None,
                 keep_records=True, prepare=True, pipeline=True):
        self.scene_of, self.key_of = scene_of, key_of
        self.pipeline = bool(pipeline)
        self.rounds_per_call, self.cycle, self.mode, self.record = int(rounds_per_call), bool(cycle), mode, record
        self.protocol = protocol
        self.on_record, self.keep_records = on_record, keep_records
        self.results = {}          # job -> its (latest) TrialRecord
        self.finished = []         # (job, TrialRecord) in completion order (cycled jobs repeat)
        self.finished_order = []
        self._lock = threading.Lock()
        self._scenes = {}
        self._payloads = AssetCache()
        by_key = {}
        for j in jobs:
            by_key.setdefault(key_of(j), []).append(j)
        self.lanes = []
        for key in sorted(by_key, key=repr):
            kj = by_key[key]
            n = len(kj) if slots is None else (slots.get(key, len(kj)) if isinstance(slots, dict) else int(slots))
            if not self.cycle:
                n = min(n, len(kj))
            if n <= 0:
                continue
            nl = max(1, min(int(lanes_per_key), n))
            per = [n // nl + (1 if i < n % nl else 0) for i in range(nl)]
            # deal the key's queue round-robin over its lanes so every lane sees the same mix
            for li in range(nl):
                q = kj[li::nl]
                if not q:
                    continue
                pr = (priority or {}).get(key, 0)
                self.lanes.append(Lane(self, key, q, per[li], device, pr))
        if prepare and self.mode in ("device", "host"):
            for ln in self.lanes:   # refill payloads of every job, outside any timed region
                for j in ln.queue:
                    self.payload(j)

    # -- jobs ---------------------------------------------------------------------------------
    def scene(self, job):
        if job not in self._scenes:
            self._scenes[job] = self.scene_of(job)
        return self._scenes[job]

    def payload(self, job):
        return self._payloads.get_or_build(("job", job), lambda: BatchedGraspTrials.scene_payload(self.scene(job)))

    def _finish(self, job, rec):
        with self._lock:
            if self.keep_records:
                self.results[job] = rec
                self.finished.append((job, rec))
            self.finished_order.append(job)
        if self.on_record is not None:
            self.on_record(job, rec)

    # -- running --------------------------------------------------------------------------------
    @property
    def main_lane(self):
        return max(range(len(self.lanes)), key=lambda i: self.lanes[i].stats.slots)

    def run(self, main_calls=None, until_done=None, timed=False, min_trials=None):
        """Every lane calls on its own thread.  main_calls: the lane with the most slots makes
        exactly that many calls and the others keep their streams busy until it is done;
        otherwise (until_done) each lane runs until its queue is empty and its slots idle.
        min_trials: additionally keep going until that many trials finished (warm-up to a
        steady phase mix).  timed: CUDA events on every lane's stream around its calls."""
        if until_done is None:
            until_done = main_calls is None and min_trials is None
        stop = threading.Event()
        errors = []
        main = self.main_lane
        n0 = len(self.finished_order)

        def lane_loop(i):
            ln = self.lanes[i]
            if timed:
                ln.dev.timer_start()
            c0 = ln.stats.calls
            while True:
                if until_done:
                    if ln.idle:
                        break
                elif i == main and main_calls is not None:
                    done = ln.stats.calls - c0
                    if done >= main_calls and (min_trials is None or len(self.finished_order) - n0 >= min_trials):
                        stop.set()
                        break
                    if min_trials is None and done == main_calls - 1:
                        ln.call(last=True)   # exactly main_calls calls complete inside the run
                        continue
                elif stop.is_set():
                    break
                elif main_calls is None and min_trials is not None and len(self.finished_order) - n0 >= min_trials:
                    stop.set()
                    break
                ln.call()
            ln.drain()
            if timed:
                ln.stats.device_ms += ln.dev.timer_stop()

        def work(i):
            try:
                lane_loop(i)
            except BaseException as exc:   # surface a lane's failure in the caller
                errors.append(exc)
                stop.set()

        th = [threading.Thread(target=work, args=(i,)) for i in range(len(self.lanes))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errors:
            raise errors[0]
        return self.results

    def reset_stats(self):
        for ln in self.lanes:
            ln.stats = LaneStats(slots=ln.stats.slots)

    def set_profiling(self, on=True):
        for ln in self.lanes:
            ln.dev.set_profiling(on)

    @property
    def n_slots(self):
        return sum(ln.stats.slots for ln in self.lanes)
