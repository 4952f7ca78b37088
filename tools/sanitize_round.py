"""One small device-protocol workload for compute-sanitizer (memcheck / racecheck / synccheck):
3 envs (box, cylinder, sphere) through grip_run_rounds with refills, plus one host-protocol round,
the contact readout and the quarantine check -- every kernel of the product path runs at least
once, including the cluster broad phase (supersets rebuilt in the closing phase).

  compute-sanitizer --tool memcheck --target-processes all python tools/sanitize_round.py
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main(rounds=int(sys.argv[1]) if len(sys.argv) > 1 else 24):
    from paper_2503_05020_b200 import protocol as pt
    from paper_2503_05020_b200 import scene as sc
    from paper_2503_05020_b200.runner import TrialRunner
    c = sc.load_cfg2_candidates()
    kinds = c["kind"]
    jobs = [0, 1, 2, 3, 4, 5]
    r = TrialRunner(jobs, lambda j: sc.cfg2_scene(j, c), lambda j: int(kinds[j]), slots=1, rounds_per_call=4)
    r.run(main_calls=max(1, rounds // 4))
    ln = r.lanes[0]
    env = ln.group.envs[0]
    ev = pt.contact_events_now(env)
    md = env.min_contact_distance()
    bad = ln.group.dev.check_finite()
    hr = TrialRunner([6, 7, 8], lambda j: sc.cfg2_scene(j, c), lambda j: int(kinds[j]), slots=1, mode="host")
    hr.run(main_calls=3)
    print("sanitize workload done:", len(r.finished), "trials,", len(ev), "events, min d", md, "nonfinite", bad.tolist())


if __name__ == "__main__":
    main()
