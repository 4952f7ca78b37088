"""Diagnostic (not collected): cProfile of the recording bench loop (single batch)."""
import cProfile, pstats, sys, io
sys.path.insert(0, '.')
import bench
sys.argv = ["bench.py", "--no-cpu", "--steps", "150", "--warmup", "50", "--lanes", "1", "--record", "/tmp/ds_prof"]
pr = cProfile.Profile()
pr.enable()
bench.main()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue()[:6000])
