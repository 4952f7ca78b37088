"""Diagnostic (not collected): cProfile of the host side of the single-batch bench loop."""
import cProfile, pstats, sys, io
sys.path.insert(0, '.')
import bench
sys.argv = ["bench.py", "--no-cpu", "--steps", "200", "--warmup", "100", "--lanes", "1"]
pr = cProfile.Profile()
pr.enable()
bench.main()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumtime").print_stats("protocol|_native|bench|multienv", 30)
print(s.getvalue()[:7000])
