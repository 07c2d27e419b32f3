import sys, time, cProfile, pstats, pathlib
sys.path.insert(0, "/root/repo")
import bench
pr = cProfile.Profile()
r = bench.v_callable_rate(bench.GOLD / "v0.ckpt")
print(r)
pr.enable()
r = bench.v_callable_rate(bench.GOLD / "v0.ckpt", seed=91)
pr.disable()
print(r)
pstats.Stats(pr).sort_stats("cumtime").print_stats(25)
