import cProfile, pstats, sys
sys.argv = ["engine_bench.py", "40", "1"]
sys.path.insert(0, "tools")
import engine_bench
cProfile.run("engine_bench.main(40, 1)", "gpurun_out/engine.prof")
p = pstats.Stats("gpurun_out/engine.prof"); p.sort_stats("cumulative").print_stats(35)
