import cProfile, pstats, os, sys, runpy, io
sys.argv = ["x"]
sys.path.insert(0, os.getcwd())
import bench
orig = bench.run_e2e
n = [0]
def wrap(*a, **k):
    pr = cProfile.Profile(); pr.enable()
    r = orig(*a, **k)
    pr.disable()
    s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(14)
    print("REP", n[0], r["ms_per_step"], r["host_enqueue_ms_per_step"]); print(s.getvalue()[:3500]); n[0] += 1
    return r
bench.run_e2e = wrap
os.environ["REPS"] = "2"
runpy.run_path("tools/e2e_probe.py", run_name="__main__")
