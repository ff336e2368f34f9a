"""cProfile of the synchronous drop-in loop (submit / release / on_release
per probe) in ring mode: where a reference user's per-call time goes."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.argv.append("--ring")
import sched_timing as T  # noqa: E402
cProfile.run("T.ring_latency('mgb-warps', 2000)", "/tmp/dropin.prof")
pstats.Stats("/tmp/dropin.prof").sort_stats("tottime").print_stats(18)
