"""cProfile of the per-call drop-in loop (bench.api_loop_rate: row_scores -> draw_samples -> track_step ->
reconstruct_frame on host arrays) at a bench config: where the host time of one iteration goes."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"])
ks, _ = bench.make_data(dict(cfg, T=26), [0])
A0, B0 = bench.init_factors(cfg, [0])
print("warm", bench.api_loop_rate(cfg, ks[:, 0], A0[0], B0[0], frames=24))
pr = cProfile.Profile()
pr.enable()
fps = bench.api_loop_rate(cfg, ks[:, 0], A0[0], B0[0], frames=100)
pr.disable()
print("frames/s under cProfile", fps)
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
