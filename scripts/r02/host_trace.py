"""cfg2 frames 0-24 with DS_TRACE_HOST=1: host-side timings per frame (graph
build, pattern build, waits) next to the GPU frame time."""
import os, sys
os.environ["DS_TRACE_HOST"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_1904_13073_b200 as pkg
spec = bench.CONFIGS["cfg2"]
cfg = bench.make_cfg(spec)
frames = bench.render_frames(spec, cfg, 25, 0)
pipe = pkg.Pipeline(cfg)
for t in range(25):
    pipe.process_frame(frames[t], t)
