"""Per-frame wall time of config 3 through the production Pipeline, with the
surfel / node capacities (growth events) -- to find frame-level stalls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_1904_13073_b200 as pkg
import torch
spec = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
cfg = bench.make_cfg(spec)
n = spec["seq_frames"]
frames = bench.render_frames(spec, cfg, n, 0)
pipe = pkg.Pipeline(cfg)
ctx = pipe.context
last = None
for t in range(n):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = pipe.process_frame(frames[t], t)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    cap = ctx.capacity()
    flag = " GROW" if last is not None and cap != last else ""
    last = cap
    print(f"{t:3d} {dt:8.2f} ms solve {st['solve_ms']:6.2f} fusion {st['fusion_ms']:6.2f} rigid {st['rigid_ms']:5.2f} total {st['total_ms']:7.2f} surfels {st['surfel_count']} nodes {st['node_count']} cap {cap}{flag}", flush=True)
