"""Pairs per assembly tile at cfg2 frame 20 (how many staging passes)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1904_13073_b200 as pkg
spec = bench.CONFIGS["cfg2"]
cfg = bench.make_cfg(spec)
frames = bench.render_frames(spec, cfg, 22, 0)
pipe = pkg.Pipeline(cfg)
for t in range(21):
    pipe.process_frame(frames[t], t)
ctx = pipe.context
pose = ctx.get_pose()
ctx.frame_maps(frames[21], 21)
ne = ctx.build_normal_equations(pose, 21, 20)
pl = ctx.associate(pose)
s = np.asarray(pl["surfel"])
cnt = np.bincount(s)
m = ctx.download_model()
print("pairs", len(s), "surfels with pairs", (cnt > 0).sum(), "max pairs per surfel", cnt.max(),
      "surfels with > 10 pairs", (cnt > 10).sum(), "mean pairs of paired surfels", cnt[cnt > 0].mean())
