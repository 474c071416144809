import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import bench
import paper_1904_13073_b200 as pkg
for name in ("cfg2", "cfg3"):
    spec = bench.CONFIGS[name]; cfg = bench.make_cfg(spec)
    frames = bench.render_frames(spec, cfg, 21, 0)
    pipe = pkg.Pipeline(cfg)
    for t in range(21):
        pipe.process_frame(frames[t], t)
    ctx = pipe.context
    ctx.frame_maps(frames[20], 20)
    a = ctx.associate(pipe.pose())
    s = a["surfel"]; s = s[s >= 0]
    u, c = np.unique(s, return_counts=True)
    h = np.bincount(c)
    print(name, "pairs", len(s), "surfels", len(u), "hist", h[:12].tolist(), "max", c.max(), ">4:", (c > 4).sum(), ">8:", (c > 8).sum())
    pipe.close()
