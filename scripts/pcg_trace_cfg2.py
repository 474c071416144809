"""PCG phase timestamps (DS_PCG_TRACE) on the cfg2 system after `skip` frames."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main(skip=40):
    import paper_1904_13073_b200 as pkg
    spec = bench.CONFIGS["cfg2"]
    cfg = bench.make_cfg(spec)
    frames = bench.render_frames(spec, cfg, skip + 1, 0)
    pipe = pkg.Pipeline(cfg)
    for t in range(skip):
        pipe.process_frame(frames[t], t)
    ctx = pipe.context
    ctx.frame_maps(frames[skip], skip)
    ne = ctx.build_normal_equations(pipe.pose(), skip, 0)
    print("nodes", ctx.num_nodes(), "blocks", len(ne["col"]), file=sys.stderr)
    for _ in range(4):
        ctx.pcg_solve(1e-3, 10, 0.0)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:2]))
