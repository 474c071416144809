"""cfg2 sequence for profiling: `skip` frames outside the profiler range, then
`count` frames inside cudaProfilerStart/Stop (use ncu --profile-from-start off)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench


def main(skip=40, count=2, config="cfg2"):
    import paper_1904_13073_b200 as pkg

    spec = bench.CONFIGS[config]
    cfg = bench.make_cfg(spec)
    frames = bench.render_frames(spec, cfg, skip + count, 0)
    pipe = pkg.Pipeline(cfg)
    for t in range(skip):
        pipe.process_frame(frames[t], t)
    import torch
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for t in range(skip, skip + count):
        d = pipe.process_frame(frames[t], t)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print({k: d[k] for k in ("surfel_count", "node_count", "correspondences", "total_ms")})


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:3]), *sys.argv[3:4])
