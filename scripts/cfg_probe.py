"""Per-frame stats of a bench config (node growth, appends) for profiling."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench


def main(config="cfg3", frames=24):
    import paper_1904_13073_b200 as pkg

    spec = bench.CONFIGS[config]
    cfg = bench.make_cfg(spec)
    fr = bench.render_frames(spec, cfg, frames, 0)
    pipe = pkg.Pipeline(cfg)
    for t in range(frames):
        d = pipe.process_frame(fr[t], t)
        if t == 0:
            print(sorted(d.keys()))
        print(t, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items()
                  if not isinstance(v, (list, dict))})


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "cfg3", int(sys.argv[2]) if len(sys.argv) > 2 else 24)
