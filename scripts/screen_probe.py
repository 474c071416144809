"""Per-frame fusion/screening counts on the cfg2 workload (first frames)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench


def main(n=12):
    import paper_1904_13073_b200 as pkg
    spec = bench.CFG2
    cfg = bench.make_cfg(spec)
    frames = bench.render_frames(spec, cfg, n, 0)
    pipe = pkg.Pipeline(cfg)
    for t, f in enumerate(frames):
        d = pipe.process_frame(f, t)
        keys = ("surfel_count", "node_count", "valid_pixels", "fused", "appended", "removed",
                "compressive_rejected", "low_support_rejected", "new_nodes", "fusion_ms")
        print(t, {k: d[k] for k in keys}, flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 12)
