"""Run a few frames of a config through the C-ABI (for ncu launch lists / captures).

  python tools/profile_frames.py --config cloth256 --frames 2 [--precision fp32] [--resetup-at 1 5]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_13390_b200 import mgpbd, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cloth256")
    ap.add_argument("--frames", type=int, default=2)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--n-iters", type=int, default=0)
    ap.add_argument("--resetup-at", type=int, nargs="*", default=[],
                    help="mark the hierarchy stale before these frames (setup from that frame's state)")
    ap.add_argument("--no-profile", action="store_true", help="graph replay instead of eager profiled launches")
    a = ap.parse_args()
    sc = scenes.make(a.config)
    n_iters = a.n_iters or sc.n_iters
    ctx = mgpbd.Context.from_scene(sc, precision=1 if a.precision == "fp32" else 0, profile=0 if a.no_profile else 1)
    for f in range(a.frames):
        if f in a.resetup_at:
            ctx.setup_hierarchy()
        t = time.perf_counter()
        ctx.step(sc.dt, n_iters)
        s = ctx.stats()
        print(f"frame {f}: wall {1e3 * (time.perf_counter() - t):.1f} ms, event {s.ms_frame:.1f} ms, setup "
              f"{s.ms_setup:.1f} ms, l0 passes {s.l0_pass_ms:.1f} ms / {s.l0_pass_launches} launches "
              f"({s.l0_pass_bytes / max(s.l0_pass_ms, 1e-9) / 1e6:.0f} GB/s), launches {s.kernel_launches}, "
              f"indef {s.indefinite_events}, levels {[(s.n[l], s.nnz[l]) for l in range(s.n_levels)]}, "
              f"omega {[round(s.omega[l], 4) for l in range(s.n_levels)]}, |b| {s.b_norm[0]:.3e}->"
              f"{s.b_norm[n_iters - 1]:.3e}", flush=True)


if __name__ == "__main__":
    main()
