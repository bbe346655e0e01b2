"""Per-frame hierarchy shape and frame time (A/B of the lazily rebuilt hierarchies).

  python tools/hier_report.py --config block1.67M --frames 12 [--precision fp32] [--phases]
One line per frame: ms, setup flag, indefinite events, level sizes / nnz, omega per level; with
--phases the context runs with profiling on (no graph replay) and adds the per-phase ms.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_13390_b200 import mgpbd, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="block1.67M")
    ap.add_argument("--frames", type=int, default=12)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--phases", action="store_true")
    a = ap.parse_args()
    sc = scenes.make(a.config)
    ctx = mgpbd.Context.from_scene(sc, precision=1 if a.precision == "fp32" else 0)
    if a.phases:
        ctx.set_profiling(True)
    for f in range(a.frames):
        ctx.step(sc.dt, sc.n_iters)
        s = ctx.stats()
        nl = s.n_levels
        sizes = " ".join(f"{s.n[l]}/{s.nnz[l]}" for l in range(nl))
        om = " ".join(f"{s.omega[l]:.3f}" for l in range(nl))
        ph = ""
        if a.phases:
            ph = (f" | asm {s.ms_assemble:.1f} gal {s.ms_galerkin:.1f} vc {s.ms_vcycle:.1f}"
                  f" pcg {s.ms_pcg_other:.1f} upd {s.ms_update:.1f} setup {s.ms_setup:.1f}")
        print(f"frame {f:2d} {s.ms_frame:7.1f} ms {'S' if s.setup_ran else ' '} ind {s.indefinite_events:2d}"
              f" | L={nl} {sizes} | omega {om}{ph}", flush=True)


if __name__ == "__main__":
    main()
